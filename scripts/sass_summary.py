#!/usr/bin/env python
"""Instruction-level evidence of the production kernels.

For every kernel in libwave25.so whose name matches the production
instantiations (k_stream interior / x walls / y walls, the source, the peer
flag kernels, and whatever else is given with --all), count the SASS
mnemonics that prove the design: UTMALDG (TMA tensor loads), UTMAPF (TMA L2
prefetch), SYNCS (mbarrier ops), USETMAXREG (warp-specialised register
reallocation), FFMA / FFMA2 / FADD / FADD2 (scalar vs packed fp32 math),
LDS / STG, and LDL / STL (local-memory spills: must be 0), plus the
registers / stack / local bytes of `cuobjdump -res-usage`.

    python scripts/sass_summary.py [--all] > profiles/sass_rNN.txt
"""
import collections
import re
import subprocess
import sys

LIB = "paper_2009_04619_b200/libwave25.so"
KEYS = ["UTMALDG", "UTMAPF", "UBLKCP", "SYNCS", "USETMAXREG", "FFMA2", "FFMA", "FADD2", "FADD", "FMUL2",
        "FMUL", "MUFU", "LDS", "STS", "LDG", "STG", "LDL", "STL", "BAR", "BRA"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.strip().splitlines()


def main():
    everything = "--all" in sys.argv
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    usage, fn = {}, None
    for ln in res.splitlines():
        m = re.search(r"Function (\S+):", ln)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", ln)
        if m and fn:
            usage[fn] = tuple(int(x) for x in m.groups())
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    counts, fn = {}, None
    for ln in sass.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            fn = m.group(1)
            counts[fn] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", ln)
        if m and fn:
            op = m.group(1)
            counts[fn][op] += 1
            counts[fn]["_total"] += 1
    names = sorted(counts)
    dem = dict(zip(names, demangle(names)))
    # HEAD's production instantiations (wave.cu init_kernels defaults): fp32 interior, seam x walls,
    # two-region x walls (non-16 PML widths), y walls; fp64 interior / walls; the stored-eta walls
    prod = re.compile(r"k_stream<248, 248, 8, 1, 0, 1, 112, float, 0, 1>|k_stream<240, 240, 8, 1, 0, 1, 112, float, 0, 1>|k_stream<32, 32, 64, 1, 7, 1, 112, float, 0, 1>|"
                      r"k_stream<24, 16, 128, 1, 5, 1, 112, float, 0, 1>|k_stream<128, 128, 16, 1, 6, 1, 112, float, 0, 1>|"
                      r"k_stream<124, 124, 8, 1, 0, 1, 112, double, 0, 1>|k_stream<24, 16, 64, 1, 5, 1, 112, double, 0, 1>|"
                      r"k_stream<64, 64, 16, 1, 6, 1, 112, double, 0, 1>|k_stream<24, 16, 64, 1, 4, 1, 112, float, 0, 1>|"
                      r"k_stream<128, 128, 16, 1, 4, 1, 112, float, 0, 1>|k_source<float>|k_peer_wait|k_peer_signal|"
                      r"k_vdt2<float>|k_inc<float>|k_stats<float>")
    print(f"# SASS summary of {LIB} (cuobjdump -sass / -res-usage), sm_100a")
    print("# kernel | regs stack shared local | total instr | " + " ".join(KEYS))
    for n in names:
        d = dem[n]
        if not everything and not prod.search(d):
            continue
        u = usage.get(n, (0, 0, 0, 0))
        c = counts[n]
        print(f"{d[:110]} | {u[0]} {u[1]} {u[2]} {u[3]} | {c['_total']} | " + " ".join(f"{k}={c[k]}" for k in KEYS))


if __name__ == "__main__":
    main()
