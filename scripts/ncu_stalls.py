"""Per-kernel stall samples by SASS opcode from an ncu report's source page
(development aid): python scripts/ncu_stalls.py report.ncu-rep
A `@!P BRA` right after `SYNCS.PHASECHK...TRYWAIT` (or whose predicate a hoisted
TRYWAIT set) is a consumer waiting on a TMA full barrier, i.e. waiting for data."""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kern, data, hdr = None, collections.OrderedDict(), None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Kernel Name":
        kern, hdr = r[1][:90], None
        data.setdefault(kern, [])
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and kern:
        data[kern].append(r)
for k, v in data.items():
    seen, vv = set(), []
    for r in v:
        if r[0] not in seen:
            seen.add(r[0])
            vv.append(r)
    tot = sum(int(r[2] or 0) for r in vv) or 1
    print(f"===== {k}  ({len(vv)} SASS instructions, {tot} stall samples)")
    cat = collections.Counter()
    for i, r in enumerate(vv):
        op = r[1].strip()
        opn = op.split()[1] if op.startswith("@") else op.split()[0]
        if opn == "BRA" and i > 0 and "SYNCS" in vv[i - 1][1]:
            opn = "BRA after SYNCS.TRYWAIT"
        cat[opn] += int(r[2] or 0)
    print("  by opcode: " + ", ".join(f"{o} {s / tot * 100:.1f}%" for o, s in cat.most_common(12)))
    for i, r in enumerate(vv):
        if int(r[2] or 0) / tot > 0.012:
            print(f"  {int(r[2]) / tot * 100:5.1f}%  {r[1].strip()[:64]:64s} | prev: {vv[i - 1][1].strip()[:56]}")
