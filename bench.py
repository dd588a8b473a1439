#!/usr/bin/env python
"""Benchmark of the 25-point acoustic wave step (arXiv 2009.04619 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

One JSON line on rank 0.  A "step" is one time step of the whole hot path
(interior 25-point stencil + PML walls + source injection) over the grid.

* N = 1: workload C3 = BASELINE.json configs[2] (1024^3 extended grid, layered
  V, 16-cell PML) -- the 1-GPU point of the configs[3]/[4] scaling runs.
* N > 1 (torchrun, one process per GPU, NCCL): weak scaling, configs[4]: a
  1024 x 1024 x (1024 N) grid in z-slabs of 1024 planes per rank, 4-plane halo
  exchange per step overlapped with the interior kernel.

value      = points x steps / device time (CUDA events, max over ranks), Gpoints/s
e2e        = same metric through the public API with HOST buffers: H2D of the
             velocity model + wavelet from pinned memory, K steps, D2H of u^K
roofline   = the interior kernel (dominant): 16 B x its points per launch / its
             average launch time measured with CUDA events on its stream in a
             profiled pass of K steps; peak = MEASURED_PEAKS.json hbm_gbs
cpu_baseline = the CPU oracle (oracle/, as it stands) on a bounded z-slab sample
             of the same workload on this host's cores (rank 0, N = 1)
--impl reference: the oracle as the reference arm (no GPU), same metric/config.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Gpoints/s per step and % of HBM roofline (GB/s) at 1/2/4/8 B200"
UNIT = "Gpoints/s"
BYTES_PER_POINT = 16        # read u, u_prev, vdt2; write u_next


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(config: str, world: int, scaling: str = "weak"):
    import synth
    if world > 1 and scaling == "strong":
        s = synth.scenario("C3")
        desc = (f"C4 strong scaling: the C3 1024^3 grid (layered V, 16-cell PML, Ricker 15 Hz at the "
                f"centre) cut into {world} z-slabs of ~{1024 // world} planes (BASELINE.json configs[3])")
        return s, desc
    if world > 1:
        s = synth.scenario("C5")
        s = s.with_(nz=s.nz * world)
        desc = (f"C5 weak scaling: 1024x1024x{1024 * world} extended grid, z-slabs of 1024 planes "
                f"per GPU, 16-cell PML, layered V 1500->4500 m/s in 8 z-layers, Ricker 15 Hz at the "
                f"global centre, fp32")
        return s, desc
    s = synth.scenario(config)
    if config == "C3":
        desc = ("C3: 1024^3 extended grid (992^3 inner + 16-cell PML on every face), layered V "
                "1500->4500 m/s in 8 z-layers, Ricker 15 Hz at the centre (BASELINE.json configs[2])")
    elif config == "C2":
        desc = "C2: 512^3 extended grid, 16-cell PML, constant V 2000 m/s, Ricker 20 Hz, fp32 (configs[1])"
    else:
        desc = f"{config}: {s.nx}x{s.ny}x{s.nz} extended grid, w={s.w}, fp32"
    return s, desc


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        lines = open(self.f.name).read().strip().splitlines()
        os.unlink(self.f.name)
        sm, smax, reasons = [], [], set()
        for ln in lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                smax.append(float(p[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "samples": len(sm),
                "reasons": sorted(reasons)}


def clocks_rejected(c):
    if not c:
        return False
    if any(r in c["reasons"] for r in ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")):
        return True
    return c["sm_mhz"] < 0.6 * c["sm_max_mhz"] and "sw_power_cap" not in c["reasons"]


# ---------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def oracle_slab_setup(s, planes: int):
    import numpy as np
    import oracle
    import synth
    off = max(0, s.nz // 2 - planes // 2)
    g = oracle.make_geom(s.nx, s.ny, planes, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
    V = synth.velocity(s, nz_global=s.nz, z_offset=off, nz_local=planes)
    vd = oracle.vdt2(V, s.dt)
    u = np.zeros((planes + 8, s.ny + 8, s.nx + 8), np.float32)
    up = np.zeros_like(u)
    u[4:-4, 4:-4, 4:-4] = synth.random_state((planes, s.ny, s.nx), 7)
    wl = synth.wavelet_for(s, 4096)
    return g, u, up, vd, wl, off


def oracle_steps(s, state, nsteps: int) -> float:
    """Run nsteps oracle steps on the slab sample; returns seconds."""
    import oracle
    g, u, up, vd, wl, off = state
    t0 = time.perf_counter()
    for n in range(nsteps):
        st = oracle.step_padded(g, u, up, vd, s.source, wl[n % len(wl)])
        assert st == 0
        u, up = up, u
    dt = time.perf_counter() - t0
    state[1], state[2] = u, up
    return dt


def cpu_baseline(s, planes=48, target_s=12.0) -> dict:
    """Oracle on a 48-plane z-slab of the workload, as many steps as fit in
    ~target_s seconds (bounded: 2..400 steps)."""
    import oracle
    oracle.build()
    state = list(oracle_slab_setup(s, planes))
    t1 = oracle_steps(s, state, 2) / 2             # warm-up + rate estimate
    steps = int(max(2, min(400, target_s / max(t1, 1e-3))))
    secs = oracle_steps(s, state, steps)
    pts = planes * s.ny * s.nx * steps
    return {"value": pts / secs / 1e9, "unit": UNIT, "cores": oracle.get_threads(), "kind": "oracle",
            "sample": (f"z-slab of {planes} planes (k={state[5]}..{state[5] + planes - 1}) of the "
                       f"{s.nx}x{s.ny}x{s.nz} grid x {steps} steps, fp32 oracle, {secs:.1f} s")}


def run_reference(args, rank, world):
    """The oracle as the reference arm: each step = one oracle time step on a
    bounded z-slab sample of the workload, sized so the run takes ~1-2 min."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    s, desc = workload(args.config, world, args.scaling)
    total = args.steps + args.warmup
    planes = int(min(64, max(4, round(48 * 200 / max(total, 1)))))
    state = list(oracle_slab_setup(s, planes))
    oracle_steps(s, state, args.warmup)
    secs = oracle_steps(s, state, args.steps)
    pts = planes * s.ny * s.nx * args.steps
    val = pts / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": desc, "sample_planes": planes},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle.get_threads(), "kind": "oracle",
                         "sample": f"z-slab of {planes} planes x {args.steps} steps (+{args.warmup} warm-up)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def measured_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (STREAM-style copy, measured)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(kernel_tag: str):
    """Per-launch DRAM bytes of the interior kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
        return d.get(kernel_tag)
    except Exception:
        return None


def kind_roof(bytes_per_step: float, ms_per_step: float, peak: float) -> dict:
    """Algorithmic GB/s of one kernel kind (its points x bytes per point over
    its serialized time per step) and its fraction of the roofline peak."""
    gbs = bytes_per_step / (ms_per_step / 1e3) / 1e9
    return {"gbs": gbs, "frac": gbs / peak, "ms_per_step": ms_per_step}


def roof_probe(torch):
    """3-read / 1-write streaming probe (out = a + b*c) over 2^28 fp32: the
    stencil's exact byte mix with zero halo -- the practical HBM roof."""
    n = 1 << 28
    a, b, c, o = (torch.empty(n, device="cuda").uniform_() for _ in range(4))
    for _ in range(3):
        torch.addcmul(a, b, c, out=o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        torch.addcmul(a, b, c, out=o)
    e1.record()
    torch.cuda.synchronize()
    gbs = 16 * n * 20 / (e0.elapsed_time(e1) / 1e3) / 1e9
    del a, b, c, o
    torch.cuda.empty_cache()
    return gbs


PARITY_STEPS = 12       # steps of the in-line multi-GPU parity check
PARITY_PLANES = 8       # planes compared on each side of every slab face


def seeded_planes(torch, z0: int, z1: int, ny: int, nx: int, seed: int, device):
    """Global planes [z0, z1) of a seeded U(-1, 1) field, generated on the
    device plane by plane (each plane's generator seeded by its global index),
    so any slab or window of the same global field is bitwise identical."""
    out = torch.empty((z1 - z0, ny, nx), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    for k in range(z0, z1):
        g.manual_seed(seed * 1_000_003 + k)
        out[k - z0].uniform_(-1.0, 1.0, generator=g)
    return out


def multi_gpu_parity(s, plan, runner, halo, rank, world, dist, barrier):
    """In-line correctness bit of an N>1 run.

    All ranks re-initialise the wired run collectively to a seeded random
    state (O(1) everywhere, so every face carries signal), step PARITY_STEPS
    steps through the production exchange path, and then every face between
    rank r-1 and rank r is checked BITWISE against a recompute on rank r by one
    plan of the window [b - 4K - 16, b + 4K + 16) of the same global grid
    (b = the face, K = PARITY_STEPS): the stencil reaches 4 planes per step,
    so the window's own cut ends cannot reach the 2 x 8 planes compared.
    Rank r-1's planes next to the face come over torch.distributed."""
    import torch
    from paper_2009_04619_b200.dist import SlabRunner, slab_bounds
    from paper_2009_04619_b200.wave import WavePlan
    import synth

    K, M = PARITY_STEPS, PARITY_PLANES
    dev = plan.device
    off, nzl = slab_bounds(s.nz, rank, world)
    wl = synth.wavelet_for(s, K)
    seed_u, seed_p = 101, 202
    u0 = seeded_planes(torch, off, off + nzl, s.ny, s.nx, seed_u, dev)
    um1 = seeded_planes(torch, off, off + nzl, s.ny, s.nx, seed_p, dev)
    if halo == "peer":
        runner.reset(um1, u0, source=(*s.source, wl))
        runner.step(K)
    else:
        barrier()
        plan.set_source(*s.source, wl)
        plan.set_state(um1, u0)
        runner.exchange_current()
        runner.step(K)
    torch.cuda.synchronize()
    del u0, um1
    peer_ok = True
    if halo == "peer":
        try:
            runner.check()
        except Exception:
            peer_ok = False
    got = plan.field(0)
    gloo = dist.get_backend() != "nccl"
    # rank r-1 sends its last M planes to rank r
    below = None
    if rank < world - 1:
        t = got[nzl - M:].contiguous()
        dist.send(t.cpu() if gloo else t, rank + 1)
    if rank > 0:
        below = torch.empty((M, s.ny, s.nx), dtype=torch.float32, device="cpu" if gloo else dev)
        dist.recv(below, rank - 1)
    ok = True
    if rank > 0:
        z0, z1 = max(0, off - 4 * K - 2 * M), min(s.nz, off + 4 * K + 2 * M)
        win = WavePlan(s.nx, s.ny, z1 - z0, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=z0)
        win.set_velocity(synth.velocity(s, nz_global=s.nz, z_offset=z0, nz_local=z1 - z0))
        win.set_source(*s.source, wl)
        win.set_state(seeded_planes(torch, z0, z1, s.ny, s.nx, seed_p, dev),
                      seeded_planes(torch, z0, z1, s.ny, s.nx, seed_u, dev))
        SlabRunner(win, 0, 1).step(K)          # one plan, no exchange: ghost planes stay zero
        torch.cuda.synchronize()
        ref = win.field(0)
        ok = bool(torch.equal(ref[off - z0:off - z0 + M], got[:M]))
        ok = ok and bool(torch.equal(ref[off - z0 - M:off - z0].to(below.device), below))
        del ref
        win.close()
    flag = torch.tensor([1 if (ok and peer_ok) else 0], dtype=torch.int32, device="cpu" if gloo else dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    barrier()
    return {"bitwise_faces_ok": bool(int(flag.item()) == 1), "faces": world - 1, "steps": K,
            "planes_per_face": 2 * M, "exchange": halo,
            "how": ("after the timed runs: collective reset to a seeded U(-1,1) state, K steps through the "
                    "production exchange, every slab face compared bitwise with one plan of the window "
                    "[b-4K-16, b+4K+16) recomputed on the face's upper rank")}


def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    import synth
    import __graft_entry__
    from paper_2009_04619_b200.wave import WavePlan
    from paper_2009_04619_b200.dist import PeerSlabRunner, SlabRunner, slab_bounds

    __graft_entry__.build_cuda()
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("WAVE25_DIST_BACKEND", "nccl")   # gloo: smoke-test on 1 GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    s, desc = workload(args.config, world, args.scaling)
    off, nzl = slab_bounds(s.nz, rank, world) if world > 1 else (0, s.nz)
    V = synth.velocity(s, nz_global=s.nz, z_offset=off, nz_local=nzl)
    total_steps = args.warmup + 3 * args.steps + 8
    wl = synth.wavelet_for(s, total_steps)

    def barrier():
        if dist is not None:
            if dist.get_backend() == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    def maxall(x: float) -> float:
        if dist is None:
            return x
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    kern = args.kernel if world == 1 else "stream"
    plan = WavePlan(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off, kernel=kern,
                    precision=args.precision)
    bpp = BYTES_PER_POINT * (2 if args.precision == "fp64" else 1)   # algorithmic bytes per point-step
    plan.set_velocity(V)
    plan.set_source(*s.source, wl)
    halo = os.environ.get("WAVE25_HALO", "peer")     # peer: fused peer stores; nccl: send/recv
    if world == 1:
        runner = None
    elif halo == "peer":
        try:
            runner = PeerSlabRunner(plan, rank, world)
        except RuntimeError as e:       # no P2P path: the NCCL send/recv path instead (all ranks agree)
            print(f"[bench] fused peer exchange unavailable ({e}); using NCCL send/recv", file=sys.stderr)
            halo = "nccl"
            runner = SlabRunner(plan, rank, world,
                                stage_on_host=os.environ.get("WAVE25_DIST_BACKEND", "nccl") != "nccl")
    else:
        runner = SlabRunner(plan, rank, world,
                            stage_on_host=os.environ.get("WAVE25_DIST_BACKEND", "nccl") != "nccl")
    stream = torch.cuda.current_stream()

    def steps(n):
        if runner is not None:
            runner.step(n)
        else:
            plan.step(n, stream=stream)

    steps(args.warmup)
    pts_total = s.nx * s.ny * s.nz

    def timed():
        clk = Clocks(local)
        barrier()
        clk.start()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        steps(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        c = clk.stop()
        return maxall(e0.elapsed_time(e1)), c

    ms, clocks = timed()
    remeasured = False
    if clocks_rejected(clocks):
        ms, clocks = timed()
        remeasured = True
    value = pts_total * args.steps / (ms / 1e3) / 1e9
    launches = plan.launches(args.steps) if (world == 1 or halo == "peer") else plan.launches_per_step * args.steps

    # ---- roofline of the dominant (interior) kernel: profiled pass -------
    roof = None
    kpts = plan.kernel_points()
    if world == 1 and not args.no_profile:
        kms, kn = plan.step_profiled(args.steps - args.steps % plan.steps_per_launch, stream=stream)
        t_launch = kms["interior"] / max(kn["interior"], 1)            # ms per launch
        # a two-step (TB2) launch reads u^n, u^{n-1}, vdt2 once and writes two levels: 20 B per point
        bpl = 20 if plan.steps_per_launch == 2 else bpp                  # algorithmic bytes per point per launch
        achieved = bpl * kpts["interior"] / (t_launch / 1e3) / 1e9
        peak, peak_src = measured_peak()
        step_ms_prof = sum(kms.values()) / max(args.steps, 1)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic("interior") if (args.precision == "fp32" and args.kernel == "stream") else None,
                "kernel": ("k_tb2 interior (two-step temporal blocking)" if args.kernel == "tb2"
                           else "k_stream PAIR interior (two steps through L2)" if args.kernel == "pair"
                           else "k_stream interior (TMA z-streaming, 25-pt)"),
                "points_per_launch": kpts["interior"], "bytes_per_point": bpl,
                "ms_per_launch": t_launch, "peak_source": peak_src,
                "kernel_ms_per_step": {k: v / max(args.steps, 1) for k, v in kms.items()},
                "kernel_points_per_step": kpts,
                "share_of_step": kms["interior"] / max(sum(kms.values()), 1e-9),
                # every kernel kind's algorithmic GB/s and fraction of the same peak (the walls:
                # their points x the same bytes per point / their serialized launch time)
                "per_kind": {k: kind_roof(bpl * kpts[k], kms[k] / max(args.steps, 1), peak)
                             for k in ("interior", "xwalls", "ywalls") if kpts.get(k) and kms.get(k)},
                "how": "CUDA events around each launch on the launching stream, profiled pass of K steps right after the first timed run "
                       "(direct launches serialized on that stream, so each event pair times one kernel)"}
        if not args.no_probe:
            roof["practical_roof_gbs_3r1w"] = roof_probe(torch)
            roof["frac_of_practical_roof"] = achieved / roof["practical_roof_gbs_3r1w"]

    # the paper's protocol: repeat the timed run, report
    # mean +- stddev (after the profiled pass, so that pass sees the thermal
    # state of the reported first run, not that of the repeats)
    reps = [ms]
    for _ in range(max(args.repeats - 1, 0)):
        reps.append(timed()[0])
    rep_ms = [r / args.steps for r in reps]

    # ---- end to end through the public API with host buffers -------------
    e2e = None
    if not args.no_e2e:
        Vh = torch.from_numpy(V).pin_memory()
        outh = torch.empty((nzl, s.ny, s.nx), dtype=plan.dtype).pin_memory()
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if isinstance(runner, PeerSlabRunner):
            # a wired run is re-initialised collectively (barriers around the
            # set_* calls, flag protocol restarted)
            runner.reset(None, None, velocity=Vh, source=(*s.source, wl))
        else:
            plan.set_state(None, None, stream=stream)        # u^0 = u^-1 = 0
            plan.set_velocity(Vh, stream=stream)              # H2D from pinned memory (+ vdt2 kernel)
            plan.set_source(*s.source, wl, stream=stream)     # wavelet H2D
            if runner is not None:
                barrier()
        steps(args.steps)
        plan.read(0, out=outh, stream=stream)             # D2H of u^K
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e_ms = maxall(max(e0.elapsed_time(e1), 1e3 * wall))
        h2d = V.nbytes + 4 * len(wl)
        e2e = {"value": pts_total * args.steps / (e_ms / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": outh.numel() * outh.element_size() / args.steps,
               "ms_total": e_ms, "api": "WavePlan.set_state/set_velocity(host)/set_source/step/read(host) "
                                         "-> libwave25.so C ABI"}

    parity = None
    if world > 1 and not args.no_parity:
        parity = multi_gpu_parity(s, plan, runner, halo, rank, world, dist, barrier)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(s)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic",
            "config": {"workload": desc, "grid": [s.nx, s.ny, s.nz], "points_per_step": pts_total,
                       "pml_width": s.w, "parallelism": f"z-slab x{world}" if world > 1 else "1 GPU",
                       "l2": f"no flush: {bpp * pts_total / 1e9:.1f} GB streamed per step >> 126 MB L2",
                       "precision": args.precision, "kernel_family": kern,
                       "kernels": "interior + x-walls + y-walls (2 streams, joined) + source, CUDA graph"
                                  if world == 1 else (
                                      "fused halo: stencil kernels store edge planes into the neighbours' ghost "
                                      "planes over NVLink (IPC peer mapping) + device step flags, CUDA graph"
                                      if halo == "peer" else "edges -> NCCL send/recv || interior, joined")},
            "hbm_gbs_at_algorithmic_bytes": value * bpp,
            "frac_of_measured_hbm": value * bpp / measured_peak()[0],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "parity": parity,
            "clocks": clocks, "remeasured": remeasured,
            "repeats": {"n": len(rep_ms), "ms_per_step": rep_ms,
                        "ms_per_step_mean": statistics.fmean(rep_ms),
                        "ms_per_step_stddev": statistics.pstdev(rep_ms) if len(rep_ms) > 1 else 0.0,
                        "note": "value is the first timed run (driver contract); repeats follow PAPER.md L885-888"},
        }
        print(json.dumps(line), flush=True)
    if hasattr(runner, "close"):
        runner.close()                 # unmap the neighbours' buffers (collective)
    plan.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="N>1: skip the in-line slab-face parity check")
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="N>1: weak = C5 (1024 planes per GPU), strong = C4 (the 1024^3 grid split N ways)")
    ap.add_argument("--repeats", type=int, default=5, help="timed runs (the first is `value`)")
    ap.add_argument("--kernel", choices=["stream", "tb2", "pair"], default="stream",
                    help="1 GPU: stream (default), tb2 (two-step temporal blocking) or pair (two steps through L2)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = env_rank()
    if world != args.gpus and args.gpus > 1 and world == 1:
        print(json.dumps({"error": f"--gpus {args.gpus} needs torchrun with {args.gpus} processes"}))
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
