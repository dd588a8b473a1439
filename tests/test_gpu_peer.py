"""The fused peer-store halo exchange with
several processes time-sharing one GPU: every rank maps its neighbours'
buffers over CUDA IPC exactly as on an NVLink node, so ranks 1..N-2 run the
both-neighbours-mapped path that N >= 3 runs.  Every result is compared
bitwise with ONE plan of the whole grid (the multi-GPU parity contract,
SURVEY.md §8(c) last bullet).

Covered: slabs thinner than 2R = 8 planes (a plane is an edge of both faces
and must reach both neighbours), the strong-scaling geometry (thin
slabs, z-PML only on the end ranks, source on a thin slab's edge plane), a
collective re-initialisation in the middle of a run, and a peer wait that
expires (reported, no trap)."""
import os
import socket

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def one_plan(s, steps, u0, um1, wl):
    from paper_2009_04619_b200.wave import WavePlan
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, wl)
    p.set_state(um1, u0)
    p.step(steps)
    out = p.read(0).cpu().numpy(), p.read(1).cpu().numpy()
    p.close()
    return out


def _worker(rank, world, port, scen, bounds, phases, q):
    """phases: list of (steps, state_seed or None).  A phase with a seed starts
    with a collective reset to the seeded random state (the first phase
    always does)."""
    import torch.distributed as dist
    from paper_2009_04619_b200.dist import PeerSlabRunner
    from paper_2009_04619_b200.wave import WavePlan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        s = synth.scenario(scen[0], **scen[1])
        sh = (s.nz, s.ny, s.nx)
        off, nzl = bounds[rank], bounds[rank + 1] - bounds[rank]
        total = sum(p[0] for p in phases)
        wl = synth.wavelet_for(s, total)
        p = WavePlan(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
        p.set_velocity(synth.velocity(s)[off:off + nzl])
        p.set_source(*s.source, wl)
        runner = PeerSlabRunner(p, rank, world)
        for steps, seed in phases:
            if seed is not None:
                u0, um1 = synth.random_state(sh, seed), synth.random_state(sh, seed + 1)
                runner.reset(um1[off:off + nzl], u0[off:off + nzl])
            runner.step(steps)
        torch.cuda.synchronize()
        runner.check()
        q.put((rank, p.read(0).cpu().numpy(), p.read(1).cpu().numpy()))
        runner.close()
        p.close()
    finally:
        dist.destroy_process_group()


def run_world(scen, bounds, phases, timeout=600):
    import torch.multiprocessing as mp
    world = len(bounds) - 1
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scen, bounds, phases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    parts = sorted((q.get(timeout=timeout) for _ in range(world)), key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    return (np.concatenate([a for _, a, _ in parts], axis=0), np.concatenate([b for _, _, b in parts], axis=0))


def reference(scen, phases):
    """One plan of the whole grid, started from the last phase's state."""
    s = synth.scenario(scen[0], **scen[1])
    sh = (s.nz, s.ny, s.nx)
    last = max(i for i, (_, seed) in enumerate(phases) if seed is not None)
    steps = sum(p[0] for p in phases[last:])
    seed = phases[last][1]
    # the source counter restarts at every reset, so the reference replays the
    # wavelet from sample 0
    wl = synth.wavelet_for(s, sum(p[0] for p in phases))
    return one_plan(s, steps, synth.random_state(sh, seed), synth.random_state(sh, seed + 1), wl)


@pytest.mark.parametrize("scen,bounds,phases,env", [
    # 3 ranks, the middle slab 5 planes (< 2R): both neighbours mapped over IPC
    (("RAGGED", {}), [0, 20, 25, 53], [(19, 71)], {}),
    # 3 ranks, middle slab of exactly R planes (every plane an edge of both faces)
    (("RAGGED", {}), [0, 24, 28, 53], [(15, 73)], {}),
    # 4 ranks, two adjacent R-plane slabs (a thin slab's neighbour is thin too)
    (("RAGGED", {}), [0, 24, 28, 32, 53], [(13, 77)], {}),
    # the seam x walls (opt-in WAVE25_SEAM=1; w = 16, rows of exactly nx: DESIGN.md §5a) on slabs: 3
    # ranks, a 4-plane middle slab holding the source (C1: 64^3, centre source)
    (("C1", {}), [0, 30, 34, 64], [(17, 79)], {"WAVE25_SEAM": "1"}),
    (("C1", {}), [0, 30, 34, 64], [(17, 79)], {}),
    # 4 ranks, strong-scaling geometry: thin slabs, the z-PML (w=5) only on the
    # end ranks, the source on plane 20 = the first plane of a 7-plane slab (an
    # edge plane of both of its faces: mirrored into both neighbours)
    (("RAGGED", dict(nz=48, w=5, src=(35, 22, 20))), [0, 14, 20, 27, 48], [(21, 75)], {}),
])
def test_peer_processes_bitwise(scen, bounds, phases, env, monkeypatch):
    for k, v in env.items():       # (inherited by the spawned ranks; the reference plan reads it too)
        monkeypatch.setenv(k, v)
    got, gotp = run_world(scen, bounds, phases)
    ref, refp = reference(scen, phases)
    assert np.array_equal(got, ref) and np.array_equal(gotp, refp)


def test_peer_reset_mid_run_bitwise():
    # re-initialising a wired run (PeerSlabRunner.reset: barrier, set_state
    # restarts the flag protocol, barrier, halo push, barrier) after 9 steps,
    # then 11 more == one plan started from the new state
    scen = ("RAGGED", {})
    phases = [(9, 81), (11, 83)]
    got, gotp = run_world(scen, [0, 18, 36, 53], phases)
    ref, refp = reference(scen, phases)
    assert np.array_equal(got, ref) and np.array_equal(gotp, refp)


@pytest.mark.parametrize("bounds", [[0, 20, 25, 53]])
def test_peer_store_thin_slabs_one_process_bitwise(bounds):
    # a thin-slab case with all slabs in one process (device pointers, each
    # slab on its own stream).  Kept to <= 3 slabs: every plan drives 3 streams
    # (interior + two wall side streams), and once more streams than the
    # device's hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS, default 8)
    # are busy, two plans' streams can share a queue, so one plan's spinning
    # peer-wait kernel can block its neighbour's wall kernels behind it -- a
    # false dependency of the single-process test harness only (one process
    # per GPU in production; the 4-slab cases run as 4 processes above)
    from paper_2009_04619_b200.wave import WavePlan
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 91), synth.random_state(sh, 92)
    V = synth.velocity(s)
    steps = 17
    wl = synth.wavelet_for(s, steps)
    n = len(bounds) - 1
    plans = []
    for r in range(n):
        off, nzl = bounds[r], bounds[r + 1] - bounds[r]
        p = WavePlan(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
        p.set_velocity(V[off:off + nzl])
        p.set_source(*s.source, wl)
        p.set_state(um1[off:off + nzl], u0[off:off + nzl])
        p.flags = torch.zeros(2, dtype=torch.int64, device="cuda")
        plans.append(p)
    for r, p in enumerate(plans):
        lo = plans[r - 1] if r > 0 else None
        hi = plans[r + 1] if r < n - 1 else None
        p.set_peers(lo_bufs=lo.bufs if lo else None, hi_bufs=hi.bufs if hi else None,
                    lo_nz=lo.nz if lo else 0, lo_flags=lo.flags if lo else None,
                    hi_flags=hi.flags if hi else None)
    for p in plans:
        p.push_halo(1)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in plans]
    for p, st in zip(plans, streams):
        p.step_peer(steps, stream=st)
    torch.cuda.synchronize()
    got = np.concatenate([p.read(0).cpu().numpy() for p in plans], axis=0)
    ref, _ = one_plan(s, steps, u0, um1, wl)
    for p in plans:
        p.peer_check()
        p.close()
    assert np.array_equal(got, ref)


def test_peer_wait_timeout_is_reported_not_trapped():
    # the lower slab steps, its upper neighbour never does: the second step's
    # wait expires after the (short) bound, peer_check raises WAVE_ERR_PEER, and
    # the CUDA context is still usable (no __trap)
    from paper_2009_04619_b200 import _abi
    from paper_2009_04619_b200.wave import WavePlan
    s = synth.scenario("RAGGED")
    plans = []
    for off, nzl in ((0, 30), (30, 23)):
        p = WavePlan(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
        p.set_velocity(synth.velocity(s)[off:off + nzl])
        p.flags = torch.zeros(2, dtype=torch.int64, device="cuda")
        plans.append(p)
    a, b = plans
    a.set_peers(hi_bufs=b.bufs, hi_flags=b.flags)
    b.set_peers(lo_bufs=a.bufs, lo_nz=a.nz, lo_flags=a.flags)
    a.set_peer_timeout(0.2)
    a.step_peer(3)
    torch.cuda.synchronize()
    with pytest.raises(_abi.WaveError) as ei:
        a.peer_check()
    assert ei.value.status == _abi.WAVE_ERR_PEER and "upper" in ei.value.message
    b.peer_check()                                   # the idle neighbour saw no timeout
    assert float(torch.ones(8, device="cuda").sum().item()) == 8.0
    # a collective reset clears the error word
    for p in plans:
        p.set_state(None, None)
    a.peer_check()
    for p in plans:
        p.close()
