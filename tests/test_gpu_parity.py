"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element on identical seeded inputs.  Gate (BASELINE.json north_star): fp32,
max |u_gpu - u_oracle| / max |u_oracle| <= 1e-5 after the configured steps.
Stream and naive kernels must agree bitwise; z-slab plans must agree bitwise
with the single-slab plan."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def WavePlan(*a, **k):
    from paper_2009_04619_b200.wave import WavePlan as WP
    return WP(*a, **k)


def rel_linf(got, ref):
    m = float(np.abs(ref).max())
    return float(np.abs(got.astype(np.float64) - ref).max()) / (m if m > 0 else 1.0)


def run_gpu(s, steps, u0=None, um1=None, kernel="stream", V=None, wl=None, precision="fp32"):
    V = synth.velocity(s) if V is None else V
    wl = synth.wavelet_for(s, max(steps, 1)) if wl is None else wl
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel, precision=precision)
    p.set_velocity(V)
    p.set_source(*s.source, wl)
    if u0 is not None or um1 is not None:
        p.set_state(um1, u0)
    p.step(steps)
    out = (p.read(0).cpu().numpy(), p.read(1).cpu().numpy())
    p.close()
    return out


def run_oracle(s, steps, u0=None, um1=None, V=None, wl=None):
    V = synth.velocity(s) if V is None else V
    wl = synth.wavelet_for(s, max(steps, 1)) if wl is None else wl
    g = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    u, up, st, _ = oracle.propagate(g, V, wl, steps, s.source, u0=u0, uprev0=um1)
    assert st == 0
    return u, up


@pytest.mark.parametrize("kernel", ["stream", "naive"])
def test_c1_point_source(kernel):
    # BASELINE.json configs[0]: 64^3, const V, Ricker, 10 steps
    s = synth.scenario("C1")
    g, gp = run_gpu(s, s.steps, kernel=kernel)
    r, rp = run_oracle(s, s.steps)
    assert rel_linf(g, r) <= TOL and rel_linf(gp, rp) <= TOL


def test_c2_full_run_vs_oracle():
    # BASELINE.json configs[1] exactly: 512^3, const V, PML, Ricker, all 500
    # steps, in the launch configuration bench.py times (stream kernels, CUDA
    # graphs) -- the whole field against the oracle (~30 s on 16 host cores)
    s = synth.scenario("C2")
    g, gp = run_gpu(s, s.steps)
    r, rp = run_oracle(s, s.steps)
    e, ep = rel_linf(g, r), rel_linf(gp, rp)
    print(f"C2 500 steps: rel Linf u^T {e:.3e}, u^(T-1) {ep:.3e}, max|u| {float(np.abs(r).max()):.4e}")
    assert float(np.abs(r).max()) > 0 and e <= TOL and ep <= TOL, (e, ep)


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("steps", [1, 10, 100])
def test_c1_random_state(seed, steps):
    # O(1) amplitude everywhere, incl. the PML (SURVEY.md §8(d) C1 extras)
    s = synth.scenario("C1")
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 2 * seed), synth.random_state(sh, 2 * seed + 1)
    g, _ = run_gpu(s, steps, u0, um1)
    r, _ = run_oracle(s, steps, u0, um1)
    assert rel_linf(g, r) <= TOL, rel_linf(g, r)


@pytest.mark.parametrize("name,steps", [("RAGGED", 40), ("SPEC48", 50)])
def test_ragged_and_spec_scenarios(name, steps):
    s = synth.scenario(name)
    sh = (s.nz, s.ny, s.nx)
    u0 = synth.random_state(sh, 3)
    g, gp = run_gpu(s, steps, u0)
    r, rp = run_oracle(s, steps, u0)
    assert rel_linf(g, r) <= TOL and rel_linf(gp, rp) <= TOL


@pytest.mark.parametrize("name,kw", [
    ("RAGGED", dict(w=0)),                               # no PML at all
    ("RAGGED", dict(nx=9, ny=11, nz=10, w=2, src=(4, 5, 5))),   # smaller than one tile
    ("RAGGED", dict(nx=37, ny=70, nz=12, w=3, src=(18, 35, 6))),  # nz < 2*9, thin slab
    ("RAGGED", dict(w=20, nx=70, ny=45, nz=53, src=(35, 22, 26))),  # w wider than a wall tile
    ("C1", dict(h=(10.0, 7.5, 12.5), eta_max=30.0)),      # anisotropic spacing, strong PML
])
def test_edge_geometries(name, kw):
    s = synth.scenario(name, **kw)
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 11), synth.random_state(sh, 12)
    g, _ = run_gpu(s, 7, u0, um1)
    r, _ = run_oracle(s, 7, u0, um1)
    assert rel_linf(g, r) <= TOL


@pytest.mark.parametrize("name", ["C1", "RAGGED"])
def test_stream_equals_naive_bitwise(name):
    s = synth.scenario(name)
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 21), synth.random_state(sh, 22)
    a, ap = run_gpu(s, 20, u0, um1, kernel="stream")
    b, bp = run_gpu(s, 20, u0, um1, kernel="naive")
    assert np.array_equal(a, b) and np.array_equal(ap, bp)


def test_mirror_symmetry_bitwise():
    n = 33
    s = synth.scenario("C1", nx=n, ny=n, nz=n, w=8, steps=60)
    g, _ = run_gpu(s, s.steps)
    assert np.abs(g).max() > 0
    for ax in range(3):
        assert np.array_equal(g, np.flip(g, axis=ax)), ax


def test_zero_and_one_step():
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 1), synth.random_state(sh, 2)
    g0, gp0 = run_gpu(s, 0, u0, um1)
    assert np.array_equal(g0, u0) and np.array_equal(gp0, um1)
    g1, gp1 = run_gpu(s, 1, u0, um1)
    r1, _ = run_oracle(s, 1, u0, um1)
    assert rel_linf(g1, r1) <= TOL and np.array_equal(gp1, u0)


def test_source_only_first_step_exact():
    # from the zero state one step leaves exactly fp32(vdt2[src] w[0]) at the source
    s = synth.scenario("RAGGED")
    wl = np.array([0.75], np.float32)
    g, _ = run_gpu(s, 1, wl=wl)
    r, _ = run_oracle(s, 1, wl=wl)
    assert np.array_equal(g, r)
    assert np.count_nonzero(g) == 1


def test_graph_replay_matches_stepwise():
    s = synth.scenario("C1")
    sh = (s.nz, s.ny, s.nx)
    u0 = synth.random_state(sh, 4)
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, 30))
    p.set_state(None, u0)
    p.step(13)                       # 6 graph pairs + 1
    a = p.read(0).cpu().numpy()
    p.set_state(None, u0)
    for _ in range(13):
        p.step(1)
    b = p.read(0).cpu().numpy()
    assert p.step_index == 13
    p.close()
    assert np.array_equal(a, b)


@pytest.mark.parametrize("nslab,precision", [(2, "fp32"), (3, "fp32"), (2, "fp64")])
def test_slabs_on_one_gpu_bitwise(nslab, precision):
    # z-slab plans + edges/interior split + device-to-device halo exchange == single plan
    from paper_2009_04619_b200.dist import slab_bounds
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 7), synth.random_state(sh, 8)
    if precision == "fp64":
        u0, um1 = u0.astype(np.float64), um1.astype(np.float64)
    V = synth.velocity(s)
    wl = synth.wavelet_for(s, 25)
    plans = []
    for r in range(nslab):
        off, nzl = slab_bounds(s.nz, r, nslab)
        p = WavePlan(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off,
                     precision=precision)
        p.set_velocity(V[off:off + nzl])
        p.set_source(*s.source, wl)
        p.set_state(um1[off:off + nzl], u0[off:off + nzl])
        plans.append((p, off, nzl))
    # initial halos: ghosts of u^0 come from the neighbours' edge planes
    for r, (p, off, nzl) in enumerate(plans):
        cur = p.field(0)
        full = torch.from_numpy(u0).cuda()
        buf = [b for b in p.bufs
               if b.data_ptr() <= cur.data_ptr() < b.data_ptr() + b.element_size() * b.numel()][0]
        plane = s.ny * p.layout.pitch_x
        v = buf[p.layout.origin:].view(-1, s.ny, p.layout.pitch_x)
        if r > 0:
            v[0:4, :, :s.nx] = full[off - 4:off]
        if r < nslab - 1:
            v[nzl + 4:nzl + 8, :, :s.nx] = full[off + nzl:off + nzl + 4]
    for n in range(25):
        for p, _, _ in plans:
            p.step_edges()
        for r, (p, off, nzl) in enumerate(plans):
            send_lo, send_hi, recv_lo, recv_hi = p.halo_views(0)
            if r > 0:
                plans[r - 1][0].halo_views(0)[3].copy_(send_lo)
            if r < nslab - 1:
                plans[r + 1][0].halo_views(0)[2].copy_(send_hi)
        for p, _, _ in plans:
            p.step_interior()
            p.step_finish()
    got = np.concatenate([p.read(0).cpu().numpy() for p, _, _ in plans], axis=0)
    ref, _ = run_gpu(s, 25, u0, um1, wl=wl, precision=precision)
    for p, _, _ in plans:
        p.close()
    assert np.array_equal(got, ref)


def test_unstable_eta_max_detected():
    from paper_2009_04619_b200 import WaveError
    from paper_2009_04619_b200._abi import WAVE_ERR_UNSTABLE
    s = synth.scenario("C1", nx=24, ny=24, nz=24, w=6, eta_max=100.0, src=(12, 12, 12))
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_velocity(synth.velocity(s))
    p.set_state(None, synth.random_state((24, 24, 24), 3))
    p.step(400)
    with pytest.raises(WaveError) as e:
        p.check_finite()
    assert e.value.status == WAVE_ERR_UNSTABLE
    p.close()


def test_courant_rejected():
    from paper_2009_04619_b200 import WaveError
    s = synth.scenario("C1", dt=5e-3)           # dt V / h = 1.0 > 0.4529
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    with pytest.raises(WaveError):
        p.set_velocity(synth.velocity(s))
    p.close()


def test_auto_dt_matches_oracle_rule():
    s = synth.scenario("SPEC48")
    V = synth.velocity(s)
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, 0.0, s.eta_max)
    p.set_velocity(V)
    assert np.float32(p.dt) == oracle.dt_auto(s.h, V)
    p.close()


def _full_size_slab_check(sname, steps, zt_list, seed=0, kernel="stream", **kw):
    """Full-size GPU run; oracle recomputes sampled z-slabs.  The oracle slab
    is the target planes plus 4*steps planes of margin on each side, whose
    ghost planes hold the initial state: after `steps` steps the target planes
    are exact (the contamination from stale ghosts moves 4 planes per step)."""
    s = synth.scenario(sname, **kw)
    sh = (s.nz, s.ny, s.nx)
    u0 = synth.random_state(sh, seed)
    um1 = synth.random_state(sh, seed + 1)
    V = synth.velocity(s)
    wl = synth.wavelet_for(s, steps)
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel)
    p.set_velocity(V)
    p.set_source(*s.source, wl)
    p.set_state(um1, u0)
    p.step(steps)
    assert kernel == "stream" or p.steps_per_launch == 2
    gpu = p.field(0)
    R = 4
    M = R * steps
    worst = 0.0
    for zt0, zt1 in zt_list:
        a, b = max(zt0 - M, 0), min(zt1 + M, s.nz)
        nzl = b - a
        g = oracle.make_geom(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=a)

        def padded(full):
            q = np.zeros((nzl + 8, s.ny + 8, s.nx + 8), np.float32)
            lo, hi = max(a - R, 0), min(b + R, s.nz)
            q[lo - (a - R):hi - (a - R), R:-R, R:-R] = full[lo:hi]
            return q
        uu, upp = padded(u0), padded(um1)
        vd = oracle.vdt2(V[a:b], s.dt)
        for n in range(steps):
            assert oracle.step_padded(g, uu, upp, vd, s.source, wl[n]) == 0
            uu, upp = upp, uu
        ref = uu[R + zt0 - a:R + zt1 - a, R:-R, R:-R]
        got = gpu[zt0:zt1].cpu().numpy()
        worst = max(worst, rel_linf(got, ref))
    p.close()
    return worst


@pytest.mark.parametrize("kernel", ["stream", "pair", "tb2"])
def test_beyond_2g_elements_sampled_slabs(kernel):
    # 2048 x 2048 x 520 (2.18e9 points per buffer > 2^31): every index and
    # offset on the path must be 64-bit; sampled slabs incl. both z caps
    err = _full_size_slab_check("C2", 4, [(0, 12), (254, 266), (508, 520)], seed=5, kernel=kernel,
                                nx=2048, ny=2048, nz=520)
    assert err <= TOL, err


@pytest.mark.parametrize("sname,kernel", [("C2", "stream"), ("C3", "stream"), ("C2", "tb2"), ("C3", "tb2"),
                                          ("C2", "pair"), ("C3", "pair")])
def test_full_size_sampled_slabs(sname, kernel):
    # BASELINE.json configs[1] / configs[2] at full size, the bench's launch
    # configuration (stream kernels, CUDA graphs); sampled z ranges cover the
    # top cap, the middle (source plane) and the bottom cap.
    s = synth.scenario(sname)
    n = s.nz
    zt = [(0, 6), (n // 2 - 3, n // 2 + 3), (n - 6, n)]
    err = _full_size_slab_check(sname, 5 if kernel == "stream" else 6, zt, kernel=kernel)
    assert err <= TOL, err


def _slab_worker(rank, world, port, steps, q):
    import os
    import torch.distributed as dist
    from paper_2009_04619_b200.dist import SlabRunner, slab_bounds
    from paper_2009_04619_b200.wave import WavePlan as WP
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        s = synth.scenario("RAGGED")
        sh = (s.nz, s.ny, s.nx)
        u0, um1 = synth.random_state(sh, 31), synth.random_state(sh, 32)
        off, nzl = slab_bounds(s.nz, rank, world)
        p = WP(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
        p.set_velocity(synth.velocity(s)[off:off + nzl])
        p.set_source(*s.source, synth.wavelet_for(s, steps))
        p.set_state(um1[off:off + nzl], u0[off:off + nzl])
        runner = SlabRunner(p, rank, world, stage_on_host=True)
        runner.exchange_current()
        runner.step(steps)
        torch.cuda.synchronize()
        q.put((rank, p.read(0).cpu().numpy()))
        p.close()
    finally:
        dist.destroy_process_group()


def test_slab_runner_two_processes_bitwise():
    # the multi-process driver (SlabRunner: edges -> halo exchange || interior)
    # with 2 ranks on one GPU over gloo == the single-plan run, bitwise
    import socket
    import torch.multiprocessing as mp
    steps = 17
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, steps, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    parts = sorted(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    got = np.concatenate([a for _, a in parts], axis=0)
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    ref, _ = run_gpu(s, steps, synth.random_state(sh, 31), synth.random_state(sh, 32),
                     wl=synth.wavelet_for(s, steps))
    assert np.array_equal(got, ref)


VARIANT_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, synth
from paper_2009_04619_b200.wave import WavePlan
for name in ("RAGGED", "C1"):
    s = synth.scenario(name)
    sh = (s.nz, s.ny, s.nx)
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, 12))
    p.set_state(synth.random_state(sh, 41), synth.random_state(sh, 42))
    p.step(12)
    print(name, hashlib.sha256(p.read(0).cpu().numpy().tobytes()).hexdigest())
    p.close()
"""


@pytest.mark.parametrize("env", [
    {"WAVE25_INNER_TILE": "128x16x1"}, {"WAVE25_INNER_TILE": "64x16x1"},
    {"WAVE25_INNER_TILE": "128x8x1"}, {"WAVE25_INNER_TILE": "248x8x1"}, {"WAVE25_INNER_TILE": "224x8x1"},
    {"WAVE25_INNER_TILE": "248x8x2"}, {"WAVE25_INNER_TILE": "248x8x2r"}, {"WAVE25_INNER_TILE": "256x8x1r"},
    {"WAVE25_INNER_TILE": "248x8x1rc2"}, {"WAVE25_INNER_TILE": "248x8x1rc4"},
    {"WAVE25_INNER_TILE": "248x8x1r"}, {"WAVE25_INNER_TILE": "240x8x1r"}, {"WAVE25_INNER_TILE": "248x8x1r104"}, {"WAVE25_INNER_TILE": "128x8x1r2"}, {"WAVE25_INNER_TILE": "c124x8x1r2"},
    {"WAVE25_WALLX_TILE": "x24c16x64x1r2"}, {"WAVE25_WALLY_TILE": "y128x8x1r2"}, {"WAVE25_WALLY_TILE": "y248x8x1ry"},
    {"WAVE25_WALLS_ALT": "1", "WAVE25_WALL_STKEEP": "1"},
    {"WAVE25_FASTDIV": "0"}, {"WAVE25_NO_ORIGIN": "1"}, {"WAVE25_XINTER": "0"},
    {"WAVE25_WALLX_TILE": "x24c16x128x1rg"}, {"WAVE25_WALLY_TILE": "y128x16x1rg"},
    {"WAVE25_SEAM": "1"}, {"WAVE25_SEAM": "1", "WAVE25_NO_SEAM": "1"},
    {"WAVE25_SEAM": "1", "WAVE25_SEAM_TILE": "seam32x32"},
    {"WAVE25_FUSED": "1", "WAVE25_FUSED_TILE": "fused128x8x1"},
    {"WAVE25_ABLATION": "gmem_32x4x1"}, {"WAVE25_ABLATION": "gmem_8x8x8"}, {"WAVE25_ABLATION": "smem_u"},
    {"WAVE25_ABLATION": "st_smem_32x16"}, {"WAVE25_ABLATION": "st_reg_shft_32x16"},
    {"WAVE25_ABLATION": "st_reg_fixed_32x16"}, {"WAVE25_ABLATION": "st_reg_fixed_32x32"},
    {"WAVE25_WALLX_TILE": "x32c16x32x1"}, {"WAVE25_WALLX_TILE": "x24c16x64x1"},
    {"WAVE25_WALLX_TILE": "x24c16x32x1"}, {"WAVE25_WALLX_TILE": "x24c16x64x1r"},
    {"WAVE25_WALLY_TILE": "y128x8x1"}, {"WAVE25_WALLY_TILE": "y128x16x1"},
    {"WAVE25_WALLY_TILE": "y64x8x1m3"}, {"WAVE25_XFUSE": "1"},
    {"WAVE25_FUSED": "1"}, {"WAVE25_FORK": "0", "WAVE25_PF": "0"}, {"WAVE25_CZ": "7"},
    {"WAVE25_ORDER": "-3"}, {"WAVE25_ORDER": "2"}, {"WAVE25_MIX": "1"}, {"WAVE25_MIX": "2"}, {"WAVE25_SIDE2": "0"}, {"WAVE25_WALL_CZ": "114"},
    # embedded wall warps: default pacing, 1-plane units, every
    # unit claimed at once, every unit left to the last wave's mop-up
    {"WAVE25_EW": "1"}, {"WAVE25_EW": "1", "WAVE25_EW_CZ": "1"}, {"WAVE25_EW": "1", "WAVE25_EW_CZ": "5"},
    {"WAVE25_EW": "1", "WAVE25_EW_REM": "0"}, {"WAVE25_EW": "1", "WAVE25_EW_REM": "1000000"},
], ids=lambda e: ",".join(f"{k[7:]}={v}" for k, v in e.items()))
def test_kernel_variants_bitwise(env):
    # (WAVE25_FASTDIV=0: IEEE divisions instead of the verified table
    # reciprocal -- bitwise the same by the setup check, R9)
    # every tile / scheduling variant used in the DESIGN.md ablations computes
    # the same values as the default configuration, bitwise
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    base = {k: v for k, v in os.environ.items() if not k.startswith("WAVE25_")}
    ref = subprocess.run([sys.executable, "-c", VARIANT_SCRIPT, root], env=base, capture_output=True,
                         text=True, check=True).stdout
    got = subprocess.run([sys.executable, "-c", VARIANT_SCRIPT, root], env={**base, **env},
                         capture_output=True, text=True, check=True).stdout
    assert ref.count("\n") == 2 and got == ref


@pytest.mark.parametrize("nslab", [2, 3])
def test_peer_store_slabs_one_process_bitwise(nslab):
    # fused halo exchange: edge planes stored straight into the neighbours'
    # ghost planes by the stencil kernels, device-side step flags; each slab
    # stepped on its own stream == the single-plan run, bitwise
    from paper_2009_04619_b200.dist import slab_bounds
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 51), synth.random_state(sh, 52)
    V = synth.velocity(s)
    steps = 23
    wl = synth.wavelet_for(s, steps)
    plans = []
    for r in range(nslab):
        off, nzl = slab_bounds(s.nz, r, nslab)
        p = WavePlan(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
        p.set_velocity(V[off:off + nzl])
        p.set_source(*s.source, wl)
        p.set_state(um1[off:off + nzl], u0[off:off + nzl])
        p.flags = torch.zeros(2, dtype=torch.int64, device="cuda")
        plans.append(p)
    for r, p in enumerate(plans):
        lo = plans[r - 1] if r > 0 else None
        hi = plans[r + 1] if r < nslab - 1 else None
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
    ref, _ = run_gpu(s, steps, u0, um1, wl=wl)
    for p in plans:
        p.close()
    assert np.array_equal(got, ref)


def _peer_worker(rank, world, port, steps, q):
    import os
    import torch.distributed as dist
    from paper_2009_04619_b200.dist import PeerSlabRunner, slab_bounds
    from paper_2009_04619_b200.wave import WavePlan as WP
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        s = synth.scenario("RAGGED")
        sh = (s.nz, s.ny, s.nx)
        u0, um1 = synth.random_state(sh, 61), synth.random_state(sh, 62)
        off, nzl = slab_bounds(s.nz, rank, world)
        p = WP(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
        p.set_velocity(synth.velocity(s)[off:off + nzl])
        p.set_source(*s.source, synth.wavelet_for(s, steps))
        p.set_state(um1[off:off + nzl], u0[off:off + nzl])
        runner = PeerSlabRunner(p, rank, world)
        runner.exchange_current()
        runner.step(steps)
        torch.cuda.synchronize()
        q.put((rank, p.read(0).cpu().numpy()))
        runner.close()            # collective: keeps buffers mapped until every rank is done
        p.close()
    finally:
        dist.destroy_process_group()


def _peer_fail_worker(rank, world, port, q):
    # rank 1 cannot wire its peers: both ranks must get the error (no hang),
    # unwire, and the NCCL-path SlabRunner (gloo here) still gives the right field
    import os
    import torch.distributed as dist
    from paper_2009_04619_b200.dist import PeerSlabRunner, SlabRunner, slab_bounds
    from paper_2009_04619_b200.wave import WavePlan as WP
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        s = synth.scenario("RAGGED")
        off, nzl = slab_bounds(s.nz, rank, world)
        p = WP(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
        p.set_velocity(synth.velocity(s)[off:off + nzl])
        p.set_source(*s.source, synth.wavelet_for(s, 7))
        if rank == 1:
            def boom(*a, **k):
                raise RuntimeError("simulated: no P2P path")
            p.set_peers = boom
        raised = False
        try:
            PeerSlabRunner(p, rank, world)
        except RuntimeError:
            raised = True
        runner = SlabRunner(p, rank, world, stage_on_host=True)
        runner.step(7)
        torch.cuda.synchronize()
        q.put((rank, raised, p.read(0).cpu().numpy()))
        dist.barrier()
        p.close()
    finally:
        dist.destroy_process_group()


def test_peer_wiring_failure_is_collective():
    import socket
    import torch.multiprocessing as mp
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    parts = sorted((q.get(timeout=300) for _ in range(2)), key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert all(raised for _, raised, _ in parts)
    got = np.concatenate([a for _, _, a in parts], axis=0)
    s = synth.scenario("RAGGED")
    ref, _ = run_gpu(s, 7, wl=synth.wavelet_for(s, 7))
    assert np.array_equal(got, ref)


def test_peer_slab_runner_two_processes_bitwise():
    # the production multi-GPU path (IPC-mapped neighbour buffers, peer stores,
    # device flags) with 2 processes sharing one GPU == the single-plan run
    import socket
    import torch.multiprocessing as mp
    steps = 19
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, steps, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    parts = sorted(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    got = np.concatenate([a for _, a in parts], axis=0)
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    ref, _ = run_gpu(s, steps, synth.random_state(sh, 61), synth.random_state(sh, 62),
                     wl=synth.wavelet_for(s, steps))
    assert np.array_equal(got, ref)


RACE_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, sys.argv[1])
import synth
from paper_2009_04619_b200.wave import WavePlan
s = synth.scenario("RAGGED")
sh = (s.nz, s.ny, s.nx)
for t in range(int(sys.argv[2])):
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, 12))
    p.set_state(synth.random_state(sh, 41), synth.random_state(sh, 42))
    for n in range(12):
        p.step(1)
    print(hashlib.sha256(p.read(0).cpu().numpy().tobytes()).hexdigest())
    p.close()
"""


def test_concurrent_walls_repeatable():
    # Regression test for a cross-proxy WAR hazard: consumer warps read a ring
    # stage with generic loads, release it, and the producer's TMA (async
    # proxy) refilled it -- without fence.proxy.async the overwrite could land
    # before slow loads completed.  It showed (~4 % of runs) when the x-wall
    # kernel shared SMs with many short interior blocks (the gmem ablation
    # shape) and steps were enqueued back to back.  30 such runs must all equal
    # the serial (one-stream) reference.
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    base = {k: v for k, v in os.environ.items() if not k.startswith("WAVE25_")}
    ref = subprocess.run([sys.executable, "-c", RACE_SCRIPT, root, "1"], env={**base, "WAVE25_SERIAL": "1"},
                         capture_output=True, text=True, check=True).stdout.split()
    got = subprocess.run([sys.executable, "-c", RACE_SCRIPT, root, "30"],
                         env={**base, "WAVE25_ABLATION": "gmem_8x8x8"}, capture_output=True, text=True,
                         check=True).stdout.split()
    assert len(got) == 30 and set(got) == set(ref), (len(set(got)), got.count(ref[0]))


SEMI_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import synth, oracle
from paper_2009_04619_b200.wave import WavePlan
worst = 0.0
for name in ("RAGGED", "C1"):
    s = synth.scenario(name)
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 41), synth.random_state(sh, 42)
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, 12))
    p.set_state(um1, u0)
    p.step(12)
    got = p.read(0).cpu().numpy()
    p.close()
    g = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    ref, _, st, _ = oracle.propagate(g, synth.velocity(s), synth.wavelet_for(s, 12), 12, s.source, u0=u0, uprev0=um1)
    worst = max(worst, float(np.abs(got - ref).max() / np.abs(ref).max()))
print(worst)
"""


def test_semi_stencil_shape_within_gate():
    # the paper's semi-stencil shape sums the z pairs in
    # forward/backward halves: a different fp32 order, so it is held to the
    # 1e-5 oracle gate instead of bitwise equality
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    base = {k: v for k, v in os.environ.items() if not k.startswith("WAVE25_")}
    out = subprocess.run([sys.executable, "-c", SEMI_SCRIPT, root], env={**base, "WAVE25_ABLATION": "semi_32x16"},
                         capture_output=True, text=True, check=True).stdout
    assert float(out.split()[-1]) <= TOL, out


def test_ipc_export_offsets():
    # wave_ipc_export: handle of the whole allocation + the byte offset of an
    # interior pointer (what PeerSlabRunner ships to the neighbours)
    from paper_2009_04619_b200 import _abi
    t = torch.zeros(1 << 20, dtype=torch.float32, device="cuda")
    h0, o0 = _abi.wave_ipc_export(t.data_ptr())
    h1, o1 = _abi.wave_ipc_export(t[1000:].data_ptr())
    assert len(h0) == 64 and h0 == h1 and o1 - o0 == 4000


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_mirror_symmetry_bitwise_full_size(precision):
    # odd extents (511^3), centred source, constant V, a mirror-symmetric O(1)
    # initial state that loads every PML wall from step 1: the field stays
    # bitwise mirror-symmetric along every axis (pair sums before multiplying,
    # the eta star's two differences flip sign together).  Catches an
    # off-by-one in a wall region, a one-sided tile edge or halo, or an
    # asymmetric z cap, on the full-size launch configuration.
    n, h = 511, 256
    s = synth.scenario("C2", nx=n, ny=n, nz=n, src=(n // 2, n // 2, n // 2))
    rng = np.random.Generator(np.random.PCG64(91))
    q = rng.uniform(-1, 1, size=(h, h, h))
    for ax in range(3):
        q = np.concatenate([q, np.flip(q, axis=ax).take(range(1, h), axis=ax)], axis=ax)
    dtype = np.float64 if precision == "fp64" else np.float32
    u0 = q.astype(dtype)
    assert all(np.array_equal(u0, np.flip(u0, axis=ax)) for ax in range(3))
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, precision=precision)
    p.set_velocity(np.full((n, n, n), 2000.0, np.float32))
    p.set_source(*s.source, synth.wavelet_for(s, 30))
    p.set_state(u0, u0)
    p.step(30)
    u = p.read(0).cpu().numpy()
    p.close()
    assert np.isfinite(u).all() and np.abs(u).max() > 0
    for ax in range(3):
        assert np.array_equal(u, np.flip(u, axis=ax)), ax


@pytest.mark.parametrize("name", ["C1", "RAGGED", "SPEC48"])
def test_table_division_verified_and_used(name):
    # the plan's exhaustive device check (k_divcheck over every fp32
    # significand, R9) accepted the Markstein table division for the
    # fp32 configurations, and fp64 plans keep the IEEE division
    s = synth.scenario(name)
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_velocity(synth.velocity(s))
    assert p.fastdiv
    p.close()
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, precision="fp64")
    p.set_velocity(synth.velocity(s))
    assert not p.fastdiv
    p.close()
