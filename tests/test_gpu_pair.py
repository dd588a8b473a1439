"""GPU parity of the two-steps-through-L2 path (WAVE_KERNEL_PAIR,
csrc/stream.cuh PAIR blocks).

Its per-point arithmetic is the single-step kernels' (common.cuh), so a PAIR
run must equal the STREAM run bitwise (values compare equal; +0/-0 may differ)
for every geometry, source position and step count, and both are within the
1e-5 gate of the CPU oracle."""
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


def _plan(s, kernel):
    from paper_2009_04619_b200.wave import WavePlan
    return WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel)


def run(s, steps, kernel, u0=None, um1=None, chunks=None):
    p = _plan(s, kernel)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, max(steps, 1)))
    if u0 is not None or um1 is not None:
        p.set_state(um1, u0)
    spl = p.steps_per_launch
    for n in (chunks or [steps]):
        p.step(n)
    out = (p.read(0).cpu().numpy(), p.read(1).cpu().numpy())
    p.close()
    return out, spl


def rel_linf(got, ref):
    m = float(np.abs(ref).max())
    return float(np.abs(got.astype(np.float64) - ref).max()) / (m if m > 0 else 1.0)


CASES = [
    ("C1", {}),                                                     # 64^3, w = 16
    ("RAGGED", {}),                                                 # 70x45x53, w = 5, h = 7.5
    ("RAGGED", dict(nx=203, ny=150, nz=40, w=16, src=(101, 75, 20))),   # several tiles + ragged tails
    ("RAGGED", dict(w=0)),                                          # no PML
    ("RAGGED", dict(src=(6, 7, 9))),                                # source in both wall frames
    ("RAGGED", dict(src=(12, 30, 40))),                             # source in the (w+8) frame only
    ("RAGGED", dict(src=(35, 22, 5))),                              # source on the first inner plane
    ("C1", dict(h=(10.0, 7.5, 12.5), eta_max=30.0)),                # anisotropic spacing, strong PML
    ("C1", dict(nx=57, ny=33, nz=19, w=8, src=(28, 16, 10))),       # smallest supported xy, thin z
]


@pytest.mark.parametrize("name,kw", CASES)
@pytest.mark.parametrize("steps", [2, 9, 20])
def test_pair_equals_stream(name, kw, steps):
    s = synth.scenario(name, **kw)
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 41), synth.random_state(sh, 42)
    (a, ap), spl_a = run(s, steps, "stream", u0, um1)
    (b, bp), spl_b = run(s, steps, "pair", u0, um1)
    assert spl_a == 1 and spl_b == 2
    assert np.array_equal(a, b), np.abs(a - b).max()
    assert np.array_equal(ap, bp), np.abs(ap - bp).max()


def test_pair_point_source_vs_oracle():
    # BASELINE.json configs[0] through the two-step path, against the oracle
    s = synth.scenario("C1")
    (g, gp), spl = run(s, s.steps, "pair")
    assert spl == 2
    V = synth.velocity(s)
    geom = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    r, rp, st, _ = oracle.propagate(geom, V, synth.wavelet_for(s, s.steps), s.steps, s.source)
    assert st == 0
    assert rel_linf(g, r) <= TOL and rel_linf(gp, rp) <= TOL


@pytest.mark.parametrize("seed", [0, 1])
def test_pair_random_state_vs_oracle(seed):
    s = synth.scenario("C1")
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 2 * seed), synth.random_state(sh, 2 * seed + 1)
    (g, _), _ = run(s, 30, "pair", u0, um1)
    geom = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    r, _, st, _ = oracle.propagate(geom, synth.velocity(s), synth.wavelet_for(s, 30), 30, s.source,
                                   u0=u0, uprev0=um1)
    assert st == 0 and rel_linf(g, r) <= TOL


def test_pair_mixed_step_calls_bitwise():
    # odd step counts (pair + single step) and repeated calls walk the 4 buffers
    # through several (u^n, u^{n-1}) states and CUDA graphs
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 5), synth.random_state(sh, 6)
    (a, ap), _ = run(s, 23, "stream", u0, um1)
    (b, bp), _ = run(s, 23, "pair", u0, um1, chunks=[3, 1, 4, 2, 5, 6, 2])
    assert np.array_equal(a, b) and np.array_equal(ap, bp)


def test_pair_launch_accounting():
    s = synth.scenario("RAGGED")
    p = _plan(s, "pair")
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, 10))
    single = p.launches_per_step
    pair = p.launches(2)
    assert p.launches(7) == 3 * pair + single
    kms, kn = p.step_profiled(4)
    assert kn["interior"] == 2 and kms["interior"] > 0
    assert p.step_index == 4
    p.close()


@pytest.mark.parametrize("cz,pk", [(8, 3), (8, 8), (16, 1), (24, 5)])
@pytest.mark.parametrize("name,kw", [("RAGGED", {}), ("RAGGED", dict(nx=203, ny=150, nz=40, w=16, src=(101, 75, 20))),
                                     ("C1", dict(nx=57, ny=33, nz=19, w=8, src=(28, 16, 10)))])
def test_pair_z_chunks_and_publication_bitwise(monkeypatch, cz, pk, name, kw):
    # several z chunks per column (step-2 chunks shifted by 4 planes, per-chunk
    # progress counters) and publication every pk planes, incl. ragged last ones
    monkeypatch.setenv("WAVE25_PAIR_CZ", str(cz))
    monkeypatch.setenv("WAVE25_PAIR_PK", str(pk))
    s = synth.scenario(name, **kw)
    sh = (s.nz, s.ny, s.nx)
    u0, um1 = synth.random_state(sh, 43), synth.random_state(sh, 44)
    (a, ap), _ = run(s, 10, "stream", u0, um1)
    (b, bp), spl = run(s, 10, "pair", u0, um1)
    assert spl == 2 and np.array_equal(a, b) and np.array_equal(ap, bp)


@pytest.mark.parametrize("name,kw", [("C1", {}), ("RAGGED", {}), ("RAGGED", dict(src=(6, 7, 9)))])
def test_pair_fp64_equals_stream_fp64(name, kw):
    # the fp64 instantiation of the pair kernel (124-wide tiles, double2 lanes)
    from paper_2009_04619_b200.wave import WavePlan
    s = synth.scenario(name, **kw)
    sh = (s.nz, s.ny, s.nx)
    u0 = synth.random_state(sh, 45).astype(np.float64)
    outs = []
    for kernel in ("stream", "pair"):
        p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel, precision="fp64")
        p.set_velocity(synth.velocity(s))
        p.set_source(*s.source, synth.wavelet_for(s, 11))
        p.set_state(None, u0)
        p.step(11)
        outs.append((p.read(0).cpu().numpy(), p.read(1).cpu().numpy(), p.steps_per_launch))
        p.close()
    (a, ap, sa), (b, bp, sb) = outs
    assert sa == 1 and sb == 2 and a.dtype == np.float64
    assert np.array_equal(a, b) and np.array_equal(ap, bp)


def test_pair_with_stored_eta_falls_back_bitwise():
    # a stored eta field disables the pair path (single steps, same values)
    from paper_2009_04619_b200.wave import WavePlan
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    eta = np.full(sh, 1.5, np.float32)
    u0 = synth.random_state(sh, 46)
    outs = []
    for kernel in ("stream", "pair"):
        p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel)
        p.set_eta(eta)
        p.set_velocity(synth.velocity(s))
        p.set_source(*s.source, synth.wavelet_for(s, 9))
        p.set_state(None, u0)
        p.step(9)
        outs.append((p.read(0).cpu().numpy(), p.steps_per_launch))
        p.close()
    assert outs[1][1] == 1 and np.array_equal(outs[0][0], outs[1][0])


def test_pair_multislab_rejected():
    from paper_2009_04619_b200._abi import WaveError
    from paper_2009_04619_b200.wave import WavePlan
    s = synth.scenario("RAGGED")
    with pytest.raises(WaveError):
        WavePlan(s.nx, s.ny, 30, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=0, kernel="pair")
