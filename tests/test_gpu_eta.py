"""GPU parity of the stored (user-supplied) eta path (SURVEY.md §8(f) rank 3,
DESIGN.md §5f, reading R16) against the oracle's stored-eta variant
(oracle.propagate(..., eta=...)), fp32 gate 1e-5, fp64 gate 1e-12; stream
and naive kernels bitwise equal."""
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


def eta_field(s, seed, scale=4.0):
    """A user-style damping field: the smooth (d/w)^2 ramp times a random
    per-point factor in [0.5, 1.5], plus random values inside (ignored there)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    def d1(n):
        i = np.arange(n)
        return np.maximum(np.maximum(s.w - i, 0), i - (n - s.w - 1))
    d = np.maximum(np.maximum(d1(s.nx)[None, None, :], d1(s.ny)[None, :, None]), d1(s.nz)[:, None, None])
    ramp = (d / max(s.w, 1)) ** 2
    f = scale * ramp * rng.uniform(0.5, 1.5, size=d.shape) + (d == 0) * rng.uniform(0, 1, size=d.shape)
    return f.astype(np.float32)


def run_gpu(s, steps, eta, u0=None, um1=None, kernel="stream", precision="fp32"):
    from paper_2009_04619_b200.wave import WavePlan
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel, precision=precision)
    if eta is not None:
        p.set_eta(eta)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, max(steps, 1)))
    if u0 is not None or um1 is not None:
        p.set_state(um1, u0)
    p.step(steps)
    out = (p.read(0).cpu().numpy(), p.read(1).cpu().numpy(), p.steps_per_launch)
    p.close()
    return out


def run_oracle(s, steps, eta, u0=None, um1=None, dtype=np.float32, round32=True):
    g = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    u, up, st, _ = oracle.propagate(g, synth.velocity(s), synth.wavelet_for(s, max(steps, 1)), steps, s.source,
                                    u0=u0, uprev0=um1, dtype=dtype, round32=round32, eta=eta)
    assert st == 0
    return u, up


def rel_linf(got, ref):
    m = float(np.abs(ref).max())
    return float(np.abs(got.astype(np.float64) - ref).max()) / (m if m > 0 else 1.0)


CASES = [("C1", {}, 20), ("RAGGED", {}, 15), ("RAGGED", dict(w=2, nx=23, ny=19, nz=21, src=(11, 9, 10)), 9),
         ("C1", dict(h=(10.0, 7.5, 12.5)), 12)]


@pytest.mark.parametrize("name,kw,steps", CASES)
def test_stored_eta_vs_oracle(name, kw, steps):
    s = synth.scenario(name, **kw)
    sh = (s.nz, s.ny, s.nx)
    eta = eta_field(s, 3)
    u0, um1 = synth.random_state(sh, 31), synth.random_state(sh, 32)
    g, gp, _ = run_gpu(s, steps, eta, u0, um1)
    r, rp = run_oracle(s, steps, eta, u0, um1)
    assert rel_linf(g, r) <= TOL and rel_linf(gp, rp) <= TOL, (rel_linf(g, r), rel_linf(gp, rp))
    # the field matters: the profile path gives a different answer
    g0, _, _ = run_gpu(s, steps, None, u0, um1)
    assert rel_linf(g0, r) > 10 * TOL


@pytest.mark.parametrize("name", ["C1", "RAGGED"])
def test_stored_eta_stream_equals_naive_bitwise(name):
    s = synth.scenario(name)
    sh = (s.nz, s.ny, s.nx)
    eta = eta_field(s, 4)
    u0 = synth.random_state(sh, 33)
    a, ap, _ = run_gpu(s, 14, eta, u0, kernel="stream")
    b, bp, _ = run_gpu(s, 14, eta, u0, kernel="naive")
    assert np.array_equal(a, b) and np.array_equal(ap, bp)


def test_stored_eta_fp64_vs_oracle():
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    eta = eta_field(s, 5)
    u0 = synth.random_state(sh, 34).astype(np.float64)
    g, _, _ = run_gpu(s, 10, eta, u0, precision="fp64")
    r, _ = run_oracle(s, 10, eta, u0, dtype=np.float64, round32=False)
    assert rel_linf(g, r) <= 1e-12, rel_linf(g, r)


def test_stored_eta_reset_to_profile_bitwise():
    from paper_2009_04619_b200.wave import WavePlan
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    u0 = synth.random_state(sh, 35)
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, 8))
    p.set_eta(eta_field(s, 6))
    p.set_eta(None)
    p.set_state(None, u0)
    p.step(8)
    a = p.read(0).cpu().numpy()
    p.close()
    b, _, _ = run_gpu(s, 8, None, u0)
    assert np.array_equal(a, b)


def test_stored_eta_rejects_negative():
    from paper_2009_04619_b200._abi import WaveError
    from paper_2009_04619_b200.wave import WavePlan
    s = synth.scenario("RAGGED")
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    eta = eta_field(s, 7)
    eta[3, 4, 5] = -1.0
    with pytest.raises(WaveError):
        p.set_eta(eta)
    p.close()


def test_stored_eta_tb2_falls_back_bitwise():
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    eta = eta_field(s, 8)
    u0 = synth.random_state(sh, 36)
    a, _, spl_a = run_gpu(s, 10, eta, u0, kernel="stream")
    b, _, spl_b = run_gpu(s, 10, eta, u0, kernel="tb2")
    assert spl_b == 1 and np.array_equal(a, b)


ETA_VARIANT_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import numpy as np, synth
from test_gpu_eta import eta_field
from paper_2009_04619_b200.wave import WavePlan
for name in ("RAGGED", "C1"):
    s = synth.scenario(name)
    sh = (s.nz, s.ny, s.nx)
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_eta(eta_field(s, 5))
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, 9))
    p.set_state(synth.random_state(sh, 43), synth.random_state(sh, 44))
    p.step(9)
    print(name, hashlib.sha256(p.read(0).cpu().numpy().tobytes()).hexdigest())
    p.close()
"""


@pytest.mark.parametrize("env", [{"WAVE25_EWALLX_TILE": "ex24c16x32x1"}, {"WAVE25_EWALLY_TILE": "ey64x8x1m3"},
                                 {"WAVE25_EWALLY_TILE": "ey128x8x1r"}],
                         ids=lambda e: ",".join(f"{k[7:]}={v}" for k, v in e.items()))
def test_eta_wall_variants_bitwise(env):
    # the stored-eta wall tile variants compute bitwise the default's values
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    base = {k: v for k, v in os.environ.items() if not k.startswith("WAVE25_")}
    ref = subprocess.run([sys.executable, "-c", ETA_VARIANT_SCRIPT, root], env=base, capture_output=True, text=True,
                         check=True).stdout
    got = subprocess.run([sys.executable, "-c", ETA_VARIANT_SCRIPT, root], env={**base, **env}, capture_output=True,
                         text=True, check=True).stdout
    assert ref.count("\n") == 2 and got == ref
