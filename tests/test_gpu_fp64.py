"""GPU parity of the fp64 path (WAVE_PREC_FP64, SPEC.md
L82 verification precision) against the fp64 CPU oracle with unrounded fp64
constants (oracle round32 = False).  Gate: max|Δ| / max|u_oracle| <= 1e-12
(the two sides differ only by FMA contraction: ~1 ulp per operation, measured
well below the gate); stream and naive fp64 kernels must agree bitwise."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL64 = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _plan(s, kernel="stream", precision="fp64"):
    from paper_2009_04619_b200.wave import WavePlan
    return WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel, precision=precision)


def run_gpu(s, steps, u0=None, um1=None, kernel="stream", precision="fp64"):
    p = _plan(s, kernel, precision)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, max(steps, 1)))
    if u0 is not None or um1 is not None:
        p.set_state(um1, u0)
    p.step(steps)
    out = (p.read(0).cpu().numpy(), p.read(1).cpu().numpy())
    p.close()
    return out


def run_oracle64(s, steps, u0=None, um1=None):
    g = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    u, up, st, _ = oracle.propagate(g, synth.velocity(s), synth.wavelet_for(s, max(steps, 1)), steps, s.source,
                                    u0=u0, uprev0=um1, dtype=np.float64, round32=False)
    assert st == 0
    return u, up


def rel_linf(got, ref):
    m = float(np.abs(ref).max())
    return float(np.abs(got - ref).max()) / (m if m > 0 else 1.0)


def test_fp64_point_source_c1():
    s = synth.scenario("C1")
    g, gp = run_gpu(s, s.steps)
    assert g.dtype == np.float64
    r, rp = run_oracle64(s, s.steps)
    assert rel_linf(g, r) <= TOL64 and rel_linf(gp, rp) <= TOL64, (rel_linf(g, r), rel_linf(gp, rp))


@pytest.mark.parametrize("name,kw,steps", [
    ("C1", {}, 30),
    ("RAGGED", {}, 25),
    ("RAGGED", dict(w=0), 9),
    ("RAGGED", dict(nx=9, ny=11, nz=10, w=2, src=(4, 5, 5)), 7),
    ("RAGGED", dict(w=20, nx=70, ny=45, nz=53, src=(35, 22, 26)), 7),
    ("C1", dict(h=(10.0, 7.5, 12.5), eta_max=30.0), 12),
    ("RAGGED", dict(nx=203, ny=150, nz=40, w=16, src=(101, 75, 20)), 6),
])
def test_fp64_random_state(name, kw, steps):
    s = synth.scenario(name, **kw)
    sh = (s.nz, s.ny, s.nx)
    u0 = synth.random_state(sh, 51).astype(np.float64)
    um1 = synth.random_state(sh, 52).astype(np.float64)
    g, _ = run_gpu(s, steps, u0, um1)
    r, _ = run_oracle64(s, steps, u0, um1)
    assert rel_linf(g, r) <= TOL64, rel_linf(g, r)


@pytest.mark.parametrize("name", ["C1", "RAGGED"])
def test_fp64_stream_equals_naive_bitwise(name):
    s = synth.scenario(name)
    sh = (s.nz, s.ny, s.nx)
    u0 = synth.random_state(sh, 61).astype(np.float64)
    a, ap = run_gpu(s, 14, u0, None, kernel="stream")
    b, bp = run_gpu(s, 14, u0, None, kernel="naive")
    assert np.array_equal(a, b) and np.array_equal(ap, bp)


def test_fp64_differs_from_fp32_by_fp32_rounding_only():
    # same scheme in two precisions: O(1e-6) apart after a few steps, never more
    s = synth.scenario("C1")
    sh = (s.nz, s.ny, s.nx)
    u0 = synth.random_state(sh, 71)
    g64, _ = run_gpu(s, 10, u0.astype(np.float64))
    g32, _ = run_gpu(s, 10, u0, precision="fp32")
    d = rel_linf(g32.astype(np.float64), g64)
    assert 0 < d < 1e-5, d


def test_fp64_source_first_step_exact():
    # from the zero state one step leaves exactly (V dt)^2 w[0] (fp64) at the source
    s = synth.scenario("RAGGED")
    wl = np.array([0.75], np.float32)
    p = _plan(s)
    V = synth.velocity(s)
    p.set_velocity(V)
    p.set_source(*s.source, wl)
    p.step(1)
    u = p.read(0).cpu().numpy()
    i, j, k = s.source
    vdt = float(V[k, j, i]) * float(np.float32(s.dt))
    assert u[k, j, i] == vdt * vdt * 0.75
    u[k, j, i] = 0
    assert not u.any()
    p.close()


def test_fp64_tb2_rejected():
    from paper_2009_04619_b200._abi import WaveError
    s = synth.scenario("C1")
    with pytest.raises(WaveError):
        _plan(s, kernel="tb2")


def test_fp64_full_size_c2_sampled():
    # BASELINE.json configs[1] (512^3) in fp64 through the production kernels:
    # 4 steps from a random state, compared on a z-slab of the oracle (the
    # slab's 4-plane halos of the full-grid state make it exact for 1 step per
    # halo plane; 4 steps need 16 extra planes each side)
    s = synth.scenario("C2")
    steps, z0, z1 = 4, 250, 262
    sh = (s.nz, s.ny, s.nx)
    rng = np.random.Generator(np.random.PCG64(81))
    u0 = rng.uniform(-1, 1, size=sh)
    p = _plan(s)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, steps))
    p.set_state(None, u0)
    p.step(steps)
    got = p.read(0)[z0:z1].cpu().numpy()
    p.close()
    a, b = z0 - 4 * steps, z1 + 4 * steps
    g = oracle.make_geom(s.nx, s.ny, b - a, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=a)
    V = synth.velocity(s)[a:b]
    vd = oracle.vdt2(V, s.dt, round32=False, dtype=np.float64)
    uu = oracle.pad(u0[a - 4:b + 4][4:-4], np.float64)
    uu[:4, 4:-4, 4:-4] = u0[a - 4:a]
    uu[-4:, 4:-4, 4:-4] = u0[b:b + 4]
    up = np.zeros_like(uu)
    wl = synth.wavelet_for(s, steps)
    for n in range(steps):
        assert oracle.step_padded(g, uu, up, vd, s.source, float(wl[n]), round32=False) == 0
        uu, up = up, uu
        # the slab's own z halos are stale after a step; the sampled planes stay
        # exact because they are >= 4*(steps-n) planes from the slab ends
    ref = uu[4 + z0 - a:4 + z1 - a, 4:-4, 4:-4]
    assert rel_linf(got, ref) <= TOL64


@pytest.mark.parametrize("n,precision,tol", [(512, "fp64", 1e-11), (512, "fp32", 2e-5), (1024, "fp32", 2e-5)])
def test_plane_wave_closed_form_full_size(n, precision, tol):
    # The scheme's own discrete plane wave: with
    # u^0 = cos(k.x), u^-1 = cos(k.x + w dt) and w from the dispersion relation
    # 4 sin^2(w dt/2)/dt^2 = V^2 sum_a -(w0 + 2 sum_m w_m cos(m k_a h))/h^2, the
    # exact solution is u^s = cos(k.x - w s dt) on cells >= 4s from the zero
    # fringe.  At the C2 and C3 sizes (512^3 / 1024^3, no PML) through the
    # production kernels -- pins at full size that need no oracle run
    # (measured: fp64 2.0e-13, fp32 2.2e-6 at 512^3).
    import math
    h, V, T = 10.0, 2000.0, 24
    dt = float(np.float32(2e-3))
    wts = [-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0]
    k = [2 * math.pi / (8 * h), 2 * math.pi / (13 * h), 2 * math.pi / (21 * h)]
    S = sum(-(wts[0] + 2 * sum(wts[m] * math.cos(m * ka * h) for m in range(1, 5))) / h ** 2 for ka in k)
    omega = 2 / dt * math.asin(math.sqrt(V * V * dt * dt * S / 4))
    x = np.arange(n) * h
    ph = k[0] * x[None, None, :] + k[1] * x[None, :, None] + k[2] * x[:, None, None]
    dtype = np.float64 if precision == "fp64" else np.float32
    s = synth.scenario("C2").with_(nx=n, ny=n, nz=n, w=0)   # h = 10 m, dt = 2 ms as above
    p = _plan(s, precision=precision)
    p.set_velocity(np.full((n, n, n), V, np.float32))
    p.set_source(n // 2, n // 2, n // 2, np.zeros(1, np.float32))
    p.set_state(np.cos(ph + omega * dt).astype(dtype), np.cos(ph).astype(dtype))
    p.step(T)
    got = p.read(0).cpu().numpy()
    p.close()
    c = slice(4 * T, n - 4 * T)
    err = float(np.abs(got[c, c, c] - np.cos(ph[c, c, c] - omega * T * dt)).max())
    print(f"plane wave {precision} {n}^3 x {T} steps: max |u - exact| = {err:.3e}")
    assert err <= tol, err


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_linear_ramp_pml_closed_form_full_size(precision):
    # u = u_prev = C + a x + b y + c z: Lap u = 0 and grad u = (a, b, c) exactly,
    # so one step gives u + vdt2 (a d_x eta + b d_y eta + c d_z eta) / (1 + eta dt)
    # in the PML and u inside (the oracle's own pin, here on
    # the C2 grid with anisotropic spacing through the production wall kernels
    # and z caps, no oracle run).  Pins the grad-eta.grad-u term per axis,
    # A = 1 - eta dt, B = 1 + eta dt, the eta profile and the Chebyshev distance.
    n, w = 512, 16
    hx, hy, hz = 10.0, 7.5, 12.5
    s = synth.scenario("C2").with_(h=(hx, hy, hz), eta_max=50.0)   # strong PML: a large correction
    dt, eta_max, V = float(np.float32(s.dt)), s.eta_max, 2000.0
    C, a, b, c = 0.7, 0.037, -0.021, 0.029
    X = (np.arange(n)[None, None, :] - n / 2) * hx
    Y = (np.arange(n)[None, :, None] - n / 2) * hy
    Z = (np.arange(n)[:, None, None] - n / 2) * hz
    dtype = np.float64 if precision == "fp64" else np.float32
    u = (C + a * X + b * Y + c * Z).astype(dtype)
    p = _plan(s, precision=precision)
    p.set_velocity(np.full((n, n, n), V, np.float32))
    p.set_source(n // 2, n // 2, n // 2, np.zeros(1, np.float32))
    p.set_state(u, u)
    p.step(1)
    got = p.read(0).cpu().numpy().astype(np.float64)
    p.close()
    def d1(m):
        i = np.arange(m)
        return np.maximum(np.maximum(w - i, 0), i - (m - w - 1))
    d = np.maximum(np.maximum(d1(n)[None, None, :], d1(n)[None, :, None]), d1(n)[:, None, None])
    etap = np.pad(eta_max * (d / w) ** 2, 1)          # eta = 0 outside the domain
    gx = (etap[1:-1, 1:-1, 2:] - etap[1:-1, 1:-1, :-2]) / (2 * hx)
    gy = (etap[1:-1, 2:, 1:-1] - etap[1:-1, :-2, 1:-1]) / (2 * hy)
    gz = (etap[2:, 1:-1, 1:-1] - etap[:-2, 1:-1, 1:-1]) / (2 * hz)
    u64 = u.astype(np.float64)
    vdt2 = (V * dt) ** 2
    exp = u64 + vdt2 * (a * gx + b * gy + c * gz) / (1 + etap[1:-1, 1:-1, 1:-1] * dt)
    exp[d == 0] = u64[d == 0]
    sl = (slice(4, -4),) * 3
    corr = float(np.abs(exp - u64)[sl].max())
    err = float(np.abs(got - exp)[sl].max())
    scale = float(np.abs(u64).max())
    print(f"linear ramp {precision} 512^3: max correction {corr:.3e}, max |u - exact| {err:.3e}, max|u| {scale:.1f}")
    assert corr > 1e-1                                 # the probe is not vacuous
    tol = 1e-14 * scale if precision == "fp64" else 1e-6 * scale
    assert err <= tol, (err, tol)
