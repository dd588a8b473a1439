"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these retypes the oracle's loop: each checks the oracle's OUTPUT
against an independent fact -- exact rational weights from the Vandermonde
system, closed-form solutions of the discrete scheme (polynomials, plane
waves, linear ramps), invariants (energy, symmetry, time reversal), a dense
brute-force operator built from Kronecker products, or values printed in
SPEC.md (tests/golden/spec_examples.json).  A plausible mistake in the oracle
(a dropped term, a wrong sign or index, a transposed axis, a wrong PML
coefficient) fails at least one of them; the comment on each test says which.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def fd_weights_second_derivative(R=4):
    """Central 2R+1-point weights of d2/dx2 by solving the moment system
    sum_m w_m m^d = 2*[d==2], d = 0,2,..,2R (even moments; symmetric weights)
    in exact rationals.  Independent of any table in the oracle."""
    # unknowns: w0, w1..wR ; equations for d = 0, 2, ..., 2R
    n = R + 1
    M = [[Fraction(0)] * n for _ in range(n)]
    rhs = [Fraction(0)] * n
    for r, d in enumerate(range(0, 2 * R + 1, 2)):
        M[r][0] = Fraction(1 if d == 0 else 0)
        for m in range(1, R + 1):
            M[r][m] = Fraction(2 * m ** d)      # w_m (m^d + (-m)^d)
        rhs[r] = Fraction(2 if d == 2 else 0)
    # Gauss-Jordan in rationals
    for c in range(n):
        piv = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[piv] = M[piv], M[c]
        rhs[c], rhs[piv] = rhs[piv], rhs[c]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c] / M[c][c]
                M[r] = [a - f * b for a, b in zip(M[r], M[c])]
                rhs[r] -= f * rhs[c]
    return [rhs[i] / M[i][i] for i in range(n)]


W = fd_weights_second_derivative()


def geom(nx, ny, nz, w=0, h=1.0, dt=1.0, eta_max=0.0, **kw):
    return oracle.make_geom(nx, ny, nz, w, h, dt, eta_max, **kw)


# --------------------------------------------------------------------------
# Coefficients
# --------------------------------------------------------------------------

def test_weights_match_spec_and_vandermonde():
    # SPEC.md L125 values == solution of the moment system (pins the weight table)
    g = GOLD["weights"]
    spec = [Fraction(n, d) for n, d in zip(g["num"], g["den"])]
    assert W == spec
    # 8th order: moment 10 is the first non-vanishing error term
    assert sum(2 * w * m ** 10 for m, w in enumerate(W) if m) != 0


@pytest.mark.parametrize("h", [(1.0, 1.0, 1.0), (2.0, 3.0, 5.0), (10.0, 10.0, 7.5)])
def test_oracle_coefficients_fp64(oracle_lib, h):
    # per-axis c_am = w_m/h_a^2, c_xyz = w0 * sum 1/h_a^2 (catches axis swaps, scaling)
    c = oracle.constants(geom(8, 8, 8, h=h), round32=False, dtype=np.float64)
    for a, key in enumerate(("c_x", "c_y", "c_z")):
        for m in range(1, 5):
            assert c[key][m - 1] == pytest.approx(float(W[m] / Fraction(h[a]) ** 2), rel=1e-15)
    exp0 = float(W[0] * sum(1 / Fraction(x) ** 2 for x in h))
    assert c["c_xyz"] == pytest.approx(exp0, rel=1e-15)
    # constant annihilation
    tot = c["c_xyz"] + 2 * (c["c_x"].sum() + c["c_y"].sum() + c["c_z"].sum())
    assert abs(tot) < 1e-12 * abs(c["c_xyz"])


def test_oracle_coefficients_fp32_rounded_once(oracle_lib):
    # fp32 constants = the exact value rounded once (R8)
    c = oracle.constants(geom(8, 8, 8, h=(10.0, 10.0, 10.0)), round32=True, dtype=np.float32)
    for m in range(1, 5):
        assert c["c_x"][m - 1] == np.float32(float(W[m] / 100))
    g = GOLD["coeffs_h1"]
    c1 = oracle.constants(geom(8, 8, 8, h=1.0), round32=True, dtype=np.float32)
    assert c1["c_x"][0] == np.float32(g["c_x1"])
    assert abs(float(c1["c_x"][3]) - g["c_x4"]) < g["c_x4_tol"]
    c2 = oracle.constants(geom(8, 8, 8, h=GOLD["coeffs_scaling"]["h"]), round32=False, dtype=np.float64)
    c1d = oracle.constants(geom(8, 8, 8, h=1.0), round32=False, dtype=np.float64)
    np.testing.assert_allclose(c2["c_x"], c1d["c_x"] * GOLD["coeffs_scaling"]["ratio"], rtol=1e-15)


def test_pml_tables(oracle_lib):
    # eta_d = eta_max (d/w)^2 increasing from 0 at the inner interface (R2)
    g = geom(40, 40, 40, w=8, h=10.0, dt=2e-3, eta_max=4.0)
    c = oracle.constants(g, round32=False, dtype=np.float64)
    d = np.arange(9)
    np.testing.assert_allclose(c["eta"], 4.0 * (d / 8.0) ** 2, rtol=1e-15)
    dt = float(np.float32(2e-3))
    np.testing.assert_allclose(c["A"], 1 - c["eta"] * dt, rtol=1e-15)
    np.testing.assert_allclose(c["B"], 1 + c["eta"] * dt, rtol=1e-15)
    assert c["eta"][0] == 0.0 and c["A"][0] == 1.0 and c["B"][0] == 1.0
    np.testing.assert_allclose(c["inv2h"], [0.05, 0.05, 0.05], rtol=1e-15)


# --------------------------------------------------------------------------
# One step: impulse, polynomials
# --------------------------------------------------------------------------

def _one_step(g, u0, up0=None, V=None, dtype=np.float64, round32=False):
    shape = (g.nz, g.ny, g.nx)
    V = np.ones(shape, np.float32) if V is None else V
    u, up, st, _ = oracle.propagate(g, V, np.zeros(1, np.float32), 1, (0, 0, 0) if False else
                                    (g.nx // 2, g.ny // 2, g.nz // 2), u0=u0, uprev0=up0,
                                    dtype=dtype, round32=round32)
    assert st == 0
    return u


@pytest.mark.parametrize("h", [(1.0, 1.0, 1.0), (1.0, 2.0, 4.0)])
def test_impulse_response(oracle_lib, h):
    # u = delta_p, u_prev = 0, (V dt)^2 = 1  ->  u_next(p) = 2 + c_xyz,
    # u_next(p +- m e_a) = w_m / h_a^2, zero elsewhere.
    n = 17
    g = geom(n, n, n, h=h, dt=1.0)
    u0 = np.zeros((n, n, n))
    c = n // 2
    u0[c, c, c] = 1.0
    out = _one_step(g, u0)
    exp = np.zeros_like(out)
    exp[c, c, c] = 2 + float(W[0] * sum(1 / Fraction(x) ** 2 for x in h))
    for m in range(1, 5):
        exp[c, c, c + m] = exp[c, c, c - m] = float(W[m] / Fraction(h[0]) ** 2)   # x innermost
        exp[c, c + m, c] = exp[c, c - m, c] = float(W[m] / Fraction(h[1]) ** 2)
        exp[c + m, c, c] = exp[c - m, c, c] = float(W[m] / Fraction(h[2]) ** 2)
    np.testing.assert_allclose(out, exp, rtol=1e-14, atol=1e-15)


def _poly_case(n, h, terms):
    """u = sum of products of monomials; returns (u, analytic Laplacian) on a
    grid with centred coordinates x = (i - n//2) h."""
    x = (np.arange(n) - n // 2) * h
    X = x[None, None, :]
    Y = x[None, :, None]
    Z = x[:, None, None]
    u = np.zeros((n, n, n))
    lap = np.zeros((n, n, n))
    for (a, b, c) in terms:
        mono = lambda v, p: v ** p if p >= 0 else 0 * v
        dd = lambda v, p: p * (p - 1) * v ** (p - 2) if p >= 2 else 0 * v
        u = u + mono(X, a) * mono(Y, b) * mono(Z, c)
        lap = lap + dd(X, a) * mono(Y, b) * mono(Z, c) + mono(X, a) * dd(Y, b) * mono(Z, c) \
            + mono(X, a) * mono(Y, b) * dd(Z, c)
    return u, lap


@pytest.mark.parametrize("terms", [
    [(9, 0, 0)], [(0, 9, 0)], [(0, 0, 9)],
    [(2, 0, 0), (0, 4, 0), (0, 0, 6)],
    [(3, 7, 5), (9, 2, 8), (1, 1, 1)],
])
def test_polynomial_exactness(oracle_lib, terms):
    # Lap8 is exact on per-axis degree <= 9; checked on cells >= 4
    # from the zero fringe.  Lap(u) = u_next - 2u with u_prev = 0, (V dt)^2 = 1.
    n, h = 21, 0.1
    g = geom(n, n, n, h=h, dt=1.0)
    u, lap = _poly_case(n, h, terms)
    out = _one_step(g, u)
    got = (out - 2 * u)[4:-4, 4:-4, 4:-4]
    ref = lap[4:-4, 4:-4, 4:-4]
    assert np.max(np.abs(got - ref)) < 1e-8 * max(1.0, np.max(np.abs(ref)))


def test_polynomial_degree10_is_not_exact(oracle_lib):
    # sharpness of the previous pin: degree 10 leaves the h^8 truncation term
    # (-1152/10!) h^8 u^(10) per axis -> -1152 h^8 for u = x^10.
    n, h = 21, 0.1
    g = geom(n, n, n, h=h, dt=1.0)
    u, lap = _poly_case(n, h, [(10, 0, 0)])
    out = _one_step(g, u)
    err = ((out - 2 * u) - lap)[4:-4, 4:-4, 4:-4]
    np.testing.assert_allclose(err, -1152 * h ** 8, rtol=1e-4)


# --------------------------------------------------------------------------
# Multi-step closed forms
# --------------------------------------------------------------------------

def test_discrete_plane_wave(oracle_lib):
    # u^0 = cos(k.x), u^-1 = cos(k.x + w dt) with w from the scheme's own
    # dispersion relation 4 sin^2(w dt/2)/dt^2 = V^2 sum_a -(w0 + 2 sum_m w_m cos(m k_a h))/h^2
    # => u^s = cos(k.x - w s dt) exactly on cells >= 4s from the fringe.
    # Pins the leapfrog update (2u - u_prev), (V dt)^2 and all 13 coefficients.
    n, h, V = 48, 10.0, 2000.0
    dt = float(np.float32(2e-3))
    g = geom(n, n, n, h=h, dt=dt)
    k = [2 * math.pi / (8 * h), 2 * math.pi / (13 * h), 2 * math.pi / (21 * h)]
    wf = [float(x) for x in W]
    S = sum(-(wf[0] + 2 * sum(wf[m] * math.cos(m * ka * h) for m in range(1, 5))) / h ** 2 for ka in k)
    omega = 2 / dt * math.asin(math.sqrt(V * V * dt * dt * S / 4))
    i = np.arange(n) * h
    phase = k[0] * i[None, None, :] + k[1] * i[None, :, None] + k[2] * i[:, None, None]
    u0 = np.cos(phase)
    um1 = np.cos(phase + omega * dt)
    Varr = np.full((n, n, n), V, np.float32)
    for T in (1, 3, 5):
        u, up, st, _ = oracle.propagate(g, Varr, np.zeros(T, np.float32), T, (0, 0, 0),
                                        u0=u0, uprev0=um1, dtype=np.float64, round32=False)
        assert st == 0
        s = slice(4 * T, n - 4 * T)
        err = np.abs(u - np.cos(phase - omega * T * dt))[s, s, s]
        assert err.max() < 1e-12, (T, err.max())
        errp = np.abs(up - np.cos(phase - omega * (T - 1) * dt))[s, s, s]
        assert errp.max() < 1e-12


def _eta_field(nx, ny, nz, w, eta_max):
    """eta on the extended grid from the Chebyshev distance to the inner box,
    computed with numpy broadcasting (an independent spelling of DESIGN.md R2/R3),
    plus one zero cell of padding on every side (eta = 0 outside, R4)."""
    def d1(n):
        i = np.arange(n)
        return np.maximum(np.maximum(w - i, 0), i - (n - w - 1))
    d = np.maximum(np.maximum(d1(nx)[None, None, :], d1(ny)[None, :, None]), d1(nz)[:, None, None])
    eta = eta_max * (d / w) ** 2
    return np.pad(eta, 1), d


def test_linear_ramp_pml_probe(oracle_lib):
    # u = u_prev = C + a x + b y + c z: Lap u = 0, d_a u = (a,b,c) exactly, so one
    # step gives  u_next = u + vdt2 (a d_x eta + b d_y eta + c d_z eta) / (1 + eta dt)
    # in the PML and u inside.  Pins the grad-eta.grad-u term
    # (each axis with its own h), A = 1 - eta dt, B = 1 + eta dt, the eta profile,
    # the Chebyshev distance and the per-point vdt2.
    nx, ny, nz, w = 35, 31, 33, 8
    hx, hy, hz = 10.0, 7.5, 12.5
    eta_max, dt = 50.0, float(np.float32(1.5e-3))
    g = geom(nx, ny, nz, w=w, h=(hx, hy, hz), dt=dt, eta_max=eta_max)
    C, a, b, c = 0.7, 0.37, -0.21, 0.29
    X = np.arange(nx)[None, None, :] * hx
    Y = np.arange(ny)[None, :, None] * hy
    Z = np.arange(nz)[:, None, None] * hz
    u = C + a * X + b * Y + c * Z + np.zeros((nz, ny, nx))
    V = synth.velocity(synth.scenario("RAGGED", nx=nx, ny=ny, nz=nz, seed=3))
    out = _one_step(g, u, u.copy(), V=V)
    etap, d = _eta_field(nx, ny, nz, w, eta_max)
    gx = (etap[1:-1, 1:-1, 2:] - etap[1:-1, 1:-1, :-2]) / (2 * hx)
    gy = (etap[1:-1, 2:, 1:-1] - etap[1:-1, :-2, 1:-1]) / (2 * hy)
    gz = (etap[2:, 1:-1, 1:-1] - etap[:-2, 1:-1, 1:-1]) / (2 * hz)
    eta = etap[1:-1, 1:-1, 1:-1]
    vdt2 = (V.astype(np.float64) * dt) ** 2
    exp = u + vdt2 * (a * gx + b * gy + c * gz) / (1 + eta * dt)
    exp[d == 0] = u[d == 0]
    s = (slice(4, -4),) * 3
    corr = np.abs(exp - u)[s]
    assert corr.max() > 1e-2                      # the probe is not vacuous
    np.testing.assert_allclose(out[s], exp[s], rtol=0, atol=1e-11)


# --------------------------------------------------------------------------
# Invariants
# --------------------------------------------------------------------------

def test_energy_conservation_and_symmetric_operator(oracle_lib):
    # Leapfrog energy E^{n+1/2} = <d+, D^-1 d+> - <u^{n+1}, A u^n>, d+ = u^{n+1}-u^n,
    # D = diag(vdt2), is exactly conserved iff the Laplacian A (zero fringe) is
    # symmetric.  A u^n is read off the oracle's own states as
    # D^-1 (u^{n+1} - 2u^n + u^{n-1}) -- no stencil is retyped here.  Catches
    # any asymmetric index error (e.g. u(+m) used twice).
    n = 20
    g = geom(n, n, n, h=10.0, dt=float(np.float32(8e-4)))
    s = synth.scenario("SPEC48", nx=n, ny=n, nz=n, seed=5)
    V = synth.velocity(s)
    vdt2 = (V.astype(np.float64) * float(np.float32(8e-4))) ** 2
    u0 = synth.random_state((n, n, n), 11).astype(np.float64)
    um1 = synth.random_state((n, n, n), 12).astype(np.float64)
    states = [um1, u0]
    for T in range(1, 5):
        u, up, st, _ = oracle.propagate(g, V, np.zeros(T, np.float32), T, (0, 0, 0), u0=u0,
                                        uprev0=um1, dtype=np.float64, round32=False)
        states.append(u)
    Au = [None] + [(states[i + 1] - 2 * states[i] + states[i - 1]) / vdt2 for i in range(1, 5)]
    E = []
    for i in range(1, 4):      # E^{i+1/2} uses states i, i+1 and A u^i
        dp = states[i + 1] - states[i]
        E.append(np.sum(dp * dp / vdt2) - np.sum(states[i + 1] * Au[i]))
    assert abs(E[1] - E[0]) < 1e-10 * abs(E[0])
    assert abs(E[2] - E[1]) < 1e-10 * abs(E[0])


def test_time_reversal(oracle_lib):
    # leapfrog is time-symmetric: from (u^{n+1}, u^n) one step returns u^{n-1}
    n = 16
    g = geom(n, n, n, h=10.0, dt=float(np.float32(1e-3)))
    V = synth.velocity(synth.scenario("SPEC48", nx=n, ny=n, nz=n, seed=2))
    a = synth.random_state((n, n, n), 1).astype(np.float64)
    b = synth.random_state((n, n, n), 2).astype(np.float64)
    c, _, st, _ = oracle.propagate(g, V, np.zeros(1, np.float32), 1, (0, 0, 0), u0=b, uprev0=a,
                                   dtype=np.float64, round32=False)
    back, _, st, _ = oracle.propagate(g, V, np.zeros(1, np.float32), 1, (0, 0, 0), u0=b, uprev0=c,
                                      dtype=np.float64, round32=False)
    np.testing.assert_allclose(back, a, atol=1e-13)


def test_mirror_symmetry_bitwise_fp32(oracle_lib):
    # odd extents, centred source, constant V, symmetric eta: the fp32 field is
    # bitwise mirror-symmetric along every axis (pair sums before multiplying;
    # SPEC.md L183 states it to 1e-12 in fp64).  Catches an off-by-one in the
    # distance d or the eta star, and any one-sided stencil term.
    n = 33
    s = synth.scenario("C1", nx=n, ny=n, nz=n, w=8, steps=60)
    g = oracle.make_geom(n, n, n, s.w, s.h, s.dt, s.eta_max)
    u, up, st, _ = oracle.propagate(g, synth.velocity(s), synth.wavelet_for(s), s.steps,
                                    s.source, dtype=np.float32)
    assert st == 0 and np.abs(u).max() > 0
    for ax in range(3):
        assert np.array_equal(u, np.flip(u, axis=ax)), ax


def test_eta_zero_reduces_to_inner(oracle_lib):
    # eta_max = 0 with w > 0 must equal w = 0 (bitwise)
    s = synth.scenario("RAGGED", steps=15)
    V = synth.velocity(s)
    wl = synth.wavelet_for(s)
    g0 = oracle.make_geom(s.nx, s.ny, s.nz, 0, s.h, s.dt, 0.0)
    g1 = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, 0.0)
    u0 = synth.random_state((s.nz, s.ny, s.nx), 7)
    a, _, _, _ = oracle.propagate(g0, V, wl, s.steps, s.source, u0=u0)
    b, _, _, _ = oracle.propagate(g1, V, wl, s.steps, s.source, u0=u0)
    assert np.array_equal(a, b)


def test_linearity_and_source_additivity(oracle_lib):
    s = synth.scenario("RAGGED", steps=12)
    g = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    V = synth.velocity(s)
    wl = synth.wavelet_for(s).astype(np.float32)
    u0 = synth.random_state((s.nz, s.ny, s.nx), 4)
    z = np.zeros(s.steps, np.float32)
    a, _, _, _ = oracle.propagate(g, V, z, s.steps, s.source, u0=u0, dtype=np.float64, round32=False)
    b, _, _, _ = oracle.propagate(g, V, z, s.steps, s.source, u0=2.5 * u0.astype(np.float64),
                                  dtype=np.float64, round32=False)
    np.testing.assert_allclose(b, 2.5 * a, rtol=1e-12, atol=1e-13)
    # field(u0, wavelet) = field(u0, 0) + field(0, wavelet)
    c, _, _, _ = oracle.propagate(g, V, wl, s.steps, s.source, dtype=np.float64, round32=False)
    d, _, _, _ = oracle.propagate(g, V, wl, s.steps, s.source, u0=u0, dtype=np.float64, round32=False)
    np.testing.assert_allclose(d, a + c, rtol=1e-12, atol=1e-13)
    # zero wavelet, zero state -> zero
    e, _, _, _ = oracle.propagate(g, V, z, s.steps, s.source)
    assert not e.any()


def test_source_increment_spec_example(oracle_lib):
    # wavelet 1, V = 2, dt = 1e-3 -> +4e-6 at the source, once
    gd = GOLD["inject"]
    n = 12
    g = oracle.make_geom(n, n, n, 2, 1.0, gd["dt"], 0.0)
    V = np.full((n, n, n), gd["V"], np.float32)
    u, up, st, _ = oracle.propagate(g, V, np.array([gd["w"]], np.float32), 1, (6, 6, 6),
                                    dtype=np.float64, round32=False)
    exp = (gd["V"] * float(np.float32(gd["dt"]))) ** 2 * gd["w"]
    assert u[6, 6, 6] == pytest.approx(gd["increment"], rel=1e-6)
    assert u[6, 6, 6] == pytest.approx(exp, rel=1e-15)
    u[6, 6, 6] = 0
    assert not u.any()


def test_zero_steps_returns_initial_state(oracle_lib):
    n = 10
    g = oracle.make_geom(n, n, n, 2, 10.0, 1e-3, 4.0)
    u0 = synth.random_state((n, n, n), 9)
    up0 = synth.random_state((n, n, n), 8)
    u, up, st, _ = oracle.propagate(g, np.full((n, n, n), 2000, np.float32), np.zeros(1, np.float32),
                                    0, (5, 5, 5), u0=u0, uprev0=up0)
    assert st == 0 and np.array_equal(u, u0) and np.array_equal(up, up0)


def test_dense_operator_brute_force(oracle_lib):
    # The one-step map (u, u_prev) -> u_next assembled as a dense matrix from
    # 1-D difference operators with Kronecker products (an independent
    # formulation: no per-point loop, no padding) and compared with the oracle
    # over 3 steps on a 9x10x11 grid with a 2-cell PML.
    nx, ny, nz, w = 9, 10, 11, 2
    hx, hy, hz = 10.0, 8.0, 12.0
    dt = float(np.float32(1e-3))
    eta_max = 30.0
    g = geom(nx, ny, nz, w=w, h=(hx, hy, hz), dt=dt, eta_max=eta_max)
    wf = [float(x) for x in W]

    def d2(n, h):
        M = np.zeros((n, n))
        for i in range(n):
            M[i, i] = wf[0] / h ** 2
            for m in range(1, 5):
                for j in (i - m, i + m):
                    if 0 <= j < n:
                        M[i, j] = wf[m] / h ** 2
        return M

    def d1(n, h):
        M = np.zeros((n, n))
        for i in range(n):
            if i + 1 < n:
                M[i, i + 1] = 1 / (2 * h)
            if i - 1 >= 0:
                M[i, i - 1] = -1 / (2 * h)
        return M

    Ix, Iy, Iz = np.eye(nx), np.eye(ny), np.eye(nz)
    kron3 = lambda A, B, C: np.kron(A, np.kron(B, C))   # z (outer) x y x x (inner)
    Lap = kron3(Iz, Iy, d2(nx, hx)) + kron3(Iz, d2(ny, hy), Ix) + kron3(d2(nz, hz), Iy, Ix)
    Gx, Gy, Gz = kron3(Iz, Iy, d1(nx, hx)), kron3(Iz, d1(ny, hy), Ix), kron3(d1(nz, hz), Iy, Ix)
    etap, d = _eta_field(nx, ny, nz, w, eta_max)
    # grad eta with eta = 0 outside the domain
    ge = [((etap[1:-1, 1:-1, 2:] - etap[1:-1, 1:-1, :-2]) / (2 * hx)).ravel(),
          ((etap[1:-1, 2:, 1:-1] - etap[1:-1, :-2, 1:-1]) / (2 * hy)).ravel(),
          ((etap[2:, 1:-1, 1:-1] - etap[:-2, 1:-1, 1:-1]) / (2 * hz)).ravel()]
    eta = etap[1:-1, 1:-1, 1:-1].ravel()
    pml = d.ravel() > 0
    V = synth.velocity(synth.scenario("RAGGED", nx=nx, ny=ny, nz=nz, seed=8))
    D = ((V.astype(np.float64) * dt) ** 2).ravel()
    Op = Lap + pml[:, None] * (ge[0][:, None] * Gx + ge[1][:, None] * Gy + ge[2][:, None] * Gz)
    Acoef = np.where(pml, 1 - eta * dt, 1.0)
    Bcoef = np.where(pml, 1 + eta * dt, 1.0)
    u = synth.random_state((nz, ny, nx), 21).astype(np.float64).ravel()
    up = synth.random_state((nz, ny, nx), 22).astype(np.float64).ravel()
    u0, up0 = u.copy(), up.copy()
    for _ in range(3):
        un = (2 * u - Acoef * up + D * (Op @ u)) / Bcoef
        u, up = un, u
    got, gotp, st, _ = oracle.propagate(g, V, np.zeros(3, np.float32), 3, (4, 5, 5),
                                        u0=u0.reshape(nz, ny, nx), uprev0=up0.reshape(nz, ny, nx),
                                        dtype=np.float64, round32=False)
    np.testing.assert_allclose(got.ravel(), u, rtol=0, atol=1e-12)
    np.testing.assert_allclose(gotp.ravel(), up, rtol=0, atol=1e-12)


# --------------------------------------------------------------------------
# Stability (R5: SPEC's eta_max = 100 is unstable; 4 is stable)
# --------------------------------------------------------------------------

def test_eta_max_100_diverges_and_is_detected(oracle_lib):
    n, w = 24, 6
    g = oracle.make_geom(n, n, n, w, 10.0, 2e-3, 100.0)
    V = np.full((n, n, n), 2000.0, np.float32)
    u0 = synth.random_state((n, n, n), 3)
    u, up, st, fail = oracle.propagate(g, V, np.zeros(400, np.float32), 400, (12, 12, 12),
                                       u0=u0, check_every=10)
    assert st == oracle.ERR_UNSTABLE and 0 < fail <= 400


def test_eta_max_4_is_stable(oracle_lib):
    n, w = 24, 6
    g = oracle.make_geom(n, n, n, w, 10.0, 2e-3, 4.0)
    V = np.full((n, n, n), 2000.0, np.float32)
    u0 = synth.random_state((n, n, n), 3)
    u, up, st, fail = oracle.propagate(g, V, np.zeros(400, np.float32), 400, (12, 12, 12),
                                       u0=u0, check_every=10)
    assert st == 0 and np.abs(u).max() < 10.0


def test_fp32_tracks_fp64_on_same_constants(oracle_lib):
    # information-level check of R8: fp32 vs fp64 arithmetic on the same
    # fp32-rounded constants stays far below the 1e-5 parity gate (C1 setup)
    s = synth.scenario("C1", steps=40)
    g = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    V, wl = synth.velocity(s), synth.wavelet_for(s)
    a, _, _, _ = oracle.propagate(g, V, wl, s.steps, s.source, dtype=np.float32)
    b, _, _, _ = oracle.propagate(g, V, wl, s.steps, s.source, dtype=np.float64, round32=True)
    assert np.abs(a - b).max() / np.abs(b).max() < 2e-6


# --------------------------------------------------------------------------
# Input generators (synth) -- the pins of the wavelet input
# --------------------------------------------------------------------------

def test_ricker_examples():
    gp = GOLD["ricker_n150"]
    w = synth.ricker_samples(gp["f_peak"], gp["t0"], gp["dt"], 300)
    t = 150 * float(np.float32(gp["dt"]))
    a = (math.pi * gp["f_peak"] * (t - gp["t0"])) ** 2
    assert w[150] == np.float32((1 - 2 * a) * math.exp(-a))
    # peak normalised: t0 on the sampling grid -> 1
    w2 = synth.ricker_samples(20.0, 0.05, 0.001, 100)
    assert abs(float(w2[50]) - GOLD["ricker_peak"]["value"]) < 1e-6
    # even about t0
    np.testing.assert_allclose(w2[50 - 20:50], w2[51:71][::-1], rtol=0, atol=2e-6)  # t0 only ~on grid (fp32 dt)


def test_dt_auto(oracle_lib):
    V = np.array([1500.0, 4500.0, 3000.0], np.float32)
    assert oracle.dt_auto(10.0, V) == np.float32(0.4 * 10.0 / 4500.0)
    assert oracle.dt_auto((10.0, 5.0, 20.0), V) == np.float32(0.4 * 5.0 / 4500.0)


def test_source_location_and_scaling_asymmetric(oracle_lib):
    # From the zero state, one step leaves exactly fp32((V(src) dt)^2 w[0]) at the
    # (i, j, k) source cell and zero elsewhere; an asymmetric source and a random
    # V pin the index order of the source cell and of the V lookup (PAPER.md L238
    # Eq. 2 RHS dt^2 V^2 f).
    s = synth.scenario("RAGGED")
    g = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    V = synth.velocity(s)
    i, j, k = 29, 17, 33
    u, _, st, _ = oracle.propagate(g, V, np.array([0.75], np.float32), 1, (i, j, k),
                                   dtype=np.float64, round32=False)
    exp = (float(V[k, j, i]) * float(s.dt32)) ** 2 * 0.75
    assert u[k, j, i] == pytest.approx(exp, rel=1e-15)
    u[k, j, i] = 0
    assert not u.any()


# --------------------------------------------------------------------------
# Stored (user-supplied) eta -- SURVEY.md §8(f) rank 3, R16
# --------------------------------------------------------------------------

def _random_eta(shape, seed, scale=20.0):
    rng = np.random.Generator(np.random.PCG64(seed))
    return (scale * rng.random(shape)).astype(np.float32)


def test_stored_eta_dense_operator_brute_force(oracle_lib):
    # Same independent Kronecker formulation as above, with an arbitrary
    # (random, non-smooth) stored eta field: grad eta from the stored values
    # with 0 outside the domain, A = 1 - eta dt and B = 1 + eta dt per PML point.
    # A transposed eta index or a wrong neighbour fails at O(1).
    nx, ny, nz, w = 9, 10, 11, 2
    hx, hy, hz = 10.0, 8.0, 12.0
    dt = float(np.float32(1e-3))
    g = geom(nx, ny, nz, w=w, h=(hx, hy, hz), dt=dt, eta_max=7.0)   # eta_max unused by stored eta
    wf = [float(x) for x in W]

    def d2(n, h):
        M = np.zeros((n, n))
        for i in range(n):
            M[i, i] = wf[0] / h ** 2
            for m in range(1, 5):
                for j in (i - m, i + m):
                    if 0 <= j < n:
                        M[i, j] = wf[m] / h ** 2
        return M

    def d1(n, h):
        return (np.eye(n, k=1) - np.eye(n, k=-1)) / (2 * h)

    Ix, Iy, Iz = np.eye(nx), np.eye(ny), np.eye(nz)
    kron3 = lambda A, B, C: np.kron(A, np.kron(B, C))
    Lap = kron3(Iz, Iy, d2(nx, hx)) + kron3(Iz, d2(ny, hy), Ix) + kron3(d2(nz, hz), Iy, Ix)
    G = [kron3(Iz, Iy, d1(nx, hx)), kron3(Iz, d1(ny, hy), Ix), kron3(d1(nz, hz), Iy, Ix)]
    eta32 = _random_eta((nz, ny, nx), 9)
    eta = eta32.astype(np.float64).ravel()
    ge = [Gk @ eta for Gk in G]                        # central differences, eta = 0 outside
    _, d = _eta_field(nx, ny, nz, w, 1.0)
    pml = d.ravel() > 0
    V = synth.velocity(synth.scenario("RAGGED", nx=nx, ny=ny, nz=nz, seed=8))
    D = ((V.astype(np.float64) * dt) ** 2).ravel()
    Op = Lap + pml[:, None] * (ge[0][:, None] * G[0] + ge[1][:, None] * G[1] + ge[2][:, None] * G[2])
    Acoef = np.where(pml, 1 - eta * dt, 1.0)
    Bcoef = np.where(pml, 1 + eta * dt, 1.0)
    u = synth.random_state((nz, ny, nx), 23).astype(np.float64).ravel()
    up = synth.random_state((nz, ny, nx), 24).astype(np.float64).ravel()
    u0, up0 = u.copy(), up.copy()
    for _ in range(3):
        un = (2 * u - Acoef * up + D * (Op @ u)) / Bcoef
        u, up = un, u
    got, gotp, st, _ = oracle.propagate(g, V, np.zeros(3, np.float32), 3, (4, 5, 5),
                                        u0=u0.reshape(nz, ny, nx), uprev0=up0.reshape(nz, ny, nx),
                                        dtype=np.float64, round32=False, eta=eta32)
    assert st == 0
    np.testing.assert_allclose(got.ravel(), u, rtol=0, atol=1e-12)
    np.testing.assert_allclose(gotp.ravel(), up, rtol=0, atol=1e-12)


def test_stored_eta_linear_ramp_probe(oracle_lib):
    # closed form of the ramp probe with an arbitrary stored eta field
    nx, ny, nz, w = 27, 25, 23, 6
    hx, hy, hz = 10.0, 7.5, 12.5
    dt = float(np.float32(1.5e-3))
    g = geom(nx, ny, nz, w=w, h=(hx, hy, hz), dt=dt, eta_max=0.0)
    C, a, b, c = 0.7, 0.37, -0.21, 0.29
    X = np.arange(nx)[None, None, :] * hx
    Y = np.arange(ny)[None, :, None] * hy
    Z = np.arange(nz)[:, None, None] * hz
    u = C + a * X + b * Y + c * Z + np.zeros((nz, ny, nx))
    V = synth.velocity(synth.scenario("RAGGED", nx=nx, ny=ny, nz=nz, seed=3))
    eta32 = _random_eta((nz, ny, nx), 10, scale=40.0)
    out, _, st, _ = oracle.propagate(g, V, np.zeros(1, np.float32), 1, (nx // 2, ny // 2, nz // 2), u0=u,
                                     uprev0=u.copy(), dtype=np.float64, round32=False, eta=eta32)
    assert st == 0
    ep = np.pad(eta32.astype(np.float64), 1)
    gx = (ep[1:-1, 1:-1, 2:] - ep[1:-1, 1:-1, :-2]) / (2 * hx)
    gy = (ep[1:-1, 2:, 1:-1] - ep[1:-1, :-2, 1:-1]) / (2 * hy)
    gz = (ep[2:, 1:-1, 1:-1] - ep[:-2, 1:-1, 1:-1]) / (2 * hz)
    e = eta32.astype(np.float64)
    vdt2 = (V.astype(np.float64) * dt) ** 2
    exp = u + vdt2 * (a * gx + b * gy + c * gz) / (1 + e * dt)
    _, d = _eta_field(nx, ny, nz, w, 1.0)
    exp[d == 0] = u[d == 0]
    s = (slice(4, -4),) * 3
    assert np.abs(exp - u)[s].max() > 1e-2
    np.testing.assert_allclose(out[s], exp[s], rtol=0, atol=1e-11)


def test_stored_eta_zero_equals_profile_eta_zero_bitwise(oracle_lib):
    s = synth.scenario("RAGGED")
    sh = (s.nz, s.ny, s.nx)
    g0 = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, 0.0)
    u0 = synth.random_state(sh, 1)
    a, ap, _, _ = oracle.propagate(g0, synth.velocity(s), synth.wavelet_for(s, 6), 6, s.source, u0=u0)
    b, bp, _, _ = oracle.propagate(g0, synth.velocity(s), synth.wavelet_for(s, 6), 6, s.source, u0=u0,
                                   eta=np.zeros(sh, np.float32))
    assert np.array_equal(a, b) and np.array_equal(ap, bp)
