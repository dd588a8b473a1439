"""Whole-field oracle parity at the CONFIGURED horizon (BASELINE.json
north_star: rel L-inf <= 1e-5 "after the configured number of steps"; the
paper's runs are 1000 iterations, §V-B).

The layered-medium configurations run 1000 steps: C3 (configs[2], 1024^3) and
its recipe on smaller grids the oracle finishes in seconds (L128, L256; the
SURVEY.md §8(d) fallback).  Systematic per-step rounding differences between
the fp32 kernels (FMA chains, pair sums first) and the fp32 oracle (S:L376
order, no contraction) accumulate with the step count, so this horizon is
where the gate is tightest.  Each test prints its margin; DESIGN.md §2 lists
the measured values.

The C3 x 1000 comparison (~10 min of oracle time on the box's host cores,
~17 GB of host memory) runs only with WAVE25_SLOW=1.
"""
import os

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


def rel_linf(got, ref):
    m = float(np.abs(ref).max())
    return float(np.abs(got.astype(np.float64) - ref).max()) / (m if m > 0 else 1.0)


def gpu_run(s, kernel="stream"):
    from paper_2009_04619_b200.wave import WavePlan
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s))
    p.step(s.steps)            # CUDA graphs of 2 steps: the launch configuration bench.py times
    out = p.read(0).cpu().numpy(), p.read(1).cpu().numpy()
    p.close()
    return out


def oracle_run(s):
    g = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    u, up, st, _ = oracle.propagate(g, synth.velocity(s), synth.wavelet_for(s), s.steps, s.source)
    assert st == 0
    return u, up


_cache = {}


def _oracle_cached(name):
    if name not in _cache:
        _cache[name] = oracle_run(synth.scenario(name))
    return _cache[name]


def _report(tag, s, e, ep, ref):
    print(f"\n[horizon] {tag}: {s.nx}x{s.ny}x{s.nz} {s.vmodel} x {s.steps} steps: rel Linf u^T {e:.3e}, "
          f"u^(T-1) {ep:.3e} (gate {TOL:g}, margin {TOL / max(e, ep, 1e-30):.2f}x), max|u| "
          f"{float(np.abs(ref).max()):.4e}")


@pytest.mark.parametrize("name", ["L128", "L256"])
@pytest.mark.parametrize("kernel", ["stream", "pair", "tb2"])
def test_layered_1000_steps_whole_field(name, kernel):
    s = synth.scenario(name)
    assert s.steps == 1000 and s.vmodel == "layered"
    if kernel != "stream" and name != "L128":
        pytest.skip("the two-step variants are bitwise equal to stream (test_gpu_tb2/pair); one size suffices")
    g, gp = gpu_run(s, kernel)
    r, rp = _oracle_cached(name)
    e, ep = rel_linf(g, r), rel_linf(gp, rp)
    _report(f"{name}/{kernel}", s, e, ep, r)
    assert float(np.abs(r).max()) > 0
    assert e <= TOL and ep <= TOL, (e, ep)


@pytest.mark.skipif(os.environ.get("WAVE25_SLOW") != "1", reason="C3 x 1000 whole field: set WAVE25_SLOW=1")
def test_c3_1000_steps_whole_field():
    # BASELINE.json configs[2] exactly: 1024^3, layered V, 16-cell PML, Ricker
    # 15 Hz at the centre, all 1000 steps through the default kernels and graphs
    s = synth.scenario("C3")
    assert s.steps == 1000
    g, gp = gpu_run(s)
    torch.cuda.empty_cache()
    r, rp = oracle_run(s)
    e, ep = rel_linf(g, r), rel_linf(gp, rp)
    _report("C3", s, e, ep, r)
    assert float(np.abs(r).max()) > 0
    assert e <= TOL and ep <= TOL, (e, ep)
