"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no stencil coefficients, no
PML profile, no dt rule, no source scaling).  It only produces the raw inputs
the method consumes, so that `oracle/` and `paper_2009_04619_b200/` can be fed
identical bytes without importing each other:

* velocity models V[nz][ny][nx] (fp32, m/s)          -- PAPER.md L236 ("V is the Earth model")
* wavelet samples w[n] (fp32)                        -- SPEC.md L167-175 (Ricker, "invented plumbing")
* random initial states u^{-1}, u^0 ~ U(-1, 1) (fp32) -- SURVEY.md §8(d) C1 extras
* the workload table (grid, PML width, spacing, dt, source, steps) of
  BASELINE.json configs[0..4] plus extra parity scenarios; every number in it
  is a literal stated in DESIGN.md §"Input recipe".

The Ricker wavelet is an input signal (the paper never fixes f's waveform,
SPEC.md L168 marks it "invented -- artifact plumbing"); it is generated here in
fp64 and rounded once to fp32 (last bullet).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = ["Scenario", "SCENARIOS", "scenario", "velocity", "ricker_samples",
           "random_state", "wavelet_for"]


@dataclasses.dataclass(frozen=True)
class Scenario:
    """One synthetic workload.  All values are inputs of the method."""
    name: str
    nx: int
    ny: int
    nz: int
    w: int                    # PML width (cells), uniform on all faces
    h: float                  # grid spacing (m), hx = hy = hz
    dt: float                 # time step (s); stored as the fp32 value np.float32(dt)
    eta_max: float            # PML damping maximum (1/s)
    vmodel: str               # "const" | "layered" | "random"
    v0: float = 2000.0        # const velocity / layered & random lower bound (m/s)
    v1: float = 4500.0        # layered & random upper bound (m/s)
    layers: int = 8           # layered model: equal z-layers
    f_peak: float = 20.0      # Ricker peak frequency (Hz)
    t0: float = 0.05          # Ricker delay (s)
    steps: int = 10
    src: Optional[tuple] = None   # global (i, j, k); None = domain centre
    seed: int = 0

    @property
    def source(self) -> tuple:
        if self.src is not None:
            return tuple(int(v) for v in self.src)
        return (self.nx // 2, self.ny // 2, self.nz // 2)

    @property
    def dt32(self) -> np.float32:
        return np.float32(self.dt)

    def with_(self, **kw) -> "Scenario":
        return dataclasses.replace(self, **kw)


# The workload table.  dt values are literals (0.4*h/Vmax written out), see
# DESIGN.md "Input recipe"; both implementations receive exactly np.float32(dt).
SCENARIOS = {
    # BASELINE.json configs[0]: 64^3, const V, Ricker, 10 steps (oracle in seconds)
    "C1": Scenario("C1", 64, 64, 64, w=16, h=10.0, dt=2.0e-3, eta_max=4.0,
                   vmodel="const", v0=2000.0, f_peak=20.0, t0=0.05, steps=10),
    # configs[1]: 512^3 const V, 500 steps, full absorbing region
    "C2": Scenario("C2", 512, 512, 512, w=16, h=10.0, dt=2.0e-3, eta_max=4.0,
                   vmodel="const", v0=2000.0, f_peak=20.0, t0=0.05, steps=500),
    # configs[2]: 1024^3 layered V (8 layers 1500 -> 4500 m/s), 1000 steps
    "C3": Scenario("C3", 1024, 1024, 1024, w=16, h=10.0, dt=8.888889e-4,
                   eta_max=4.0, vmodel="layered", v0=1500.0, v1=4500.0,
                   f_peak=15.0, t0=0.0666667, steps=1000),
    # configs[4] per-rank block of the weak-scaling run (nz = 1024*N globally)
    "C5": Scenario("C5", 1024, 1024, 1024, w=16, h=10.0, dt=8.888889e-4,
                   eta_max=4.0, vmodel="layered", v0=1500.0, v1=4500.0,
                   f_peak=15.0, t0=0.0666667, steps=1000),
    # SPEC.md L602 acceptance scenario: 48^3, w=4, V ~ U(1500,4500), 50 steps
    "SPEC48": Scenario("SPEC48", 48, 48, 48, w=4, h=10.0, dt=8.888889e-4,
                       eta_max=4.0, vmodel="random", v0=1500.0, v1=4500.0,
                       f_peak=15.0, t0=0.0666667, steps=50),
    # ragged, non-cubic, misaligned extents for tile-edge coverage
    "RAGGED": Scenario("RAGGED", 70, 45, 53, w=5, h=7.5, dt=6.0e-4,
                       eta_max=4.0, vmodel="random", v0=1500.0, v1=4500.0,
                       f_peak=25.0, t0=0.04, steps=40, src=(31, 20, 27)),
    # 128^3 layered, the SURVEY A.8 drift study grid
    "L128": Scenario("L128", 128, 128, 128, w=16, h=10.0, dt=8.888889e-4,
                     eta_max=4.0, vmodel="layered", v0=1500.0, v1=4500.0,
                     f_peak=15.0, t0=0.0666667, steps=1000),
    # 256^3 layered x 1000 steps: the C3 recipe (V, dt, wavelet, w) on a grid
    # the oracle finishes in seconds (SURVEY.md §8(d) oracle-timing bullet)
    "L256": Scenario("L256", 256, 256, 256, w=16, h=10.0, dt=8.888889e-4,
                     eta_max=4.0, vmodel="layered", v0=1500.0, v1=4500.0,
                     f_peak=15.0, t0=0.0666667, steps=1000),
}


def scenario(name: str, **overrides) -> Scenario:
    s = SCENARIOS[name]
    return s.with_(**overrides) if overrides else s


def velocity(s: Scenario, nz_global: Optional[int] = None, z_offset: int = 0,
             nz_local: Optional[int] = None) -> np.ndarray:
    """V[nz_local][ny][nx] fp32 for the z-slab [z_offset, z_offset+nz_local).

    const:   V = v0 everywhere.
    layered: `layers` equal z-layers over the GLOBAL z extent, layer l has
             V = v0 + l*(v1-v0)/(layers-1)  (1500, 1928.57, ..., 4500 m/s).
    random:  V ~ U(v0, v1) i.i.d., numpy PCG64(seed), drawn over the global
             grid so that slabs of one run agree with the full grid.
    """
    nzg = s.nz if nz_global is None else nz_global
    nzl = nzg - z_offset if nz_local is None else nz_local
    if s.vmodel == "const":
        return np.full((nzl, s.ny, s.nx), s.v0, dtype=np.float32)
    if s.vmodel == "layered":
        k = np.arange(z_offset, z_offset + nzl)
        layer = (k * s.layers) // nzg
        vals = (s.v0 + layer * ((s.v1 - s.v0) / (s.layers - 1))).astype(np.float32)
        return np.ascontiguousarray(
            np.broadcast_to(vals[:, None, None], (nzl, s.ny, s.nx)), dtype=np.float32)
    if s.vmodel == "random":
        rng = np.random.Generator(np.random.PCG64(s.seed))
        full = rng.uniform(s.v0, s.v1, size=(nzg, s.ny, s.nx)).astype(np.float32)
        return np.ascontiguousarray(full[z_offset:z_offset + nzl])
    raise ValueError(f"unknown velocity model {s.vmodel!r}")


def ricker_samples(f_peak: float, t0: float, dt: float, nsamples: int) -> np.ndarray:
    """Ricker wavelet w(t) = (1 - 2 pi^2 f^2 (t-t0)^2) exp(-pi^2 f^2 (t-t0)^2)
    sampled at t = n*dt, computed in fp64 with dt taken as
    the fp32 value, rounded once to fp32."""
    dt64 = float(np.float32(dt))
    t = np.arange(nsamples, dtype=np.float64) * dt64
    a = (math.pi * f_peak * (t - t0)) ** 2
    return ((1.0 - 2.0 * a) * np.exp(-a)).astype(np.float32)


def wavelet_for(s: Scenario, nsamples: Optional[int] = None) -> np.ndarray:
    return ricker_samples(s.f_peak, s.t0, s.dt, s.steps if nsamples is None else nsamples)


def random_state(shape, seed: int) -> np.ndarray:
    """fp32 array ~ U(-1, 1) from numpy PCG64(seed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=shape).astype(np.float32)
