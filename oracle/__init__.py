"""CPU oracle for the 25-point acoustic wave step (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product package
(paper_2009_04619_b200) never imports it and shares no code with it.

The arithmetic lives in plain C (wave_oracle.c, oracle_body.h,
oracle_consts.h); this module only builds the shared library and marshals
numpy arrays through ctypes.  See wave_oracle.c's header for the passages each
function follows and DESIGN.md §3 for the readings of the paper it adopts.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SOURCES = ["wave_oracle.c", "oracle_body.h", "oracle_consts.h"]
R = 4

OK, ERR_CONFIG, ERR_UNSTABLE, ERR_ALLOC = 0, 1, 2, 5

_lock = threading.Lock()
_lib = None


class Geom(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("w", ctypes.c_int32),
                ("hx", ctypes.c_double), ("hy", ctypes.c_double), ("hz", ctypes.c_double),
                ("dt", ctypes.c_float), ("eta_max", ctypes.c_double),
                ("nz_global", ctypes.c_int64), ("z_offset", ctypes.c_int64)]


def make_geom(nx, ny, nz, w, h, dt, eta_max, nz_global=None, z_offset=0) -> Geom:
    hx, hy, hz = (h, h, h) if np.isscalar(h) else tuple(h)
    return Geom(int(nx), int(ny), int(nz), int(w), float(hx), float(hy), float(hz),
                float(np.float32(dt)), float(eta_max),
                int(nz if nz_global is None else nz_global), int(z_offset))


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, OpenMP, -ffp-contract=off, no fast-math)."""
    srcs = [os.path.join(HERE, s) for s in SOURCES]
    if not force and os.path.exists(LIB_PATH):
        newest = max(os.path.getmtime(s) for s in srcs)
        if os.path.getmtime(LIB_PATH) >= newest:
            return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
           "-shared", "-Wall", os.path.join(HERE, "wave_oracle.c"), "-o", tmp, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(LIB_PATH)
            P = ctypes.c_void_p
            i64, i32 = ctypes.c_int64, ctypes.c_int
            for sfx in ("f32", "f64"):
                f = getattr(L, f"oracle_step_{sfx}")
                f.argtypes = [ctypes.POINTER(Geom), i32, P, P, P, i64, i64, i64, ctypes.c_float]
                f.restype = i32
                f = getattr(L, f"oracle_propagate_{sfx}")
                f.argtypes = [ctypes.POINTER(Geom), i32, P, P, i64, i64, i64, i64, P, P, i64,
                              ctypes.POINTER(i64)]
                f.restype = i32
                f = getattr(L, f"oracle_propagate_eta_{sfx}")
                f.argtypes = [ctypes.POINTER(Geom), i32, P, P, P, i64, i64, i64, i64, P, P, i64,
                              ctypes.POINTER(i64)]
                f.restype = i32
                f = getattr(L, f"oracle_constants_{sfx}")
                f.argtypes = [ctypes.POINTER(Geom), i32, P, P, P, P, P]
                f.restype = i32
                f = getattr(L, f"oracle_vdt2_{sfx}")
                f.argtypes = [P, i64, ctypes.c_float, i32, P]
                f.restype = None
            L.oracle_dt_auto.argtypes = [ctypes.c_double] * 3 + [P, i64]
            L.oracle_dt_auto.restype = ctypes.c_float
            L.oracle_set_threads.argtypes = [i32]
            L.oracle_get_threads.restype = i32
            _lib = L
        return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _sfx(dtype) -> str:
    return "f32" if np.dtype(dtype) == np.float32 else "f64"


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def constants(g: Geom, round32: bool = True, dtype=np.float32) -> dict:
    """The constants the oracle uses: c_xyz, c_x/y/z[1..4], eta/A/B[0..w], 1/(2h)."""
    dt_ = np.dtype(dtype)
    c = np.zeros(13, dt_)
    eta, A, B = (np.zeros(g.w + 1, dt_) for _ in range(3))
    i2h = np.zeros(3, dt_)
    st = getattr(lib(), f"oracle_constants_{_sfx(dt_)}")(ctypes.byref(g), int(round32), _ptr(c),
                                                          _ptr(eta), _ptr(A), _ptr(B), _ptr(i2h))
    assert st == OK, st
    return {"c_xyz": c[0], "c_x": c[1:5], "c_y": c[5:9], "c_z": c[9:13],
            "eta": eta, "A": A, "B": B, "inv2h": i2h}


def vdt2(V: np.ndarray, dt: float, round32: bool = True, dtype=np.float32) -> np.ndarray:
    V = np.ascontiguousarray(V, dtype=np.float32)
    out = np.empty(V.shape, np.dtype(dtype))
    getattr(lib(), f"oracle_vdt2_{_sfx(dtype)}")(_ptr(V), V.size, float(np.float32(dt)),
                                                int(round32), _ptr(out))
    return out


def dt_auto(h, V: np.ndarray) -> np.float32:
    hx, hy, hz = (h, h, h) if np.isscalar(h) else tuple(h)
    V = np.ascontiguousarray(V, dtype=np.float32)
    return np.float32(lib().oracle_dt_auto(hx, hy, hz, _ptr(V), V.size))


def propagate(g: Geom, V: np.ndarray, wavelet: np.ndarray, T: int, src,
              u0: Optional[np.ndarray] = None, uprev0: Optional[np.ndarray] = None,
              dtype=np.float32, round32: bool = True, check_every: int = 0,
              eta: Optional[np.ndarray] = None):
    """Algorithm 1 for T steps on a full (single-slab) grid.

    Returns (u^T, u^{T-1}, status, fail_step) as dense [nz][ny][nx] arrays of
    `dtype`.  Inputs u0 = u^0 and uprev0 = u^{-1} default to zero.
    eta: None (the eta_max (d/w)^2 profile) or a user-supplied fp32 eta field
    [nz][ny][nx] (stored-eta variant, R16).
    """
    dt_ = np.dtype(dtype)
    shape = (g.nz, g.ny, g.nx)
    u = np.zeros(shape, dt_) if u0 is None else np.array(u0, dtype=dt_, order="C", copy=True)
    up = np.zeros(shape, dt_) if uprev0 is None else np.array(uprev0, dtype=dt_, order="C", copy=True)
    V = np.ascontiguousarray(V, dtype=np.float32)
    assert V.shape == shape, (V.shape, shape)
    wl = np.ascontiguousarray(wavelet, dtype=np.float32)
    if wl.size < T:
        wl = np.concatenate([wl, np.zeros(T - wl.size, np.float32)])
    fail = ctypes.c_int64(-1)
    si, sj, sk = (int(v) for v in src)
    if eta is not None:
        eta = np.ascontiguousarray(eta, dtype=np.float32)
        assert eta.shape == shape, (eta.shape, shape)
    st = getattr(lib(), f"oracle_propagate_eta_{_sfx(dt_)}")(
        ctypes.byref(g), int(round32), _ptr(V), None if eta is None else _ptr(eta), _ptr(wl), int(T),
        si, sj, sk, _ptr(u), _ptr(up), int(check_every), ctypes.byref(fail))
    return u, up, int(st), int(fail.value)


def pad(a: np.ndarray, dtype=None) -> np.ndarray:
    """Dense [nz][ny][nx] -> zero-padded [nz+8][ny+8][nx+8] (SPEC.md L31 layout)."""
    dt_ = a.dtype if dtype is None else np.dtype(dtype)
    out = np.zeros(tuple(n + 2 * R for n in a.shape), dt_)
    out[R:-R, R:-R, R:-R] = a
    return out


def unpad(p: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(p[R:-R, R:-R, R:-R])


def step_padded(g: Geom, u_pad: np.ndarray, up_pad: np.ndarray, vdt2_dense: np.ndarray,
                src, wn: float, round32: bool = True) -> int:
    """One Algorithm-1 step on a padded (slab) grid: up_pad <- u^{n+1} (+ source
    if the global source plane lies in this slab).  The z pad of u_pad carries
    the neighbouring slabs' planes (ghosts) or zeros at the global ends."""
    dt_ = u_pad.dtype
    assert up_pad.dtype == dt_ and vdt2_dense.dtype == dt_
    si, sj, sk = (int(v) for v in src)
    return int(getattr(lib(), f"oracle_step_{_sfx(dt_)}")(
        ctypes.byref(g), int(round32), _ptr(u_pad), _ptr(up_pad), _ptr(vdt2_dense),
        si, sj, sk, float(np.float32(wn))))
