"""ctypes binding of include/wave.h -- argument marshalling only.

Every function here has the name of the C entry point it calls and does no
arithmetic of the method: all of the time step runs in the CUDA kernels of
libwave25.so.  There is no CPU fallback: if the library is missing, importing
`lib()` raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libwave25.so")
# A/B measurement builds only (e.g. the scalar-arithmetic build of
# scripts/build_variant.sh): another in-tree library of the same ABI
if os.environ.get("WAVE25_LIB"):
    LIB_PATH = os.path.join(HERE, os.path.basename(os.environ["WAVE25_LIB"]))

(WAVE_OK, WAVE_ERR_CONFIG, WAVE_ERR_UNSTABLE, WAVE_ERR_VERIFY, WAVE_ERR_CUDA, WAVE_ERR_ALLOC, WAVE_ERR_STATE,
 WAVE_ERR_PEER) = range(8)
STATUS_NAMES = {0: "WAVE_OK", 1: "WAVE_ERR_CONFIG", 2: "WAVE_ERR_UNSTABLE", 3: "WAVE_ERR_VERIFY",
                4: "WAVE_ERR_CUDA", 5: "WAVE_ERR_ALLOC", 6: "WAVE_ERR_STATE", 7: "WAVE_ERR_PEER"}
WAVE_MEM_HOST, WAVE_MEM_DEVICE = 0, 1
WAVE_KERNEL_STREAM, WAVE_KERNEL_NAIVE, WAVE_KERNEL_TB2, WAVE_KERNEL_PAIR = 0, 1, 2, 3
WAVE_PREC_FP32, WAVE_PREC_FP64 = 0, 1
REGION_NAMES = ["inner", "top", "bottom", "front", "back", "left", "right"]

EXPORTS = [
    "wave_version", "wave_last_error", "wave_layout", "wave_decompose", "wave_constants",
    "wave_plan_create", "wave_plan_bind", "wave_plan_destroy", "wave_set_velocity",
    "wave_set_source", "wave_set_state", "wave_step", "wave_step_edges", "wave_step_interior",
    "wave_step_finish", "wave_halo_views", "wave_read", "wave_field_ptr", "wave_check_finite",
    "wave_step_index", "wave_get_dt", "wave_launches_per_step", "wave_kernel_points",
    "wave_step_profiled", "wave_set_peers", "wave_step_peer", "wave_push_halo",
    "wave_plan_bind_aux", "wave_launches", "wave_steps_per_launch", "wave_plan_bind_eta", "wave_set_eta",
    "wave_ipc_export", "wave_ipc_import", "wave_ipc_release", "wave_set_peer_timeout", "wave_peer_check",
    "wave_division_table", "wave_fastdiv",
]
KERNEL_KINDS = ["interior", "xwalls", "ywalls", "source"]


class WaveDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("pml_width", ctypes.c_int32), ("kernel", ctypes.c_int32),
                ("hx", ctypes.c_double), ("hy", ctypes.c_double), ("hz", ctypes.c_double),
                ("dt", ctypes.c_float), ("precision", ctypes.c_int32),
                ("eta_max", ctypes.c_double),
                ("nz_global", ctypes.c_int64), ("z_offset", ctypes.c_int64)]


class WaveLayout(ctypes.Structure):
    _fields_ = [("pitch_x", ctypes.c_int64), ("ghost_z", ctypes.c_int64), ("planes", ctypes.c_int64),
                ("elems_u", ctypes.c_int64), ("elems_vdt2", ctypes.c_int64), ("align_bytes", ctypes.c_int64),
                ("elem_bytes", ctypes.c_int64), ("origin", ctypes.c_int64), ("seam", ctypes.c_int64)]


class WaveRegion(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("lo", ctypes.c_int64 * 3), ("ext", ctypes.c_int64 * 3)]


class WavePeers(ctypes.Structure):
    _fields_ = [("lo_buf", ctypes.c_void_p * 2), ("hi_buf", ctypes.c_void_p * 2), ("lo_nz", ctypes.c_int64),
                ("my_flags", ctypes.c_void_p), ("lo_flags", ctypes.c_void_p), ("hi_flags", ctypes.c_void_p)]


class WaveError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load libwave25.so (build it with __graft_entry__.build()).  Raises if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: the CUDA library must be built "
                                  "(python -c 'import __graft_entry__ as g; g.build()'); "
                                  "there is no CPU fallback")
            L = ctypes.CDLL(LIB_PATH)
            P, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
            DP = ctypes.POINTER(WaveDesc)
            sig = {
                "wave_version": ([], ctypes.c_char_p),
                "wave_last_error": ([], ctypes.c_char_p),
                "wave_layout": ([DP, ctypes.POINTER(WaveLayout)], i32),
                "wave_decompose": ([DP, ctypes.POINTER(WaveRegion)], i32),
                "wave_constants": ([DP, P, P, P, P, P], i32),
                "wave_plan_create": ([DP, ctypes.POINTER(P)], i32),
                "wave_plan_bind": ([P, P, P, P, P], i32),
                "wave_plan_destroy": ([P], None),
                "wave_set_velocity": ([P, P, i32, P], i32),
                "wave_set_source": ([P, i64, i64, i64, P, i64, P], i32),
                "wave_set_state": ([P, P, P, i32, P], i32),
                "wave_step": ([P, i64, P], i32),
                "wave_step_edges": ([P, P], i32),
                "wave_step_interior": ([P, P], i32),
                "wave_step_finish": ([P], i32),
                "wave_halo_views": ([P, i32, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P),
                                     ctypes.POINTER(P), ctypes.POINTER(i64)], i32),
                "wave_read": ([P, i32, P, i32, P], i32),
                "wave_field_ptr": ([P, i32, ctypes.POINTER(P)], i32),
                "wave_check_finite": ([P, ctypes.POINTER(f32), P], i32),
                "wave_step_index": ([P], i64),
                "wave_get_dt": ([P], f32),
                "wave_launches_per_step": ([P], i32),
                "wave_kernel_points": ([P, P], i32),
                "wave_step_profiled": ([P, i64, P, P, P], i32),
                "wave_set_peers": ([P, ctypes.POINTER(WavePeers)], i32),
                "wave_step_peer": ([P, i64, P], i32),
                "wave_push_halo": ([P, i32, P], i32),
                "wave_plan_bind_aux": ([P, P, P, P], i32),
                "wave_launches": ([P, i64], i64),
                "wave_steps_per_launch": ([P], i32),
                "wave_plan_bind_eta": ([P, P, P], i32),
                "wave_set_eta": ([P, P, i32, P], i32),
                "wave_ipc_export": ([P, P, ctypes.POINTER(i64)], i32),
                "wave_ipc_import": ([P, i64, ctypes.POINTER(P), ctypes.POINTER(P)], i32),
                "wave_ipc_release": ([P], i32),
                "wave_set_peer_timeout": ([P, ctypes.c_double], i32),
                "wave_peer_check": ([P, P], i32),
                "wave_division_table": ([DP, P, P], i32),
                "wave_fastdiv": ([P], i32),
            }
            for name, (args, res) in sig.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
        return _lib


def check(status: int) -> None:
    if status != WAVE_OK:
        raise WaveError(status, lib().wave_last_error().decode(errors="replace"))


def make_desc(nx, ny, nz, pml_width, h, dt, eta_max=4.0, kernel=WAVE_KERNEL_STREAM,
              nz_global=None, z_offset=0, precision=WAVE_PREC_FP32) -> WaveDesc:
    hx, hy, hz = (h, h, h) if isinstance(h, (int, float)) else tuple(h)
    return WaveDesc(int(nx), int(ny), int(nz), int(pml_width), int(kernel), float(hx), float(hy),
                    float(hz), float(dt), int(precision), float(eta_max),
                    int(nz if nz_global is None else nz_global), int(z_offset))


# ---- thin wrappers, same names as the C ABI ------------------------------------------------

def wave_version() -> str:
    return lib().wave_version().decode()


def wave_layout(desc: WaveDesc) -> WaveLayout:
    out = WaveLayout()
    check(lib().wave_layout(ctypes.byref(desc), ctypes.byref(out)))
    return out


def wave_decompose(desc: WaveDesc):
    out = (WaveRegion * 7)()
    check(lib().wave_decompose(ctypes.byref(desc), out))
    return [dict(kind=REGION_NAMES[r.kind], lo=tuple(r.lo), ext=tuple(r.ext)) for r in out]


def wave_constants(desc: WaveDesc) -> dict:
    import numpy as np
    w = desc.pml_width
    c13 = np.zeros(13, np.float32)
    eta, A, B = (np.zeros(w + 1, np.float32) for _ in range(3))
    i2h = np.zeros(3, np.float32)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    check(lib().wave_constants(ctypes.byref(desc), p(c13), p(eta), p(A), p(B), p(i2h)))
    return {"c_xyz": c13[0], "c_x": c13[1:5], "c_y": c13[5:9], "c_z": c13[9:13],
            "eta": eta, "A": A, "B": B, "inv2h": i2h}


def wave_division_table(desc: WaveDesc):
    """(B[w+1], rB[w+1]): the PML divisors of an fp32 plan and their RN reciprocals."""
    import numpy as np
    w = desc.pml_width
    B, rB = np.zeros(w + 1, np.float32), np.zeros(w + 1, np.float32)
    check(lib().wave_division_table(ctypes.byref(desc), B.ctypes.data_as(ctypes.c_void_p),
                                    rB.ctypes.data_as(ctypes.c_void_p)))
    return B, rB


def wave_fastdiv(plan) -> int:
    return int(lib().wave_fastdiv(plan))


def wave_plan_create(desc: WaveDesc) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    check(lib().wave_plan_create(ctypes.byref(desc), ctypes.byref(h)))
    return h


def wave_plan_bind(plan, u0: int, u1: int, vdt2: int, stream: int) -> None:
    check(lib().wave_plan_bind(plan, u0, u1, vdt2, stream))


def wave_plan_bind_aux(plan, u2: int, u3: int, stream: int) -> None:
    check(lib().wave_plan_bind_aux(plan, u2, u3, stream))


def wave_plan_bind_eta(plan, eta_buf: int, stream: int) -> None:
    check(lib().wave_plan_bind_eta(plan, eta_buf, stream))


def wave_set_eta(plan, eta_ptr, where: int, stream: int) -> None:
    check(lib().wave_set_eta(plan, eta_ptr, where, stream))


def wave_launches(plan, nsteps: int) -> int:
    return int(lib().wave_launches(plan, int(nsteps)))


def wave_steps_per_launch(plan) -> int:
    return int(lib().wave_steps_per_launch(plan))


def wave_plan_destroy(plan) -> None:
    lib().wave_plan_destroy(plan)


def wave_set_velocity(plan, vel_ptr: int, where: int, stream: int) -> None:
    check(lib().wave_set_velocity(plan, vel_ptr, where, stream))


def wave_set_source(plan, i, j, k, wavelet_ptr: int, nsamples: int, stream: int) -> None:
    check(lib().wave_set_source(plan, int(i), int(j), int(k), wavelet_ptr, int(nsamples), stream))


def wave_set_state(plan, uprev_ptr, ucur_ptr, where: int, stream: int) -> None:
    check(lib().wave_set_state(plan, uprev_ptr, ucur_ptr, where, stream))


def wave_step(plan, nsteps: int, stream: int) -> None:
    check(lib().wave_step(plan, int(nsteps), stream))


def wave_step_edges(plan, stream: int) -> None:
    check(lib().wave_step_edges(plan, stream))


def wave_step_interior(plan, stream: int) -> None:
    check(lib().wave_step_interior(plan, stream))


def wave_step_finish(plan) -> None:
    check(lib().wave_step_finish(plan))


def wave_halo_views(plan, which: int = 0):
    a, b, c, d = (ctypes.c_void_p() for _ in range(4))
    n = ctypes.c_int64()
    check(lib().wave_halo_views(plan, int(which), ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                ctypes.byref(d), ctypes.byref(n)))
    return a.value, b.value, c.value, d.value, n.value


def wave_read(plan, which: int, dst_ptr: int, where: int, stream: int) -> None:
    check(lib().wave_read(plan, int(which), dst_ptr, where, stream))


def wave_field_ptr(plan, which: int) -> int:
    out = ctypes.c_void_p()
    check(lib().wave_field_ptr(plan, int(which), ctypes.byref(out)))
    return out.value


def wave_check_finite(plan, stream: int) -> float:
    v = ctypes.c_float()
    check(lib().wave_check_finite(plan, ctypes.byref(v), stream))
    return v.value


def wave_step_index(plan) -> int:
    return int(lib().wave_step_index(plan))


def wave_get_dt(plan) -> float:
    return float(lib().wave_get_dt(plan))


def wave_launches_per_step(plan) -> int:
    return int(lib().wave_launches_per_step(plan))


def wave_kernel_points(plan) -> dict:
    import numpy as np
    out = np.zeros(4, np.int64)
    check(lib().wave_kernel_points(plan, out.ctypes.data))
    return dict(zip(KERNEL_KINDS, (int(v) for v in out)))


def wave_step_profiled(plan, nsteps: int, stream: int):
    """Returns ({kind: summed ms}, {kind: launches}) over nsteps profiled steps."""
    import numpy as np
    ms = np.zeros(4, np.float64)
    n = np.zeros(4, np.int64)
    check(lib().wave_step_profiled(plan, int(nsteps), stream, ms.ctypes.data, n.ctypes.data))
    return dict(zip(KERNEL_KINDS, (float(v) for v in ms))), dict(zip(KERNEL_KINDS, (int(v) for v in n)))


def wave_set_peers(plan, peers) -> None:
    """peers: WavePeers or None (clears)."""
    check(lib().wave_set_peers(plan, ctypes.byref(peers) if peers is not None else None))


def wave_step_peer(plan, nsteps: int, stream: int) -> None:
    check(lib().wave_step_peer(plan, int(nsteps), stream))


def wave_push_halo(plan, which: int, stream: int) -> None:
    check(lib().wave_push_halo(plan, int(which), stream))


def wave_set_peer_timeout(plan, seconds: float) -> None:
    check(lib().wave_set_peer_timeout(plan, float(seconds)))


def wave_peer_check(plan, stream: int) -> None:
    """Raises WaveError(WAVE_ERR_PEER) if a peer wait of this plan expired."""
    check(lib().wave_peer_check(plan, stream))


def wave_ipc_export(dptr: int) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding dptr, byte offset of dptr in it)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    check(lib().wave_ipc_export(ctypes.c_void_p(dptr), h, ctypes.byref(off)))
    return h.raw, int(off.value)


def wave_ipc_import(handle: bytes, offset: int) -> tuple[int, int]:
    """Map another process's exported allocation on the current device: (base, dptr)."""
    if len(handle) != 64:
        raise ValueError("CUDA IPC handles are 64 bytes")
    base, ptr = ctypes.c_void_p(), ctypes.c_void_p()
    check(lib().wave_ipc_import(handle, int(offset), ctypes.byref(base), ctypes.byref(ptr)))
    return int(base.value), int(ptr.value)


def wave_ipc_release(base: int) -> None:
    check(lib().wave_ipc_release(ctypes.c_void_p(base)))
