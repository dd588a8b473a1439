"""WavePlan: torch-owned device buffers + the C ABI (marshalling only).

PyTorch provides device memory and streams; every step of the method runs in
libwave25.so's CUDA kernels (include/wave.h).  Arrays passed in are copied to
the device by the library (host pointers) or read in place (device tensors).
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _abi


def _stream_handle(stream: Optional[torch.cuda.Stream]) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def _as_input(a, shape, device, dtype=torch.float32):
    """Return (pointer, where, keepalive) for a dense array of `shape` and `dtype`."""
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"shape {tuple(t.shape)} != {tuple(shape)}")
        t = t.to(dtype=dtype).contiguous()
        if t.is_cuda:
            if t.device != device:
                t = t.to(device)
            return t.data_ptr(), _abi.WAVE_MEM_DEVICE, t
        return t.data_ptr(), _abi.WAVE_MEM_HOST, t
    arr = np.ascontiguousarray(a, dtype=np.float64 if dtype == torch.float64 else np.float32)
    if arr.shape != tuple(shape):
        raise ValueError(f"shape {arr.shape} != {tuple(shape)}")
    return arr.ctypes.data, _abi.WAVE_MEM_HOST, arr


class WavePlan:
    """One grid (or one z-slab of a grid) on one GPU.

    nx, ny, nz   extended extents of this plan (nz = slab planes)
    w            PML width;  h spacing (scalar or (hx, hy, hz));  dt (0 = auto)
    eta_max      PML damping maximum (1/s);  kernel "stream" | "naive" | "tb2"
                 ("tb2": two-step temporal blocking, 4 wavefield buffers)
    nz_global, z_offset   slab position (defaults: single slab)
    precision    "fp32" (default) or "fp64" (wavefields, vdt2 and arithmetic in
                 double; the velocity and wavelet are still given in fp32)
    """

    def __init__(self, nx, ny, nz, w, h, dt, eta_max=4.0, kernel="stream",
                 nz_global=None, z_offset=0, device=None, stream=None, precision="fp32"):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        kern = {"stream": _abi.WAVE_KERNEL_STREAM, "naive": _abi.WAVE_KERNEL_NAIVE,
                "tb2": _abi.WAVE_KERNEL_TB2, "pair": _abi.WAVE_KERNEL_PAIR}[kernel]
        prec = {"fp32": _abi.WAVE_PREC_FP32, "fp64": _abi.WAVE_PREC_FP64}[precision]
        self.dtype = torch.float64 if prec == _abi.WAVE_PREC_FP64 else torch.float32
        self.desc = _abi.make_desc(nx, ny, nz, w, h, float(np.float32(dt)), eta_max, kern,
                                   nz_global, z_offset, prec)
        self.layout = _abi.wave_layout(self.desc)
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.shape = (self.nz, self.ny, self.nx)
        self._plan = None
        with torch.cuda.device(self.device):
            L = self.layout
            nb = 4 if kern == _abi.WAVE_KERNEL_TB2 else 2
            self.bufs = [torch.empty(L.elems_u, dtype=self.dtype, device=self.device) for _ in range(nb)]
            self.vdt2 = torch.empty(L.elems_vdt2, dtype=self.dtype, device=self.device)
            self._plan = _abi.wave_plan_create(self.desc)
            _abi.wave_plan_bind(self._plan, self.bufs[0].data_ptr(), self.bufs[1].data_ptr(),
                                self.vdt2.data_ptr(), _stream_handle(stream))
            if nb == 4:
                _abi.wave_plan_bind_aux(self._plan, self.bufs[2].data_ptr(), self.bufs[3].data_ptr(),
                                        _stream_handle(stream))
        self._keep = []

    # ---- inputs ---------------------------------------------------------
    def set_velocity(self, vel, stream=None) -> None:
        ptr, where, keep = _as_input(vel, self.shape, self.device)
        with torch.cuda.device(self.device):
            _abi.wave_set_velocity(self._plan, ptr, where, _stream_handle(stream))
        del keep

    def set_eta(self, eta, stream=None) -> None:
        """Stored (user-supplied) PML damping field eta [nz, ny, nx] (fp32, >= 0)
        instead of the eta_max (d/w)^2 profile; None returns to the profile.
        The plan allocates (once) the device buffer the field is copied into."""
        with torch.cuda.device(self.device):
            if eta is None:
                _abi.wave_set_eta(self._plan, None, _abi.WAVE_MEM_HOST, _stream_handle(stream))
                return
            if not hasattr(self, "eta_buf"):
                self.eta_buf = torch.empty(self.layout.elems_vdt2, dtype=torch.float32, device=self.device)
                _abi.wave_plan_bind_eta(self._plan, self.eta_buf.data_ptr(), _stream_handle(stream))
            ptr, where, keep = _as_input(eta, self.shape, self.device, torch.float32)
            _abi.wave_set_eta(self._plan, ptr, where, _stream_handle(stream))
            del keep

    def set_source(self, i, j, k, wavelet, stream=None) -> None:
        wl = np.ascontiguousarray(np.asarray(wavelet, dtype=np.float32).ravel())
        with torch.cuda.device(self.device):
            _abi.wave_set_source(self._plan, i, j, k, wl.ctypes.data, wl.size, _stream_handle(stream))

    def set_state(self, uprev=None, ucur=None, stream=None) -> None:
        """Initial u^{-1} / u^0 (None = zero); both host or both device arrays."""
        given = [a for a in (uprev, ucur) if a is not None]
        conv = [_as_input(a, self.shape, self.device, self.dtype) for a in given]
        if len({c[1] for c in conv}) > 1:
            raise ValueError("uprev and ucur must both be host or both device arrays")
        where = conv[0][1] if conv else _abi.WAVE_MEM_HOST
        it = iter(conv)
        ptrs = [None if a is None else next(it)[0] for a in (uprev, ucur)]
        with torch.cuda.device(self.device):
            _abi.wave_set_state(self._plan, ptrs[0], ptrs[1], where, _stream_handle(stream))
        del conv

    # ---- stepping -------------------------------------------------------
    def step(self, n: int = 1, stream=None) -> None:
        with torch.cuda.device(self.device):
            _abi.wave_step(self._plan, n, _stream_handle(stream))

    def step_edges(self, stream=None) -> None:
        _abi.wave_step_edges(self._plan, _stream_handle(stream))

    def step_interior(self, stream=None) -> None:
        _abi.wave_step_interior(self._plan, _stream_handle(stream))

    def step_finish(self) -> None:
        _abi.wave_step_finish(self._plan)

    # ---- fused peer-store halo exchange ----------------------------------
    def set_peers(self, lo_bufs=None, hi_bufs=None, lo_nz: int = 0, lo_flags=None, hi_flags=None) -> None:
        """Wire the z-neighbours for step_peer: their two wavefield buffers and
        flag words (torch tensors, or anything with data_ptr() -- e.g. the
        IPC mappings of dist.PeerSlabRunner -- on this or a peer device); None
        where there is no neighbour.  Allocates this plan's zeroed flag words."""
        if not hasattr(self, "flags"):
            self.flags = torch.zeros(2, dtype=torch.int64, device=self.device)
        else:
            self.flags.zero_()
        pe = _abi.WavePeers()
        if lo_bufs is not None:
            pe.lo_buf[0], pe.lo_buf[1] = lo_bufs[0].data_ptr(), lo_bufs[1].data_ptr()
            pe.lo_flags = lo_flags.data_ptr()
        if hi_bufs is not None:
            pe.hi_buf[0], pe.hi_buf[1] = hi_bufs[0].data_ptr(), hi_bufs[1].data_ptr()
            pe.hi_flags = hi_flags.data_ptr()
        pe.lo_nz = int(lo_nz)
        pe.my_flags = self.flags.data_ptr()
        self._peer_refs = (lo_bufs, hi_bufs, lo_flags, hi_flags)
        torch.cuda.synchronize(self.device)
        with torch.cuda.device(self.device):
            _abi.wave_set_peers(self._plan, pe)

    def clear_peers(self) -> None:
        """Remove the neighbour wiring (before the neighbours' mappings go away)."""
        with torch.cuda.device(self.device):
            _abi.wave_set_peers(self._plan, None)
        self._peer_refs = None

    def step_peer(self, n: int = 1, stream=None) -> None:
        with torch.cuda.device(self.device):
            _abi.wave_step_peer(self._plan, n, _stream_handle(stream))

    def set_peer_timeout(self, seconds: float) -> None:
        """Bound of each peer wait (device time); an expired wait is reported
        by peer_check, it never traps."""
        with torch.cuda.device(self.device):
            _abi.wave_set_peer_timeout(self._plan, seconds)

    def peer_check(self, stream=None) -> None:
        """Synchronise and raise if any peer wait expired (results invalid)."""
        with torch.cuda.device(self.device):
            _abi.wave_peer_check(self._plan, _stream_handle(stream))

    def push_halo(self, which: int = 1, stream=None) -> None:
        with torch.cuda.device(self.device):
            _abi.wave_push_halo(self._plan, which, _stream_handle(stream))

    # ---- outputs --------------------------------------------------------
    def _buffer_view(self, ptr: int) -> torch.Tensor:
        L = self.layout
        for b in self.bufs:
            off = ptr - b.data_ptr()
            es = b.element_size()
            if 0 <= off < b.numel() * es:
                start = off // es
                v = b[start:start + self.nz * self.ny * L.pitch_x]
                return v.view(self.nz, self.ny, L.pitch_x)[:, :, :self.nx]
        raise RuntimeError("field pointer outside the plan's buffers")

    def field(self, which: int = 0) -> torch.Tensor:
        """Zero-copy [nz, ny, nx] view of u^n (which=0) or u^{n-1} (which=1)."""
        return self._buffer_view(_abi.wave_field_ptr(self._plan, which))

    def read(self, which: int = 0, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Dense copy of u^n / u^{n-1}; `out` may be a CUDA or (pinned) CPU tensor."""
        if out is None:
            out = torch.empty(self.shape, dtype=self.dtype, device=self.device)
        if out.dtype != self.dtype:
            raise ValueError(f"out must be {self.dtype}")
        where = _abi.WAVE_MEM_DEVICE if out.is_cuda else _abi.WAVE_MEM_HOST
        with torch.cuda.device(self.device):
            _abi.wave_read(self._plan, which, out.data_ptr(), where, _stream_handle(stream))
        return out

    def halo_views(self, which: int = 0):
        """(send_lo, send_hi, recv_lo, recv_hi) torch views of 4-plane blocks;
        which = 0: in the buffer the edges step writes, 1: in the current u^n."""
        a, b, c, d, n = _abi.wave_halo_views(self._plan, which)
        out = []
        for p in (a, b, c, d):
            for buf in self.bufs:
                off = p - buf.data_ptr()
                es = buf.element_size()
                if 0 <= off < buf.numel() * es:
                    out.append(buf[off // es: off // es + n])
                    break
        return tuple(out)

    def check_finite(self, stream=None) -> float:
        with torch.cuda.device(self.device):
            return _abi.wave_check_finite(self._plan, _stream_handle(stream))

    @property
    def step_index(self) -> int:
        return _abi.wave_step_index(self._plan)

    @property
    def dt(self) -> float:
        return _abi.wave_get_dt(self._plan)

    @property
    def launches_per_step(self) -> int:
        return _abi.wave_launches_per_step(self._plan)

    def launches(self, nsteps: int) -> int:
        """Exact number of kernel launches step(nsteps) enqueues from the current state."""
        return _abi.wave_launches(self._plan, nsteps)

    @property
    def fastdiv(self) -> bool:
        """True when the PML divisions use the verified table reciprocal (wave_fastdiv)."""
        return _abi.wave_fastdiv(self._plan) == 1

    @property
    def steps_per_launch(self) -> int:
        """2 when step() runs two-step temporal blocking, else 1."""
        return _abi.wave_steps_per_launch(self._plan)

    def kernel_points(self) -> dict:
        return _abi.wave_kernel_points(self._plan)

    def step_profiled(self, n: int, stream=None):
        """n steps with a CUDA event pair around every kernel launch (each on
        its launching stream); returns ({kind: ms summed}, {kind: launches})."""
        with torch.cuda.device(self.device):
            return _abi.wave_step_profiled(self._plan, n, _stream_handle(stream))

    def close(self) -> None:
        if self._plan is not None:
            torch.cuda.synchronize(self.device)
            _abi.wave_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            if self._plan is not None:
                _abi.wave_plan_destroy(self._plan)
                self._plan = None
        except Exception:
            pass
