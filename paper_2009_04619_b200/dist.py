"""z-slab domain decomposition across GPUs (not in the paper,
which is single-GPU).

Two exchange paths:

* PeerSlabRunner (default): the exchange is fused into the compute.  Each
  rank maps its neighbours' wavefield buffers and flag words (CUDA IPC handles
  exported and opened by libwave25 on the rank's own device with lazy peer
  access; wave_set_peers enables peer access over NVLink / NVSwitch); the
  streaming kernels store the 4 edge planes of u_next
  straight into the neighbours' ghost planes as they compute them, and
  system-scope release/acquire step flags order consecutive steps
  (wave_step_peer).  torch.distributed is used only to swap the IPC handles
  at setup.
* SlabRunner: edges -> NCCL send/recv of the 4-plane blocks (overlapped with
  the interior kernel) -> join; the collective-library baseline.

The extended domain is cut into contiguous z-slabs, one per rank (z is the
outermost axis, so a slab face is one contiguous block of 4 planes).  Per time
step only u^n's 4 boundary planes cross ranks: u^{n-1} and vdt2 are read at
the centre only and eta is computed in-register.  The exchange is a pairwise
send/recv with no reduction:

    edges kernel (planes [0,4) and [nz-4,nz))  -> stream E
    send those planes to the neighbours' ghost planes, receive theirs
                                                  (NCCL over NVLink, after E)
    interior kernel (planes [4, nz-4))          -> stream I (overlaps the exchange)
    join, role swap

`slab_bounds` and `halo_exchange` are backend-agnostic (NCCL with CUDA
tensors, gloo with CPU tensors) so the decomposition logic is tested on CPU
with world_size 2 (tests/test_dist_cpu.py).
"""
from __future__ import annotations

from typing import Optional, Sequence

import torch
import torch.distributed as dist

GHOST = 4   # stencil radius R = 4


def slab_bounds(nz_global: int, rank: int, world: int) -> tuple[int, int]:
    """(z_offset, nz_local) of `rank`: near-equal contiguous slabs, the first
    nz_global % world ranks one plane thicker.  Every slab needs >= 4 planes so
    that its ghost planes come from one neighbour."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(nz_global, world)
    if base < GHOST:
        raise ValueError(f"nz_global={nz_global} too small for {world} slabs (need >= {GHOST} planes each)")
    nz = base + (1 if rank < extra else 0)
    off = rank * base + min(rank, extra)
    return off, nz


def halo_exchange(send_lo: Optional[torch.Tensor], send_hi: Optional[torch.Tensor],
                  recv_lo: Optional[torch.Tensor], recv_hi: Optional[torch.Tensor],
                  rank: int, world: int, group=None, stage_on_host: bool = False):
    """Send my lowest/highest 4 planes to rank-1 / rank+1 and receive theirs
    into my lower/upper ghost planes.  Returns the list of work handles
    (call .wait() on each).  With stage_on_host, CUDA blocks go through host
    copies (for gloo, which has no CUDA P2P)."""
    ops = []
    staged = []
    def _s(t):
        if stage_on_host and t.is_cuda:
            h = t.detach().cpu()
            return h
        return t
    def _r(t):
        if stage_on_host and t.is_cuda:
            h = torch.empty(t.shape, dtype=t.dtype)
            staged.append((h, t))
            return h
        return t
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, _s(send_lo), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, _r(recv_lo), rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, _s(send_hi), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, _r(recv_hi), rank + 1, group))
    if not ops:
        return []
    works = dist.batch_isend_irecv(ops)
    if staged:
        for wk in works:
            wk.wait()
        for h, t in staged:
            t.copy_(h)
        return []
    return works


class SlabRunner:
    """One rank's slab of a distributed run (NCCL, one process per GPU).

    The step is split so the halo exchange of the 4 edge planes overlaps the
    interior kernel: edges on `s_edge` -> NCCL send/recv (ordered after the
    edges by running under `s_edge`) while the interior runs on the current
    stream; both are joined before the role swap.
    """

    def __init__(self, plan, rank: int, world: int, group=None, stage_on_host: bool = False):
        self.plan = plan
        self.rank, self.world, self.group = rank, world, group
        self.stage_on_host = stage_on_host
        self.s_edge = torch.cuda.Stream(device=plan.device)

    def exchange_current(self) -> None:
        """Fill the ghost planes of the current u^n from the neighbours (needed
        once when the run starts from a non-zero state)."""
        if self.world == 1:
            return
        main = torch.cuda.current_stream(self.plan.device)
        send_lo, send_hi, recv_lo, recv_hi = self.plan.halo_views(1)
        works = halo_exchange(send_lo, send_hi, recv_lo, recv_hi, self.rank, self.world, self.group,
                              self.stage_on_host)
        for wk in works:
            wk.wait()
        main.synchronize()

    def step(self, n: int = 1) -> None:
        main = torch.cuda.current_stream(self.plan.device)
        for _ in range(n):
            self.s_edge.wait_stream(main)
            self.plan.step_edges(stream=self.s_edge)
            if self.world > 1:
                send_lo, send_hi, recv_lo, recv_hi = self.plan.halo_views()
                with torch.cuda.stream(self.s_edge):
                    works = halo_exchange(send_lo, send_hi, recv_lo, recv_hi, self.rank, self.world,
                                          self.group, self.stage_on_host)
                    for wk in works:
                        wk.wait()      # makes s_edge wait for the NCCL kernels
            self.plan.step_interior(stream=main)
            main.wait_stream(self.s_edge)
            self.plan.step_finish()


class _PeerBuf:
    """A neighbour's device buffer mapped into this process (CUDA IPC, opened
    on this rank's device with lazy peer access); quacks like a tensor for
    WavePlan.set_peers (data_ptr())."""

    def __init__(self, desc, device):
        from . import _abi
        handle, offset = desc
        with torch.cuda.device(device):
            self.base, self.ptr = _abi.wave_ipc_import(handle, offset)

    def data_ptr(self) -> int:
        return self.ptr

    def release(self) -> None:
        from . import _abi
        if self.base:
            _abi.wave_ipc_release(self.base)
            self.base = self.ptr = 0


def _export(t: torch.Tensor):
    """(IPC handle, byte offset) of a CUDA tensor's memory."""
    from . import _abi
    with torch.cuda.device(t.device):
        return _abi.wave_ipc_export(t.data_ptr())


class PeerSlabRunner:
    """One rank's slab with the halo exchange fused into the compute kernels
    (peer stores over NVLink + device-side step flags); see the module doc."""

    def __init__(self, plan, rank: int, world: int, group=None):
        self.plan, self.rank, self.world, self.group = plan, rank, world, group
        if not hasattr(plan, "flags"):
            plan.flags = torch.zeros(2, dtype=torch.int64, device=plan.device)
        torch.cuda.synchronize(plan.device)
        mine = (_export(plan.bufs[0]), _export(plan.bufs[1]), _export(plan.flags), plan.nz)
        allv = [None] * world
        dist.all_gather_object(allv, mine, group=group)
        lo = allv[rank - 1] if rank > 0 else None
        hi = allv[rank + 1] if rank < world - 1 else None
        dev = plan.device
        self._lo = self._hi = None
        err = None
        try:
            self._lo = (_PeerBuf(lo[0], dev), _PeerBuf(lo[1], dev), _PeerBuf(lo[2], dev), lo[3]) if lo else None
            self._hi = (_PeerBuf(hi[0], dev), _PeerBuf(hi[1], dev), _PeerBuf(hi[2], dev), hi[3]) if hi else None
            plan.set_peers(lo_bufs=self._lo[:2] if self._lo else None,
                           hi_bufs=self._hi[:2] if self._hi else None,
                           lo_nz=self._lo[3] if self._lo else 0, lo_flags=self._lo[2] if self._lo else None,
                           hi_flags=self._hi[2] if self._hi else None)
        except Exception as e:          # e.g. no P2P path between two GPUs
            err = e
        # every rank learns whether every rank is wired (a collective all reach,
        # so a failure on one rank cannot leave the others waiting)
        flag = torch.tensor([0 if err else 1], dtype=torch.int32,
                            device=plan.device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag.item()) == 0:
            self._unwire()
            raise RuntimeError(f"peer wiring failed on at least one rank (this rank: {err!r})")
        self._barrier()

    def _unwire(self) -> None:
        try:
            self.plan.clear_peers()
        finally:
            for side in (self._lo, self._hi):
                if side:
                    for b in side[:3]:
                        if isinstance(b, _PeerBuf):
                            b.release()
            self._lo = self._hi = None

    def close(self) -> None:
        """Unwire the plan and unmap the neighbours' buffers (collective: every
        rank calls it after its last step; the barrier keeps each mapping alive
        until no rank can still be storing through it)."""
        self._barrier()
        self._unwire()

    def _barrier(self):
        torch.cuda.synchronize(self.plan.device)
        dist.barrier(group=self.group)

    def exchange_current(self) -> None:
        """Push the current u^n edge planes into the neighbours' ghosts (once,
        for a non-zero starting state)."""
        self.plan.push_halo(1)
        self._barrier()

    def reset(self, uprev=None, ucur=None, velocity=None, source=None) -> None:
        """Collective re-initialisation of the wired run (every rank calls it).

        barrier (no rank is still stepping or storing into a neighbour's
        ghost planes) -> each rank installs the new velocity / source / state;
        wave_set_state zeroes the ghost planes and restarts the step-flag
        protocol (done count, flag words, peer-wait error word) -> barrier
        (every memset has landed before any neighbour writes into the ghosts)
        -> push the new u^0 edge planes into the neighbours' ghosts -> barrier.
        source = (i, j, k, wavelet) in global coordinates."""
        self._barrier()
        if velocity is not None:
            self.plan.set_velocity(velocity)
        if source is not None:
            self.plan.set_source(*source)
        self.plan.set_state(uprev, ucur)
        self._barrier()
        if ucur is not None:
            self.plan.push_halo(1)
        self._barrier()

    def check(self) -> None:
        """Raise (WAVE_ERR_PEER) if a peer wait of this rank expired."""
        self.plan.peer_check()

    def step(self, n: int = 1) -> None:
        self.plan.step_peer(n)
