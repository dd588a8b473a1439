"""Multi-GPU z-slab host logic on CPU: slab bounds, and a world_size-2 gloo run
in which each rank steps its slab with the oracle and exchanges the 4-plane
halos with paper_2009_04619_b200.dist.halo_exchange -- the result must be
bitwise equal to the single-grid oracle run (SURVEY.md §4 "N-GPU = 1-GPU")."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_04619_b200.dist import slab_bounds, halo_exchange


def test_slab_bounds_partition():
    for nzg in (8, 9, 33, 64, 1000, 1024):
        for world in (1, 2, 3, 4, 8):
            if nzg // world < 4:
                with pytest.raises(ValueError):
                    slab_bounds(nzg, 0, world)
                continue
            covered = []
            for r in range(world):
                off, n = slab_bounds(nzg, r, world)
                assert n >= 4
                covered.extend(range(off, off + n))
            assert covered == list(range(nzg))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sname, steps, out_q):
    import oracle
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = synth.scenario(sname)
        off, nzl = slab_bounds(s.nz, rank, world)
        g = oracle.make_geom(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
        V = synth.velocity(s, nz_global=s.nz, z_offset=off, nz_local=nzl)
        vd = oracle.vdt2(V, s.dt)
        full_u0 = synth.random_state((s.nz, s.ny, s.nx), 5)
        full_um1 = synth.random_state((s.nz, s.ny, s.nx), 6)
        wl = synth.wavelet_for(s, steps)
        R = 4
        # padded slabs; z pads carry the neighbours' planes (initial halo)
        def padded(full):
            p = np.zeros((nzl + 8, s.ny + 8, s.nx + 8), np.float32)
            lo, hi = max(off - R, 0), min(off + nzl + R, s.nz)
            p[lo - (off - R):hi - (off - R), R:-R, R:-R] = full[lo:hi]
            return p
        u, up = padded(full_u0), padded(full_um1)
        for n in range(steps):
            st = oracle.step_padded(g, u, up, vd, s.source, wl[n])
            assert st == 0
            # up now holds u^{n+1}; exchange its 4 edge planes into the ghosts
            T = torch.from_numpy(up)
            works = halo_exchange(T[R:2 * R], T[nzl:nzl + R], T[0:R], T[nzl + R:nzl + 2 * R],
                                  rank, world)
            for wk in works:
                wk.wait()
            u, up = up, u
        out_q.put((rank, off, nzl, np.ascontiguousarray(u[R:-R, R:-R, R:-R])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sname,world", [("RAGGED", 2), ("C1", 2)])
def test_two_rank_gloo_slabs_equal_single_grid(oracle_lib, sname, world):
    import oracle
    import synth
    steps = 12
    s = synth.scenario(sname)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sname, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts.sort()
    got = np.concatenate([p[3] for p in parts], axis=0)
    g = oracle.make_geom(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    ref, _, st, _ = oracle.propagate(g, synth.velocity(s), synth.wavelet_for(s, steps), steps, s.source,
                                     u0=synth.random_state((s.nz, s.ny, s.nx), 5),
                                     uprev0=synth.random_state((s.nz, s.ny, s.nx), 6))
    assert st == 0
    assert np.array_equal(got, ref)
