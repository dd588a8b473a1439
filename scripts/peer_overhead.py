"""In-process cost of the fused peer-store halo exchange (development aid):
two z-slab plans of a 1024 x 1024 x 2048 grid (C5 at N = 2) stepped on their
own streams on ONE GPU with peer stores + device flags, vs the same two slabs
stepped without peers (independent plans), vs one plan of the whole grid.
On one GPU the two slabs share the SMs, so the comparison isolates the extra
work of the exchange (edge-plane stores, flag kernels, cross-stream waits)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2009_04619_b200.wave import WavePlan
from paper_2009_04619_b200.dist import slab_bounds

s = synth.scenario("C5")
s = s.with_(nz=s.nz * 2)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40


def mk(nzl, off, peer):
    p = WavePlan(s.nx, s.ny, nzl, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=off)
    p.set_velocity(synth.velocity(s, nz_global=s.nz, z_offset=off, nz_local=nzl))
    p.set_source(*s.source, synth.wavelet_for(s, 4 * steps + 20))
    return p


def timed(fn, side=()):
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for st in side:
        st.wait_stream(main)
    fn()
    for st in side:
        main.wait_stream(st)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


plans = []
for r in range(2):
    off, nzl = slab_bounds(s.nz, r, 2)
    p = mk(nzl, off, True)
    p.flags = torch.zeros(2, dtype=torch.int64, device="cuda")
    plans.append(p)
a, b = plans
a.set_peers(hi_bufs=b.bufs, hi_flags=b.flags)
b.set_peers(lo_bufs=a.bufs, lo_nz=a.nz, lo_flags=a.flags)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def peer_steps(n):
    a.step_peer(n, stream=sa)
    b.step_peer(n, stream=sb)


peer_steps(6)
ms_peer = timed(lambda: peer_steps(steps), side=(sa, sb))
for p in plans:
    p.close()
torch.cuda.empty_cache()
one = mk(s.nz, 0, False)
one.step(6)
ms_one = timed(lambda: one.step(steps))
print(f"2 slabs x 1024 planes, fused peer exchange, 2 streams: {ms_peer:.3f} ms/step")
print(f"1 plan of 2048 planes (no exchange):                   {ms_one:.3f} ms/step")
print(f"exchange overhead on one GPU: {100 * (ms_peer / ms_one - 1):.1f} %")
