"""Small end-to-end runs for compute-sanitizer (development aid): C1 and RAGGED
geometries, stream + naive kernels, graph replay, slab split path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2009_04619_b200.wave import WavePlan

for name, kw in [("C1", {}), ("RAGGED", {}), ("RAGGED", dict(nx=9, ny=11, nz=10, w=2, src=(4, 5, 5)))]:
    s = synth.scenario(name, **kw)
    for kernel in ("stream", "naive"):
        p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel)
        p.set_velocity(synth.velocity(s))
        p.set_source(*s.source, synth.wavelet_for(s, 8))
        p.set_state(None, synth.random_state((s.nz, s.ny, s.nx), 1))
        p.step(5)
        p.check_finite()
        _ = p.read(0).cpu()
        p.close()
# slab split path
s = synth.scenario("RAGGED")
p = WavePlan(s.nx, s.ny, 30, s.w, s.h, s.dt, s.eta_max, nz_global=s.nz, z_offset=0)
p.set_velocity(synth.velocity(s)[:30])
p.set_source(*s.source, synth.wavelet_for(s, 8))
for _ in range(3):
    p.step_edges(); p.step_interior(); p.step_finish()
torch.cuda.synchronize()
p.close()
print("sanitize_run done")
