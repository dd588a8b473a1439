import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_2009_04619_b200.wave import WavePlan
which = sys.argv[1]
for name, kw in [("C1", {}), ("RAGGED", {}), ("RAGGED", dict(nx=9, ny=11, nz=10, w=2, src=(4, 5, 5)))]:
    s = synth.scenario(name, **kw)
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=which)
    p.set_velocity(synth.velocity(s)); p.set_source(*s.source, synth.wavelet_for(s, 8))
    p.set_state(None, synth.random_state((s.nz, s.ny, s.nx), 1)); p.step(4); p.check_finite(); p.close()
print("done", which)
