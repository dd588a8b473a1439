import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2009_04619_b200.wave import WavePlan
s = synth.scenario("C1")
p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=os.environ.get("K", "tb2"))
p.set_velocity(synth.velocity(s))
p.set_source(*s.source, synth.wavelet_for(s, 8))
p.set_state(None, synth.random_state((s.nz, s.ny, s.nx), 1))
p.step(2)
torch.cuda.synchronize()
p.close()
print("done")
