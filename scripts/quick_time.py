"""Quick device timing of wave_step on a scenario (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2009_04619_b200.wave import WavePlan

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
kernel = sys.argv[2] if len(sys.argv) > 2 else "stream"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
s = synth.scenario(name)
p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel)
p.set_velocity(synth.velocity(s))
p.set_source(*s.source, synth.wavelet_for(s, 4000))
p.step(10)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); p.step(steps); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
pts = s.nx * s.ny * s.nz
print(f"{name} {kernel}: {ms:.4f} ms/step  {pts/ms/1e6:.1f} Gpt/s  {16*pts/ms/1e6:.1f} GB/s@16B  launches/step={p.launches_per_step}  maxabs={p.check_finite():.3e}")
