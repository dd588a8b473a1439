"""Quick device timing of wave_step on a scenario (development aid):
python scripts/quick_time.py [C3] [stream|tb2|naive] [steps] [fp32|fp64]"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2009_04619_b200.wave import WavePlan

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
kernel = sys.argv[2] if len(sys.argv) > 2 else "stream"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
prec = sys.argv[4] if len(sys.argv) > 4 else "fp32"
s = synth.scenario(name)
p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel, precision=prec)
p.set_velocity(synth.velocity(s))
p.set_source(*s.source, synth.wavelet_for(s, 4000))
p.step(10)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); p.step(steps); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
pts = s.nx * s.ny * s.nz
bpp = 32 if prec == "fp64" else 16
print(f"{name} {kernel} {prec}: {ms:.4f} ms/step  {pts/ms/1e6:.1f} Gpt/s  {bpp*pts/ms/1e6:.1f} GB/s@{bpp}B  launches/step={p.launches_per_step}  maxabs={p.check_finite():.3e}")
