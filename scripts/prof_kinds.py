"""Per-kernel-kind device times of a plan (development aid): python scripts/prof_kinds.py C3 tb2 [steps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2009_04619_b200.wave import WavePlan

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
kernel = sys.argv[2] if len(sys.argv) > 2 else "stream"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
prec = sys.argv[4] if len(sys.argv) > 4 else "fp32"
s = synth.scenario(name)
p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel, precision=prec)
if os.environ.get("PROF_ETA"):
    import numpy as np
    def d1(n):
        i = np.arange(n)
        return np.maximum(np.maximum(s.w - i, 0), i - (n - s.w - 1))
    d = np.maximum(np.maximum(d1(s.nx)[None, None, :], d1(s.ny)[None, :, None]), d1(s.nz)[:, None, None])
    p.set_eta((s.eta_max * (d / s.w) ** 2).astype(np.float32))
p.set_velocity(synth.velocity(s))
p.set_source(*s.source, synth.wavelet_for(s, 4000))
p.step(4)
p.step_profiled(2)
ms, n = p.step_profiled(steps)
pts = p.kernel_points()
print(f"{name} {kernel} steps/launch={p.steps_per_launch}")
for k in ms:
    if n[k]:
        print(f"  {k:9s} {ms[k]/steps:8.4f} ms/step  launches={n[k]}  {ms[k]/n[k]:.4f} ms/launch  points/step={pts[k]}")
print(f"  total    {sum(ms.values())/steps:8.4f} ms/step (serialized)")
