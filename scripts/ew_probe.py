"""Embedded-wall timing probe (development aid): step time plus the wall
warps' per-plane time during the interior vs in the last wave's mop-up
(WAVE25_EW_DBG=1 counters, printed at plan close).
python scripts/ew_probe.py C3 50"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("WAVE25_EW", "1")
os.environ.setdefault("WAVE25_EW_DBG", "1")
import torch
import synth
from paper_2009_04619_b200.wave import WavePlan

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
s = synth.scenario(name)
p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
p.set_velocity(synth.velocity(s))
p.set_source(*s.source, synth.wavelet_for(s, 4000))
p.step(4)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); p.step(steps); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"{name} EW {' '.join(k + '=' + v for k, v in sorted(os.environ.items()) if k.startswith('WAVE25_'))}: "
      f"{ms:.4f} ms/step {s.nx * s.ny * s.nz / ms / 1e6:.1f} Gpt/s", flush=True)
p.close()
