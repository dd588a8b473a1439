"""Timeline of one pair-kernel launch (development aid; WAVE25_PAIR_DBG=8 makes
the library record per-block start/end times and dump them at plan close to
./pair_timeline.txt): python scripts/pair_timeline.py [C3]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["WAVE25_PAIR_DBG"] = os.environ.get("WAVE25_PAIR_DBG", "8")
import torch
import synth
from paper_2009_04619_b200.wave import WavePlan

s = synth.scenario(sys.argv[1] if len(sys.argv) > 1 else "C3")
p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel="pair")
p.set_velocity(synth.velocity(s))
p.set_source(*s.source, synth.wavelet_for(s, 100))
p.step(6)
torch.cuda.synchronize()
p.close()
