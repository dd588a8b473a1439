"""Bitwise check of an env variant against the default path on a full-size
scenario from a random O(1) state (every wall point active), development aid:
python scripts/ew_check.py C2 8 WAVE25_EW=1 [WAVE25_EW_CZ=16 ...]   (CHECK_PREC=fp64: an fp64 plan)"""
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BODY = r"""
import hashlib, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, synth
from paper_2009_04619_b200.wave import WavePlan
s = synth.scenario(sys.argv[2]); n = int(sys.argv[3])
sh = (s.nz, s.ny, s.nx)
import os
prec = os.environ.get("CHECK_PREC", "fp32")
p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, precision=prec)
p.set_velocity(synth.velocity(s))
p.set_source(*s.source, synth.wavelet_for(s, n))
g = torch.Generator(device="cuda").manual_seed(7)
dt_ = torch.float64 if prec == "fp64" else torch.float32
um1 = torch.rand(sh, generator=g, device="cuda", dtype=dt_) - 0.5
u0 = torch.rand(sh, generator=g, device="cuda", dtype=dt_) - 0.5
p.set_state(um1, u0)
p.step(n)
a = p.read(0).cpu().numpy(); b = p.read(1).cpu().numpy()
print(hashlib.sha256(a.tobytes() + b.tobytes()).hexdigest(), float(np.abs(a).max()))
"""
name, n, envs = sys.argv[1], sys.argv[2], sys.argv[3:]
base = {k: v for k, v in os.environ.items() if not k.startswith("WAVE25_")}
ref = subprocess.run([sys.executable, "-c", BODY, ROOT, name, n], env=base, capture_output=True, text=True)
var = dict(base)
for e in envs:
    k, v = e.split("=", 1)
    var[k] = v
got = subprocess.run([sys.executable, "-c", BODY, ROOT, name, n], env=var, capture_output=True, text=True)
ok = ref.returncode == 0 and got.returncode == 0 and ref.stdout.split()[:1] == got.stdout.split()[:1]
print(f"{name} {n} steps {' '.join(envs)}: {'BITWISE EQUAL' if ok else 'DIFFERENT'}  ref={ref.stdout.strip()[:20]} got={got.stdout.strip()[:20]}")
if not ok:
    print(ref.stderr[-2000:], got.stderr[-2000:])
sys.exit(0 if ok else 1)
