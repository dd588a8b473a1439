import os, subprocess, sys
import numpy as np
script = r'''
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2009_04619_b200.wave import WavePlan
s = synth.scenario("RAGGED")
sh = (s.nz, s.ny, s.nx)
mode = sys.argv[2]
for t in range(int(sys.argv[3])):
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max)
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, 12))
    p.set_state(synth.random_state(sh, 41), synth.random_state(sh, 42))
    if mode == "single":
        for n in range(12): p.step(1)
    elif mode == "graph":
        p.step(12)
    elif mode == "graphsync":
        for n in range(6): p.step(2); torch.cuda.synchronize()
    np.save(f"/tmp/r_{sys.argv[1]}_{t}.npy", p.read(0).cpu().numpy())
    p.close()
'''
base = {k: v for k, v in os.environ.items() if not k.startswith("WAVE25_")}
N = 30
subprocess.run([sys.executable, "-c", script, "ref", "graph", "1"], env={**base, "WAVE25_SERIAL": "1"}, check=True)
ref = np.load("/tmp/r_ref_0.npy")
for mode in ("single", "graph", "gsingle", "ggraph"):
    extra = {"WAVE25_GMAPS": "1"} if mode.startswith("g") and mode != "graph" else {}
    m = {"gsingle": "single", "ggraph": "graph"}.get(mode, mode)
    subprocess.run([sys.executable, "-c", script, "gm" + mode, m, str(N)], env={**base, "WAVE25_ABLATION": "gmem_8x8x8", **extra}, check=True)
    nbad = sum(1 for t in range(N) if not np.array_equal(np.load(f"/tmp/r_gm{mode}_{t}.npy"), ref))
    print(mode, "nbad", nbad, "of", N)
