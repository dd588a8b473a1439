"""Small end-to-end runs for compute-sanitizer (development aid): every kernel
family (stream / naive / tb2 / pair), fp32 and fp64, stored eta, the paper-shape
ablation kernels, graph replay and the slab split path, on C1 / RAGGED-size
grids; the round-2 variants (embedded wall warps, seams, tile choices) on C1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2009_04619_b200.wave import WavePlan


def run(s, kernel="stream", precision="fp32", eta=False, steps=5):
    p = WavePlan(s.nx, s.ny, s.nz, s.w, s.h, s.dt, s.eta_max, kernel=kernel, precision=precision)
    if eta:
        p.set_eta(np.full((s.nz, s.ny, s.nx), 2.0, np.float32))
    p.set_velocity(synth.velocity(s))
    p.set_source(*s.source, synth.wavelet_for(s, 8))
    u0 = synth.random_state((s.nz, s.ny, s.nx), 1)
    p.set_state(None, u0 if precision == "fp32" else u0.astype(np.float64))
    p.step(steps)
    p.check_finite()
    _ = p.read(0).cpu()
    p.close()


cases = [("C1", {}), ("RAGGED", {}), ("RAGGED", dict(nx=9, ny=11, nz=10, w=2, src=(4, 5, 5)))]
for name, kw in cases:
    s = synth.scenario(name, **kw)
    for kernel in ("stream", "naive", "tb2", "pair"):
        run(s, kernel)
    run(s, "stream", "fp64")
    run(s, "naive", "fp64")
    run(s, "stream", eta=True)
# round-2 variants on C1 (64^3, w = 16): embedded wall warps (several pacing
# settings, incl. 1-plane units and an all-mop-up run), seam x walls, the 248
# tile (C1 picks 240 by default), two CTAs per SM
for env in ({"WAVE25_EW": "1"}, {"WAVE25_EW": "1", "WAVE25_EW_CZ": "1"}, {"WAVE25_EW": "1", "WAVE25_EW_REM": "1000000"},
            {"WAVE25_SEAM": "1"}, {"WAVE25_INNER_TILE": "248x8x1r"}, {"WAVE25_INNER_TILE": "128x8x1r2"},
            {"WAVE25_WALLX_TILE": "x24c16x64x1r2", "WAVE25_WALLY_TILE": "y128x8x1r2"}):
    os.environ.update(env)
    run(synth.scenario("C1"), "stream")
    for k in env:
        del os.environ[k]
if os.environ.get("WAVE25_ABLATION"):
    run(synth.scenario("RAGGED"), "stream")
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
