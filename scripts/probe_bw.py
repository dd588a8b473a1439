"""Practical HBM roofs (development aid): 1R1W copy and the stencil's exact 3R1W
byte mix (out = a + b*c, 16 B/element) over 1024^3 fp32 arrays."""
import torch
n = 1024 ** 3
a, b, c, o = (torch.rand(n, device="cuda") for _ in range(4))
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: o.copy_(a)); print(f"copy 1R1W: {ms:.3f} ms  {8*n/ms/1e6:.0f} GB/s")
ms = t(lambda: torch.addcmul(a, b, c, out=o)); print(f"addcmul 3R1W: {ms:.3f} ms  {16*n/ms/1e6:.0f} GB/s  -> {n/ms/1e6:.1f} Gpt/s at 16 B/pt")
