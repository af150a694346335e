"""Time FlashAdamW.step() on GPT-2-medium parameters with synthetic grads, at
early (t ~ 1) and steady-state (t ~ 1000) step counters."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from bench_gpt2_train import make_model, HP
from paper_2602_23349_b200.torch_optim import FlashAdamW

m = make_model(torch.bfloat16)
ps = list(m.parameters())
n = sum(p.numel() for p in ps)
opt = FlashAdamW(ps, check_errors=False, **HP)
g = torch.Generator(device="cuda").manual_seed(0)
for p in ps:
    p.grad = (torch.randn(p.shape, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
for t0 in (0, 1000):
    for p in ps:
        opt.state[p]["step"] = t0
    for _ in range(3):
        opt.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        opt.step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"t0={t0}: {ms:.3f} ms/step, {n / ms / 1e6:.1f} Gparams/s")
