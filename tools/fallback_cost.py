"""Cost of the exact fallback tile: FlashAdamW on GPT-2-medium shapes with
synthetic grads, then the same with one tiny gradient (|g| = 1e-12 < 2^-35)
planted in every k-th 512-element slice."""
import os, sys
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
base = [(torch.randn(p.shape, device="cuda", generator=g) * 1e-3).to(torch.bfloat16) for p in ps]

def timeit():
    for _ in range(3):
        opt.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        opt.step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 10

for p in ps:
    opt.state[p]["step"] = 1000
for every in (0, 1000, 100, 10, 1):
    for p, gb in zip(ps, base):
        gg = gb.clone().reshape(-1)
        if every:
            gg[::512 * every] = 1e-12
        p.grad = gg.view(p.shape)
    ms = timeit()
    print(f"tiny grad in every {every or 'no'} slice(s): {ms:.3f} ms  ({n / ms / 1e6:.1f} Gparams/s)")
# clustered: the leading 1% / 10% of every tensor holds tiny gradients (like
# embedding rows of tokens absent from the batch)
for frac in (0.01, 0.1):
    for p, gb in zip(ps, base):
        gg = gb.clone().reshape(-1)
        gg[:int(gg.numel() * frac)] = 1e-12
        p.grad = gg.view(p.shape)
    ms = timeit()
    print(f"tiny grads in the leading {frac:.0%} of every tensor: {ms:.3f} ms  ({n / ms / 1e6:.1f} Gparams/s)")
