"""How often do real GPT-2-medium gradients trip the fused tile's tiny-gradient
guard (0 < |g| < 2^-35), and how many 512-element slices contain one?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_gpt2_train import make_model

m = make_model(torch.bfloat16)
x = torch.randint(0, 50257, (8, 1024), device="cuda")
m(input_ids=x, labels=x).loss.backward()
tot = tiny = slices = bad_slices = 0
for name, p in m.named_parameters():
    g = p.grad.reshape(-1).float().abs()
    t = (g > 0) & (g < 2.0**-35)
    n = g.numel()
    tot += n
    tiny += int(t.sum())
    ns = -(-n // 512)
    pad = ns * 512 - n
    tb = torch.nn.functional.pad(t.float(), (0, pad)).view(ns, 512).amax(1)
    slices += ns
    bad_slices += int(tb.sum())
    if int(tb.sum()):
        print(f"{name:40s} n={n:9d} tiny={int(t.sum()):8d} slices_hit={int(tb.sum())}/{ns}")
print(f"tiny fraction {tiny/tot:.2e}; slices with a tiny gradient {bad_slices}/{slices} = {bad_slices/slices:.3%}")
