"""A few real GPT-2-medium training steps with FlashAdamW, then one more
optimizer step (the one to profile: launch index 7)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from bench_gpt2_train import make_model, HP
from paper_2602_23349_b200.torch_optim import FlashAdamW

m = make_model(torch.bfloat16)
opt = FlashAdamW(list(m.parameters()), check_errors=False, **HP)
x = torch.randint(0, 50257, (8, 1024), device="cuda")
for i in range(8):
    m(input_ids=x, labels=x).loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=True)
torch.cuda.synchronize()
print("done")
