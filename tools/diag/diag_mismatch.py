"""Debug helper: run one fused step vs the oracle and print the first mismatches."""
import os
import sys
import numpy as np
import torch
_R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, _R); sys.path.insert(0, os.path.join(_R, "tests"))
import helpers as H
from devstate import from_device, oracle_dict, oracle_state, to_device, bits
from oracle import oracle as O
from paper_2602_23349_b200 import optim as FO

def run(opt, n, seed, t=7):
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(seed)
    st = H.random_state(rng, n, opt)
    g = H.random_grad(rng, n)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1) if opt == "adamw" else H.random_hparams(rng, opt)
    fs = to_device(st, t, dev)
    FO.STEP_FUNCTIONS_INPLACE[opt](fs, torch.from_numpy(g).to(dev).bfloat16(), FO.HP_TYPES[opt](**hp))
    got = from_device(fs)
    ost = oracle_state(st, t)
    O.step_inplace(opt, ost, g, **hp)
    ref = oracle_dict(ost)
    for k in ref:
        d = np.nonzero(bits(got[k]) != bits(ref[k]))[0]
        if len(d):
            print(opt, k, len(d), "first idx", d[:8])
            for i in d[:4]:
                gi = i if "scales" not in k else i * 32
                print("   i", i, "got", got[k][i], "ref", ref[k][i], "in lp", hex(st["weights.lp"][gi]), "rho", st["weights.rho"][gi],
                      "mc", st["momentum.codes"][gi], "g", g[gi])
                if "scales" in k:
                    sl = slice(i * 32, i * 32 + 32)
                    print("   group m codes got", got["momentum.codes"][sl].tolist())
                    print("   group m codes ref", ref["momentum.codes"][sl].tolist())
                    print("   grads", g[sl].tolist())

for opt in ("adamw", "sgd", "lion"):
    run(opt, 70001, 2602)
    run(opt, 1 << 20, 5)
