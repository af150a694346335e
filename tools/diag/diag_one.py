"""Debug helper: step tiny AdamW states without raising; print mask + outputs vs oracle."""
import os
import sys
import numpy as np
import torch
_R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, _R); sys.path.insert(0, os.path.join(_R, "tests"))
import helpers as H
from devstate import from_device, oracle_dict, oracle_state, to_device
from oracle import oracle as O
from paper_2602_23349_b200 import optim as FO
from paper_2602_23349_b200._errors import DeviceErrors

dev = torch.device("cuda:0")
for n in (1, 2, 17, 31, 33):
    opt = "adamw"
    rng = np.random.default_rng(1000 + n)
    st = H.random_state(rng, n, opt)
    g = H.random_grad(rng, n, std=float(10 ** rng.uniform(-5, -1)))
    hp = H.random_hparams(rng, opt)
    t = int(rng.integers(0, 3000))
    fs = to_device(st, t, dev)
    err = DeviceErrors(dev)
    FO.step_many(opt, [fs], [torch.from_numpy(g).to(dev).bfloat16()], FO.HP_TYPES[opt](**hp), errors=err)
    got = from_device(fs)
    ost = oracle_state(st, t)
    e2 = O.step_inplace(opt, ost, g, **hp)
    ref = oracle_dict(ost)
    print("n", n, "mask", hex(err.mask()), "oracle mask", e2, "hp", hp, "t", t)
    for k in ref:
        print("  ", k, "got", got[k][:4], "ref", ref[k][:4], "in", st[k][:4])
    print("   g", g[:4])
