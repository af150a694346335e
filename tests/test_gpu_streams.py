"""Concurrent fused launches on two streams ("different
parameter tensors may be stepped in parallel"): each stream has its own
fix-up bitmap, so slices flagged by one list are never re-run with the
other list's tensor table.  AdamW from the zero state with tiny gradients
trips the operand guards in many slices, which exercises the fix-up on
both streams at once.  Bitwise against the oracle."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import helpers as H
from devstate import from_device, mismatches, oracle_dict, oracle_state, to_device

pytestmark = pytest.mark.gpu


def _list(rng, sizes, dev, hp, oracle_mod):
    states, grads, refs = [], [], []
    for n in sizes:
        st = H.random_state(rng, n, "adamw")
        for k in st:
            if k not in ("weights.lp", "weights.rho"):
                st[k] = np.zeros_like(st[k])
        g = H.random_grad(rng, n, std=1e-3)
        pick = rng.random(n) < 0.05
        g[pick] = (np.sign(rng.standard_normal(int(pick.sum()))) *
                   2.0 ** rng.uniform(-120, -60, int(pick.sum()))).astype(np.float32)
        g = (g.view(np.uint32) & 0xFFFF0000).view(np.float32)
        states.append(to_device(st, 0, dev))
        grads.append(torch.from_numpy(g).to(dev).bfloat16())
        ost = oracle_state(st, 0)
        assert oracle_mod.step_inplace("adamw", ost, g, **hp) == 0
        refs.append(oracle_dict(ost))
    return states, grads, refs


def test_two_streams_with_fixups(cuda_dev, oracle_mod):
    from paper_2602_23349_b200 import optim as FO

    rng = np.random.default_rng(4711)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    a = _list(rng, [300000, 7680 * 5 + 100, 4096, 131072], cuda_dev, hp, oracle_mod)
    b = _list(rng, [65536, 250000, 999, 7680 * 9], cuda_dev, hp, oracle_mod)
    s1, s2 = torch.cuda.Stream(cuda_dev), torch.cuda.Stream(cuda_dev)
    cur = torch.cuda.current_stream(cuda_dev)
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    hpo = FO.AdamHyperParams(**hp)
    FO.step_many("adamw", a[0], a[1], hpo, stream=s1)
    FO.step_many("adamw", b[0], b[1], hpo, stream=s2)
    torch.cuda.synchronize(cuda_dev)
    for states, _, refs in (a, b):
        for fs, ref in zip(states, refs):
            mm = mismatches(from_device(fs), ref)
            assert all(v == 0 for v in mm.values()), mm
