"""GPU parity for the group-32 exact kernel (step_g32_kernel): the lists the
fast tile does not take -- int16 corrections (formats.py:94-95, N = 32767),
the linear-variance ablation (quantize.py:161-185), views that are not
16-byte aligned and hyper-parameters outside the fast tile's guard ranges --
as one multi-tensor launch per parameter group, bitwise against the oracle.
Error cases are compared byte for byte with the one-thread-per-group kernel
(FO_GENERIC=pergroup) that the group-32 kernel replaces for G = 32.
"""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import helpers as H
from devstate import from_device, mismatches, oracle_dict, oracle_state, to_device

pytestmark = pytest.mark.gpu

OPTS = ["adamw", "sgd", "lion"]
SIZES = [1, 31, 32, 33, 127, 128, 129, 1000, 4096 + 5, 70001, 262144 + 96]


def _hp_obj(opt, hp):
    from paper_2602_23349_b200 import optim as FO

    return FO.HP_TYPES[opt](**hp)


def _int16_state(rng, n, opt):
    st = H.random_state(rng, n, opt)
    st["weights.rho"] = rng.integers(-32767, 32768, n).astype(np.int16)
    return st


def _many(opt, make_state, sizes, hps, dev, oracle_mod, scheme="companded", grad_dtype=torch.bfloat16, t0=5):
    from paper_2602_23349_b200 import optim as FO

    rng = np.random.default_rng(len(sizes) * 31 + OPTS.index(opt))
    states, grads, hpo, refs = [], [], [], []
    for i, n in enumerate(sizes):
        st = make_state(rng, n, opt)
        g = H.random_grad(rng, n, std=float(10 ** rng.uniform(-4, -2)))
        if grad_dtype == torch.float32:
            g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        t = t0 + (i % 3)
        states.append(to_device(st, t, dev, 32, scheme))
        gd = torch.from_numpy(g).to(dev)
        grads.append(gd.bfloat16() if grad_dtype == torch.bfloat16 else gd)
        hp = hps[i % len(hps)]
        hpo.append(_hp_obj(opt, hp))
        ost = oracle_state(st, t, 32, scheme)
        assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
        refs.append(oracle_dict(ost))
    FO.step_many(opt, states, grads, hpo)
    for n, fs, ref in zip(sizes, states, refs):
        mm = mismatches(from_device(fs), ref)
        assert all(v == 0 for v in mm.values()), (n, mm)


@pytest.mark.parametrize("opt", OPTS)
@pytest.mark.parametrize("grad_dtype", [torch.bfloat16, torch.float32])
def test_int16_multi_tensor(opt, grad_dtype, cuda_dev, oracle_mod):
    rng = np.random.default_rng(160 + OPTS.index(opt))
    hps = [H.random_hparams(rng, opt), H.random_hparams(rng, opt)]
    _many(opt, _int16_state, SIZES, hps, cuda_dev, oracle_mod, grad_dtype=grad_dtype)


@pytest.mark.parametrize("rho_bits", [8, 16])
def test_linear_variance_multi_tensor(rho_bits, cuda_dev, oracle_mod):
    rng = np.random.default_rng(170 + rho_bits)
    make = _int16_state if rho_bits == 16 else (lambda r, n, o: H.random_state(r, n, o))
    _many("adamw", make, SIZES, [H.random_hparams(rng, "adamw")], cuda_dev, oracle_mod, scheme="linear")


@pytest.mark.parametrize("opt", OPTS)
def test_hparams_outside_fast_ranges(opt, cuda_dev, oracle_mod):
    """Scalars the fast tile's guards do not cover: tiny
    betas / momentum, subnormal eps, huge learning rates."""
    hp = {"adamw": [dict(lr=1e-3, beta1=1e-35, beta2=0.5, eps=1e-40, weight_decay=0.1),
                    dict(lr=1e3, beta1=0.9, beta2=0.999999, eps=1e30, weight_decay=0.0)],
          "sgd": [dict(lr=1e-3, momentum=1e-36, weight_decay=0.01), dict(lr=3e4, momentum=0.9999999, weight_decay=0.0)],
          "lion": [dict(lr=1e-3, beta1=1e-37, beta2=0.5, weight_decay=0.1),
                   dict(lr=1e-4, beta1=0.9, beta2=0.9999999, weight_decay=0.0)]}[opt]
    _many(opt, lambda r, n, o: H.random_state(r, n, o), SIZES[:8], hp, cuda_dev, oracle_mod, t0=1)


@pytest.mark.parametrize("opt", OPTS)
def test_misaligned_multi_tensor(opt, cuda_dev, oracle_mod):
    """Views offset by one element (2-byte aligned only) in one call."""
    from paper_2602_23349_b200 import optim as FO
    from paper_2602_23349_b200.formats import SplitTensor

    rng = np.random.default_rng(180 + OPTS.index(opt))
    hp = H.random_hparams(rng, opt)
    states, grads, refs = [], [], []
    for n in SIZES:
        st = H.random_state(rng, n, opt)
        g = H.random_grad(rng, n)
        fs = to_device(st, 3, cuda_dev)
        big = torch.empty(n + 1, dtype=torch.bfloat16, device=cuda_dev)
        big[1:].copy_(fs.weights.lp_values)
        fs.weights = SplitTensor(big[1:], fs.weights.corrections)
        gb = torch.empty(n + 1, dtype=torch.bfloat16, device=cuda_dev)
        gb[1:].copy_(torch.from_numpy(g).bfloat16())
        states.append(fs)
        grads.append(gb[1:])
        ost = oracle_state(st, 3)
        assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
        refs.append(oracle_dict(ost))
    FO.step_many(opt, states, grads, [_hp_obj(opt, hp)] * len(SIZES))
    for n, fs, ref in zip(SIZES, states, refs):
        mm = mismatches(from_device(fs), ref)
        assert all(v == 0 for v in mm.values()), (n, mm)


_ERR_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {tests!r}); sys.path.insert(0, {root!r})
import helpers as H
from devstate import from_device, to_device
from paper_2602_23349_b200 import optim as FO
dev = torch.device("cuda:0")
out = {{}}
for case, opt in enumerate(["adamw", "sgd", "lion", "adamw", "adamw"]):
    rng = np.random.default_rng(500 + case)
    n = 4096 + 77
    st = H.random_state(rng, n, opt)
    st["weights.rho"] = rng.integers(-32768, 32768, n).astype(np.int16)   # includes -32768 (invalid)
    g = H.random_grad(rng, n)
    g[rng.integers(0, n, 9)] = np.float32("nan")
    g[rng.integers(0, n, 5)] = np.float32("inf")
    g[rng.integers(0, n, 5)] = np.float32(1e30)                          # scale overflow
    fs = to_device(st, 2, dev, 32, "linear" if case == 4 else "companded")
    hp = FO.HP_TYPES[opt](**H.random_hparams(rng, opt))
    try:
        FO.STEP_FUNCTIONS_INPLACE[opt](fs, torch.from_numpy(g).to(dev), hp)
        msg = ""
    except ValueError as e:
        msg = str(e)
    for k, v in from_device(fs).items():
        out["%d/%s" % (case, k)] = np.ascontiguousarray(v).view(np.uint8)
    out["%d/msg" % case] = np.frombuffer(msg.encode(), np.uint8)
np.savez(sys.argv[1], **out)
"""


def test_error_cases_match_pergroup_kernel(tmp_path, cuda_dev):
    """Non-finite gradients, invalid int16 codes and scale overflow: the
    group-32 kernel writes the same bytes and raises the same error as the
    one-thread-per-group kernel."""
    here = os.path.dirname(os.path.abspath(__file__))
    script = tmp_path / "err.py"
    script.write_text(_ERR_SCRIPT.format(tests=here, root=os.path.dirname(here)))
    res = {}
    for mode in ("g32", "pergroup"):
        env = dict(os.environ)
        if mode == "pergroup":
            env["FO_GENERIC"] = "pergroup"
        out = tmp_path / f"{mode}.npz"
        r = subprocess.run([sys.executable, str(script), str(out)], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-3000:]
        res[mode] = dict(np.load(out))
    a, b = res["g32"], res["pergroup"]
    assert sorted(a) == sorted(b)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert any(a[f"{c}/msg"].size for c in range(5))


def test_pergroup_kernel_still_matches(cuda_dev):
    """FO_GENERIC=pergroup: the one-thread-per-group kernel passes the same
    int16 / linear / misaligned parity cases."""
    env = dict(os.environ, FO_GENERIC="pergroup")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_g32.py"), "-k", "int16 or linear or misaligned or outside"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("opt", OPTS)
def test_int16_every_code(opt, cuda_dev, oracle_mod):
    """Every valid int16 correction code once (the reconstruct's division by
    32767 is a Markstein quotient on the fast variant)."""
    rng = np.random.default_rng(190 + OPTS.index(opt))
    n = 65535
    st = H.random_state(rng, n, opt)
    st["weights.rho"] = rng.permutation(np.arange(-32767, 32768)).astype(np.int16)
    g = H.random_grad(rng, n)
    hp = H.random_hparams(rng, opt)
    from paper_2602_23349_b200 import optim as FO

    fs = to_device(st, 7, cuda_dev)
    FO.STEP_FUNCTIONS_INPLACE[opt](fs, torch.from_numpy(g).to(cuda_dev).bfloat16(), _hp_obj(opt, hp))
    ost = oracle_state(st, 7)
    assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
    mm = mismatches(from_device(fs), oracle_dict(ost))
    assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
def test_int16_tiny_gradients(opt, cuda_dev, oracle_mod):
    """Tiny and subnormal gradients through the group-32 kernel's shortcuts
    (per-element fallback to the IEEE intrinsics), live and zero state."""
    rng = np.random.default_rng(195 + OPTS.index(opt))
    for zero in (False, True):
        n = 40000 + 17
        st = _int16_state(rng, n, opt)
        if zero:
            for k in st:
                if k not in ("weights.lp", "weights.rho"):
                    st[k] = np.zeros_like(st[k])
        g = H.random_grad(rng, n, std=1e-3)
        pick = rng.random(n) < 0.3
        g[pick] = (np.sign(rng.standard_normal(int(pick.sum()))) *
                   2.0 ** rng.uniform(-149, -30, int(pick.sum()))).astype(np.float32)
        g = (g.view(np.uint32) & 0xFFFF0000).view(np.float32)
        hp = H.random_hparams(rng, opt)
        from paper_2602_23349_b200 import optim as FO

        t = 0 if zero else 30
        fs = to_device(st, t, cuda_dev)
        FO.STEP_FUNCTIONS_INPLACE[opt](fs, torch.from_numpy(g).to(cuda_dev).bfloat16(), _hp_obj(opt, hp))
        ost = oracle_state(st, t)
        assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
        mm = mismatches(from_device(fs), oracle_dict(ost))
        assert all(v == 0 for v in mm.values()), (zero, mm)


def test_ieee_variant_still_matches(cuda_dev):
    """FO_G32_FAST=0: the group-32 kernel on IEEE intrinsics throughout passes
    the same parity cases."""
    env = dict(os.environ, FO_G32_FAST="0")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_g32.py"), "-k", "int16 or linear or misaligned or outside"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
