"""GPU parity of the optional layouts on the fused warp-specialised kernel:
int16 corrections (formats.py:94-95, N = 32767) and the linear-variance
ablation (quantize.py:161-185, selected by optim.py:164-175), bitwise against
the oracle.  The fused kernel takes them when the views are 16-byte aligned
(step_ws_kernel<..., NCORR, LINEAR>); the fix-up share shows the fused tile,
not the straight restatement, stored the checked bytes.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import helpers as H
from devstate import from_device, mismatches, oracle_dict, oracle_state, to_device

pytestmark = pytest.mark.gpu

OPTS = ["adamw", "sgd", "lion"]
SIZES = [1, 33, 511, 512, 513, 8192, 8192 * 16 + 5, 1_000_003]


def _hp_obj(opt, hp):
    from paper_2602_23349_b200 import optim as FO

    return FO.HP_TYPES[opt](**hp)


def _state(rng, n, opt, rho_bits, training_like):
    lp = H.bf16_codes((rng.standard_normal(n) * 0.02).astype(np.float32)) if training_like else None
    st = H.random_state(rng, n, opt, lp=lp)
    if rho_bits == 16:
        st["weights.rho"] = rng.integers(-32767, 32768, n).astype(np.int16)
    return st


def _run(opt, st, g, t, hp, dev, oracle_mod, scheme, grad_dtype=torch.bfloat16):
    from paper_2602_23349_b200 import optim as FO

    fs = to_device(st, t, dev, 32, scheme)
    gd = torch.from_numpy(g).to(dev)
    if grad_dtype == torch.bfloat16:
        gd = gd.to(torch.bfloat16)
    FO.STEP_FUNCTIONS_INPLACE[opt](fs, gd, _hp_obj(opt, hp))
    got = from_device(fs)
    ost = oracle_state(st, t, 32, scheme)
    assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
    return mismatches(got, oracle_dict(ost))


CASES = [("adamw", 16, "companded"), ("adamw", 8, "linear"), ("adamw", 16, "linear"),
         ("sgd", 16, "companded"), ("lion", 16, "companded")]


@pytest.mark.parametrize("opt,rho_bits,scheme", CASES)
@pytest.mark.parametrize("n", SIZES)
def test_layout_bitwise(opt, rho_bits, scheme, n, cuda_dev, oracle_mod):
    rng = np.random.default_rng(9000 + n + 13 * CASES.index((opt, rho_bits, scheme)))
    st = _state(rng, n, opt, rho_bits, training_like=False)
    g = H.random_grad(rng, n, std=float(10 ** rng.uniform(-5, -1)))
    hp = H.random_hparams(rng, opt)
    t = int(rng.integers(0, 3000))
    mm = _run(opt, st, g, t, hp, cuda_dev, oracle_mod, scheme)
    assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt,rho_bits,scheme", CASES)
@pytest.mark.parametrize("t", [0, 1000])
def test_layout_fast_share(opt, rho_bits, scheme, t, cuda_dev, oracle_mod):
    """Training-like weights: >= 99% of the slices are stored by the fused
    tile of the layout (both the general and the steady-state instance),
    bitwise equal to the oracle."""
    from paper_2602_23349_b200 import _lib

    rng = np.random.default_rng(9100 + t + CASES.index((opt, rho_bits, scheme)))
    n = (1 << 21) + 4321
    st = _state(rng, n, opt, rho_bits, training_like=True)
    g = H.random_grad(rng, n)
    hp = dict(lr=1e-5, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1) if opt == "adamw" else \
        H.random_hparams(rng, opt)
    _lib.fixup_stats(reset=True)
    mm = _run(opt, st, g, t, hp, cuda_dev, oracle_mod, scheme)
    flagged, slices = _lib.fixup_stats(reset=True)
    assert all(v == 0 for v in mm.values()), mm
    assert slices >= n // 512, (flagged, slices)  # the fused launch ran
    assert flagged <= 0.01 * slices, (flagged, slices)


@pytest.mark.parametrize("opt", OPTS)
def test_int16_every_code_fused(opt, cuda_dev, oracle_mod):
    """Every valid int16 correction code against every sign of weight, through
    the fused tile's computed R(rho) (no table)."""
    rng = np.random.default_rng(9200 + OPTS.index(opt))
    codes = np.arange(-32767, 32768, dtype=np.int32)
    n = 2 * codes.size + 1000
    lp = H.bf16_codes((rng.standard_normal(n) * 0.02).astype(np.float32))
    st = H.random_state(rng, n, opt, lp=lp)
    rho = np.concatenate([codes, codes[::-1], rng.integers(-32767, 32768, 1000)]).astype(np.int16)
    st["weights.rho"] = rho
    g = H.random_grad(rng, n)
    mm = _run(opt, st, g, 7, H.random_hparams(rng, opt), cuda_dev, oracle_mod, "companded")
    assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
def test_int16_f32_grads(opt, cuda_dev, oracle_mod):
    rng = np.random.default_rng(9300 + OPTS.index(opt))
    n = 70_001
    st = _state(rng, n, opt, 16, training_like=True)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    mm = _run(opt, st, g, 3, H.random_hparams(rng, opt), cuda_dev, oracle_mod, "companded", torch.float32)
    assert all(v == 0 for v in mm.values()), mm


def test_int16_invalid_code_raises(cuda_dev):
    """rho = -32768 (formats.py:270-271) reaches the fix-up restatement, which
    reports the reference's error."""
    from paper_2602_23349_b200 import optim as FO

    rng = np.random.default_rng(9400)
    n = 4096
    st = _state(rng, n, "adamw", 16, training_like=True)
    st["weights.rho"][1234] = -32768
    fs = to_device(st, 5, cuda_dev, 32, "companded")
    g = torch.from_numpy(H.random_grad(rng, n)).to(cuda_dev).bfloat16()
    with pytest.raises(ValueError, match="invalid-correction-code"):
        FO.adamw_step(fs, g, FO.AdamHyperParams(lr=1e-3))


@pytest.mark.parametrize("scheme", ["companded", "linear"])
def test_layout_trajectory(scheme, cuda_dev, oracle_mod):
    """Ten steps of an int16 state, compared after each step."""
    from paper_2602_23349_b200 import optim as FO

    rng = np.random.default_rng(9500)
    n = 50_000 + 17
    st = _state(rng, n, "adamw", 16, training_like=True)
    fs = to_device(st, 0, cuda_dev, 32, scheme)
    ost = oracle_state(st, 0, 32, scheme)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    for _ in range(10):
        g = H.random_grad(rng, n, std=1e-2)
        FO.adamw_step_(fs, torch.from_numpy(g).to(cuda_dev).bfloat16(), FO.AdamHyperParams(**hp))
        assert oracle_mod.step_inplace("adamw", ost, g, **hp) == 0
        mm = mismatches(from_device(fs), oracle_dict(ost))
        assert all(v == 0 for v in mm.values()), mm
