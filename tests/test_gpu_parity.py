"""GPU parity: the CUDA step (through the C ABI) vs the C oracle, bitwise.

Bar: bf16 weights, int8 corrections, int8/uint8 codes and fp16 scales all
bit-identical (0 mismatches).  The oracle itself is pinned to the reference
in tests/test_oracle_golden.py.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import helpers as H
from devstate import from_device, mismatches, oracle_dict, oracle_state, to_device

pytestmark = pytest.mark.gpu

OPTS = ["adamw", "sgd", "lion"]
SIZES = [1, 31, 32, 33, 500, 511, 512, 513, 1000, 4096, 70001]


def _hp_obj(opt, hp):
    from paper_2602_23349_b200 import optim as FO

    return FO.HP_TYPES[opt](**hp)


def _run_pair(opt, st, g, t, hp, dev, oracle_mod, grad_dtype=torch.bfloat16, G=32, scheme="companded"):
    from paper_2602_23349_b200 import optim as FO

    fs = to_device(st, t, dev, G, scheme)
    gd = torch.from_numpy(g).to(dev)
    if grad_dtype == torch.bfloat16:
        gd = gd.to(torch.bfloat16)
    FO.STEP_FUNCTIONS_INPLACE[opt](fs, gd, _hp_obj(opt, hp))
    got = from_device(fs)
    ost = oracle_state(st, t, G, scheme)
    err = oracle_mod.step_inplace(opt, ost, g, **hp)
    assert err == 0
    assert fs.t == ost.t == t + 1
    return mismatches(got, oracle_dict(ost))


@pytest.mark.parametrize("opt", OPTS)
@pytest.mark.parametrize("n", SIZES)
def test_fused_step_bitwise(opt, n, cuda_dev, oracle_mod):
    rng = np.random.default_rng(1000 + n + 7 * OPTS.index(opt))
    st = H.random_state(rng, n, opt)
    g = H.random_grad(rng, n, std=float(10 ** rng.uniform(-5, -1)))
    hp = H.random_hparams(rng, opt)
    t = int(rng.integers(0, 3000))
    mm = _run_pair(opt, st, g, t, hp, cuda_dev, oracle_mod)
    assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
def test_fused_step_1m_and_odd(opt, cuda_dev, oracle_mod):
    """BASELINE config 1 sizes: 2^20 and 1,000,003 (partial trailing group)."""
    for n in (1 << 20, 1_000_003):
        rng = np.random.default_rng(n)
        st = H.random_state(rng, n, opt)
        g = H.random_grad(rng, n)
        hp = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1) if opt == "adamw" else \
            H.random_hparams(rng, opt)
        mm = _run_pair(opt, st, g, 10, hp, cuda_dev, oracle_mod)
        assert all(v == 0 for v in mm.values()), (n, mm)


@pytest.mark.parametrize("opt", OPTS)
def test_fast_path_share(opt, cuda_dev, oracle_mod):
    """The fused tile, not the fix-up re-run, computes the parity cases: on a
    state with training-like weights (N(0, 0.02^2), no +-0 codes) at least 99%
    of the 512-element slices are stored by the fast tile (fo_fixup_stats),
    and the result is still bitwise equal to the oracle.  The standard random
    state (0.5% exact zeros, magnitudes down to 1e-40) sends most slices to
    the fix-up launch; both paths are covered."""
    from paper_2602_23349_b200 import _lib

    rng = np.random.default_rng(4242 + OPTS.index(opt))
    n = (1 << 21) + 12345
    lp = H.bf16_codes((rng.standard_normal(n) * 0.02).astype(np.float32))
    st = H.random_state(rng, n, opt, lp=lp)
    g = H.random_grad(rng, n)
    hp = dict(lr=1e-5, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1) if opt == "adamw" else \
        H.random_hparams(rng, opt)
    _lib.fixup_stats(reset=True)
    mm = _run_pair(opt, st, g, 1000, hp, cuda_dev, oracle_mod)
    flagged, slices = _lib.fixup_stats(reset=True)
    assert all(v == 0 for v in mm.values()), mm
    assert slices >= n // 512, (flagged, slices)
    assert flagged <= 0.01 * slices, (flagged, slices)

    st2 = H.random_state(rng, 1 << 20, opt)
    g2 = H.random_grad(rng, 1 << 20)
    mm = _run_pair(opt, st2, g2, 10, hp, cuda_dev, oracle_mod)
    flagged2, slices2 = _lib.fixup_stats(reset=True)
    assert all(v == 0 for v in mm.values()), mm
    assert 0 < flagged2 <= slices2


@pytest.mark.parametrize("opt", OPTS)
def test_f32_gradients(opt, cuda_dev, oracle_mod):
    """f32 grads that are not bf16-representable (the reference's own input type)."""
    rng = np.random.default_rng(5)
    n = 8192 + 77
    st = H.random_state(rng, n, opt)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    mm = _run_pair(opt, st, g, 3, H.random_hparams(rng, opt), cuda_dev, oracle_mod, grad_dtype=torch.float32)
    assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
def test_multi_step_from_init(opt, cuda_dev, oracle_mod):
    """t = 1 from the zero state, then more steps; compares after each step."""
    from paper_2602_23349_b200 import optim as FO

    rng = np.random.default_rng(77)
    n = 20000 + 13
    theta0 = H.random_weights(rng, n)
    fs = FO.init_flash_state(torch.from_numpy(theta0).to(cuda_dev), opt)
    ost = oracle_mod.init_state(theta0, opt)
    assert mismatches(from_device(fs), oracle_dict(ost)) == {k: 0 for k in oracle_dict(ost)}
    hp = H.random_hparams(rng, opt)
    for _ in range(4):
        g = H.random_grad(rng, n, std=1e-2)
        FO.STEP_FUNCTIONS_INPLACE[opt](fs, torch.from_numpy(g).to(cuda_dev).bfloat16(), _hp_obj(opt, hp))
        assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
        mm = mismatches(from_device(fs), oracle_dict(ost))
        assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
def test_multi_tensor_fused_launch(opt, cuda_dev, oracle_mod):
    """Many tensors of mixed sizes (incl. partial groups) and two param
    groups with different hyper-parameters in one fo_step_mt call."""
    from paper_2602_23349_b200 import optim as FO

    rng = np.random.default_rng(11)
    sizes = [64, 1000, 4096, 9, 147456, 256, 1, 2048 + 31, 589824, 33]
    hps = [H.random_hparams(rng, opt), H.random_hparams(rng, opt)]
    states, grads, hpo, refs = [], [], [], []
    for i, n in enumerate(sizes):
        st = H.random_state(rng, n, opt)
        g = H.random_grad(rng, n)
        t = 5 + (i % 3)
        states.append(to_device(st, t, cuda_dev))
        grads.append(torch.from_numpy(g).to(cuda_dev).bfloat16())
        hpo.append(_hp_obj(opt, hps[i % 2]))
        ost = oracle_state(st, t)
        assert oracle_mod.step_inplace(opt, ost, g, **hps[i % 2]) == 0
        refs.append(oracle_dict(ost))
    FO.step_many(opt, states, grads, hpo)
    for fs, ref in zip(states, refs):
        mm = mismatches(from_device(fs), ref)
        assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
@pytest.mark.parametrize("G", [1, 7, 16, 64, 100])
def test_generic_group_sizes(opt, G, cuda_dev, oracle_mod):
    rng = np.random.default_rng(G)
    n = 5000 + G
    st = H.random_state(rng, n, opt, G=G)
    g = H.random_grad(rng, n)
    mm = _run_pair(opt, st, g, 2, H.random_hparams(rng, opt), cuda_dev, oracle_mod, G=G)
    assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
def test_int16_corrections(opt, cuda_dev, oracle_mod):
    rng = np.random.default_rng(16)
    n = 3000 + 5
    st = H.random_state(rng, n, opt)
    st["weights.rho"] = rng.integers(-32767, 32768, n).astype(np.int16)
    g = H.random_grad(rng, n)
    mm = _run_pair(opt, st, g, 4, H.random_hparams(rng, opt), cuda_dev, oracle_mod)
    assert all(v == 0 for v in mm.values()), mm


def test_linear_variance_scheme(cuda_dev, oracle_mod):
    rng = np.random.default_rng(21)
    n = 4096 + 3
    st = H.random_state(rng, n, "adamw")
    g = H.random_grad(rng, n)
    mm = _run_pair("adamw", st, g, 6, H.random_hparams(rng, "adamw"), cuda_dev, oracle_mod, scheme="linear")
    assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
def test_misaligned_views_take_generic_path(opt, cuda_dev, oracle_mod):
    """Tensors whose storage is not 16-byte aligned still step correctly."""
    from paper_2602_23349_b200 import optim as FO
    from paper_2602_23349_b200.formats import SplitTensor

    rng = np.random.default_rng(3)
    n = 2000
    st = H.random_state(rng, n, opt)
    g = H.random_grad(rng, n)
    fs = to_device(st, 1, cuda_dev)
    big_lp = torch.empty(n + 1, dtype=torch.bfloat16, device=cuda_dev)
    big_lp[1:].copy_(fs.weights.lp_values)
    fs.weights = SplitTensor(big_lp[1:], fs.weights.corrections)
    FO.STEP_FUNCTIONS_INPLACE[opt](fs, torch.from_numpy(g).to(cuda_dev).bfloat16(), _hp_obj(opt, H.random_hparams(
        np.random.default_rng(9), opt)))
    ost = oracle_state(st, 1)
    oracle_mod.step_inplace(opt, ost, g, **H.random_hparams(np.random.default_rng(9), opt))
    mm = mismatches(from_device(fs), oracle_dict(ost))
    assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
def test_zero_gradient_keeps_weights(opt, cuda_dev):
    """tests/test_optim.py:142-153: zero grads from init leave lp/rho bitwise unchanged."""
    from paper_2602_23349_b200 import optim as FO

    rng = np.random.default_rng(8)
    theta0 = rng.standard_normal(256).astype(np.float32)
    fs0 = FO.init_flash_state(torch.from_numpy(theta0).to(cuda_dev), opt)
    hp = {"sgd": FO.SgdHyperParams(lr=0.1), "adamw": FO.AdamHyperParams(lr=0.1),
          "lion": FO.LionHyperParams(lr=0.1)}[opt]
    fs1 = FO.STEP_FUNCTIONS[opt](fs0, torch.zeros(256, device=cuda_dev), hp)
    assert torch.equal(fs0.weights.lp_values, fs1.weights.lp_values)
    assert torch.equal(fs0.weights.corrections, fs1.weights.corrections)
    assert fs0.t == 0 and fs1.t == 1  # functional form leaves the input untouched


class TestErrors:
    def _state(self, opt, dev, n=256):
        rng = np.random.default_rng(1)
        return H.random_state(rng, n, opt), to_device

    @pytest.mark.parametrize("opt", OPTS)
    def test_nonfinite_gradient(self, opt, cuda_dev):
        from paper_2602_23349_b200 import optim as FO

        rng = np.random.default_rng(2)
        st = H.random_state(rng, 300, opt)
        fs = to_device(st, 0, cuda_dev)
        g = torch.zeros(300, device=cuda_dev)
        g[77] = float("nan")
        with pytest.raises(ValueError, match="gradient-nonfinite"):
            FO.STEP_FUNCTIONS[opt](fs, g, _hp_obj(opt, H.random_hparams(rng, opt)))
        assert fs.t == 0

    @pytest.mark.parametrize("opt", OPTS)
    def test_invalid_correction_code(self, opt, cuda_dev):
        from paper_2602_23349_b200 import optim as FO

        rng = np.random.default_rng(3)
        st = H.random_state(rng, 300, opt)
        st["weights.rho"][5] = -128
        fs = to_device(st, 0, cuda_dev)
        with pytest.raises(ValueError, match="invalid-correction-code"):
            FO.STEP_FUNCTIONS[opt](fs, torch.zeros(300, device=cuda_dev), _hp_obj(opt, H.random_hparams(rng, opt)))

    def test_scale_overflow(self, cuda_dev):
        from paper_2602_23349_b200 import optim as FO

        rng = np.random.default_rng(4)
        st = H.random_state(rng, 64, "sgd")
        fs = to_device(st, 0, cuda_dev)
        g = torch.zeros(64, device=cuda_dev)
        g[3] = 1e6
        with pytest.raises(ValueError, match="scale-overflow"):
            FO.sgd_step(fs, g, FO.SgdHyperParams(lr=1e-3))

    def test_length_mismatch(self, cuda_dev):
        from paper_2602_23349_b200 import optim as FO

        fs = FO.init_flash_state(torch.ones(10, device=cuda_dev), "sgd")
        with pytest.raises(ValueError, match="length"):
            FO.sgd_step(fs, torch.ones(11, device=cuda_dev), FO.SgdHyperParams(lr=0.1))


@pytest.mark.parametrize("opt", OPTS)
def test_special_weight_codes(opt, cuda_dev, oracle_mod):
    """Weight codes where the fused tile's shortcuts need their guards: +-0
    with every correction sign (the integer reconstruct's two wrong cases),
    subnormal codes, binade bottoms (the formats.py:147-154 refinement),
    the largest finite bf16, and tiny gradients (|g| < 2^-35)."""
    rng = np.random.default_rng(4242 + OPTS.index(opt))
    special = np.array([0x0000, 0x8000, 0x0001, 0x8001, 0x007F, 0x0080, 0x8080, 0x0100, 0x8100, 0x3F80, 0xBF80,
                        0x4000, 0xC000, 0x7F7F, 0xFF7F, 0x0700, 0x0701, 0x8700], np.uint16)
    n = 16384 + 96
    st = H.random_state(rng, n, opt)
    lp = st["weights.lp"].copy()
    pick = rng.random(n) < 0.25
    lp[pick] = special[rng.integers(0, special.size, int(pick.sum()))]
    st["weights.lp"] = lp
    rho = st["weights.rho"]
    rho[rng.random(n) < 0.05] = 0
    g = H.random_grad(rng, n, std=1e-3)
    tiny = rng.random(n) < 0.01
    g[tiny] = (rng.standard_normal(int(tiny.sum())) * 2.0**-40).astype(np.float32)
    g = H.bf16_round(g) if hasattr(H, "bf16_round") else g
    mm = _run_pair(opt, st, g, 50, H.random_hparams(rng, opt), cuda_dev, oracle_mod)
    assert all(v == 0 for v in mm.values()), mm


@pytest.mark.parametrize("opt", ["adamw"])
def test_more_tensors_than_one_launch(opt, cuda_dev, oracle_mod):
    """> 384 tensors (FO_MT_MAX_TENSORS) in one call: several launches."""
    from paper_2602_23349_b200 import optim as FO

    rng = np.random.default_rng(99)
    sizes = [int(x) for x in rng.integers(1, 3000, 450)] + [7680 * 3 + 517]
    hp = H.random_hparams(rng, opt)
    states, grads, refs = [], [], []
    for n in sizes:
        st = H.random_state(rng, n, opt)
        g = H.random_grad(rng, n)
        states.append(to_device(st, 700, cuda_dev))
        grads.append(torch.from_numpy(g).to(cuda_dev).bfloat16())
        ost = oracle_state(st, 700)
        assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
        refs.append(oracle_dict(ost))
    FO.step_many(opt, states, grads, [_hp_obj(opt, hp)] * len(sizes))
    for fs, ref in zip(states, refs):
        mm = mismatches(from_device(fs), ref)
        assert all(v == 0 for v in mm.values()), mm


def test_ldg_kernel_matches_too(cuda_dev):
    """The LDG kernel (taken when a list's scale runs are not 16-byte aligned,
    FO_KERNEL=mt forces it) passes the same bitwise parity cases."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, FO_KERNEL="mt")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_parity.py"), "-k",
                        "fused_step_bitwise or multi_tensor or special or f32_gradients"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("opt", OPTS)
@pytest.mark.parametrize("case", ["live_state", "zero_state", "subnormal"])
def test_tiny_gradients(opt, case, cuda_dev, oracle_mod):
    """Gradients far below the typical scale (real bf16 backward passes have
    them): on a live state the fast tile takes them (its guards look at the
    m / v operands, not at g); from the zero state m and v are tiny too and
    the guards must send the slices to the exact re-run.  Bitwise."""
    rng = np.random.default_rng(9000 + 10 * OPTS.index(opt) + ["live_state", "zero_state", "subnormal"].index(case))
    n = 65536 + 1000
    st = H.random_state(rng, n, opt)
    t = 40
    if case == "zero_state":
        for k in st:
            if k not in ("weights.lp", "weights.rho"):
                st[k] = np.zeros_like(st[k])
        t = 0
    g = H.random_grad(rng, n, std=1e-3)
    pick = rng.random(n) < 0.3
    exps = rng.uniform(-60, -30, int(pick.sum())) if case != "subnormal" else rng.uniform(-149, -120, int(pick.sum()))
    tiny = (np.sign(rng.standard_normal(int(pick.sum()))) * 2.0 ** exps).astype(np.float32)
    g[pick] = tiny
    g = (g.view(np.uint32) & 0xFFFF0000).view(np.float32)  # bf16-exact
    hp = H.random_hparams(rng, opt)
    mm = _run_pair(opt, st, g, t, hp, cuda_dev, oracle_mod)
    assert all(v == 0 for v in mm.values()), mm
