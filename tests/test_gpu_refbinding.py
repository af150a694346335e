"""GPU: the reference-side binding (paper_2602_23349_b200/flashopt_binding.py,
INTEGRATION.md §2) routes the reference's own `flashopt.optim.*_step` calls
on reference FlashState objects through fo_step_host; the result must be
bit-identical to the reference's NumPy step on the same inputs.  Uses the
unmodified reference installed in baseline/_ref (it travels to the box)."""

from __future__ import annotations

import numpy as np
import pytest

import helpers as H
import refbridge as RB

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not RB.available(), reason="reference not installed")]

OPTS = ["adamw", "sgd", "lion"]


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view({1: np.uint8, 2: np.uint16, 4: np.uint32}[a.itemsize])


def _same(a: dict, b: dict):
    return {k: int((_bits(a[k]) != _bits(b[k])).sum()) for k in a}


@pytest.mark.parametrize("opt", OPTS)
@pytest.mark.parametrize("n", [1, 33, 4096, 70_001, 1 << 20])
def test_binding_matches_reference(opt, n, cuda_dev):
    from paper_2602_23349_b200 import flashopt_binding as B

    fo = RB.flashopt()
    rng = np.random.default_rng(31 * n + OPTS.index(opt))
    st = H.random_state(rng, n, opt)
    g = H.random_grad(rng, n)
    hp = H.random_hparams(rng, opt)
    t = int(rng.integers(0, 2000))
    ref_in = RB.to_ref_state(st, t)
    want = RB.from_ref_state(fo.optim.STEP_FUNCTIONS[opt](ref_in, g, RB.hp_object(opt, hp)))
    snap = RB.from_ref_state(ref_in)
    snap = {k: v.copy() for k, v in snap.items()}
    got_state = B.step(opt, ref_in, g, RB.hp_object(opt, hp))
    assert got_state.t == t + 1
    assert all(v == 0 for v in _same(RB.from_ref_state(got_state), want).values())
    # pure contract: the input state is untouched
    assert all(v == 0 for v in _same(RB.from_ref_state(ref_in), snap).values())
    assert ref_in.t == t


def test_install_routes_reference_api(cuda_dev):
    """After install(), the reference's public API (STEP_FUNCTIONS and the
    module functions) runs on the GPU, multi-step trajectories from
    init_flash_state stay bitwise equal to the untouched NumPy path, and
    errors are the reference's ValueErrors, raised with the input intact."""
    from paper_2602_23349_b200 import flashopt_binding as B

    fo = RB.flashopt()
    O = fo.optim
    rng = np.random.default_rng(5)
    n = 50_017
    theta0 = H.random_weights(rng, n)
    orig = B.install(fo)
    try:
        assert O.adamw_step.__wrapped__ is orig["adamw"]
        for opt in OPTS:
            hp = RB.hp_object(opt, H.random_hparams(rng, opt))
            a = O.init_flash_state(theta0, opt)
            b = O.init_flash_state(theta0, opt)
            for _ in range(4):
                g = H.random_grad(rng, n, std=1e-2)
                a = O.STEP_FUNCTIONS[opt](a, g, hp)          # B200
                b = orig[opt](b, g, hp)                       # reference NumPy
                mm = _same(RB.from_ref_state(a), RB.from_ref_state(b))
                assert all(v == 0 for v in mm.values()), (opt, mm)
                assert a.t == b.t
        st = O.init_flash_state(theta0, "adamw")
        bad = np.zeros(n, np.float32)
        bad[7] = np.inf
        with pytest.raises(ValueError, match="gradient-nonfinite"):
            O.adamw_step(st, bad, O.AdamHyperParams(lr=1e-3))
        with pytest.raises(ValueError, match="gradient-nonfinite"):
            orig["adamw"](st, bad, O.AdamHyperParams(lr=1e-3))
        assert st.t == 0 and not st.momentum.codes.any()
        with pytest.raises(ValueError, match="gradient length"):
            O.adamw_step(st, np.zeros(n + 1, np.float32), O.AdamHyperParams(lr=1e-3))
        # ReferenceState (fp32 comparator) stays on NumPy
        rs = O.init_reference_state(theta0, "sgd")
        out = O.sgd_step(rs, np.zeros(n, np.float32), O.SgdHyperParams(lr=0.1))
        assert isinstance(out, O.ReferenceState)
    finally:
        B.uninstall(fo, orig)
    assert O.adamw_step is orig["adamw"]


@pytest.mark.parametrize("width_bits", [8, 16])
@pytest.mark.parametrize("scheme", ["companded", "linear"])
def test_binding_optional_layouts_trajectory(width_bits, scheme, cuda_dev):
    """The reference's optional layouts through the binding: INT16_CORRECTION
    weights (formats.py:94-95) and the linear variance scheme
    (optim.py:164-175), ten AdamW steps from init, bitwise equal to the
    reference's NumPy trajectory after every step."""
    from paper_2602_23349_b200 import flashopt_binding as B

    fo = RB.flashopt()
    O, F = fo.optim, fo.formats
    rng = np.random.default_rng(700 + width_bits + (1 if scheme == "linear" else 0))
    n = 40_003
    theta0 = H.random_weights(rng, n)
    width = F.INT16_CORRECTION if width_bits == 16 else F.INT8_CORRECTION
    a = O.init_flash_state(theta0, "adamw", variance_scheme=scheme)
    a.weights = F.SplitTensor.from_values(theta0, F.BF16, width)
    b = O.init_flash_state(theta0, "adamw", variance_scheme=scheme)
    b.weights = F.SplitTensor.from_values(theta0, F.BF16, width)
    hp = O.AdamHyperParams(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    for _ in range(10):
        g = H.random_grad(rng, n, std=1e-2)
        a = B.step("adamw", a, g, hp)
        b = O.adamw_step(b, g, hp)
        assert a.weights.corrections.dtype == b.weights.corrections.dtype
        mm = _same(RB.from_ref_state(a), RB.from_ref_state(b))
        assert all(v == 0 for v in mm.values()), mm
