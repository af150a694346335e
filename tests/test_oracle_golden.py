"""CPU: pin the C oracle (oracle/flashopt_oracle.c) to the reference.

Three independent anchors:
  * the reference's own known-answer tests (hand traces) re-run through the
    oracle (pkg/tests/test_formats.py, test_quantize.py, test_optim.py);
  * golden vectors generated from the live reference (tests/golden/*.npz,
    tests/golden/make_golden.py), compared bit for bit;
  * when /root/reference is importable, fresh random cases against the live
    reference.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import helpers as H
import refbridge as R
from devstate import bits, mismatches, oracle_dict, oracle_state

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _index():
    with open(os.path.join(GOLD, "index.json")) as f:
        return json.load(f)


# ----------------------------------------------------------------- known answers
class TestKnownAnswers:
    def test_split_hand_traces(self, oracle_mod):
        """test_formats.py:169-180."""
        lp, rho = oracle_mod.split(np.array([1.00390625, 1.0, 1.001953125], np.float32))
        assert (lp.astype(np.uint32) << 16).view(np.float32).tolist() == [1.0, 1.0, 1.0]
        assert rho.tolist() == [127, 0, 64]

    def test_reconstruct_hand_traces(self, oracle_mod):
        """test_formats.py:222-246."""
        out = oracle_mod.reconstruct(np.array([0x3F80, 0x3F80, 0x3F80, 0x7F80], np.uint16),
                                     np.array([0, 64, 127, 93], np.int8))
        assert out[0] == 1.0
        assert out[1] == np.float32(1.0) + np.float32((np.float32(64) / np.float32(127)) * np.float32(2.0 ** -8))
        assert out[2] == np.float32(1.00390625)
        assert np.isposinf(out[3])
        with pytest.raises(ValueError, match="invalid-correction-code"):
            oracle_mod.reconstruct(np.array([0x3F80], np.uint16), np.array([-128], np.int8))

    def test_saturated_split(self, oracle_mod):
        lp, rho = oracle_mod.split(np.array([3.4e38, -3.4e38], np.float32))
        assert lp.tolist() == [0x7F80, 0xFF80] and rho.tolist() == [0, 0]

    def test_split_rejects_nonfinite(self, oracle_mod):
        with pytest.raises(ValueError, match="split-nonfinite"):
            oracle_mod.split(np.array([1.0, np.inf], np.float32))

    def test_quantize_hand_traces(self, oracle_mod):
        """test_quantize.py:20-25, :43-53, :80-86, :98-108, :120-125, :167-171."""
        c, s = oracle_mod.quantize_momentum(np.array([0.5, -1.0, 0.25, 0.0], np.float32), 4)
        assert s.tolist() == [1.0] and c.tolist() == [85, -127, 51, 0]
        d = oracle_mod.dequantize_momentum(np.array([85, -127, 0], np.int8), np.array([1.0], np.float16), 3)
        assert abs(d[0] - 85.0 / 169.0) < 1e-7 and d[1] == -1.0 and d[2] == 0.0
        c, s = oracle_mod.quantize_variance(np.array([4.0, 1.0, 0.25, 0.0], np.float32), 4)
        assert s.tolist() == [2.0] and c.tolist() == [255, 128, 64, 0]
        d = oracle_mod.dequantize_variance(np.array([255, 128, 64], np.uint8), np.array([2.0], np.float16), 3)
        assert d[0] == 4.0 and abs(d[1] - 1.0078585) < 1e-6 and abs(d[2] - 0.2519646) < 1e-6
        _, s = oracle_mod.quantize_variance(np.array([0.25, 0.01, 16.0, 4.0], np.float32), 2)
        assert s.tolist() == [0.5, 4.0]
        x = np.ones(33, np.float32)
        x[32] = 0.25
        assert oracle_mod.quantize_momentum(x)[1].tolist() == [1.0, 0.25]
        with pytest.raises(ValueError, match="scale-overflow"):
            oracle_mod.quantize_momentum(np.array([65505.0], np.float32), 1)
        with pytest.raises(ValueError, match="quantize-nonfinite"):
            oracle_mod.quantize_momentum(np.array([1.0, np.nan], np.float32))

    def test_fp16_round_up_subnormals(self, oracle_mod):
        """SURVEY Appendix B probe 8: 2^-25 -> 2^-24, 6e-8 -> 1.19e-7."""
        _, s = oracle_mod.quantize_momentum(np.array([2.0 ** -25, 6e-8], np.float32), 1)
        assert s.astype(np.float32).tolist() == [2.0 ** -24, np.float32(np.float16(1.1920929e-07))]

    @pytest.mark.parametrize("opt", ["sgd", "adamw", "lion"])
    def test_zero_gradient_keeps_weights(self, opt, oracle_mod):
        """test_optim.py:142-153."""
        rng = np.random.default_rng(8)
        theta0 = rng.standard_normal(256).astype(np.float32)
        st0 = oracle_mod.init_state(theta0, opt)
        hp = {"sgd": dict(lr=0.1), "adamw": dict(lr=0.1), "lion": dict(lr=0.1)}[opt]
        st1 = oracle_mod.step(opt, st0, np.zeros(256, np.float32), **hp)
        assert np.array_equal(st0.lp, st1.lp) and np.array_equal(st0.rho, st1.rho)
        assert st0.t == 0 and st1.t == 1

    def test_init_records_correction(self, oracle_mod):
        """test_optim.py:47-51."""
        st = oracle_mod.init_state(np.array([1.001953125], np.float32), "sgd")
        assert st.rho.tolist() == [64] and st.v_codes is None

    def test_gradient_errors(self, oracle_mod):
        st = oracle_mod.init_state(np.array([1.0, 2.0], np.float32), "sgd")
        with pytest.raises(ValueError, match="length"):
            oracle_mod.step("sgd", st, np.array([1.0], np.float32), lr=0.1)
        with pytest.raises(ValueError, match="gradient-nonfinite"):
            oracle_mod.step("sgd", st, np.array([np.nan, 0.0], np.float32), lr=0.1)


# ----------------------------------------------------------------- golden vectors
def _case_state(z, name):
    prefix = f"{name}/in."
    return {k[len(prefix):]: z[k] for k in z.files if k.startswith(prefix)}


def _case_out(z, name):
    prefix = f"{name}/out."
    return {k[len(prefix):]: z[k] for k in z.files if k.startswith(prefix)}


def test_oracle_matches_golden_steps(oracle_mod):
    idx = _index()
    z = np.load(os.path.join(GOLD, "steps.npz"))
    names = sorted(k for k in idx if not k.startswith("traj_"))
    assert len(names) >= 24
    for name in names:
        meta = idx[name]
        ost = oracle_state(_case_state(z, name), meta["t"])
        assert oracle_mod.step_inplace(meta["optimizer"], ost, z[f"{name}/grad"], **meta["hp"]) == 0
        mm = mismatches(oracle_dict(ost), _case_out(z, name))
        assert all(v == 0 for v in mm.values()), (name, mm)


def test_oracle_matches_golden_trajectories(oracle_mod):
    idx = _index()
    z = np.load(os.path.join(GOLD, "trajectories.npz"))
    for opt in ("adamw", "sgd", "lion"):
        meta = idx[f"traj_{opt}"]
        st = oracle_mod.init_state(z[f"{opt}/theta0"], opt)
        for s in range(meta["steps"]):
            assert oracle_mod.step_inplace(opt, st, z[f"{opt}/grad{s}"], **meta["hp"]) == 0
            ref = {k.split(".", 1)[1]: z[k] for k in z.files if k.startswith(f"{opt}/step{s}.")}
            mm = mismatches(oracle_dict(st), ref)
            assert all(v == 0 for v in mm.values()), (opt, s, mm)


def test_oracle_matches_golden_codecs(oracle_mod):
    z = np.load(os.path.join(GOLD, "codecs.npz"))
    lp, rho = oracle_mod.split(z["split_x"])
    assert np.array_equal(lp, z["split_lp"]) and np.array_equal(rho, z["split_rho"])
    lp16, rho16 = oracle_mod.split(z["split_x"], 16)
    assert np.array_equal(lp16, z["split_lp16"]) and np.array_equal(rho16, z["split_rho16"])
    rec = oracle_mod.reconstruct(z["rec_lp"], z["rec_rho"])
    ref = z["rec_out"]
    fin = np.isfinite(ref)
    assert np.array_equal(bits(rec)[fin], bits(ref)[fin])
    c, s = oracle_mod.quantize_momentum(z["qm_x"])
    assert np.array_equal(c, z["qm_codes"]) and np.array_equal(bits(s), bits(z["qm_scales"]))
    assert np.array_equal(bits(oracle_mod.dequantize_momentum(c, s)), bits(z["qm_deq"]))
    c, s = oracle_mod.quantize_variance(z["qv_x"])
    assert np.array_equal(c, z["qv_codes"]) and np.array_equal(bits(s), bits(z["qv_scales"]))
    assert np.array_equal(bits(oracle_mod.dequantize_variance(c, s)), bits(z["qv_deq"]))


def test_chunked_stepping_is_bit_identical(oracle_mod):
    """SURVEY Appendix B probe 6: 32-aligned chunks == whole tensor (the basis
    of multi-tensor chunking and ZeRO-1 sharding)."""
    rng = np.random.default_rng(6)
    n = 32_017
    st = H.random_state(rng, n, "adamw")
    g = H.random_grad(rng, n)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    whole = oracle_state(st, 3)
    oracle_mod.step_inplace("adamw", whole, g, **hp)
    parts = []
    for b in range(0, n, 4096):
        e = min(n, b + 4096)
        sub = {k: (v[b:e] if "scales" not in k else v[b // 32:(e + 31) // 32]) for k, v in st.items()}
        ost = oracle_state(sub, 3)
        oracle_mod.step_inplace("adamw", ost, g[b:e], **hp)
        parts.append(oracle_dict(ost))
    cat = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    assert all(v == 0 for v in mismatches(oracle_dict(whole), cat).values())


def test_zero_padding_is_a_fixed_point(oracle_mod):
    """SURVEY Appendix B probe 13: zero-padding a tensor to a multiple of 32
    leaves every real output unchanged and the padding at 0 (ZeRO-1 layout)."""
    rng = np.random.default_rng(13)
    n, npad = 1000, 1024
    theta0 = H.random_weights(rng, n)
    for opt in ("adamw", "sgd", "lion"):
        a = oracle_mod.init_state(theta0, opt)
        b = oracle_mod.init_state(np.concatenate([theta0, np.zeros(npad - n, np.float32)]), opt)
        hp = H.random_hparams(rng, opt)
        for _ in range(4):
            g = H.random_grad(rng, n)
            oracle_mod.step_inplace(opt, a, g, **hp)
            oracle_mod.step_inplace(opt, b, np.concatenate([g, np.zeros(npad - n, np.float32)]), **hp)
        da, db = oracle_dict(a), oracle_dict(b)
        for k in da:
            if "scales" in k:
                assert np.array_equal(bits(da[k]), bits(db[k][: da[k].size]))
            else:
                assert np.array_equal(bits(da[k]), bits(db[k][:n]))
                assert not np.any(bits(db[k][n:]))


# ----------------------------------------------------------------- live reference
@pytest.mark.skipif(not R.available(), reason="reference not importable here")
@pytest.mark.parametrize("opt", ["adamw", "sgd", "lion"])
def test_oracle_matches_live_reference(opt, oracle_mod):
    rng = np.random.default_rng({"adamw": 1, "sgd": 2, "lion": 3}[opt])
    for _ in range(6):
        n = int(rng.integers(1, 40_000))
        st = H.random_state(rng, n, opt)
        g = H.random_grad(rng, n, std=float(10 ** rng.uniform(-5, -1)))
        hp = H.random_hparams(rng, opt)
        t = int(rng.integers(0, 5000))
        ref = R.ref_step(opt, st, g, t, hp)
        ost = oracle_state(st, t)
        assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
        mm = mismatches(oracle_dict(ost), {k: np.asarray(v) for k, v in ref.items()})
        assert all(v == 0 for v in mm.values()), mm


@pytest.mark.skipif(not R.available(), reason="reference not importable here")
def test_error_precedence_matches_live_reference(oracle_mod):
    """The reference raises the first failing stage; the oracle's mask maps to
    the same message (optim.py program order)."""
    fo = R.flashopt()
    rng = np.random.default_rng(99)
    for opt in ("adamw", "sgd", "lion"):
        st = H.random_state(rng, 64, opt)
        st["weights.rho"][3] = -128                       # invalid correction code
        g = H.random_grad(rng, 64)
        g[7] = 1e38                                        # huge grad -> overflowing m / v
        hp = H.random_hparams(rng, opt)
        try:
            R.ref_step(opt, st, g, 5, hp)
            ref_msg = None
        except ValueError as e:
            ref_msg = str(e)
        ost = oracle_state(st, 5)
        mask = oracle_mod.step_inplace(opt, ost, g, **hp)
        try:
            oracle_mod.raise_for(mask, opt)
            got = None
        except ValueError as e:
            got = str(e)
        assert got == ref_msg, (opt, got, ref_msg)
    del fo
