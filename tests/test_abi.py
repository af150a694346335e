"""CPU: the C-ABI library loads, exports every entry point include/*.h
declares, and its host-side helpers (no GPU needed) behave like the
reference: f32 step scalars (optim.py:210-226), error-message precedence
(optim.py:187-258) and synchronous argument validation."""

from __future__ import annotations

import ctypes
import glob
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols() -> set[str]:
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        syms |= set(re.findall(r"\b(fo_[a-z0-9_]+)\s*\(", text))
    return syms


def test_library_exports_every_declared_symbol():
    from paper_2602_23349_b200 import _lib

    L = _lib.lib()
    declared = _declared_symbols()
    assert {"fo_step_mt", "fo_adamw_step", "fo_sgd_step", "fo_lion_step", "fo_split", "fo_reconstruct"} <= declared
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    # and the ctypes table covers exactly the declared set
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


def test_abi_version_and_status_strings():
    from paper_2602_23349_b200 import _lib

    L = _lib.lib()
    assert L.fo_abi_version() == 2
    assert L.fo_status_string(0) == b"ok"
    assert L.fo_status_string(-1) == b"invalid argument"


@pytest.mark.parametrize("beta1,beta2,t", [(0.9, 0.999, 1), (0.9, 0.95, 10), (0.85, 0.9999, 4321), (0.0, 0.5, 3)])
def test_make_hparams_matches_python_float_semantics(beta1, beta2, t):
    """f32(1 - beta**t) computed in float64 then rounded once, like
    np.float32(1.0 - hp.beta1**t) in optim.py:212-213; f32(1-beta) like the
    NEP-50 promotion of (1.0 - hp.beta1) * f32 array."""
    from paper_2602_23349_b200 import _lib

    hp = _lib.make_hparams("adamw", 1e-3, beta1, beta2, 1e-8, 0.1, t=t)
    f32 = lambda x: float(np.float32(x))  # noqa: E731
    assert hp.lr == f32(1e-3) and hp.wd == f32(0.1) and hp.eps == f32(1e-8)
    assert hp.b1 == f32(beta1) and hp.omb1 == f32(1.0 - beta1)
    assert hp.b2 == f32(beta2) and hp.omb2 == f32(1.0 - beta2)
    assert hp.bc1 == f32(1.0 - beta1 ** t) and hp.bc2 == f32(1.0 - beta2 ** t)
    if hp.bc1 > 0:
        assert hp.rbc1 == float(np.float32(1.0) / np.float32(hp.bc1))
    assert hp.rbc2 == float(np.float32(1.0) / np.float32(hp.bc2))


def test_error_message_precedence():
    from paper_2602_23349_b200 import _lib

    E = _lib
    msg = _lib.error_message
    assert msg(0, "adamw") == ""
    assert msg(E.ERR_GRAD_NONFINITE | E.ERR_M_OVERFLOW, "adamw").startswith("gradient-nonfinite")
    assert msg(E.ERR_RHO_INVALID | E.ERR_SPLIT_NONFINITE, "lion").startswith("invalid-correction-code")
    # SGD quantises momentum before reconstructing (optim.py:195-197)
    assert msg(E.ERR_RHO_INVALID | E.ERR_M_OVERFLOW, "sgd").startswith("scale-overflow")
    assert msg(E.ERR_RHO_INVALID | E.ERR_M_OVERFLOW, "adamw").startswith("invalid-correction-code")
    assert msg(E.ERR_M_OVERFLOW | E.ERR_V_NONFINITE, "adamw").startswith("scale-overflow")
    assert msg(E.ERR_V_NONFINITE, "adamw").startswith("quantize-nonfinite")
    assert msg(E.ERR_SPLIT_NONFINITE | E.ERR_M_NONFINITE, "adamw").startswith("split-nonfinite")


def test_messages_match_oracle_table(oracle_mod):
    from paper_2602_23349_b200 import _lib

    for opt in ("adamw", "sgd", "lion"):
        for mask in range(1, 256):
            try:
                oracle_mod.raise_for(mask, opt)
                expect = None
            except ValueError as e:
                expect = str(e)
            got = _lib.error_message(mask, opt)
            if expect is not None:
                assert got == expect, (opt, hex(mask), got, expect)


def test_argument_validation_is_synchronous():
    """Bad arguments are rejected before any CUDA call (works without a GPU)."""
    from paper_2602_23349_b200 import _lib

    L = _lib.lib()
    hp = _lib.make_hparams("adamw", 1e-3)
    t = _lib.fo_tensor()
    t.n = 10  # null pointers
    assert L.fo_step_mt(1, ctypes.byref(t), 1, ctypes.byref(hp), 1, 0, 8, 32, 0, None, None) == -1
    assert L.fo_step_mt(7, None, 0, ctypes.byref(hp), 1, 0, 8, 32, 0, None, None) == -1   # unknown optimizer
    assert L.fo_step_mt(1, None, 0, ctypes.byref(hp), 1, 0, 12, 32, 0, None, None) == -1  # rho bits
    assert L.fo_step_mt(1, None, 0, ctypes.byref(hp), 1, 0, 8, 0, 0, None, None) == -1    # group size
    hps = (_lib.fo_hparams * 17)()
    assert L.fo_step_mt(1, None, 0, hps, 17, 0, 8, 32, 0, None, None) == -3               # too many sets
    t2 = _lib.fo_tensor()
    t2.n = 0  # empty tensors are a no-op
    assert L.fo_step_mt(1, ctypes.byref(t2), 1, ctypes.byref(hp), 1, 0, 8, 32, 0, None, None) == 0
    assert L.fo_split(None, 5, None, None, 8, None, None) == -1
    assert L.fo_selftest(0, 0, 1, None, None) == -1


def test_hyperparameter_validation_mirrors_reference():
    """optim.py:47-94 rules and messages."""
    from paper_2602_23349_b200 import optim as FO

    with pytest.raises(ValueError, match="momentum"):
        FO.SgdHyperParams(lr=0.1, momentum=1.0)
    with pytest.raises(ValueError, match="eps"):
        FO.AdamHyperParams(lr=0.1, eps=0.0)
    with pytest.raises(ValueError, match="betas"):
        FO.LionHyperParams(lr=0.1, beta2=1.5)
    with pytest.raises(ValueError, match="learning rate"):
        FO.SgdHyperParams(lr=math.nan)
    with pytest.raises(ValueError, match="weight decay"):
        FO.AdamHyperParams(lr=0.1, weight_decay=-1.0)
    assert FO.AdamHyperParams(lr=1.0) == FO.AdamHyperParams(lr=1.0, beta1=0.9, beta2=0.999, eps=1e-8,
                                                            weight_decay=0.0)


@pytest.mark.parametrize("beta1,beta2", [(0.9, 0.95), (0.9, 0.999), (0.5, 0.6), (0.0, 0.9)])
def test_bias_table_matches_make_hparams(beta1, beta2):
    """fo_bias_table (the capturable step's device table) holds exactly the
    bias corrections fo_make_hparams gives the host path at every t, and ends
    at the first t where both are 1.0f (optim.py:212-213)."""
    from paper_2602_23349_b200 import _lib

    L = _lib.lib()
    n = ctypes.c_int32(0)
    assert L.fo_bias_table(beta1, beta2, 1 << 22, None, ctypes.byref(n)) == 0
    n = n.value
    out = (ctypes.c_float * (4 * n))()
    m = ctypes.c_int32(0)
    assert L.fo_bias_table(beta1, beta2, n, ctypes.cast(out, ctypes.c_void_p), ctypes.byref(m)) == 0
    assert m.value == n
    tab = np.frombuffer(out, dtype=np.float32).reshape(n, 4)
    for t in list(range(min(n, 400))) + [n - 1]:
        hp = _lib.make_hparams("adamw", 1e-3, beta1, beta2, 1e-8, 0.0, t=t)
        assert (tab[t] == np.array([hp.bc1, hp.rbc1, hp.bc2, hp.rbc2], dtype=np.float32)).all(), t
    assert tab[-1][0] == 1.0 and tab[-1][2] == 1.0
    assert n == 2 or not (tab[-2][0] == 1.0 and tab[-2][2] == 1.0)
    small = ctypes.c_int32(0)
    assert L.fo_bias_table(0.9, 0.9999, 1000, None, ctypes.byref(small)) == -3  # needs ~1.7e5 entries


def test_capturable_entry_points_validate_synchronously():
    from paper_2602_23349_b200 import _lib

    L = _lib.lib()
    assert L.fo_fused_tile_elems() == 8192
    ts = (_lib.fo_tensor * 3)()
    for i, n in enumerate((1, 8192, 8193)):
        ts[i].n = n
    # 1 + 1 + 2 CTA tiles of 16 slices = 64 slices -> 2 words
    assert L.fo_fix_words(ts, 3) == 2
    hp = _lib.make_hparams("adamw", 1e-3)
    ds = _lib.fo_dev_scalars()
    assert L.fo_step_mt_dev(1, None, 0, ctypes.byref(hp), ctypes.byref(ds), 0, None, None) == -1  # no step ptr
    ds.step = 16
    assert L.fo_step_mt_dev(1, None, 0, ctypes.byref(hp), ctypes.byref(ds), 0, None, None) == -1  # adamw: no table
    ds.bc_table, ds.bc_len = 16, 40
    assert L.fo_step_mt_dev(1, None, 0, ctypes.byref(hp), ctypes.byref(ds), 0, None, None) == -1  # no bitmap


def test_peer_entry_points_validate_synchronously():
    """fo_step_mt_peers / fo_ipc_* reject bad arguments before any CUDA call."""
    from paper_2602_23349_b200 import _lib

    L = _lib.lib()
    hp = _lib.make_hparams("adamw", 1e-3)
    deltas = (ctypes.c_int64 * 8)()
    assert L.fo_step_mt_peers(1, None, 0, ctypes.byref(hp), 0, deltas, 8, None, None) == -1  # > FO_MAX_PEERS
    assert L.fo_step_mt_peers(1, None, 0, ctypes.byref(hp), 0, None, 2, None, None) == -1    # no deltas
    assert L.fo_step_mt_peers(7, None, 0, ctypes.byref(hp), 0, deltas, 1, None, None) == -1  # optimizer
    t = _lib.fo_tensor()
    t.n, t.hp_index = 10, 1
    assert L.fo_step_mt_peers(1, ctypes.byref(t), 1, ctypes.byref(hp), 0, deltas, 1, None, None) == -1
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    assert L.fo_ipc_export(None, h, ctypes.byref(off)) == -1
    ptr = ctypes.c_void_p(0)
    assert L.fo_ipc_open(None, 0, ctypes.byref(ptr)) == -1
    assert L.fo_ipc_open(h, -1, ctypes.byref(ptr)) == -1
    assert L.fo_ipc_close(None, 0) == -1
