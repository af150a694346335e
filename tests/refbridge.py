"""Bridge to the live NumPy reference (flashopt).

Looked up in baseline/_ref first -- the unmodified reference installed with
pip; it is git-ignored but travels to the GPU box with the
repo snapshot -- then in /root/reference/pkg/src (build container only).
Tests that use it skip when neither is present.  Used to pin the C oracle,
to generate tests/golden/ fixtures and to check the reference-side binding
(paper_2602_23349_b200/flashopt_binding.py) against the reference's own
NumPy output on the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATES = (os.path.join(_ROOT, "baseline", "_ref"), "/root/reference/pkg/src")
REF_SRC = next((p for p in _CANDIDATES if os.path.isdir(os.path.join(p, "flashopt"))), _CANDIDATES[-1])


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "flashopt"))


def flashopt():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    import flashopt.checkpoint  # noqa: F401
    import flashopt.formats  # noqa: F401
    import flashopt.optim  # noqa: F401
    import flashopt.quantize  # noqa: F401
    return sys.modules["flashopt"]


def to_ref_state(st: dict, t: int, G: int = 32):
    fo = flashopt()
    F, Q, O = fo.formats, fo.quantize, fo.optim
    rho = st["weights.rho"]
    width = F.INT8_CORRECTION if rho.dtype == np.int8 else F.INT16_CORRECTION
    w = F.SplitTensor(st["weights.lp"].copy(), rho.copy(), F.BF16, width)
    spec = Q.GroupSpec(G)
    m = Q.QuantizedState(st["momentum.codes"].copy(), st["momentum.scales"].copy(), spec, "momentum")
    v = None
    if "variance.codes" in st:
        v = Q.QuantizedState(st["variance.codes"].copy(), st["variance.scales"].copy(), spec, "variance")
    return O.FlashState(w, m, v, t)


def from_ref_state(fs) -> dict:
    out = {
        "weights.lp": fs.weights.lp_values,
        "weights.rho": fs.weights.corrections,
        "momentum.codes": fs.momentum.codes,
        "momentum.scales": fs.momentum.scales,
    }
    if fs.variance is not None:
        out["variance.codes"] = fs.variance.codes
        out["variance.scales"] = fs.variance.scales
    return out


def hp_object(optimizer: str, hp: dict):
    O = flashopt().optim
    if optimizer == "adamw":
        return O.AdamHyperParams(**hp)
    if optimizer == "sgd":
        return O.SgdHyperParams(**hp)
    return O.LionHyperParams(**hp)


def ref_step(optimizer: str, st: dict, grad: np.ndarray, t: int, hp: dict, G: int = 32) -> dict:
    O = flashopt().optim
    fs = to_ref_state(st, t, G)
    out = O.STEP_FUNCTIONS[optimizer](fs, grad, hp_object(optimizer, hp))
    return from_ref_state(out)
