"""numpy <-> device FlashState conversion for the GPU parity tests."""

from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O


def to_device(st: dict, t: int, dev, G: int = 32, scheme: str = "companded"):
    from paper_2602_23349_b200.formats import SplitTensor
    from paper_2602_23349_b200.optim import FlashState
    from paper_2602_23349_b200.quantize import GroupSpec, QuantizedState

    def T(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    spec = GroupSpec(G)
    w = SplitTensor(T(st["weights.lp"].view(np.int16)).view(torch.bfloat16), T(st["weights.rho"]))
    m = QuantizedState(T(st["momentum.codes"]), T(st["momentum.scales"]), spec, "momentum")
    v = None
    if "variance.codes" in st:
        kind = "variance" if scheme == "companded" else "linear-unsigned"
        v = QuantizedState(T(st["variance.codes"]), T(st["variance.scales"]), spec, kind)
    return FlashState(w, m, v, t, scheme)


def from_device(fs) -> dict:
    torch.cuda.synchronize()
    out = {
        "weights.lp": fs.weights.lp_values.view(torch.int16).cpu().numpy().view(np.uint16),
        "weights.rho": fs.weights.corrections.cpu().numpy(),
        "momentum.codes": fs.momentum.codes.cpu().numpy(),
        "momentum.scales": fs.momentum.scales.cpu().numpy(),
    }
    if fs.variance is not None:
        out["variance.codes"] = fs.variance.codes.cpu().numpy()
        out["variance.scales"] = fs.variance.scales.cpu().numpy()
    return out


def oracle_state(st: dict, t: int, G: int = 32, scheme: str = "companded") -> "O.OracleState":
    c = lambda k: None if k not in st else np.array(st[k], copy=True)  # noqa: E731
    return O.OracleState(c("weights.lp"), c("weights.rho"), c("momentum.codes"), c("momentum.scales"),
                         c("variance.codes"), c("variance.scales"), t, G, scheme)


def oracle_dict(ost) -> dict:
    out = {"weights.lp": ost.lp, "weights.rho": ost.rho, "momentum.codes": ost.m_codes,
           "momentum.scales": ost.m_scales}
    if ost.v_codes is not None:
        out["variance.codes"] = ost.v_codes
        out["variance.scales"] = ost.v_scales
    return out


def bits(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    return a.view({1: np.uint8, 2: np.uint16, 4: np.uint32}[a.itemsize])


def mismatches(a: dict, b: dict) -> dict:
    """Per-record count of bitwise-differing elements."""
    assert set(a) == set(b), (set(a), set(b))
    return {k: int((bits(a[k]) != bits(b[k])).sum()) for k in a}
