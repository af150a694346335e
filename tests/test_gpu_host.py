"""GPU: fo_step_host (host-resident state, the reference's calling
convention) against the C oracle, bitwise, including multi-slot streaming."""

from __future__ import annotations

import numpy as np
import pytest

import helpers as H
from devstate import mismatches, oracle_dict, oracle_state

pytestmark = pytest.mark.gpu


def _host_state(st: dict, t: int, pinned: bool):
    from paper_2602_23349_b200.host import HostFlashState, pinned_empty

    def arr(k):
        if k not in st:
            return None
        a = st[k]
        if pinned:
            b = pinned_empty(a.size, a.dtype)
            b[:] = a
            return b
        return a.copy()

    return HostFlashState(arr("weights.lp"), arr("weights.rho"), arr("momentum.codes"), arr("momentum.scales"),
                          arr("variance.codes"), arr("variance.scales"), t)


def _as_dict(hs) -> dict:
    d = {"weights.lp": hs.lp, "weights.rho": hs.rho, "momentum.codes": hs.m_codes, "momentum.scales": hs.m_scales}
    if hs.v_codes is not None:
        d["variance.codes"] = hs.v_codes
        d["variance.scales"] = hs.v_scales
    return d


@pytest.mark.parametrize("opt", ["adamw", "sgd", "lion"])
@pytest.mark.parametrize("pinned", [True, False])
def test_host_step_matches_oracle(opt, pinned, cuda_dev, oracle_mod):
    from paper_2602_23349_b200 import host, optim as FO

    rng = np.random.default_rng(42)
    sizes = [100_000, 33, 4096, 2_000_003, 1, 70_000]
    hp = H.random_hparams(rng, opt)
    states, grads, refs = [], [], []
    for n in sizes:
        st = H.random_state(rng, n, opt)
        g = H.random_grad(rng, n)
        t = 7
        states.append(_host_state(st, t, pinned))
        gb = (g.view(np.uint32) >> 16).astype(np.uint16)  # bf16 bit patterns
        grads.append(gb)
        ost = oracle_state(st, t)
        assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
        refs.append(oracle_dict(ost))
    # small slots: many batches, tensors split across slots, 3-slot rotation
    host.step_host(opt, states, grads, FO.HP_TYPES[opt](**hp), chunk_elems=1 << 18)
    for hs, ref in zip(states, refs):
        assert hs.t == 8
        mm = mismatches(_as_dict(hs), ref)
        assert all(v == 0 for v in mm.values()), mm


def test_host_step_raises_reference_errors(cuda_dev):
    from paper_2602_23349_b200 import host, optim as FO

    rng = np.random.default_rng(1)
    st = _host_state(H.random_state(rng, 100, "adamw"), 0, False)
    g = np.zeros(100, np.float32)
    g[5] = np.nan
    with pytest.raises(ValueError, match="gradient-nonfinite"):
        host.step_host("adamw", [st], [g], FO.AdamHyperParams(lr=1e-3))
