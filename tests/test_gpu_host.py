"""GPU: fo_step_host (host-resident state, the reference's calling
convention) against the C oracle, bitwise, including multi-slot streaming."""

from __future__ import annotations

import numpy as np
import pytest

import helpers as H
from devstate import mismatches, oracle_dict, oracle_state

pytestmark = pytest.mark.gpu


def _host_state(st: dict, t: int, pinned: bool, G: int = 32):
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
                          arr("variance.codes"), arr("variance.scales"), t, G)


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


@pytest.mark.parametrize("opt", ["adamw", "sgd", "lion"])
@pytest.mark.parametrize("G", [1, 4, 16, 33, 64, 100, 1024])
def test_host_step_any_group_size(opt, G, cuda_dev, oracle_mod):
    """Any group size >= 1 (quantize.py:33-44 accepts it), with slots small
    enough that tensors straddle slots and batches hold many pieces: every
    piece keeps its own 16-byte aligned run of scales inside the slot."""
    from paper_2602_23349_b200 import host, optim as FO

    rng = np.random.default_rng(1000 + G)
    sizes = [5000, 1, 2 * G + 3, 70_001, 4096, G, 12_345]
    hp = H.random_hparams(rng, opt)
    states, grads, refs = [], [], []
    for n in sizes:
        st = H.random_state(rng, n, opt, G=G)
        g = H.random_grad(rng, n)
        states.append(_host_state(st, 3, False, G))
        grads.append((g.view(np.uint32) >> 16).astype(np.uint16))
        ost = oracle_state(st, 3, G)
        assert oracle_mod.step_inplace(opt, ost, g, **hp) == 0
        refs.append(oracle_dict(ost))
    host.step_host(opt, states, grads, FO.HP_TYPES[opt](**hp), chunk_elems=8192)
    for hs, ref in zip(states, refs):
        mm = mismatches(_as_dict(hs), ref)
        assert all(v == 0 for v in mm.values()), (G, hs.length, mm)


def test_host_step_concurrent_threads(cuda_dev, oracle_mod):
    """fo_step_host is reentrant: concurrent calls from several host threads
    each lease their own device slots and streams."""
    import threading

    from paper_2602_23349_b200 import host, optim as FO

    hp = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    jobs = []
    for k in range(4):
        rng = np.random.default_rng(77 + k)
        n = 300_000 + 1000 * k
        st = H.random_state(rng, n, "adamw")
        g = H.random_grad(rng, n)
        ost = oracle_state(st, 5)
        assert oracle_mod.step_inplace("adamw", ost, g, **hp) == 0
        jobs.append((_host_state(st, 5, True), g, oracle_dict(ost)))
    errs = []

    def work(job):
        try:
            for _ in range(1):
                host.step_host("adamw", [job[0]], [job[1]], FO.AdamHyperParams(**hp), chunk_elems=1 << 16)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(j,)) for j in jobs]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for hs, _, ref in jobs:
        mm = mismatches(_as_dict(hs), ref)
        assert all(v == 0 for v in mm.values()), mm
