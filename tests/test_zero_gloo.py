"""CPU, world_size 2 (gloo): the ZeRO-1 layout and collectives.

The sharded optimizer (paper_2602_23349_b200/zero.py) runs with the C oracle
injected as its step (no GPU here); after several steps every rank's full
parameters and every shard's state must equal a single-process, unsharded
oracle run bit for bit.  Gradients are exact under the bf16 reduce-scatter:
rank 0 contributes g, rank 1 zeros, op=sum."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SIZES = [1000, 4096 + 7, 33, 70_000, 1]
STEPS = 3


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _np(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def _oracle_step_fn(opt, states, grads, hps):
    from oracle import oracle as O

    for st, g, hp in zip(states, grads, hps):
        ost = O.OracleState(_np(st.weights.lp_values), _np(st.weights.corrections), _np(st.momentum.codes),
                            _np(st.momentum.scales), None if st.variance is None else _np(st.variance.codes),
                            None if st.variance is None else _np(st.variance.scales), st.t)
        gf = g.float().numpy()
        err = O.step_inplace(opt, ost, gf, **hp.__dict__)
        assert err == 0
        st.t += 1


def _init_params(seed=0):
    g = torch.Generator().manual_seed(seed)
    return [(torch.randn(n, generator=g) * 0.02).to(torch.bfloat16) for n in SIZES]


def _grads(step, seed=100):
    g = torch.Generator().manual_seed(seed + step)
    return [(torch.randn(n, generator=g) * 1e-3).to(torch.bfloat16) for n in SIZES]


def _worker(rank, world, port, opt, q, zkw=None, mode="assign"):
    try:
        _worker_body(rank, world, port, opt, q, zkw, mode)
    except BaseException:  # report instead of leaving the parent waiting
        import traceback

        q.put((rank, "error", traceback.format_exc()))
        raise


def _worker_body(rank, world, port, opt, q, zkw, mode):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_23349_b200 import optim as FO
    from paper_2602_23349_b200.zero import ZeroFlashOptimizer

    params = _init_params()
    if mode != "assign":
        params = [p.requires_grad_() for p in params]
    hp = {"adamw": [FO.AdamHyperParams(lr=1e-3, beta2=0.95, weight_decay=0.1), FO.AdamHyperParams(lr=1e-3)],
          "sgd": [FO.SgdHyperParams(lr=0.1, weight_decay=1e-4), FO.SgdHyperParams(lr=0.1)],
          "lion": [FO.LionHyperParams(lr=1e-4, weight_decay=0.1), FO.LionHyperParams(lr=1e-4)]}[opt]
    zo = ZeroFlashOptimizer(params, opt, hp, group_of=[0, 1, 0, 1, 1], step_fn=_oracle_step_fn, reduce_op="sum",
                            **(zkw or {}))
    for s in range(STEPS):
        if mode == "assign":
            zo.zero_grad()
            if rank == 0:
                for p, g in zip(params, _grads(s)):
                    p.grad.copy_(g)
        else:
            # a real backward: rank 0's loss has gradient exactly g, rank 1's is
            # exactly zero; with mode "none" the user sets grads to None first
            # (torch's default zero_grad), which detaches them from the flat buffer
            if mode == "none":
                for p in params:
                    p.grad = None
            else:
                zo.zero_grad()
            gs = _grads(s)
            loss = sum((p * (g if rank == 0 else torch.zeros_like(g))).sum() for p, g in zip(params, gs))
            loss.backward()
        zo.step()
    if zkw and zkw.get("overlap_grad_reduce"):
        # every bucket's reduce-scatter was started inside backward
        assert zo.rs_launched_in_backward == STEPS * len(zo.layout.buckets) > STEPS, zo.rs_launched_in_backward
    full = [p.detach().clone() for p in params]
    shard_state = [(seg.param_index, seg.tensor_off, seg.length,
                    {"rho": st.weights.corrections.numpy().copy(), "m": st.momentum.codes.numpy().copy(),
                     "ms": st.momentum.scales.numpy().copy()}) for seg, st in zip(zo.segments, zo.states)]
    q.put((rank, [_np(f).copy() for f in full], shard_state))
    dist.barrier()
    dist.destroy_process_group()


LAYOUTS = {
    "one-bucket": (None, "assign"),
    "buckets": ({"bucket_elems": 2048}, "assign"),
    "overlap-hooks": ({"bucket_elems": 4096, "overlap_grad_reduce": True}, "backward"),
    "overlap-set-to-none": ({"bucket_elems": 4096, "overlap_grad_reduce": True}, "none"),
    "no-hooks-set-to-none": ({"bucket_elems": 8192}, "none"),
}


@pytest.mark.parametrize("layout", list(LAYOUTS))
@pytest.mark.parametrize("opt", ["adamw", "sgd", "lion"])
def test_zero1_matches_unsharded_oracle(opt, layout, oracle_mod):
    """Bucketed ownership (rank r owns piece r of every bucket), the
    reduce-scatter launched per bucket from post-accumulate-grad hooks while
    backward runs, and gradients detached by set_to_none: all bitwise equal to
    the unsharded oracle."""
    if layout != "one-bucket" and opt != "adamw":
        pytest.skip("layouts are optimizer-independent; covered with adamw")
    zkw, mode = LAYOUTS[layout]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, opt, q, zkw, mode)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    errs = [x[2] for x in got if isinstance(x[1], str)]
    assert not errs, errs[0]
    results = dict((r, (f, s)) for r, f, s in got)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # unsharded reference run
    from paper_2602_23349_b200 import optim as FO

    hp = {"adamw": [dict(lr=1e-3, beta2=0.95, weight_decay=0.1), dict(lr=1e-3)],
          "sgd": [dict(lr=0.1, weight_decay=1e-4), dict(lr=0.1)],
          "lion": [dict(lr=1e-4, weight_decay=0.1), dict(lr=1e-4)]}[opt]
    hp = [{k: v for k, v in FO.HP_TYPES[opt](**h).__dict__.items()} for h in hp]
    group_of = [0, 1, 0, 1, 1]
    states = []
    for p in _init_params():
        lp = _np(p).copy()
        n = lp.size
        ng = -(-n // 32)
        v = (np.zeros(n, np.uint8), np.zeros(ng, np.float16)) if opt == "adamw" else (None, None)
        states.append(oracle_mod.OracleState(lp, np.zeros(n, np.int8), np.zeros(n, np.int8),
                                             np.zeros(ng, np.float16), v[0], v[1], 0))
    for s in range(STEPS):
        for i, (st, g) in enumerate(zip(states, _grads(s))):
            assert oracle_mod.step_inplace(opt, st, g.float().numpy(), **hp[group_of[i]]) == 0
    for r in (0, 1):
        full, shard_state = results[r]
        for i, st in enumerate(states):
            assert np.array_equal(full[i], st.lp), (r, i)
        for pi, off, length, d in shard_state:
            st = states[pi]
            assert np.array_equal(d["rho"], st.rho[off:off + length])
            assert np.array_equal(d["m"], st.m_codes[off:off + length])
            g0 = off // 32
            assert np.array_equal(d["ms"].view(np.uint16), st.m_scales[g0:g0 + d["ms"].size].view(np.uint16))
    # the two shards together cover every element exactly once
    cover = {}
    for r in (0, 1):
        for pi, off, length, _ in results[r][1]:
            cover.setdefault(pi, []).append((off, length))
    for pi, runs in cover.items():
        runs.sort()
        assert sum(ln for _, ln in runs) == SIZES[pi]
        assert runs[0][0] == 0 and all(a + b == c for (a, b), (c, _) in zip(runs, runs[1:]))


def _worker_ckpt(rank, world, port, opt, q, directory):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_23349_b200 import optim as FO
    from paper_2602_23349_b200.zero import ZeroFlashOptimizer

    hp = {"adamw": [FO.AdamHyperParams(lr=1e-3, beta2=0.95, weight_decay=0.1), FO.AdamHyperParams(lr=1e-3)],
          "sgd": [FO.SgdHyperParams(lr=0.1, weight_decay=1e-4), FO.SgdHyperParams(lr=0.1)],
          "lion": [FO.LionHyperParams(lr=1e-4, weight_decay=0.1), FO.LionHyperParams(lr=1e-4)]}[opt]
    params = _init_params()
    zo = ZeroFlashOptimizer(params, opt, hp, group_of=[0, 1, 0, 1, 1], step_fn=_oracle_step_fn, reduce_op="sum",
                            bucket_elems=4096)
    for s in range(STEPS):
        zo.zero_grad()
        if rank == 0:
            for p, g in zip(params, _grads(s)):
                p.grad.copy_(g)
        zo.step()
    zo.save_checkpoint(directory, batch_bytes=20_000)  # several gather batches
    # restore into a fresh optimizer over zeroed parameters
    fresh = [torch.zeros_like(p) for p in _init_params()]
    z2 = ZeroFlashOptimizer(fresh, opt, hp, group_of=[0, 1, 0, 1, 1], step_fn=_oracle_step_fn, reduce_op="sum",
                            bucket_elems=4096)
    z2.load_checkpoint(directory)
    same = torch.equal(zo.flat_params.view(torch.int16), z2.flat_params.view(torch.int16)) and z2.t == zo.t
    for a, b in zip(zo.states, z2.states):
        same &= torch.equal(a.weights.corrections, b.weights.corrections)
        same &= torch.equal(a.momentum.codes, b.momentum.codes)
        same &= torch.equal(a.momentum.scales.view(torch.int16), b.momentum.scales.view(torch.int16))
        if opt == "adamw":
            same &= torch.equal(a.variance.codes, b.variance.codes)
            same &= torch.equal(a.variance.scales.view(torch.int16), b.variance.scales.view(torch.int16))
        same &= a.t == b.t
    q.put((rank, bool(same)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("opt", ["adamw", "sgd", "lion"])
def test_zero1_sharded_checkpoint(opt, oracle_mod, tmp_path):
    """SURVEY.md §8e sharded checkpoints: the shards' state is gathered into
    one FLOP v1 file per tensor, byte-identical to the file of the unsharded
    oracle state, and reloads (re-sharded) bit for bit."""
    from paper_2602_23349_b200 import optim as FO
    from paper_2602_23349_b200.checkpoint import save_checkpoint
    from paper_2602_23349_b200.host import HostFlashState

    d = str(tmp_path / "ckpt")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_ckpt, args=(r, 2, port, opt, q, d)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}
    hp = {"adamw": [dict(lr=1e-3, beta2=0.95, weight_decay=0.1), dict(lr=1e-3)],
          "sgd": [dict(lr=0.1, weight_decay=1e-4), dict(lr=0.1)],
          "lion": [dict(lr=1e-4, weight_decay=0.1), dict(lr=1e-4)]}[opt]
    hp = [{k: v for k, v in FO.HP_TYPES[opt](**h).__dict__.items()} for h in hp]
    group_of = [0, 1, 0, 1, 1]
    for i, p in enumerate(_init_params()):
        lp = _np(p).copy()
        n = lp.size
        ng = -(-n // 32)
        v = (np.zeros(n, np.uint8), np.zeros(ng, np.float16)) if opt == "adamw" else (None, None)
        st = oracle_mod.OracleState(lp, np.zeros(n, np.int8), np.zeros(n, np.int8), np.zeros(ng, np.float16),
                                    v[0], v[1], 0)
        for s in range(STEPS):
            assert oracle_mod.step_inplace(opt, st, _grads(s)[i].float().numpy(), **hp[group_of[i]]) == 0
        ref = tmp_path / f"ref{i}.flop"
        save_checkpoint(HostFlashState(st.lp, st.rho, st.m_codes, st.m_scales, st.v_codes, st.v_scales, st.t, 32),
                        ref, opt)
        with open(ref, "rb") as f1, open(os.path.join(d, f"{i:05d}.flop"), "rb") as f2:
            assert f1.read() == f2.read(), i
