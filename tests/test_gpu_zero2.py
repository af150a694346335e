"""GPU, two processes sharing cuda:0: the ZeRO-1 optimizer with the REAL
fused CUDA step (not the oracle) on every rank, gloo collectives staged
through host memory (NCCL refuses two ranks on one GPU).  After several
steps every rank's full bf16 parameters and every owned segment's state must
equal an unsharded oracle run bit for bit.  Gradients are exact under the
reduction: rank 0's backward yields g, rank 1's exactly zero.
Covers bucketed ownership, the reduce-scatter started from backward hooks,
fp32 parameters split at construction, and the batched rank-0 checkpoint.
With fused_allgather=True there is no all-gather: each rank's fused step
stores its updated weights into the other rank's parameter buffer through
CUDA IPC (two processes on one device exercise the same peer-store path
as two GPUs over NVLink), and every rank's parameters must still equal the
oracle's after every step."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SIZES = [1000, 4096 + 7, 33, 70_000, 1, 40_960, 8192]
ZERO = 6  # an all-zero tensor with zero gradients: its slices trip the fast tile's guards (fix-up path)
STEPS = 3
HP = {"adamw": dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1),
      "sgd": dict(lr=0.1, momentum=0.9, weight_decay=1e-4),
      "lion": dict(lr=1e-4, beta1=0.9, beta2=0.99, weight_decay=0.1)}


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _theta0():
    g = torch.Generator().manual_seed(11)
    t = [(torch.randn(n, generator=g) * 0.02) for n in SIZES]  # fp32 master weights
    t[ZERO].zero_()
    return t


def _grads(step):
    g = torch.Generator().manual_seed(500 + step)
    gs = [(torch.randn(n, generator=g) * 1e-3).to(torch.bfloat16) for n in SIZES]
    gs[ZERO].zero_()
    return gs


def _worker(rank, world, port, opt, q, directory, fused=False):
    try:
        import sys

        import torch.distributed as dist

        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path[:0] = [root, os.path.join(root, "tests")]
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2602_23349_b200 import optim as FO
        from paper_2602_23349_b200.zero import ZeroFlashOptimizer

        params = [t.cuda().requires_grad_() for t in _theta0()]
        zo = ZeroFlashOptimizer(params, opt, [FO.HP_TYPES[opt](**HP[opt])], reduce_op="sum", bucket_elems=8192,
                                overlap_grad_reduce=True, check_errors=True, fused_allgather=fused)
        for s in range(STEPS):
            zo.zero_grad()
            gs = [g.cuda() for g in _grads(s)]
            loss = sum((p * (g if rank == 0 else torch.zeros_like(g))).sum() for p, g in zip(params, gs))
            loss.backward()
            zo.step()
        torch.cuda.synchronize()
        assert zo.rs_launched_in_backward == STEPS * len(zo.layout.buckets)
        zo.save_checkpoint(directory, batch_bytes=50_000)
        full = [p.detach().view(torch.int16).cpu().numpy().view(np.uint16).copy() for p in params]
        segs = [(seg.param_index, seg.tensor_off, seg.length,
                 {"rho": st.weights.corrections.cpu().numpy(), "m": st.momentum.codes.cpu().numpy(),
                  "ms": st.momentum.scales.cpu().numpy(),
                  "v": None if st.variance is None else st.variance.codes.cpu().numpy(),
                  "vs": None if st.variance is None else st.variance.scales.cpu().numpy()})
                for seg, st in zip(zo.segments, zo.states)]
        from paper_2602_23349_b200 import _lib

        flagged, _ = _lib.fixup_stats()
        q.put((rank, full, segs, flagged))
        dist.barrier()
        if fused:
            zo.close()
        dist.destroy_process_group()
    except BaseException:
        import traceback

        q.put((rank, "error", traceback.format_exc()))
        raise


@pytest.mark.parametrize("fused", [False, True], ids=["nccl_allgather", "fused_allgather"])
@pytest.mark.parametrize("opt", ["adamw", "sgd", "lion"])
def test_zero1_two_ranks_cuda_step(opt, fused, cuda_dev, oracle_mod, tmp_path):
    from paper_2602_23349_b200.checkpoint import save_checkpoint
    from paper_2602_23349_b200.host import HostFlashState

    d = str(tmp_path / "ckpt")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, opt, q, d, fused)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    errs = [x[2] for x in got if isinstance(x[1], str)]
    assert not errs, errs[0]
    res = {r: (f, s) for r, f, s, _ in got}
    assert sum(x[3] for x in got) > 0  # the fix-up launch re-ran (and mirrored) flagged slices
    states = [oracle_mod.init_state(t.numpy(), opt) for t in _theta0()]
    for s in range(STEPS):
        for st, g in zip(states, _grads(s)):
            assert oracle_mod.step_inplace(opt, st, g.float().numpy(), **HP[opt]) == 0
    cover = {}
    for r in (0, 1):
        full, segs = res[r]
        for i, st in enumerate(states):
            assert np.array_equal(full[i], st.lp), (r, i)
        for pi, off, length, dd in segs:
            st = states[pi]
            g0 = off // 32
            assert np.array_equal(dd["rho"], st.rho[off:off + length]), (r, pi)
            assert np.array_equal(dd["m"], st.m_codes[off:off + length])
            assert np.array_equal(dd["ms"].view(np.uint16), st.m_scales[g0:g0 + dd["ms"].size].view(np.uint16))
            if dd["v"] is not None:
                assert np.array_equal(dd["v"], st.v_codes[off:off + length])
                assert np.array_equal(dd["vs"].view(np.uint16), st.v_scales[g0:g0 + dd["vs"].size].view(np.uint16))
            cover.setdefault(pi, []).append((off, length))
    for pi, runs in cover.items():
        assert sum(ln for _, ln in sorted(runs)) == SIZES[pi]
    # the batched rank-0 checkpoint is byte-identical to the unsharded oracle state's files
    for i, st in enumerate(states):
        ref = tmp_path / f"ref{i}.flop"
        save_checkpoint(HostFlashState(st.lp, st.rho, st.m_codes, st.m_scales, st.v_codes, st.v_scales, st.t, 32),
                        ref, opt)
        with open(ref, "rb") as f1, open(os.path.join(d, f"{i:05d}.flop"), "rb") as f2:
            assert f1.read() == f2.read(), i
