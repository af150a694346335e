"""ZeRO-1 sharded FlashOptim step over torch.distributed (NCCL on NVLink).

Layout: every parameter is a view into one flat bf16 buffer,
each tensor padded with zeros to a multiple of 32 so groups never straddle
tensors (padding is a fixed point of all three steps: SURVEY Appendix B
probe 13, tests/test_oracle_golden.py), and the total padded to a multiple of
`ALIGN * world`.  Rank r owns the contiguous slice [r*L/W, (r+1)*L/W) of the
flat buffer and allocates the correction / moment codes and scales only for
that slice -- the paper's "rho remains local with the optimizer states"
(PAPER.md:358-360).  One step is

    reduce-scatter(flat bf16 grads) -> fused step on the shard -> all-gather(flat bf16 params)

The step on a slice is bit-identical to stepping the full tensors on one GPU
because every operation is elementwise or reduces within one group
(SURVEY Appendix B probe 6).  Only the rank's shard of the grads is
materialised after the reduce-scatter.

`step_fn` is pluggable so the sharding and collective logic can be tested
with the gloo backend on CPU (tests/test_zero_gloo.py); on GPUs the default
is the fused CUDA step (paper_2602_23349_b200.optim.step_many).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import torch
import torch.distributed as dist

ALIGN = 512  # shard boundaries are tile- and group-aligned


def shard_range(n: int, rank: int, world: int, align: int = 64) -> tuple[int, int]:
    """Per-tensor contiguous slice [a, b) of rank `rank` (align-multiple starts)."""
    per = -(-n // world)
    per = -(-per // align) * align
    a = min(n, rank * per)
    return a, min(n, a + per)


@dataclass
class Segment:
    """A run of the rank's shard that belongs to one parameter."""

    param_index: int
    shard_off: int    # offset inside the rank's shard
    tensor_off: int   # offset inside the parameter (multiple of 32)
    length: int       # real (unpadded) elements of the parameter in this run
    hp_index: int


class FlatLayout:
    """Offsets of every parameter in the padded flat buffer."""

    def __init__(self, numels: Sequence[int], world: int, group: int = 32):
        self.numels = [int(n) for n in numels]
        self.offsets = []
        off = 0
        for n in self.numels:
            self.offsets.append(off)
            off += -(-n // group) * group
        unit = ALIGN * world
        self.total = -(-off // unit) * unit if off else unit
        self.world = world
        self.shard = self.total // world

    def segments(self, rank: int, hp_index: Sequence[int]) -> list[Segment]:
        lo, hi = rank * self.shard, (rank + 1) * self.shard
        segs = []
        for i, (o, n) in enumerate(zip(self.offsets, self.numels)):
            a, b = max(lo, o), min(hi, o + n)
            if a < b:
                segs.append(Segment(i, a - lo, a - o, b - a, int(hp_index[i])))
        return segs


class ZeroFlashOptimizer:
    """ZeRO-1 FlashSGD / FlashAdamW / FlashLion over a process group.

    params      : bf16 tensors, identical on every rank (they are re-pointed
                  into the flat buffer; gradients go to a flat grad buffer).
    hparams     : one hyper-parameter object per param group; `group_of[i]`
                  is parameter i's group.
    """

    def __init__(self, params: Sequence[torch.Tensor], optimizer: str, hparams: Sequence, group_of=None,
                 process_group=None, step_fn: Callable | None = None, reduce_op: str = "avg"):
        from .flat import FlatStates

        self.pg = process_group
        self.world = dist.get_world_size(self.pg)
        self.rank = dist.get_rank(self.pg)
        self.optimizer = optimizer
        self.params = list(params)
        self.hparams = list(hparams)
        self.group_of = list(group_of) if group_of is not None else [0] * len(self.params)
        dev = self.params[0].device
        self.layout = FlatLayout([p.numel() for p in self.params], self.world)
        L = self.layout
        self.flat_params = torch.zeros(L.total, dtype=torch.bfloat16, device=dev)
        self.flat_grads = torch.zeros(L.total, dtype=torch.bfloat16, device=dev)
        for p, o in zip(self.params, L.offsets):
            self.flat_params[o:o + p.numel()].copy_(p.detach().reshape(-1))
            p.data = self.flat_params[o:o + p.numel()].view_as(p)
            p.grad = self.flat_grads[o:o + p.numel()].view_as(p)
        lo = self.rank * L.shard
        self.shard_params = self.flat_params[lo:lo + L.shard]
        self.shard_grads = torch.zeros(L.shard, dtype=torch.bfloat16, device=dev)
        self.segments = L.segments(self.rank, self.group_of)
        # optimizer state for the shard only, one FlashState per segment
        sizes = [s.length for s in self.segments]
        views = [self.shard_params[s.shard_off:s.shard_off + s.length] for s in self.segments]
        self.flat_state = FlatStates(sizes, optimizer, dev, lp_views=views) if sizes else None
        self.states = self.flat_state.states if sizes else []
        self.step_fn = step_fn
        self.reduce_op = reduce_op
        self.t = 0

    # -- the three phases --------------------------------------------------------
    def reduce_scatter_grads(self) -> None:
        op = dist.ReduceOp.SUM
        if self.reduce_op == "avg" and dist.get_backend(self.pg) == "nccl":
            op = dist.ReduceOp.AVG
        dist.reduce_scatter_tensor(self.shard_grads, self.flat_grads, op=op, group=self.pg)
        if self.reduce_op == "avg" and op == dist.ReduceOp.SUM:
            self.shard_grads.div_(self.world)

    def step_shard(self) -> None:
        grads = [self.shard_grads[s.shard_off:s.shard_off + s.length] for s in self.segments]
        hps = [self.hparams[s.hp_index] for s in self.segments]
        if not self.states:
            return
        if self.step_fn is not None:
            self.step_fn(self.optimizer, self.states, grads, hps)
        else:
            from .optim import step_many

            step_many(self.optimizer, self.states, grads, hps)

    def all_gather_params(self) -> None:
        dist.all_gather_into_tensor(self.flat_params, self.shard_params, group=self.pg)

    @torch.no_grad()
    def step(self) -> None:
        self.reduce_scatter_grads()
        self.step_shard()
        self.all_gather_params()
        self.t += 1

    def zero_grad(self) -> None:
        self.flat_grads.zero_()
