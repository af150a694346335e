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

    # -- checkpoints (SURVEY.md §8e "sharded checkpoints") -----------------------
    # A tensor's state can straddle ranks.  To keep the reference layout -- one
    # FLOP v1 file per tensor with rank-1 (n,) records (checkpoint.py:73-80,
    # :98-125) -- the shards are gathered in flat-buffer coordinates, each
    # tensor's slices are cut out with the padding dropped, and rank 0 writes
    # the files: byte-identical to what a single-GPU FlashState of the whole
    # tensor writes.  Loading re-shards: every rank reads the files and keeps
    # its own segments.

    def _local_records(self) -> dict:
        L = self.layout
        dev = self.flat_params.device
        adam = self.optimizer == "adamw"
        rho_dt = self.states[0].weights.corrections.dtype if self.states else torch.int8
        loc = {"rho": torch.zeros(L.shard, dtype=rho_dt, device=dev),
               "mq": torch.zeros(L.shard, dtype=torch.int8, device=dev),
               "ms": torch.zeros(L.shard // 32, dtype=torch.float16, device=dev)}
        if adam:
            loc["vq"] = torch.zeros(L.shard, dtype=torch.uint8, device=dev)
            loc["vs"] = torch.zeros(L.shard // 32, dtype=torch.float16, device=dev)
        for seg, st in zip(self.segments, self.states):
            a, n, ga = seg.shard_off, seg.length, seg.shard_off // 32
            loc["rho"][a:a + n].copy_(st.weights.corrections)
            loc["mq"][a:a + n].copy_(st.momentum.codes)
            loc["ms"][ga:ga + st.momentum.scales.numel()].copy_(st.momentum.scales)
            if adam:
                loc["vq"][a:a + n].copy_(st.variance.codes)
                loc["vs"][ga:ga + st.variance.scales.numel()].copy_(st.variance.scales)
        return loc

    def _gather_records(self) -> dict:
        """All ranks' state records in flat-buffer coordinates (collective)."""
        out = {}
        for k, t in self._local_records().items():
            raw = t.view(torch.uint8)  # bytes: every backend gathers them, bit patterns untouched
            parts = [torch.empty_like(raw) for _ in range(self.world)]
            dist.all_gather(parts, raw, group=self.pg)
            out[k] = torch.cat(parts).view(t.dtype)
        return out

    def save_checkpoint(self, directory, names: Sequence[str] | None = None) -> dict | None:
        """Collective: one FLOP v1 file per parameter plus a manifest, written
        by rank 0 (returns the manifest there, None elsewhere)."""
        import json
        import os

        import numpy as np

        from .checkpoint import save_checkpoint
        from .host import HostFlashState

        g = self._gather_records()
        manifest = None
        if self.rank == 0:
            os.makedirs(directory, exist_ok=True)
            L = self.layout
            names = list(names) if names is not None else [f"param{i:05d}" for i in range(len(self.params))]
            host = {k: v.cpu().numpy() for k, v in g.items()}
            lp_all = self.flat_params.view(torch.int16).cpu().numpy().view(np.uint16)
            manifest = {"format": "FLOP v1 per parameter", "optimizer": self.optimizer, "params": [], "bytes": 0}
            for i, (p, o, n) in enumerate(zip(self.params, L.offsets, L.numels)):
                go, ng = o // 32, -(-n // 32)
                hs = HostFlashState(lp_all[o:o + n], host["rho"][o:o + n], host["mq"][o:o + n],
                                    host["ms"][go:go + ng], host["vq"][o:o + n] if "vq" in host else None,
                                    host["vs"][go:go + ng] if "vs" in host else None, self.t, 32)
                fname = f"{i:05d}.flop"
                manifest["bytes"] += save_checkpoint(hs, os.path.join(directory, fname), self.optimizer)
                manifest["params"].append({"index": i, "name": names[i], "file": fname, "shape": list(p.shape)})
            with open(os.path.join(directory, "manifest.json"), "w") as f:
                json.dump(manifest, f, indent=1)
        dist.barrier(group=self.pg)
        return manifest

    @torch.no_grad()
    def load_checkpoint(self, directory) -> None:
        """Restore the full bf16 parameters and this rank's state segments from
        files written by save_checkpoint (or by single-GPU save_optimizer)."""
        import json
        import os

        from .checkpoint import CheckpointError, load_checkpoint

        with open(os.path.join(directory, "manifest.json")) as f:
            manifest = json.load(f)
        if manifest["optimizer"] != self.optimizer:
            raise CheckpointError(f"checkpoint is for {manifest['optimizer']}, optimizer is {self.optimizer}")
        if len(manifest["params"]) != len(self.params):
            raise CheckpointError("parameter count differs from the checkpoint")
        L = self.layout
        dev = self.flat_params.device
        by_param: dict = {}
        for seg, st in zip(self.segments, self.states):
            by_param.setdefault(seg.param_index, []).append((seg, st))
        step = None
        for i, ent in enumerate(manifest["params"]):
            hs = load_checkpoint(os.path.join(directory, ent["file"]))
            o, n = L.offsets[i], L.numels[i]
            if hs.length != n:
                raise CheckpointError(f"parameter {i}: checkpoint has {hs.length} elements, model {n}")
            step = hs.t
            self.flat_params[o:o + n].copy_(torch.from_numpy(hs.lp.view("int16")).to(dev).view(torch.bfloat16))
            for seg, st in by_param.get(i, []):
                a, m, ga = seg.tensor_off, seg.length, seg.tensor_off // 32
                T = lambda x: torch.from_numpy(x).to(dev)  # noqa: E731
                st.weights.corrections.copy_(T(hs.rho[a:a + m]))
                st.momentum.codes.copy_(T(hs.m_codes[a:a + m]))
                st.momentum.scales.copy_(T(hs.m_scales[ga:ga + st.momentum.scales.numel()]))
                if self.optimizer == "adamw":
                    st.variance.codes.copy_(T(hs.v_codes[a:a + m]))
                    st.variance.scales.copy_(T(hs.v_scales[ga:ga + st.variance.scales.numel()]))
                st.t = hs.t
        if step is not None:
            self.t = int(step)
