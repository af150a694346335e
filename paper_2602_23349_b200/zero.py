"""ZeRO-1 sharded FlashOptim step over torch.distributed (NCCL on NVLink).

Layout: every parameter is a view into one flat bf16 buffer,
each tensor padded with zeros to a multiple of 32 so groups never straddle
tensors (padding is a fixed point of all three steps: SURVEY Appendix B
probe 13, tests/test_oracle_golden.py).  The flat buffer is cut into
buckets (one bucket by default); each bucket is split into W equal pieces
and rank r owns piece r of every bucket, allocating the correction / moment
codes and scales only for what it owns -- the paper's "rho remains local
with the optimizer states".  One step is

    reduce-scatter(bf16 grads, per bucket) -> fused step on the owned pieces
        -> all-gather(bf16 params, per bucket, in place)

The step on a piece is bit-identical to stepping the full tensors on one GPU
because every operation is elementwise or reduces within one group
(SURVEY Appendix B probe 6).  Only the owned pieces of the gradients are
kept after the reduce-scatter.

With `fused_allgather=True` there is no separate all-gather: every rank
maps the other ranks' flat parameter buffers into its address space (CUDA
IPC, fo_ipc_export / fo_ipc_open), and the fused step stores each updated
bf16 weight both locally and at the same flat offset in every peer's buffer
(fo_step_mt_peers), so the exchange of the new weights runs inside the step,
tile by tile, over NVLink; a cross-rank barrier on the stream orders the
peers' next reads.  One hyper-parameter set, the default layout.

With `overlap_grad_reduce=True` a post-accumulate-grad hook counts the
gradients that have arrived per bucket and launches that bucket's
reduce-scatter asynchronously as soon as it is complete, so the exchange
runs under the rest of the backward pass; step() only waits for it.

`step_fn` is pluggable so the sharding and collective logic can be tested
with the gloo backend on CPU (tests/test_zero_gloo.py); on GPUs the default
is the fused CUDA step through a cached launch table (flat.StepPlan).  With
gloo and CUDA tensors the collectives are staged through host memory (a test
mode: two processes can then share one GPU and still run the CUDA step).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import torch
import torch.distributed as dist

ALIGN = 512  # piece boundaries are tile- and group-aligned


def shard_range(n: int, rank: int, world: int, align: int = 64) -> tuple[int, int]:
    """Per-tensor contiguous slice [a, b) of rank `rank` (align-multiple starts)."""
    per = -(-n // world)
    per = -(-per // align) * align
    a = min(n, rank * per)
    return a, min(n, a + per)


@dataclass
class Segment:
    """A run of the rank's owned elements that belongs to one parameter."""

    param_index: int
    shard_off: int    # offset inside the rank's shard (concatenated pieces)
    tensor_off: int   # offset inside the parameter (multiple of 32)
    length: int       # real (unpadded) elements of the parameter in this run
    hp_index: int
    flat_off: int = 0  # offset inside the flat buffer


class FlatLayout:
    """Offsets of every parameter in the padded flat buffer and its buckets."""

    def __init__(self, numels: Sequence[int], world: int, group: int = 32, bucket_elems: int | None = None):
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
        b = self.total if not bucket_elems else max(unit, -(-int(bucket_elems) // unit) * unit)
        self.buckets = [(s, min(b, self.total - s)) for s in range(0, self.total, b)]  # (start, size)
        self.piece_off = []  # shard offset of each bucket's piece
        so = 0
        for _, size in self.buckets:
            self.piece_off.append(so)
            so += size // world

    def piece(self, k: int, rank: int) -> tuple[int, int]:
        """Flat range [lo, hi) of bucket k owned by `rank`."""
        s, size = self.buckets[k]
        per = size // self.world
        return s + rank * per, s + (rank + 1) * per

    def segments(self, rank: int, hp_index: Sequence[int]) -> list[Segment]:
        segs = []
        for k in range(len(self.buckets)):
            lo, hi = self.piece(k, rank)
            for i, (o, n) in enumerate(zip(self.offsets, self.numels)):
                a, b = max(lo, o), min(hi, o + n)
                if a < b:
                    segs.append(Segment(i, self.piece_off[k] + a - lo, a - o, b - a, int(hp_index[i]), a))
        return segs

    def buckets_of(self, i: int) -> list[int]:
        o, n = self.offsets[i], self.numels[i]
        return [k for k, (s, size) in enumerate(self.buckets) if s < o + n and o < s + size]


class ZeroFlashOptimizer:
    """ZeRO-1 FlashSGD / FlashAdamW / FlashLion over a process group.

    params      : bf16 (or fp32, CUDA) tensors, identical on every rank;
                  they are re-pointed into the flat buffer and their .grad
                  into a flat grad buffer.  fp32 parameters are split once
                  into bf16 + int8 correction (init_flash_state,
                  optim.py:143-161) like FlashAdamW does.
    hparams     : one hyper-parameter object per param group; `group_of[i]`
                  is parameter i's group.
    check_errors: error policy of the fused step (see _errors.ErrorPolicy).
    """

    def __init__(self, params: Sequence[torch.Tensor], optimizer: str, hparams: Sequence, group_of=None,
                 process_group=None, step_fn: Callable | None = None, reduce_op: str = "avg",
                 bucket_elems: int | None = None, overlap_grad_reduce: bool = False,
                 check_errors: bool | str = "deferred", fused_allgather: bool = False):
        from .flat import FlatStates

        self.pg = process_group
        self.world = dist.get_world_size(self.pg)
        self.rank = dist.get_rank(self.pg)
        self.backend = dist.get_backend(self.pg)
        self.optimizer = optimizer
        self.params = list(params)
        self.hparams = list(hparams)
        self.group_of = list(group_of) if group_of is not None else [0] * len(self.params)
        dev = self.params[0].device
        self.device = dev
        if overlap_grad_reduce and bucket_elems is None:
            bucket_elems = 1 << 26
        self.layout = FlatLayout([p.numel() for p in self.params], self.world, bucket_elems=bucket_elems)
        L = self.layout
        self.flat_params = torch.zeros(L.total, dtype=torch.bfloat16, device=dev)
        self.flat_grads = torch.zeros(L.total, dtype=torch.bfloat16, device=dev)
        split_rho = {}
        with torch.no_grad():
            for i, (p, o) in enumerate(zip(self.params, L.offsets)):
                src = p.detach().reshape(-1)
                if p.dtype == torch.float32:
                    from .formats import split

                    lp, rho = split(src)  # init_flash_state: fp32 -> bf16 + int8 rho (raises like the reference)
                    self.flat_params[o:o + p.numel()].copy_(lp)
                    split_rho[i] = rho
                elif p.dtype == torch.bfloat16:
                    self.flat_params[o:o + p.numel()].copy_(src)
                else:
                    raise TypeError(f"parameters must be bf16 or fp32, got {p.dtype}")
                p.data = self.flat_params[o:o + p.numel()].view(p.shape)
                p.grad = self.flat_grads[o:o + p.numel()].view(p.shape)
        self._grad_views = [self.flat_grads[o:o + p.numel()].view(p.shape) for p, o in zip(self.params, L.offsets)]
        self.shard_grads = torch.zeros(L.shard, dtype=torch.bfloat16, device=dev)
        self.segments = L.segments(self.rank, self.group_of)
        # optimizer state for the owned pieces only, one FlashState per segment
        sizes = [s.length for s in self.segments]
        views = [self.flat_params[s.flat_off:s.flat_off + s.length] for s in self.segments]
        self.flat_state = FlatStates(sizes, optimizer, dev, lp_views=views) if sizes else None
        self.states = self.flat_state.states if sizes else []
        for seg, st in zip(self.segments, self.states):
            if seg.param_index in split_rho:
                a = seg.tensor_off
                st.weights.corrections.copy_(split_rho[seg.param_index][a:a + seg.length])
        self.step_fn = step_fn
        self.reduce_op = reduce_op
        self.t = 0
        self._plan = None
        self._errors = None
        self.check_errors = check_errors
        if dev.type == "cuda" and step_fn is None:
            from ._errors import ErrorPolicy

            self._errors = ErrorPolicy(check_errors, dev)
        # overlap of the reduce-scatter with backward
        self._pending_works: dict = {}
        self.rs_launched_in_backward = 0  # bucket reduce-scatters started from the grad hooks
        self._hooks = []
        self._bucket_params = [[] for _ in L.buckets]
        for i in range(len(self.params)):
            for k in L.buckets_of(i):
                self._bucket_params[k].append(i)
        self._remaining = [len(b) for b in self._bucket_params]
        if overlap_grad_reduce:
            index = {id(p): i for i, p in enumerate(self.params)}
            for p in self.params:
                self._hooks.append(p.register_post_accumulate_grad_hook(
                    lambda p, i=index[id(p)]: self._on_grad(i)))
        self.fused_allgather = bool(fused_allgather)
        self._peer_ptrs: list = []
        self._peer_delta = None
        if self.fused_allgather:
            self._map_peers()

    # -- peer memory (fused_allgather) -------------------------------------------------
    def _map_peers(self) -> None:
        """Exchange CUDA IPC handles of the flat parameter buffers and map every
        peer's buffer: delta[r] = (peer r's buffer in this process) - (ours)."""
        import ctypes

        from . import _lib

        if self.device.type != "cuda" or self.step_fn is not None:
            raise ValueError("fused_allgather needs the CUDA step")
        if len(self.hparams) != 1:
            raise ValueError("fused_allgather takes one hyper-parameter set")
        if self.world - 1 > _lib.FO_MAX_PEERS:
            raise ValueError(f"fused_allgather maps at most {_lib.FO_MAX_PEERS} peers")
        L = _lib.lib()
        handle = ctypes.create_string_buffer(64)
        off = ctypes.c_int64(0)
        _lib.check(L.fo_ipc_export(self.flat_params.data_ptr(), handle, ctypes.byref(off)), "fo_ipc_export")
        mine = (bytes(handle.raw), int(off.value))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.pg)
        deltas = []
        for r, (h, o) in enumerate(allh):
            if r == self.rank:
                continue
            buf = ctypes.create_string_buffer(h, 64)
            ptr = ctypes.c_void_p(0)
            _lib.check(L.fo_ipc_open(buf, o, ctypes.byref(ptr)), "fo_ipc_open")
            self._peer_ptrs.append((int(ptr.value), o))
            deltas.append(int(ptr.value) - self.flat_params.data_ptr())
        self._peer_delta = (ctypes.c_int64 * max(1, len(deltas)))(*deltas)
        self._npeers = len(deltas)

    def close(self) -> None:
        """Unmap the peers' parameter buffers (fused_allgather)."""
        from . import _lib

        torch.cuda.synchronize(self.device)
        for ptr, o in self._peer_ptrs:
            _lib.lib().fo_ipc_close(ptr, o)
        self._peer_ptrs = []

    def _peer_barrier(self) -> None:
        """Every rank's fused step (and its stores into our buffer) before our
        next read of the parameters."""
        if self._staged():
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.pg)
        else:  # on the stream: completes only once every rank's step has finished
            t = torch.zeros(1, dtype=torch.int32, device=self.device)
            dist.all_reduce(t, group=self.pg)

    # -- collectives (host-staged for gloo with CUDA tensors) -----------------------
    def _staged(self) -> bool:
        return self.backend == "gloo" and self.device.type == "cuda"

    def _reduce_scatter(self, out: torch.Tensor, inp: torch.Tensor, async_op: bool = False):
        op = dist.ReduceOp.SUM
        if self.reduce_op == "avg" and self.backend == "nccl":
            op = dist.ReduceOp.AVG
        if self._staged():
            h_out = out.cpu()
            dist.reduce_scatter_tensor(h_out, inp.cpu(), op=op, group=self.pg)
            out.copy_(h_out)
            work = None
        else:
            work = dist.reduce_scatter_tensor(out, inp, op=op, group=self.pg, async_op=async_op)
        if self.reduce_op == "avg" and op == dist.ReduceOp.SUM:
            if work is not None:
                work.wait()
                work = None
            out.div_(self.world)
        return work

    def _all_gather(self, out: torch.Tensor, inp: torch.Tensor, async_op: bool = False):
        if self._staged():
            h = out.cpu()
            dist.all_gather_into_tensor(h, inp.cpu(), group=self.pg)
            out.copy_(h)
            return None
        if self.backend == "gloo":
            inp = inp.clone()  # gloo: no aliasing of input and output
        return dist.all_gather_into_tensor(out, inp, group=self.pg, async_op=async_op)

    # -- gradients ---------------------------------------------------------------------
    def _adopt_grad(self, i: int) -> None:
        """Make sure parameter i's gradient lives in its flat-buffer view (a
        user's zero_grad(set_to_none=True) or a reassignment detaches it)."""
        p, view = self.params[i], self._grad_views[i]
        g = p.grad
        if g is None:
            view.zero_()  # no gradient this step: stepped as zero (decay and momentum still apply)
            p.grad = view
        elif g.data_ptr() != view.data_ptr():
            view.copy_(g.reshape(view.shape))
            p.grad = view

    def _launch_bucket_rs(self, k: int, async_op: bool):
        s, size = self.layout.buckets[k]
        per = size // self.world
        so = self.layout.piece_off[k]
        return self._reduce_scatter(self.shard_grads[so:so + per], self.flat_grads[s:s + size], async_op)

    def _on_grad(self, i: int) -> None:
        self._adopt_grad(i)
        for k in self.layout.buckets_of(i):
            self._remaining[k] -= 1
            if self._remaining[k] == 0 and k not in self._pending_works:
                self._pending_works[k] = self._launch_bucket_rs(k, async_op=True)
                self.rs_launched_in_backward += 1

    # -- the three phases --------------------------------------------------------
    def reduce_scatter_grads(self) -> None:
        if not self._hooks:
            for i in range(len(self.params)):
                self._adopt_grad(i)
        for k in range(len(self.layout.buckets)):
            if k not in self._pending_works:
                if self._hooks:
                    for i in self._bucket_params[k]:
                        self._adopt_grad(i)
                self._pending_works[k] = self._launch_bucket_rs(k, async_op=bool(self._hooks))
        for w in self._pending_works.values():
            if w is not None:
                w.wait()
        self._pending_works = {}
        self._remaining = [len(b) for b in self._bucket_params]

    def _scalars(self) -> list:
        return [hp.scalars(self.t + 1) for hp in self.hparams]

    def step_shard(self) -> None:
        if not self.states:
            return
        grads = [self.shard_grads[s.shard_off:s.shard_off + s.length] for s in self.segments]
        if self.step_fn is not None:
            hps = [self.hparams[s.hp_index] for s in self.segments]
            self.step_fn(self.optimizer, self.states, grads, hps)
            return
        from . import _lib
        from ._errors import stream_handle
        from .flat import StepPlan

        if len(self.hparams) > _lib.FO_MAX_HPARAMS:
            raise ValueError(f"at most {_lib.FO_MAX_HPARAMS} param groups")
        if self._plan is None:
            self._plan = StepPlan(self.optimizer, self.states, [s.hp_index for s in self.segments])
            self._plan.set_grads(grads)
        if self.fused_allgather:
            self._plan.launch_peers(self._scalars()[0], self._peer_delta, self._npeers, self._errors.ptr,
                                    stream_handle(self.device))
        else:
            self._plan.launch(self._scalars(), self._errors.ptr, stream_handle(self.device))

    def all_gather_params(self) -> None:
        works = []
        for k in range(len(self.layout.buckets)):
            s, size = self.layout.buckets[k]
            lo, hi = self.layout.piece(k, self.rank)
            works.append(self._all_gather(self.flat_params[s:s + size], self.flat_params[lo:hi],
                                          async_op=len(self.layout.buckets) > 1))
        for w in works:
            if w is not None:
                w.wait()

    @torch.no_grad()
    def step(self) -> None:
        self.reduce_scatter_grads()
        self.step_shard()
        if self.fused_allgather:
            self._peer_barrier()
        else:
            self.all_gather_params()
        self.t += 1
        if self._errors is not None:
            self._errors.after_step(self.optimizer)

    def raise_errors(self) -> None:
        if self._errors is not None:
            self._errors.raise_now(self.optimizer)

    def zero_grad(self, set_to_none: bool = False) -> None:
        """Zero the flat gradient buffer (gradients stay flat-buffer views;
        set_to_none is accepted for torch.optim compatibility and ignored)."""
        self.flat_grads.zero_()
        for p, v in zip(self.params, self._grad_views):
            p.grad = v

    def remove_hooks(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks = []

    # -- checkpoints (SURVEY.md §8e "sharded checkpoints") -----------------------
    # A tensor's state can straddle ranks.  To keep the reference layout -- one
    # FLOP v1 file per tensor with rank-1 (n,) records (checkpoint.py:73-80,
    # :98-125) -- rank 0 gathers, a batch of tensors at a time, every rank's
    # segments of those tensors and writes the files: byte-identical to what a
    # single-GPU FlashState of the whole tensor writes.  Only rank 0 holds a
    # batch (bounded by `batch_bytes`); no rank ever holds the whole state of
    # another.  Loading re-shards: every rank reads the files of the tensors
    # it owns segments of (and every tensor's bf16 weights).

    def _records(self) -> list:
        adam = self.optimizer == "adamw"
        return ["rho", "mq", "ms"] + (["vq", "vs"] if adam else [])

    def _seg_bytes(self, seg: Segment) -> int:
        ng = -(-seg.length // 32)
        adam = self.optimizer == "adamw"
        return seg.length * (3 if adam else 2) + ng * 2 * (2 if adam else 1)

    def _pack(self, segs_states) -> torch.Tensor:
        parts = []
        for seg, st in segs_states:
            parts += [st.weights.corrections.view(torch.uint8), st.momentum.codes.view(torch.uint8),
                      st.momentum.scales.view(torch.uint8)]
            if self.optimizer == "adamw":
                parts += [st.variance.codes.view(torch.uint8), st.variance.scales.view(torch.uint8)]
        if not parts:
            return torch.zeros(0, dtype=torch.uint8, device=self.device)
        return torch.cat([x.reshape(-1) for x in parts])

    def save_checkpoint(self, directory, names: Sequence[str] | None = None,
                        batch_bytes: int = 1 << 30) -> dict | None:
        """Collective: one FLOP v1 file per parameter plus a manifest, written
        by rank 0 (returns the manifest there, None elsewhere)."""
        import json
        import os

        import numpy as np

        from .checkpoint import save_checkpoint
        from .host import HostFlashState

        if self.states and self.states[0].weights.corrections.dtype != torch.int8:
            raise ValueError("sharded checkpoints hold int8 corrections")
        L = self.layout
        nparams = len(self.params)
        all_segs = [L.segments(r, self.group_of) for r in range(self.world)]
        mine = list(zip(self.segments, self.states))
        names = list(names) if names is not None else [f"param{i:05d}" for i in range(nparams)]
        manifest = None
        if self.rank == 0:
            os.makedirs(directory, exist_ok=True)
            manifest = {"format": "FLOP v1 per parameter", "optimizer": self.optimizer, "params": [], "bytes": 0}
        adam = self.optimizer == "adamw"
        i0 = 0
        while i0 < nparams:
            # a batch of whole tensors of about batch_bytes of state
            i1, acc = i0, 0
            while i1 < nparams and (i1 == i0 or acc + L.numels[i1] * 3.2 <= batch_bytes):
                acc += L.numels[i1] * 3.2
                i1 += 1
            sel = lambda segs: [s for s in segs if i0 <= s.param_index < i1]  # noqa: E731
            sizes = [sum(self._seg_bytes(s) for s in sel(segs)) for segs in all_segs]
            cap = max(sizes) if sizes else 0
            buf = self._pack([(s, st) for s, st in mine if i0 <= s.param_index < i1])
            send = torch.zeros(max(cap, 1), dtype=torch.uint8, device=self.device)
            send[:buf.numel()].copy_(buf)
            gl = [torch.empty_like(send) for _ in range(self.world)] if self.rank == 0 else None
            if self._staged():
                h = send.cpu()
                hl = [torch.empty_like(h) for _ in range(self.world)] if self.rank == 0 else None
                dist.gather(h, hl, dst=0, group=self.pg)
                gl = hl
            else:
                dist.gather(send, gl, dst=0, group=self.pg)
            if self.rank == 0:
                lp_all = self.flat_params.view(torch.int16)
                arrays = {}
                for i in range(i0, i1):
                    n = L.numels[i]
                    ng = -(-n // 32)
                    arrays[i] = {"rho": np.zeros(n, np.int8), "mq": np.zeros(n, np.int8),
                                 "ms": np.zeros(ng, np.float16), "vq": np.zeros(n, np.uint8) if adam else None,
                                 "vs": np.zeros(ng, np.float16) if adam else None}
                for r in range(self.world):
                    raw = gl[r].cpu().numpy()
                    pos = 0
                    for s in sel(all_segs[r]):
                        a, m, ga, ng = s.tensor_off, s.length, s.tensor_off // 32, -(-s.length // 32)
                        d = arrays[s.param_index]

                        def take(nbytes, dt):
                            nonlocal pos
                            out = raw[pos:pos + nbytes].view(dt)
                            pos += nbytes
                            return out

                        d["rho"][a:a + m] = take(m, np.int8)
                        d["mq"][a:a + m] = take(m, np.int8)
                        d["ms"][ga:ga + ng] = take(2 * ng, np.float16)
                        if adam:
                            d["vq"][a:a + m] = take(m, np.uint8)
                            d["vs"][ga:ga + ng] = take(2 * ng, np.float16)
                for i in range(i0, i1):
                    o, n = L.offsets[i], L.numels[i]
                    lp = lp_all[o:o + n].cpu().numpy().view(np.uint16)
                    d = arrays[i]
                    hs = HostFlashState(lp, d["rho"], d["mq"], d["ms"], d["vq"], d["vs"], self.t, 32)
                    fname = f"{i:05d}.flop"
                    manifest["bytes"] += save_checkpoint(hs, os.path.join(directory, fname), self.optimizer)
                    manifest["params"].append({"index": i, "name": names[i], "file": fname,
                                               "shape": list(self.params[i].shape)})
            i0 = i1
        if self.rank == 0:
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

        import numpy as np

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
            if hs.rho.dtype != np.int8 or hs.group_size != 32:
                raise CheckpointError(f"parameter {i}: the sharded optimizer holds int8 corrections with "
                                      f"groups of 32 (file: {hs.rho.dtype}, G={hs.group_size})")
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
