"""Gradient release: the fused step runs from backward hooks, so a
parameter's gradient lives only until its own step has consumed it.

Reference: the eager loop of training.py:209-226 steps each tensor as soon as
its gradient is yielded by the lazy reverse-order backward (mlp.py:113-153)
and refreshes the compute weights at once (training.py:221-223)
states it is bitwise identical to stepping after the full backward.  PAPER.md
:353-356 gives the memory effect (7 -> 5 bytes/param for FlashAdamW).

B200 mapping:
  * `Tensor.register_post_accumulate_grad_hook` fires when a parameter's
    gradient is complete (after every use of the parameter in backward, so
    overwriting the weight is safe -- the autograd graph no longer needs it);
  * the hook hands the gradient to a bucket and drops `param.grad`; once the
    bucket holds `bucket_elems` elements (or backward ends) a side stream
    waits on the autograd stream and launches ONE fused step for every
    tensor in the bucket (fo_step_mt with a small __grid_constant__ table,
    one launch per param group), instead of one launch per parameter;
  * the gradient tensors are handed to the side stream (`record_stream`),
    so the caching allocator can reuse their memory as soon as the step
    kernel has read them: at most one bucket of gradients is alive at once;
  * a callback queued on the autograd engine flushes the last bucket and
    makes the compute stream wait for the side stream when backward ends, so
    the next forward sees the new weights.
"""

from __future__ import annotations

import torch

from ._errors import ErrorPolicy


class GradientRelease:
    """Attach to a FlashAdamW / FlashSGD / FlashLion; afterwards call only
    `loss.backward()` (no optimizer.step(), no zero_grad()).

    bucket_elems: gradients are stepped in fused launches of at least this
        many elements (the last bucket of a backward may be smaller); 0 steps
        every parameter on its own.
    check_errors: error policy (see _errors.ErrorPolicy); "deferred" reads the
        error word asynchronously at the end of each backward.
    timing: record CUDA events around every side-stream launch
        (`side_stream_ms()`).
    """

    def __init__(self, optimizer, stream: torch.cuda.Stream | None = None, bucket_elems: int = 1 << 25,
                 check_errors: bool | str = "deferred", timing: bool = False):
        self.opt = optimizer
        if getattr(optimizer, "capturable", False):
            raise ValueError("gradient release steps from backward hooks; use an optimizer with capturable=False")
        params = [p for g in optimizer.param_groups for p in g["params"]]
        if not params:
            raise ValueError("optimizer has no parameters")
        self.device = params[0].device
        self.stream = stream or torch.cuda.Stream(self.device)
        self.policy = ErrorPolicy(check_errors, self.device)
        self.errors = self.policy.errors
        self.bucket_elems = int(bucket_elems)
        self.group_of = {}
        for g in optimizer.param_groups:
            for p in g["params"]:
                self.group_of[p] = g
        self.handles = [p.register_post_accumulate_grad_hook(self._hook) for p in params]
        self._pending = False
        self._bucket: list = []
        self._bucket_n = 0
        self.steps_launched = 0   # parameters stepped
        self.launch_calls = 0     # fused launches (one per bucket and param group)
        self.timing = timing
        self._events: list = []

    def _flush(self) -> None:
        if not self._bucket:
            return
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)  # every gradient in the bucket (and every use of its param) is done
        bucket, self._bucket, self._bucket_n = self._bucket, [], 0
        by_group: dict = {}
        for p, g in bucket:
            by_group.setdefault(id(self.group_of[p]), (self.group_of[p], [], []))
            _, ps, gs = by_group[id(self.group_of[p])]
            ps.append(p)
            gs.append(g)
        with torch.cuda.stream(self.stream):
            if self.timing:
                a = torch.cuda.Event(enable_timing=True)
                a.record(self.stream)
            for group, ps, gs in by_group.values():
                self.opt._launch(ps, gs, group, stream=self.stream, errors=self.policy)
                self.launch_calls += 1
            if self.timing:
                b = torch.cuda.Event(enable_timing=True)
                b.record(self.stream)
                self._events.append((a, b))
        for _, g in bucket:
            g.record_stream(self.stream)
        self.steps_launched += len(bucket)

    def _finish(self) -> None:
        self._flush()
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        self._pending = False
        self.policy.after_step(self.opt.OPT, stream=self.stream)

    def _hook(self, p: torch.Tensor) -> None:
        if p.grad is None:
            return
        if not self._pending:
            self._pending = True
            torch.autograd.Variable._execution_engine.queue_callback(self._finish)
        g = p.grad
        self._bucket.append((p, g.reshape(-1)))
        self._bucket_n += g.numel()
        p.grad = None
        if self._bucket_n >= self.bucket_elems:
            self._flush()

    def side_stream_ms(self, reset: bool = True) -> float:
        """Device time of the side-stream launches recorded so far (syncs)."""
        self.stream.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in self._events)
        if reset:
            self._events = []
        return ms

    def check(self) -> None:
        """Raise the reference's ValueError for any flagged error (syncs)."""
        if self._pending:
            self._finish()
        self.policy.raise_now(self.opt.OPT)

    def remove(self) -> None:
        for h in self.handles:
            h.remove()
        self.handles = []
