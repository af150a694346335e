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
  * the hook records an event on the autograd stream, and a side stream
    waits on it and launches the fused step for that one tensor (a small
    __grid_constant__ parameter block, fo_step_mt);
  * the gradient tensor is handed to the side stream (`record_stream`) and
    dropped (`param.grad = None`), so the caching allocator can reuse its
    memory as soon as the step kernel has read it;
  * a callback queued on the autograd engine makes the compute stream wait
    for the side stream when backward ends, so the next forward sees the new
    weights.
"""

from __future__ import annotations

import torch

from ._errors import DeviceErrors


class GradientRelease:
    """Attach to a FlashAdamW / FlashSGD / FlashLion; afterwards call only
    `loss.backward()` (no optimizer.step(), no zero_grad())."""

    def __init__(self, optimizer, stream: torch.cuda.Stream | None = None):
        self.opt = optimizer
        params = [p for g in optimizer.param_groups for p in g["params"]]
        if not params:
            raise ValueError("optimizer has no parameters")
        self.device = params[0].device
        self.stream = stream or torch.cuda.Stream(self.device)
        self.errors = DeviceErrors(self.device)
        self.group_of = {}
        for g in optimizer.param_groups:
            for p in g["params"]:
                self.group_of[p] = g
        self.handles = [p.register_post_accumulate_grad_hook(self._hook) for p in params]
        self._pending = False
        self.steps_launched = 0

    def _finish(self) -> None:
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        self._pending = False

    def _hook(self, p: torch.Tensor) -> None:
        if p.grad is None:
            return
        cur = torch.cuda.current_stream(self.device)
        if not self._pending:
            self._pending = True
            torch.autograd.Variable._execution_engine.queue_callback(self._finish)
        self.stream.wait_stream(cur)  # the gradient (and every earlier use of p) is ready
        g = p.grad
        with torch.cuda.stream(self.stream):
            self.opt._launch([p], [g.reshape(-1)], self.group_of[p], stream=self.stream, errors=self.errors)
        g.record_stream(self.stream)
        p.grad = None
        self.steps_launched += 1

    def check(self) -> None:
        """Raise the reference's ValueError for any flagged error (syncs)."""
        self._finish() if self._pending else None
        m = self.errors.mask()
        if m:
            from ._errors import raise_for_mask

            self.errors.reset()
            raise_for_mask(m, self.opt.OPT)

    def remove(self) -> None:
        for h in self.handles:
            h.remove()
        self.handles = []
