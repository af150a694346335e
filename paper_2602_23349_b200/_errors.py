"""Device error word <-> reference ValueError mapping, plus small pointer
helpers shared by the host modules."""

from __future__ import annotations

import torch

from . import _lib


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class DeviceErrors:
    """A 4-byte device word the kernels atomicOr FO_ERR_* bits into.

    Reading it synchronises the stream; the reference raises before
    producing output, the device path reports after the fact."""

    def __init__(self, device: torch.device):
        self.word = torch.zeros(1, dtype=torch.int32, device=device)

    @property
    def ptr(self) -> int:
        return self.word.data_ptr()

    def mask(self) -> int:
        return int(self.word.item()) & 0xFFFFFFFF

    def reset(self) -> None:
        self.word.zero_()

    def raise_if_set(self, optimizer: str, variance_scheme: str = "companded") -> None:
        m = self.mask()
        if m:
            raise_for_mask(m, optimizer, variance_scheme)


class ErrorPolicy:
    """When an optimizer reads its device error word.

    "sync" (True): after every step, one device-to-host read that waits for
        the step -- the reference's timing (it raises inside the step call),
        but the host can no longer run ahead of the GPU.
    "deferred" (the default): after every step the word is copied into
        pinned host memory on the step's stream and an event is recorded; the
        next step() (or an explicit check) looks at it only if the event has
        completed, so nothing ever blocks.  An error is raised at most one
        step late; the state has been updated by then either way (device
        kernels cannot raise before writing).
    "off" (False): never read automatically; call raise_errors().
    """

    def __init__(self, mode, device: torch.device):
        if mode is True:
            mode = "sync"
        elif mode is False or mode is None:
            mode = "off"
        if mode not in ("sync", "deferred", "off"):
            raise ValueError(f"check_errors must be True, False, 'sync', 'deferred' or 'off', got {mode!r}")
        self.mode = mode
        self.errors = DeviceErrors(device)
        self._host = torch.zeros(1, dtype=torch.int32, pin_memory=True) if mode == "deferred" else None
        self._event = None

    @property
    def ptr(self) -> int:
        return self.errors.ptr

    def after_step(self, optimizer: str, stream=None, variance_scheme: str = "companded") -> None:
        if self.mode == "sync":
            self.raise_now(optimizer, variance_scheme)
        elif self.mode == "deferred":
            self.poll(optimizer, variance_scheme)
            s = stream or torch.cuda.current_stream(self.errors.word.device)
            with torch.cuda.stream(s):
                self._host.copy_(self.errors.word, non_blocking=True)
                self._event = torch.cuda.Event()
                self._event.record(s)

    def poll(self, optimizer: str, variance_scheme: str = "companded") -> None:
        """Raise if an earlier step's errors have reached the host (non-blocking)."""
        ev = self._event
        if ev is None or not ev.query():
            return
        self._event = None
        m = int(self._host.item()) & 0xFFFFFFFF
        if m:
            self.errors.reset()
            raise_for_mask(m, optimizer, variance_scheme)

    def raise_now(self, optimizer: str, variance_scheme: str = "companded") -> None:
        """Wait for the queued steps and raise for any flagged error."""
        self._event = None
        m = self.errors.mask()
        if m:
            self.errors.reset()
            raise_for_mask(m, optimizer, variance_scheme)


def raise_for_mask(mask: int, optimizer: str, variance_scheme: str = "companded") -> None:
    msg = _lib.error_message(mask, optimizer)
    if variance_scheme == "linear" and msg.startswith("negative-variance"):
        msg = "negative-unsigned: unsigned buffer has negative entries"  # quantize.py:166
    raise ValueError(msg)
