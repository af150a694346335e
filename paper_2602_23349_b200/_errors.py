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


def raise_for_mask(mask: int, optimizer: str, variance_scheme: str = "companded") -> None:
    msg = _lib.error_message(mask, optimizer)
    if variance_scheme == "linear" and msg.startswith("negative-variance"):
        msg = "negative-unsigned: unsigned buffer has negative entries"  # quantize.py:166
    raise ValueError(msg)
