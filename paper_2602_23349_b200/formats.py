"""Device-side weight split codec (mirror of flashopt.formats).

A master weight is held as a bf16 code plus a signed ULP-scaled correction
(`rho`, int8 with N = 127 or int16 with N = 32767).  The arithmetic runs in
the CUDA library (csrc/fo_math.cuh, fo_codec.cu); this module only moves
torch device tensors across the C ABI.

Reference: /root/reference/pkg/src/flashopt/formats.py
  split        :232-245  -> split()
  reconstruct  :248-276  -> reconstruct()
  SplitTensor  :300-333  -> SplitTensor
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._errors import DeviceErrors, ptr, stream_handle

__all__ = ["BF16", "INT8_CORRECTION", "INT16_CORRECTION", "CorrectionWidth", "SplitTensor", "split",
           "reconstruct", "upcast"]

BF16 = "bf16"  # the only low-precision weight format a FlashState uses (optim.py:155, checkpoint.py:251)


@dataclass(frozen=True)
class CorrectionWidth:
    """Correction code width: 8 or 16 bits, symmetric range [-N, N] (formats.py:75-95)."""

    bits: int

    def __post_init__(self) -> None:
        if self.bits not in (8, 16):
            raise ValueError("correction width must be 8 or 16 bits")

    @property
    def n(self) -> int:
        return (1 << (self.bits - 1)) - 1

    @property
    def dtype(self) -> torch.dtype:
        return torch.int8 if self.bits == 8 else torch.int16


INT8_CORRECTION = CorrectionWidth(8)
INT16_CORRECTION = CorrectionWidth(16)


def _width_of(rho: torch.Tensor) -> CorrectionWidth:
    if rho.dtype == torch.int8:
        return INT8_CORRECTION
    if rho.dtype == torch.int16:
        return INT16_CORRECTION
    raise TypeError(f"corrections must be int8 or int16, got {rho.dtype}")


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda:
            raise ValueError("FlashOptim B200 tensors must live on a CUDA device (no CPU path)")
        if not t.is_contiguous():
            raise ValueError("FlashOptim B200 tensors must be contiguous")


def upcast(lp: torch.Tensor) -> torch.Tensor:
    """Exact bf16 -> f32 widening (formats.py:183-187)."""
    return lp.float()


def split(theta: torch.Tensor, width: CorrectionWidth = INT8_CORRECTION) -> tuple[torch.Tensor, torch.Tensor]:
    """fp32 -> (bf16 codes, correction codes); raises `split-nonfinite` like
    formats.py:242-243.  Synchronises to check the device error word."""
    theta = theta.detach().contiguous().view(-1)
    if theta.dtype != torch.float32:
        raise TypeError("split expects float32 master weights")
    _require_cuda(theta)
    lp = torch.empty(theta.numel(), dtype=torch.bfloat16, device=theta.device)
    rho = torch.empty(theta.numel(), dtype=width.dtype, device=theta.device)
    err = DeviceErrors(theta.device)
    _lib.check(_lib.lib().fo_split(ptr(theta), theta.numel(), ptr(lp), ptr(rho), width.bits, err.ptr,
                                   stream_handle(theta.device)), "fo_split")
    err.raise_if_set("adamw")
    return lp, rho


def reconstruct(lp: torch.Tensor, rho: torch.Tensor) -> torch.Tensor:
    """(bf16, rho) -> fp32 master weights (formats.py:248-276)."""
    _require_cuda(lp, rho)
    if lp.numel() != rho.numel():
        raise ValueError("lp_values and corrections must have identical shape")
    width = _width_of(rho)
    out = torch.empty(lp.numel(), dtype=torch.float32, device=lp.device)
    err = DeviceErrors(lp.device)
    _lib.check(_lib.lib().fo_reconstruct(ptr(lp), ptr(rho), width.bits, lp.numel(), ptr(out), err.ptr,
                                         stream_handle(lp.device)), "fo_reconstruct")
    err.raise_if_set("adamw")
    return out


@dataclass
class SplitTensor:
    """Compressed master weights on the device: bf16 values + corrections."""

    lp_values: torch.Tensor   # torch.bfloat16, flat
    corrections: torch.Tensor  # torch.int8 / torch.int16, flat

    def __post_init__(self) -> None:
        if self.lp_values.shape != self.corrections.shape:
            raise ValueError("lp_values and corrections must have identical shape")

    @property
    def width(self) -> CorrectionWidth:
        return _width_of(self.corrections)

    @property
    def length(self) -> int:
        return int(self.lp_values.numel())

    @classmethod
    def from_values(cls, theta: torch.Tensor, width: CorrectionWidth = INT8_CORRECTION) -> "SplitTensor":
        lp, rho = split(theta, width)
        return cls(lp, rho)

    def lp_float(self) -> torch.Tensor:
        return upcast(self.lp_values)

    def reconstruct(self) -> torch.Tensor:
        return reconstruct(self.lp_values, self.corrections)

    def clone(self) -> "SplitTensor":
        return SplitTensor(self.lp_values.clone(), self.corrections.clone())
