"""Device-side group-wise companded 8-bit state codecs (mirror of
flashopt.quantize).

Reference: /root/reference/pkg/src/flashopt/quantize.py
  GroupSpec            :33-44    QuantizedState        :47-64
  quantize_momentum    :109-122  dequantize_momentum   :125-131
  quantize_variance    :134-149  dequantize_variance   :152-158
Scales are stored as fp16 rounded up (torch.float16 tensors), exactly the
reference's bits.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._errors import DeviceErrors, ptr, stream_handle

__all__ = ["GroupSpec", "QuantizedState", "quantize_momentum", "dequantize_momentum", "quantize_variance",
           "dequantize_variance"]

KINDS = ("momentum", "variance", "linear-signed", "linear-unsigned")


@dataclass(frozen=True)
class GroupSpec:
    """Contiguous groups of `group_size` elements, one fp16 scale each."""

    group_size: int = 32

    def __post_init__(self) -> None:
        if self.group_size < 1:
            raise ValueError("group size must be >= 1")

    def num_groups(self, length: int) -> int:
        return -(-length // self.group_size) if length else 0


@dataclass
class QuantizedState:
    """8-bit codes + fp16 group scales of one state buffer, on the device."""

    codes: torch.Tensor   # int8 (momentum / linear-signed) or uint8 (variance / linear-unsigned)
    scales: torch.Tensor  # float16, spec.num_groups(len(codes))
    spec: GroupSpec
    kind: str

    def __post_init__(self) -> None:
        if self.kind not in KINDS:
            raise ValueError(f"unknown state kind: {self.kind}")
        if self.scales.numel() != self.spec.num_groups(self.codes.numel()):
            raise ValueError("scale count does not match group count")

    @property
    def length(self) -> int:
        return int(self.codes.numel())

    def clone(self) -> "QuantizedState":
        return QuantizedState(self.codes.clone(), self.scales.clone(), self.spec, self.kind)


def _flat_f32(x: torch.Tensor) -> torch.Tensor:
    x = x.detach().contiguous().view(-1)
    if x.dtype != torch.float32:
        x = x.float()
    if not x.is_cuda:
        raise ValueError("FlashOptim B200 tensors must live on a CUDA device (no CPU path)")
    return x


def quantize_momentum(m: torch.Tensor, spec: GroupSpec = GroupSpec()) -> QuantizedState:
    m = _flat_f32(m)
    codes = torch.empty(m.numel(), dtype=torch.int8, device=m.device)
    scales = torch.empty(spec.num_groups(m.numel()), dtype=torch.float16, device=m.device)
    err = DeviceErrors(m.device)
    _lib.check(_lib.lib().fo_quantize_momentum(ptr(m), m.numel(), spec.group_size, ptr(codes), ptr(scales),
                                               err.ptr, stream_handle(m.device)), "fo_quantize_momentum")
    err.raise_if_set("adamw")
    return QuantizedState(codes, scales, spec, "momentum")


def dequantize_momentum(q: QuantizedState) -> torch.Tensor:
    if q.kind != "momentum":
        raise ValueError(f"kind-mismatch: expected momentum, got {q.kind}")
    out = torch.empty(q.length, dtype=torch.float32, device=q.codes.device)
    _lib.check(_lib.lib().fo_dequantize_momentum(ptr(q.codes), ptr(q.scales), q.length, q.spec.group_size,
                                                 ptr(out), stream_handle(q.codes.device)), "fo_dequantize_momentum")
    return out


def quantize_variance(v: torch.Tensor, spec: GroupSpec = GroupSpec()) -> QuantizedState:
    v = _flat_f32(v)
    codes = torch.empty(v.numel(), dtype=torch.uint8, device=v.device)
    scales = torch.empty(spec.num_groups(v.numel()), dtype=torch.float16, device=v.device)
    err = DeviceErrors(v.device)
    _lib.check(_lib.lib().fo_quantize_variance(ptr(v), v.numel(), spec.group_size, ptr(codes), ptr(scales),
                                               err.ptr, stream_handle(v.device)), "fo_quantize_variance")
    err.raise_if_set("adamw")
    return QuantizedState(codes, scales, spec, "variance")


def dequantize_variance(q: QuantizedState) -> torch.Tensor:
    if q.kind != "variance":
        raise ValueError(f"kind-mismatch: expected variance, got {q.kind}")
    out = torch.empty(q.length, dtype=torch.float32, device=q.codes.device)
    _lib.check(_lib.lib().fo_dequantize_variance(ptr(q.codes), ptr(q.scales), q.length, q.spec.group_size,
                                                 ptr(out), stream_handle(q.codes.device)), "fo_dequantize_variance")
    return out
