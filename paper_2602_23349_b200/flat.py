"""Flat HBM layout for the optimizer state of a whole parameter list, and a
cached launch plan for the fused multi-tensor step.

Layout: one contiguous buffer per record kind -- rho (i8),
momentum codes (i8), variance codes (u8), momentum scales (f16), variance
scales (f16) -- with every tensor's slice starting at a multiple of
ALIGN = 64 elements, so every slice is 16-byte aligned for 128-bit loads
and every group of 32 lies inside one tensor (groups never span tensors,
quantize.py:72-79).  The bf16 weights and the gradients stay wherever the
caller keeps them (model parameters / .grad), so the flat buffers only hold
what the optimizer owns: 3 + 4/32 bytes per parameter for FlashAdamW.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import torch

from . import _lib
from .formats import SplitTensor
from .optim import FlashState
from .quantize import GroupSpec, QuantizedState

ALIGN = 64


def _round_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


class FlatStates:
    """Optimizer-owned state buffers for `sizes`, with FlashState views."""

    def __init__(self, sizes: Sequence[int], optimizer: str, device, group_size: int = 32,
                 lp_views: Sequence[torch.Tensor] | None = None, rho_bits: int = 8,
                 variance_scheme: str = "companded"):
        if rho_bits not in (8, 16) or variance_scheme not in ("companded", "linear"):
            raise ValueError("rho_bits must be 8 or 16 and variance_scheme companded or linear")
        self.optimizer = optimizer
        self.variance_scheme = variance_scheme
        self.sizes = [int(s) for s in sizes]
        self.spec = GroupSpec(group_size)
        self.offsets, self.goffsets = [], []
        off = goff = 0
        for n in self.sizes:
            self.offsets.append(off)
            self.goffsets.append(goff)
            off += _round_up(n, ALIGN)
            goff += _round_up(self.spec.num_groups(n), ALIGN // 2)
        self.total, self.gtotal = off, goff
        dev = torch.device(device)
        self.rho = torch.zeros(off, dtype=torch.int8 if rho_bits == 8 else torch.int16, device=dev)
        self.m_codes = torch.zeros(off, dtype=torch.int8, device=dev)
        self.m_scales = torch.zeros(goff, dtype=torch.float16, device=dev)
        adam = optimizer == "adamw"
        self.v_codes = torch.zeros(off, dtype=torch.uint8, device=dev) if adam else None
        self.v_scales = torch.zeros(goff, dtype=torch.float16, device=dev) if adam else None
        if lp_views is None:
            self.lp = torch.zeros(off, dtype=torch.bfloat16, device=dev)
            lp_views = [self.lp[o:o + n] for o, n in zip(self.offsets, self.sizes)]
        else:
            self.lp = None
        self.states: list[FlashState] = []
        for i, n in enumerate(self.sizes):
            o, go, ng = self.offsets[i], self.goffsets[i], self.spec.num_groups(n)
            w = SplitTensor(lp_views[i].reshape(-1), self.rho[o:o + n])
            m = QuantizedState(self.m_codes[o:o + n], self.m_scales[go:go + ng], self.spec, "momentum")
            v = None
            if adam:
                kind = "variance" if variance_scheme == "companded" else "linear-unsigned"
                v = QuantizedState(self.v_codes[o:o + n], self.v_scales[go:go + ng], self.spec, kind)
            self.states.append(FlashState(w, m, v, 0, variance_scheme if adam else "companded"))

    @property
    def numel(self) -> int:
        return sum(self.sizes)


class StepPlan:
    """Pre-built fo_tensor table for a fixed list of states.  Per step only
    gradient pointers and the hyper-parameter table change."""

    def __init__(self, optimizer: str, states: Sequence[FlashState], hp_index: Sequence[int] | None = None):
        self.optimizer = optimizer
        self.tag = _lib.OPT_TAGS[optimizer]
        self.states = list(states)
        self.table = (_lib.fo_tensor * len(self.states))()
        adam = optimizer == "adamw"
        for i, st in enumerate(self.states):
            e = self.table[i]
            e.lp = st.weights.lp_values.data_ptr()
            e.rho = st.weights.corrections.data_ptr()
            e.m_codes = st.momentum.codes.data_ptr()
            e.m_scales = st.momentum.scales.data_ptr()
            e.v_codes = st.variance.codes.data_ptr() if adam else None
            e.v_scales = st.variance.scales.data_ptr() if adam else None
            e.n = st.length
            e.hp_index = 0 if hp_index is None else int(hp_index[i])
        st0 = self.states[0]
        self.rho_bits = st0.weights.width.bits
        self.group_size = st0.momentum.spec.group_size
        self.var_scheme = _lib.FO_VAR_LINEAR if st0.variance_scheme == "linear" else _lib.FO_VAR_COMPANDED
        for st in self.states:
            if (st.weights.width.bits, st.momentum.spec.group_size, st.variance_scheme) != \
                    (self.rho_bits, self.group_size, st0.variance_scheme):
                raise ValueError("a StepPlan needs one layout (correction width, group size, variance scheme)")
        self._grad_ptrs: tuple = ()
        self.grad_dtype = _lib.FO_GRAD_BF16

    def set_grads(self, grads: Sequence[torch.Tensor]) -> None:
        ptrs = tuple(g.data_ptr() for g in grads)
        if ptrs == self._grad_ptrs:
            return
        dts = {g.dtype for g in grads}
        if dts - {torch.bfloat16, torch.float32} or len(dts) != 1:
            raise ValueError("a StepPlan needs all-bf16 or all-f32 gradients")
        self.grad_dtype = _lib.FO_GRAD_BF16 if dts == {torch.bfloat16} else _lib.FO_GRAD_F32
        for i, (p, g) in enumerate(zip(ptrs, grads)):
            if g.numel() != self.table[i].n:
                raise ValueError("gradient length does not match state")
            self.table[i].grad = p
        self._grad_ptrs = ptrs

    def launch_peers(self, hparams: _lib.fo_hparams, peer_delta, npeers: int, err_ptr: int | None,
                     stream_handle: int) -> None:
        """The fused step + all-gather (fo_step_mt_peers): every updated
        weights.lp value is also written at the byte deltas `peer_delta`
        (one hyper-parameter set; the default layout)."""
        if self.rho_bits != 8 or self.group_size != 32 or self.var_scheme != _lib.FO_VAR_COMPANDED:
            raise ValueError("the fused all-gather takes the default layout only")
        hp = (_lib.fo_hparams * 1)(hparams)
        _lib.check(_lib.lib().fo_step_mt_peers(self.tag, self.table, len(self.states), hp, self.grad_dtype,
                                               peer_delta, npeers, err_ptr, stream_handle),
                   "fo_step_mt_peers")
        for st in self.states:
            st.t += 1

    def launch(self, hparams: Sequence[_lib.fo_hparams], err_ptr: int | None, stream_handle: int) -> None:
        hp = (_lib.fo_hparams * len(hparams))(*hparams)
        _lib.check(_lib.lib().fo_step_mt(self.tag, self.table, len(self.states), hp, len(hparams),
                                         self.grad_dtype, self.rho_bits, self.group_size, self.var_scheme,
                                         err_ptr, stream_handle), "fo_step_mt")
        for st in self.states:
            st.t += 1


def make_hparams_list(hps: Sequence, ts: Sequence[int]) -> list:
    return [hp.scalars(t) for hp, t in zip(hps, ts)]


__all__ = ["FlatStates", "StepPlan", "ALIGN", "make_hparams_list", "ctypes"]
