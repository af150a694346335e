"""Host-resident FlashState stepped on the B200 (fo_step_host).

This is the reference's own calling convention -- the state and the
gradient are NumPy arrays in host memory and `adamw_step(state, grad, hp)`
updates them (optim.py:187-261) -- executed by the CUDA library: the arrays
are streamed through device slots (H2D copy, fused step, D2H copy) with the
copies overlapping the kernels.  Use `pinned_state` for full PCIe bandwidth.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from ._errors import raise_for_mask

__all__ = ["HostFlashState", "pinned_empty", "pinned_state", "step_host"]


@dataclass
class HostFlashState:
    """FLOP v1 record arrays (checkpoint.py:111-123) in host memory."""

    lp: np.ndarray                     # uint16 bf16 codes   "weights.lp"
    rho: np.ndarray                    # int8 / int16        "weights.rho"
    m_codes: np.ndarray                # int8                "momentum.codes"
    m_scales: np.ndarray               # float16             "momentum.scales"
    v_codes: np.ndarray | None = None  # uint8               "variance.codes"
    v_scales: np.ndarray | None = None  # float16            "variance.scales"
    t: int = 0
    group_size: int = 32
    variance_scheme: str = "companded"

    @property
    def length(self) -> int:
        return int(self.lp.size)


def pinned_empty(n: int, dtype) -> np.ndarray:
    """A NumPy view of page-locked host memory (torch's pinned allocator)."""
    import torch

    tdt = {np.dtype(np.uint16): torch.int16, np.dtype(np.int16): torch.int16, np.dtype(np.int8): torch.int8,
           np.dtype(np.uint8): torch.uint8, np.dtype(np.float16): torch.float16,
           np.dtype(np.float32): torch.float32}[np.dtype(dtype)]
    t = torch.empty(int(n), dtype=tdt, pin_memory=True)
    return t.numpy().view(dtype)


def pinned_state(n: int, optimizer: str, group_size: int = 32, rho_dtype=np.int8) -> HostFlashState:
    ng = -(-n // group_size) if n else 0
    adam = optimizer == "adamw"
    return HostFlashState(pinned_empty(n, np.uint16), pinned_empty(n, rho_dtype), pinned_empty(n, np.int8),
                          pinned_empty(ng, np.float16), pinned_empty(n, np.uint8) if adam else None,
                          pinned_empty(ng, np.float16) if adam else None, 0, group_size)


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    if not a.flags.c_contiguous:
        raise ValueError("host state arrays must be C-contiguous")
    return a.ctypes.data


def step_host(optimizer: str, states: Sequence[HostFlashState], grads: Sequence[np.ndarray], hps,
              chunk_elems: int = 0, check: bool = True) -> int:
    """Step host-resident states in place on the GPU; returns the error mask
    (raising the reference's ValueError when `check`)."""
    from .optim import HP_TYPES

    if len(states) != len(grads):
        raise ValueError("states and grads differ in length")
    if not isinstance(hps, (list, tuple)):
        hps = [hps] * len(states)
    if not states:
        return 0
    table, scalars, tensors = {}, [], []
    gdt = None
    s0 = states[0]
    for st, g, hp in zip(states, grads, hps):
        if not isinstance(hp, HP_TYPES[optimizer]):
            raise TypeError(f"{optimizer} step needs {HP_TYPES[optimizer].__name__}")
        if g.size != st.length:
            raise ValueError("gradient length does not match state")
        if (st.group_size, st.rho.dtype, st.variance_scheme) != (s0.group_size, s0.rho.dtype, s0.variance_scheme):
            raise ValueError("one call needs one layout (group size, correction width, variance scheme)")
        d = g.dtype
        if d not in (np.float32, np.uint16, np.int16):
            raise TypeError("grads must be float32 or bf16 bit patterns (uint16)")
        gdt = gdt or d
        if (d == np.float32) != (gdt == np.float32):
            raise ValueError("one call needs one gradient dtype")
        key = (hp, st.t + 1)
        if key not in table:
            table[key] = len(scalars)
            scalars.append(hp.scalars(st.t + 1))
        tensors.append(_lib.fo_tensor(_ptr(st.lp), _ptr(st.rho), _ptr(st.m_codes), _ptr(st.m_scales),
                                      _ptr(st.v_codes) if optimizer == "adamw" else None,
                                      _ptr(st.v_scales) if optimizer == "adamw" else None, _ptr(g), st.length,
                                      table[key], 0))
    arr = (_lib.fo_tensor * len(tensors))(*tensors)
    hp_arr = (_lib.fo_hparams * len(scalars))(*scalars)
    err = ctypes.c_uint32(0)
    _lib.check(_lib.lib().fo_step_host(
        _lib.OPT_TAGS[optimizer], arr, len(tensors), hp_arr, len(scalars),
        _lib.FO_GRAD_F32 if gdt == np.float32 else _lib.FO_GRAD_BF16, s0.rho.dtype.itemsize * 8, s0.group_size,
        _lib.FO_VAR_LINEAR if s0.variance_scheme == "linear" else _lib.FO_VAR_COMPANDED, int(chunk_elems),
        ctypes.byref(err)), "fo_step_host")
    for st in states:
        st.t += 1
    if check and err.value:
        raise_for_mask(err.value, optimizer, s0.variance_scheme)
    return int(err.value)
