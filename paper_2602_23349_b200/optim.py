"""FlashSGD / FlashAdamW / FlashLion steps on device state (mirror of
flashopt.optim).

Reference: /root/reference/pkg/src/flashopt/optim.py
  *HyperParams      :47-94    FlashState       :114-130
  init_flash_state  :143-161  sgd_step :187-205  adamw_step :208-235
  lion_step         :238-258  STEP_FUNCTIONS   :261

Two call styles:
  * `adamw_step(state, grad, hp) -> FlashState` keeps the reference's pure
    contract: the input state is never mutated (its buffers are cloned and
    the clone is stepped), errors raise ValueError with the reference
    message and no state is returned.
  * `adamw_step_(state, grad, hp)` / `step_many(...)` step in place, which
    is what the torch.optim classes, gradient release and ZeRO-1 use; many
    tensors go to the GPU in one fused multi-tensor launch.
All arithmetic happens in libflashoptim_b200.so; there is no CPU path.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Sequence

import torch

from . import _lib
from ._errors import DeviceErrors, raise_for_mask, stream_handle
from .formats import INT8_CORRECTION, SplitTensor, split
from .quantize import GroupSpec, QuantizedState

__all__ = ["SgdHyperParams", "AdamHyperParams", "LionHyperParams", "FlashState", "init_flash_state", "sgd_step",
           "adamw_step", "lion_step", "sgd_step_", "adamw_step_", "lion_step_", "step_many", "STEP_FUNCTIONS",
           "STEP_FUNCTIONS_INPLACE", "OPTIMIZERS"]

OPTIMIZERS = ("sgd", "adamw", "lion")


def _check_lr(lr: float) -> None:
    if not math.isfinite(lr):
        raise ValueError("learning rate must be finite")


def _check_beta(*betas: float) -> None:
    if not all(0.0 <= b < 1.0 for b in betas):
        raise ValueError("betas must lie in [0, 1)")


def _check_wd(wd: float) -> None:
    if wd < 0.0:
        raise ValueError("weight decay must be >= 0")


@dataclass(frozen=True)
class SgdHyperParams:
    """optim.py:47-58."""

    lr: float
    momentum: float = 0.9
    weight_decay: float = 0.0

    def __post_init__(self) -> None:
        _check_lr(self.lr)
        if not 0.0 <= self.momentum < 1.0:
            raise ValueError("momentum must lie in [0, 1)")
        _check_wd(self.weight_decay)

    def scalars(self, t: int) -> _lib.fo_hparams:
        return _lib.make_hparams("sgd", self.lr, momentum=self.momentum, weight_decay=self.weight_decay, t=t)


@dataclass(frozen=True)
class AdamHyperParams:
    """optim.py:61-76."""

    lr: float
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0

    def __post_init__(self) -> None:
        _check_lr(self.lr)
        _check_beta(self.beta1, self.beta2)
        if self.eps <= 0.0:
            raise ValueError("eps must be > 0")
        _check_wd(self.weight_decay)

    def scalars(self, t: int) -> _lib.fo_hparams:
        return _lib.make_hparams("adamw", self.lr, self.beta1, self.beta2, self.eps, self.weight_decay, t=t)


@dataclass(frozen=True)
class LionHyperParams:
    """optim.py:79-94."""

    lr: float
    beta1: float = 0.9
    beta2: float = 0.99
    weight_decay: float = 0.0

    def __post_init__(self) -> None:
        _check_lr(self.lr)
        _check_beta(self.beta1, self.beta2)
        _check_wd(self.weight_decay)

    def scalars(self, t: int) -> _lib.fo_hparams:
        return _lib.make_hparams("lion", self.lr, self.beta1, self.beta2, weight_decay=self.weight_decay, t=t)


HP_TYPES = {"sgd": SgdHyperParams, "adamw": AdamHyperParams, "lion": LionHyperParams}


@dataclass
class FlashState:
    """Compressed optimizer state of one flat tensor, resident in HBM
    (optim.py:114-130)."""

    weights: SplitTensor
    momentum: QuantizedState
    variance: QuantizedState | None  # AdamW only
    t: int = 0
    variance_scheme: str = "companded"

    @property
    def length(self) -> int:
        return self.weights.length

    @property
    def device(self) -> torch.device:
        return self.weights.lp_values.device

    def weights_for_compute(self) -> torch.Tensor:
        """The bf16 weight component as f32 (what the reference trains on)."""
        return self.weights.lp_float()

    def clone(self) -> "FlashState":
        return FlashState(self.weights.clone(), self.momentum.clone(),
                          None if self.variance is None else self.variance.clone(), self.t, self.variance_scheme)


def init_flash_state(theta0: torch.Tensor, optimizer: str, spec: GroupSpec = GroupSpec(),
                     variance_scheme: str = "companded") -> FlashState:
    """Split fp32 master weights and zero both moments (optim.py:143-161)."""
    if optimizer not in OPTIMIZERS:
        raise ValueError(f"unknown optimizer: {optimizer}")
    if variance_scheme not in ("companded", "linear"):
        raise ValueError(f"unknown variance scheme: {variance_scheme}")
    theta0 = theta0.detach().reshape(-1).float()
    lp, rho = split(theta0, INT8_CORRECTION)
    n, dev = theta0.numel(), theta0.device
    ng = spec.num_groups(n)
    momentum = QuantizedState(torch.zeros(n, dtype=torch.int8, device=dev),
                              torch.zeros(ng, dtype=torch.float16, device=dev), spec, "momentum")
    variance = None
    if optimizer == "adamw":
        kind = "variance" if variance_scheme == "companded" else "linear-unsigned"
        variance = QuantizedState(torch.zeros(n, dtype=torch.uint8, device=dev),
                                  torch.zeros(ng, dtype=torch.float16, device=dev), spec, kind)
    return FlashState(SplitTensor(lp, rho), momentum, variance, 0, variance_scheme)


# ---------------------------------------------------------------------------
# in-place multi-tensor stepping
# ---------------------------------------------------------------------------

@dataclass
class _Batch:
    tensors: list = field(default_factory=list)
    keep: list = field(default_factory=list)  # keeps converted grads alive until the launch is enqueued


def _grad_view(grad: torch.Tensor, n: int) -> tuple[torch.Tensor, int]:
    g = grad.detach()
    if g.numel() != n:
        raise ValueError("gradient length does not match state")
    if not g.is_cuda:
        raise ValueError("FlashOptim B200 gradients must live on a CUDA device (no CPU path)")
    if g.dtype == torch.bfloat16:
        return g.contiguous().view(-1), _lib.FO_GRAD_BF16
    return g.contiguous().view(-1).float(), _lib.FO_GRAD_F32


def step_many(optimizer: str, states: Sequence[FlashState], grads: Sequence[torch.Tensor],
              hps: Sequence | object, errors: DeviceErrors | None = None,
              stream: torch.cuda.Stream | None = None) -> None:
    """Step every (state, grad) pair in place, fused into as few kernel
    launches as the layouts allow (one per FO_MT_MAX_TENSORS tensors for the
    fast layout).  `hps` is one hyper-parameter object or one per state.
    Each state's step counter t is incremented (optim.py:211).  Errors are
    ORed into `errors` (not checked here)."""
    if optimizer not in OPTIMIZERS:
        raise ValueError(f"unknown optimizer: {optimizer}")
    if len(states) != len(grads):
        raise ValueError("states and grads differ in length")
    if not isinstance(hps, (list, tuple)):
        hps = [hps] * len(states)
    if not states:
        return
    hp_type = HP_TYPES[optimizer]
    table: dict = {}
    scalars: list = []
    batches: dict = {}
    for st, g, hp in zip(states, grads, hps):
        if not isinstance(hp, hp_type):
            raise TypeError(f"{optimizer} step needs {hp_type.__name__}, got {type(hp).__name__}")
        t = st.t + 1
        key = (hp, t)
        if key not in table:
            if len(table) == _lib.FO_MAX_HPARAMS:
                raise ValueError(f"more than {_lib.FO_MAX_HPARAMS} distinct (hyper-parameter, step) sets "
                                 "in one fused call")
            table[key] = len(scalars)
            scalars.append(hp.scalars(t))
        gv, gtype = _grad_view(g, st.length)
        vs = st.variance
        if optimizer == "adamw" and vs is None:
            raise ValueError("adamw state has no variance buffer")
        layout = (gtype, st.weights.width.bits, st.momentum.spec.group_size,
                  _lib.FO_VAR_LINEAR if st.variance_scheme == "linear" else _lib.FO_VAR_COMPANDED)
        b = batches.setdefault(layout, _Batch())
        b.keep.append(gv)
        b.tensors.append(_lib.fo_tensor(
            st.weights.lp_values.data_ptr(), st.weights.corrections.data_ptr(), st.momentum.codes.data_ptr(),
            st.momentum.scales.data_ptr(), vs.codes.data_ptr() if vs is not None and optimizer == "adamw" else None,
            vs.scales.data_ptr() if vs is not None and optimizer == "adamw" else None, gv.data_ptr(), st.length,
            table[key], 0))
    hp_arr = (_lib.fo_hparams * len(scalars))(*scalars)
    dev = states[0].device
    sh = stream.cuda_stream if stream is not None else stream_handle(dev)
    L = _lib.lib()
    for (gtype, bits, gs, vscheme), b in batches.items():
        arr = (_lib.fo_tensor * len(b.tensors))(*b.tensors)
        _lib.check(L.fo_step_mt(_lib.OPT_TAGS[optimizer], arr, len(b.tensors), hp_arr, len(scalars), gtype, bits,
                                gs, vscheme, errors.ptr if errors is not None else None, sh), "fo_step_mt")
        if stream is not None:
            for gv in b.keep:
                gv.record_stream(stream)
    for st in states:
        st.t += 1


def _step_inplace(optimizer: str, state: FlashState, grad: torch.Tensor, hp) -> FlashState:
    err = DeviceErrors(state.device)
    step_many(optimizer, [state], [grad], hp, errors=err)
    m = err.mask()
    if m:
        raise_for_mask(m, optimizer, state.variance_scheme)
    return state


def sgd_step_(state: FlashState, grad: torch.Tensor, hp: SgdHyperParams) -> FlashState:
    return _step_inplace("sgd", state, grad, hp)


def adamw_step_(state: FlashState, grad: torch.Tensor, hp: AdamHyperParams) -> FlashState:
    return _step_inplace("adamw", state, grad, hp)


def lion_step_(state: FlashState, grad: torch.Tensor, hp: LionHyperParams) -> FlashState:
    return _step_inplace("lion", state, grad, hp)


def _functional(optimizer: str, state: FlashState, grad: torch.Tensor, hp) -> FlashState:
    # reference: "_check_grad" happens before anything is produced (optim.py:176-182)
    if grad.numel() != state.length:
        raise ValueError("gradient length does not match state")
    out = state.clone()
    return _step_inplace(optimizer, out, grad, hp)


def sgd_step(state: FlashState, grad: torch.Tensor, hp: SgdHyperParams) -> FlashState:
    """m <- mu*m + g; theta <- theta - lr*(m + wd*theta) (optim.py:187-205)."""
    return _functional("sgd", state, grad, hp)


def adamw_step(state: FlashState, grad: torch.Tensor, hp: AdamHyperParams) -> FlashState:
    """AdamW with decoupled decay and exact-integer bias correction (optim.py:208-235)."""
    return _functional("adamw", state, grad, hp)


def lion_step(state: FlashState, grad: torch.Tensor, hp: LionHyperParams) -> FlashState:
    """Sign update from the interpolated momentum, then EMA (optim.py:238-258)."""
    return _functional("lion", state, grad, hp)


STEP_FUNCTIONS = {"sgd": sgd_step, "adamw": adamw_step, "lion": lion_step}
STEP_FUNCTIONS_INPLACE = {"sgd": sgd_step_, "adamw": adamw_step_, "lion": lion_step_}
