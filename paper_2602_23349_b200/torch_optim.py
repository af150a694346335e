"""torch.optim front end: FlashAdamW, FlashSGD, FlashLion.

Drop-in optimizers over the fused CUDA step.  The reference package has no
torch classes (its API is optim.py's pure functions over FlashState); this is
the torch.optim surface the build promises (BASELINE.json north_star), mapped
one to one onto the reference state:

    param.data (bf16)           <-> FlashState.weights.lp_values  "weights.lp"
    state["weights.rho"]        <-> FlashState.weights.corrections
    state["momentum.codes"]     <-> FlashState.momentum.codes
    state["momentum.scales"]    <-> FlashState.momentum.scales (fp16)
    state["variance.codes"]     <-> FlashState.variance.codes  (AdamW)
    state["variance.scales"]    <-> FlashState.variance.scales (AdamW)
    state["step"]               <-> FlashState.t

(the keys are the FLOP v1 record names, checkpoint.py:111-123).  Defaults are
the reference's (optim.py:47-94): AdamW betas (0.9, 0.999), eps 1e-8,
weight_decay 0 (note: torch.optim.AdamW defaults to 0.01); SGD momentum 0.9;
Lion betas (0.9, 0.99).  Hyper-parameters are validated with the reference's
rules and messages.

fp32 parameters are split once into bf16 + int8 correction
(init_flash_state, optim.py:143-161): `param.data` becomes the bf16 tensor,
so the model trains on bf16 weights while the optimizer keeps 24-bit master
weights.  bf16 parameters start with zero corrections.

All parameters of a param group go to the GPU in one fused launch per step
(fo_step_mt).  Errors (the reference's ValueErrors) are flagged by the
kernels in a device word; `check_errors` chooses when the host reads it:
"deferred" (default: copied asynchronously after each step and raised by
the next step() once it has arrived, never blocking), True / "sync" (read
after every step, which waits for the step) or False (only when
raise_errors() is called).  See _errors.ErrorPolicy.

capturable=True (torch.optim's meaning): optimizer.step() can be captured
into a CUDA graph and replayed.  The step counter of each param group lives
in a device int32 tensor (state["step"], shared by the group's parameters)
that step() advances with a device increment, the bias corrections come from
a device table (fo_bias_table) indexed by it, and a CUDA-tensor group "lr"
is read from device memory, so a replay computes the same bytes as an eager
step (fo_step_mt_dev).  The default layout only (int8 corrections, group
size 32); errors are read with raise_errors() (nothing is read back while a
graph is being captured).
"""

from __future__ import annotations

import ctypes
from typing import Iterable

import torch

from . import _lib
from ._errors import DeviceErrors, ErrorPolicy, raise_for_mask, stream_handle
from .formats import INT8_CORRECTION, SplitTensor, split
from .optim import AdamHyperParams, FlashState, LionHyperParams, SgdHyperParams
from .quantize import GroupSpec, QuantizedState

__all__ = ["FlashAdamW", "FlashSGD", "FlashLion", "FlashOptimizer"]

RECORDS = ("weights.rho", "momentum.codes", "momentum.scales", "variance.codes", "variance.scales")


class FlashOptimizer(torch.optim.Optimizer):
    """Shared machinery; subclasses define OPT and hp(group)."""

    OPT = ""

    def __init__(self, params, defaults: dict, *, check_errors: bool | str = "deferred", group_size: int = 32,
                 capturable: bool = False):
        if check_errors not in (True, False, None, "sync", "deferred", "off"):
            raise ValueError(f"check_errors must be True, False, 'sync', 'deferred' or 'off', got {check_errors!r}")
        if capturable and group_size != 32:
            raise ValueError("capturable=True needs group_size 32 (the fused kernel's layout)")
        self.check_errors = check_errors
        self.capturable = bool(capturable)
        self.spec = GroupSpec(group_size)
        super().__init__(params, defaults)
        self._cap: dict = {}
        for group in self.param_groups:
            self.hp(group)  # validate with the reference's rules
            for p in group["params"]:
                self._init_state(p)
        self._errors: ErrorPolicy | None = None
        self._plans: dict = {}
        if self.capturable:
            for gi in range(len(self.param_groups)):
                self._cap_group(gi)

    # -- state -----------------------------------------------------------------
    def _init_state(self, p: torch.Tensor) -> None:
        st = self.state[p]
        if "weights.rho" in st:
            return
        if not p.is_cuda:
            raise ValueError("FlashOptim B200 optimizers need CUDA parameters (no CPU path)")
        n, dev = p.numel(), p.device
        with torch.no_grad():
            if p.dtype == torch.float32:
                lp, rho = split(p.detach().reshape(-1), INT8_CORRECTION)  # init_flash_state
                p.data = lp.view(p.shape)
                st["weights.rho"] = rho.view(p.shape)
            elif p.dtype == torch.bfloat16:
                st["weights.rho"] = torch.zeros(p.shape, dtype=torch.int8, device=dev)
            else:
                raise TypeError(f"parameters must be bf16 or fp32, got {p.dtype}")
        ng = self.spec.num_groups(n)
        st["momentum.codes"] = torch.zeros(p.shape, dtype=torch.int8, device=dev)
        st["momentum.scales"] = torch.zeros(ng, dtype=torch.float16, device=dev)
        if self.OPT == "adamw":
            st["variance.codes"] = torch.zeros(p.shape, dtype=torch.uint8, device=dev)
            st["variance.scales"] = torch.zeros(ng, dtype=torch.float16, device=dev)
        st["step"] = 0

    def flash_state(self, p: torch.Tensor) -> FlashState:
        """The reference-shaped FlashState view of a parameter's state (shares memory)."""
        st = self.state[p]
        w = SplitTensor(p.data.reshape(-1), st["weights.rho"].reshape(-1))
        m = QuantizedState(st["momentum.codes"].reshape(-1), st["momentum.scales"], self.spec, "momentum")
        v = None
        if self.OPT == "adamw":
            v = QuantizedState(st["variance.codes"].reshape(-1), st["variance.scales"], self.spec, "variance")
        return FlashState(w, m, v, int(st["step"]))

    def hp(self, group: dict):
        raise NotImplementedError

    # -- capturable step ----------------------------------------------------------
    def _cap_group(self, gi: int) -> dict:
        """Device step counter, bias table and fix-up bitmap of param group gi
        (built before any capture: nothing here may run inside one)."""
        c = self._cap.get(gi)
        if c is not None:
            return c
        group = self.param_groups[gi]
        ps = list(group["params"])
        if not ps:
            return {}
        dev = ps[0].device
        steps = {int(self.state[p]["step"]) for p in ps}
        if len(steps) != 1:
            raise ValueError("capturable=True needs one step counter per param group")
        step = torch.full((), steps.pop(), dtype=torch.int32, device=dev)
        for p in ps:
            if self.state[p]["weights.rho"].dtype != torch.int8:
                raise ValueError("capturable=True takes int8 corrections only")
            self.state[p]["step"] = step
        table, n = None, 0
        if self.OPT == "adamw":
            b1, b2 = (float(x) for x in group["betas"])
            ln = ctypes.c_int32(0)
            _lib.check(_lib.lib().fo_bias_table(b1, b2, 1 << 26, None, ctypes.byref(ln)), "fo_bias_table")
            n = int(ln.value)
            host = (ctypes.c_float * (4 * n))()
            _lib.check(_lib.lib().fo_bias_table(b1, b2, n, ctypes.cast(host, ctypes.c_void_p), ctypes.byref(ln)),
                       "fo_bias_table")
            table = torch.frombuffer(bytearray(host), dtype=torch.float32).to(dev)
        tens = (_lib.fo_tensor * len(ps))()
        for i, p in enumerate(ps):
            tens[i].n = p.numel()
        words = int(_lib.lib().fo_fix_words(tens, len(ps)))
        c = dict(step=step, table=table, bc_len=n, fix=torch.zeros(words, dtype=torch.int32, device=dev),
                 count=torch.zeros(1, dtype=torch.int64, device=dev), betas=group.get("betas"), key=None,
                 tensors=None, hp=None, hp_key=None)
        self._cap[gi] = c
        return c

    def _step_capturable(self, gi: int, group: dict, ps: list) -> None:
        c = self._cap_group(gi)
        if group.get("betas") != c["betas"]:
            raise ValueError("capturable=True: betas changed after the bias table was built")
        key = (tuple(id(p) for p in ps), tuple(p.data_ptr() for p in ps))
        if c["key"] != key:
            if len(ps) != len(group["params"]):
                raise ValueError("capturable=True: every parameter of a group needs a gradient")
            adam = self.OPT == "adamw"
            tens = (_lib.fo_tensor * len(ps))()
            for i, p in enumerate(ps):
                st, e = self.state[p], tens[i]
                e.lp, e.rho = p.data.data_ptr(), st["weights.rho"].data_ptr()
                e.m_codes, e.m_scales = st["momentum.codes"].data_ptr(), st["momentum.scales"].data_ptr()
                e.v_codes = st["variance.codes"].data_ptr() if adam else None
                e.v_scales = st["variance.scales"].data_ptr() if adam else None
                e.n = p.numel()
            c["key"], c["tensors"] = key, tens
        tens = c["tensors"]
        for i, p in enumerate(ps):
            g = p.grad
            if g.dtype != torch.bfloat16 or not g.is_contiguous():
                raise ValueError("capturable=True needs contiguous bf16 gradients")
            tens[i].grad = g.data_ptr()
        lr = group["lr"]
        lr_dev = isinstance(lr, torch.Tensor)
        if lr_dev and (lr.dtype != torch.float32 or lr.device != ps[0].device or lr.numel() != 1):
            raise ValueError("a tensor lr must be a one-element float32 tensor on the parameters' device")
        hp_key = tuple((k, v) for k, v in group.items() if k not in ("params", "lr")) + \
            (("lr", None if lr_dev else lr),)
        if c["hp_key"] != hp_key:
            g2 = dict(group, lr=1.0 if lr_dev else lr)  # a device lr is never read from here
            c["hp"], c["hp_key"] = (_lib.fo_hparams * 1)(self.hp(g2).scalars(1)), hp_key
        c["step"].add_(1)  # optim.py:211, t = state.t + 1, on the device
        ds = _lib.fo_dev_scalars(c["step"].data_ptr(), lr.data_ptr() if lr_dev else None,
                                 c["table"].data_ptr() if c["table"] is not None else None, c["bc_len"], 0,
                                 c["fix"].data_ptr(), c["fix"].numel(), c["count"].data_ptr())
        _lib.check(_lib.lib().fo_step_mt_dev(
            _lib.OPT_TAGS[self.OPT], tens, len(ps), c["hp"], ctypes.byref(ds), _lib.FO_GRAD_BF16,
            self._errors.ptr, stream_handle(ps[0].device)), "fo_step_mt_dev")

    # -- step ------------------------------------------------------------------
    def _rho_bits(self, p: torch.Tensor) -> int:
        return self.state[p]["weights.rho"].element_size() * 8

    def _launch(self, params: list, grads: list, group: dict, stream=None, errors=None):
        """One fused launch for `params` (all from `group`), split by
        correction width (int8, or int16 loaded from an INT16_CORRECTION
        checkpoint, formats.py:94-95)."""
        widths = {self._rho_bits(p) for p in params}
        if len(widths) > 1:
            for w in sorted(widths):
                sel = [(p, g) for p, g in zip(params, grads) if self._rho_bits(p) == w]
                self._launch([p for p, _ in sel], [g for _, g in sel], group, stream, errors)
            return
        rho_bits = widths.pop() if widths else 8
        hp = self.hp(group)
        tensors, scalars, index, keep = [], [], {}, []
        gdt = None
        all_bf16 = all(g.dtype == torch.bfloat16 for g in grads)  # else every grad goes as f32
        for p, g in zip(params, grads):
            st = self.state[p]
            t = int(st["step"]) + 1
            if t not in index:
                index[t] = len(scalars)
                scalars.append(hp.scalars(t))
            g = (g if all_bf16 else g.float()).contiguous()
            gdt = g.dtype
            keep.append(g)  # converted grads stay alive until the launch is stream-ordered
            adam = self.OPT == "adamw"
            tensors.append(_lib.fo_tensor(
                p.data.data_ptr(), st["weights.rho"].data_ptr(), st["momentum.codes"].data_ptr(),
                st["momentum.scales"].data_ptr(), st["variance.codes"].data_ptr() if adam else None,
                st["variance.scales"].data_ptr() if adam else None, g.data_ptr(), p.numel(), index[t], 0))
        if gdt is None:
            return
        if len(scalars) > _lib.FO_MAX_HPARAMS:
            raise ValueError("too many distinct step counters in one param group")
        arr = (_lib.fo_tensor * len(tensors))(*tensors)
        hp_arr = (_lib.fo_hparams * len(scalars))(*scalars)
        dev = params[0].device
        sh = stream.cuda_stream if stream is not None else stream_handle(dev)
        errs = errors or self._errors
        _lib.check(_lib.lib().fo_step_mt(
            _lib.OPT_TAGS[self.OPT], arr, len(tensors), hp_arr, len(scalars),
            _lib.FO_GRAD_BF16 if gdt == torch.bfloat16 else _lib.FO_GRAD_F32, rho_bits, self.spec.group_size,
            _lib.FO_VAR_COMPANDED, errs.ptr if errs is not None else None, sh), "fo_step_mt")
        if stream is not None:
            for g in keep:
                g.record_stream(stream)
        for p in params:
            self.state[p]["step"] = int(self.state[p]["step"]) + 1

    def _launch_cached(self, gi: int, group: dict, ps: list) -> bool:
        """Fast path for the common case (every parameter of the group has a
        contiguous bf16 gradient and the same step counter): the fo_tensor
        table is built once per group and only gradient pointers change per
        step.  Returns False when the general path must run."""
        t0 = int(self.state[ps[0]]["step"])
        grads = []
        for p in ps:
            g = p.grad
            if g.dtype != torch.bfloat16 or not g.is_contiguous() or int(self.state[p]["step"]) != t0 \
                    or self.state[p]["weights.rho"].dtype != torch.int8:
                return False
            grads.append(g)
        key = (tuple(id(p) for p in ps), tuple(p.data_ptr() for p in ps))
        plan = self._plans.get(gi)
        if plan is None or plan[0] != key:
            adam = self.OPT == "adamw"
            table = (_lib.fo_tensor * len(ps))()
            for i, p in enumerate(ps):
                st, e = self.state[p], table[i]
                e.lp = p.data.data_ptr()
                e.rho = st["weights.rho"].data_ptr()
                e.m_codes = st["momentum.codes"].data_ptr()
                e.m_scales = st["momentum.scales"].data_ptr()
                e.v_codes = st["variance.codes"].data_ptr() if adam else None
                e.v_scales = st["variance.scales"].data_ptr() if adam else None
                e.n = p.numel()
                e.hp_index = 0
            plan = (key, table)
            self._plans[gi] = plan
        table = plan[1]
        for i, g in enumerate(grads):
            table[i].grad = g.data_ptr()
        hp = (_lib.fo_hparams * 1)(self.hp(group).scalars(t0 + 1))
        dev = ps[0].device
        _lib.check(_lib.lib().fo_step_mt(
            _lib.OPT_TAGS[self.OPT], table, len(ps), hp, 1, _lib.FO_GRAD_BF16, 8, self.spec.group_size,
            _lib.FO_VAR_COMPANDED, self._errors.ptr, stream_handle(dev)), "fo_step_mt")
        for p in ps:
            self.state[p]["step"] = t0 + 1
        return True

    @torch.no_grad()
    def step(self, closure=None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        dev = None
        for gi, group in enumerate(self.param_groups):
            ps = [p for p in group["params"] if p.grad is not None]
            if not ps:
                continue
            dev = ps[0].device
            if self._errors is None or self._errors.errors.word.device != dev:
                self._errors = ErrorPolicy(self.check_errors, dev)
            if self.capturable:
                self._step_capturable(gi, group, ps)
            elif not self._launch_cached(gi, group, ps):
                self._launch(ps, [p.grad.reshape(-1) for p in ps], group)
        if dev is not None and not (self.capturable and torch.cuda.is_current_stream_capturing()):
            self._errors.after_step(self.OPT)
        return loss

    def raise_errors(self) -> None:
        """Raise the reference's ValueError for any error the kernels flagged
        since the last check (waits for the queued steps)."""
        if self._errors is None:
            return
        self._errors.raise_now(self.OPT)

    def _check_layout(self, p: torch.Tensor, st: dict) -> None:
        """A loaded state must match the optimizer's layout: its group size
        (scales hold ceil(n/G) entries) and a correction width the kernels take
        (int8, or int16 from INT16_CORRECTION, formats.py:94-95)."""
        n = p.numel()
        rho = st.get("weights.rho")
        if rho is not None:
            if rho.dtype not in (torch.int8, torch.int16):
                raise ValueError(f"weights.rho must be int8 or int16, got {rho.dtype}")
            if rho.numel() != n:
                raise ValueError(f"weights.rho has {rho.numel()} elements, parameter has {n}")
        ng = self.spec.num_groups(n)
        for k in ("momentum.scales", "variance.scales"):
            v = st.get(k)
            if v is not None and v.numel() != ng:
                raise ValueError(f"{k} has {v.numel()} entries; group size {self.spec.group_size} needs {ng} "
                                 "(checkpoint written with another group size)")

    # -- torch.optim plumbing ----------------------------------------------------
    # torch.optim.Optimizer.load_state_dict casts floating-point state to the
    # parameter dtype (bf16), which would round the fp16 scales; they travel
    # as their int16 bit patterns instead and are restored bit for bit.
    _SCALES = ("momentum.scales", "variance.scales")

    def state_dict(self) -> dict:
        sd = super().state_dict()
        packed = {}
        for pid, st in sd["state"].items():
            st = dict(st)
            for k in self._SCALES:
                if k in st and st[k].dtype == torch.float16:
                    st[k] = st[k].view(torch.int16)
            packed[pid] = st
        sd["state"] = packed
        return sd

    def load_state_dict(self, state_dict: dict) -> None:
        # torch.optim casts every state tensor of a floating-point parameter to
        # the parameter dtype; load the groups through torch and the state
        # tensors directly, in their own dtypes.
        saved = state_dict["state"]
        self._plans = {}
        super().load_state_dict({**state_dict, "state": {}})
        id_map = {}
        for g_saved, g in zip(state_dict["param_groups"], self.param_groups):
            for pid, p in zip(g_saved["params"], g["params"]):
                id_map[pid] = p
        for pid, st in saved.items():
            p = id_map[pid]
            self._check_layout(p, st)
            if p.dtype == torch.float32:  # a fresh model: the checkpoint holds bf16 weights.lp
                p.data = p.data.to(torch.bfloat16)
            new = {}
            for k, v in st.items():
                if isinstance(v, torch.Tensor):
                    v = v.to(p.device, copy=True)  # deep copy, like torch.optim
                    if k in self._SCALES and v.dtype == torch.int16:
                        v = v.view(torch.float16)
                new[k] = int(v) if k == "step" else v
            self.state[p] = new
        for g in self.param_groups:
            for p in g["params"]:
                self._init_state(p)
        self._reset_capturable()

    def _reset_capturable(self) -> None:
        """After the state tensors were replaced (load_state_dict,
        checkpoint.load_optimizer): one device step counter per group again,
        from the loaded values, and fresh launch tables."""
        if self.capturable:
            self._cap = {}
            for gi in range(len(self.param_groups)):
                self._cap_group(gi)


class FlashAdamW(FlashOptimizer):
    """FlashAdamW (optim.py:208-235): decoupled weight decay, exact-integer bias correction."""

    OPT = "adamw"

    def __init__(self, params: Iterable, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, **kw):
        super().__init__(params, dict(lr=lr, betas=tuple(betas), eps=eps, weight_decay=weight_decay), **kw)

    def hp(self, g: dict) -> AdamHyperParams:
        return AdamHyperParams(lr=float(g["lr"]), beta1=float(g["betas"][0]), beta2=float(g["betas"][1]),
                               eps=float(g["eps"]), weight_decay=float(g["weight_decay"]))


class FlashSGD(FlashOptimizer):
    """FlashSGD (optim.py:187-205): m <- mu*m + g; theta <- theta - lr*(m + wd*theta)."""

    OPT = "sgd"

    def __init__(self, params: Iterable, lr: float = 1e-2, momentum: float = 0.9, weight_decay: float = 0.0, **kw):
        super().__init__(params, dict(lr=lr, momentum=momentum, weight_decay=weight_decay), **kw)

    def hp(self, g: dict) -> SgdHyperParams:
        return SgdHyperParams(lr=float(g["lr"]), momentum=float(g["momentum"]), weight_decay=float(g["weight_decay"]))


class FlashLion(FlashOptimizer):
    """FlashLion (optim.py:238-258)."""

    OPT = "lion"

    def __init__(self, params: Iterable, lr: float = 1e-4, betas=(0.9, 0.99), weight_decay: float = 0.0, **kw):
        super().__init__(params, dict(lr=lr, betas=tuple(betas), weight_decay=weight_decay), **kw)

    def hp(self, g: dict) -> LionHyperParams:
        return LionHyperParams(lr=float(g["lr"]), beta1=float(g["betas"][0]), beta2=float(g["betas"][1]),
                               weight_decay=float(g["weight_decay"]))


# ctypes is re-exported for callers that build their own launch tables
_ = ctypes
