"""The reference-side binding: `flashopt.optim.*_step` on the B200.

This is the module a `flashopt` maintainer adds to the reference package
 -- shipped here as working code and exercised by
tests/test_gpu_refbinding.py against the reference's own NumPy output.  It
depends only on ctypes, NumPy and libflashoptim_b200.so (no torch): the
reference's FlashState objects (optim.py:114-130) keep their NumPy arrays
in host memory and `fo_step_host` streams them through the GPU.

    from paper_2602_23349_b200 import flashopt_binding
    flashopt_binding.install(flashopt)        # flashopt = the reference package
    new_state = flashopt.optim.adamw_step(state, grad, hp)   # now on the B200

`install` replaces `adamw_step` / `sgd_step` / `lion_step` (optim.py:187,
:208, :238) and the `STEP_FUNCTIONS` table (optim.py:261) with wrappers
that keep the reference contract: the input state is never mutated (a copy
is stepped and returned), hyper-parameters are the reference's own objects,
errors are the reference's ValueError messages, raised before any output is
returned.  States the library does not take (ReferenceState, non-BF16
formats) go to the original NumPy function.
"""

from __future__ import annotations

import copy
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FO_LIB_PATH") or os.path.join(_HERE, "libflashoptim_b200.so")

_TAG = {"sgd": 0, "adamw": 1, "lion": 2}
_GRAD_F32 = 1


class _HP(ctypes.Structure):
    _fields_ = [(k, ctypes.c_float) for k in
                ("lr", "wd", "eps", "b1", "omb1", "b2", "omb2", "mu", "bc1", "bc2", "rbc1", "rbc2")]


class _T(ctypes.Structure):
    _fields_ = [("lp", ctypes.c_void_p), ("rho", ctypes.c_void_p), ("m_codes", ctypes.c_void_p),
                ("m_scales", ctypes.c_void_p), ("v_codes", ctypes.c_void_p), ("v_scales", ctypes.c_void_p),
                ("grad", ctypes.c_void_p), ("n", ctypes.c_int64), ("hp_index", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


_L = None


def _lib():
    global _L
    if _L is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        L.fo_make_hparams.argtypes = [ctypes.c_int] + [ctypes.c_double] * 6 + [ctypes.c_int64, ctypes.POINTER(_HP)]
        L.fo_make_hparams.restype = None
        L.fo_step_host.argtypes = [ctypes.c_int, ctypes.POINTER(_T), ctypes.c_int32, ctypes.POINTER(_HP),
                                   ctypes.c_int32, ctypes.c_int, ctypes.c_int, ctypes.c_int32, ctypes.c_int,
                                   ctypes.c_int64, ctypes.POINTER(ctypes.c_uint32)]
        L.fo_step_host.restype = ctypes.c_int
        L.fo_error_message.argtypes = [ctypes.c_uint32, ctypes.c_int]
        L.fo_error_message.restype = ctypes.c_char_p
        L.fo_status_string.argtypes = [ctypes.c_int]
        L.fo_status_string.restype = ctypes.c_char_p
        _L = L
    return _L


def _ptr(a):
    if a is None:
        return None
    if not a.flags.c_contiguous:
        raise ValueError("state arrays must be C-contiguous")
    return a.ctypes.data


def supported(state) -> bool:
    """FlashState with BF16 weights (the library's format); anything else
    (ReferenceState, other low-precision formats) stays on NumPy."""
    w = getattr(state, "weights", None)
    if w is None or not hasattr(state, "momentum"):
        return False
    fmt = getattr(w, "fmt", None)
    return getattr(fmt, "name", "bf16").lower() in ("bf16", "bfloat16") and w.lp_values.dtype == np.uint16


def step_inplace(optimizer: str, state, grad, hp):
    """Step a reference FlashState's arrays in place on the GPU (t += 1).
    Raises the reference's ValueError (the arrays are then already written:
    use `step` for the pure contract)."""
    g = np.ascontiguousarray(np.asarray(grad, dtype=np.float32).ravel())  # optim.py:179
    if g.size != state.length:
        raise ValueError("gradient length does not match state")         # optim.py:180-181
    h = _HP()
    _lib().fo_make_hparams(_TAG[optimizer], float(hp.lr), float(getattr(hp, "beta1", 0.0)),
                           float(getattr(hp, "beta2", 0.0)), float(getattr(hp, "eps", 1.0)),
                           float(hp.weight_decay), float(getattr(hp, "momentum", 0.0)), state.t + 1,
                           ctypes.byref(h))
    v = state.variance if optimizer == "adamw" else None
    w, m = state.weights, state.momentum
    t = _T(_ptr(w.lp_values), _ptr(w.corrections), _ptr(m.codes), _ptr(m.scales), _ptr(v.codes) if v else None,
           _ptr(v.scales) if v else None, _ptr(g), g.size, 0, 0)
    err = ctypes.c_uint32(0)
    scheme = 1 if getattr(state, "variance_scheme", "companded") == "linear" else 0
    rc = _lib().fo_step_host(_TAG[optimizer], ctypes.byref(t), 1, ctypes.byref(h), 1, _GRAD_F32,
                             int(w.corrections.dtype.itemsize * 8), int(m.spec.group_size), scheme, 0,
                             ctypes.byref(err))
    if rc:
        raise RuntimeError(f"libflashoptim_b200: {_lib().fo_status_string(rc).decode()} (status {rc})")
    if err.value:
        msg = _lib().fo_error_message(err.value, _TAG[optimizer]).decode()
        if scheme == 1 and msg.startswith("negative-variance"):
            msg = "negative-unsigned: unsigned buffer has negative entries"  # quantize.py:166
        raise ValueError(msg)
    state.t += 1
    return state


def step(optimizer: str, state, grad, hp):
    """The reference's pure contract (optim.py:7-9): a new FlashState is
    returned, `state` is untouched, errors raise before anything is returned."""
    out = copy.deepcopy(state)
    return step_inplace(optimizer, out, grad, hp)


def install(flashopt_pkg) -> dict:
    """Route flashopt.optim's step functions through the B200 library.
    Returns the original functions (pass them to `uninstall`)."""
    O = flashopt_pkg.optim
    orig = {"sgd": O.sgd_step, "adamw": O.adamw_step, "lion": O.lion_step}
    hp_types = {"sgd": O.SgdHyperParams, "adamw": O.AdamHyperParams, "lion": O.LionHyperParams}

    def make(name):
        fallback = orig[name]

        def stepper(state, grad, hp):
            if not isinstance(state, O.FlashState) or not supported(state) or not isinstance(hp, hp_types[name]):
                return fallback(state, grad, hp)
            return step(name, state, grad, hp)

        stepper.__name__ = f"{name}_step"
        stepper.__doc__ = f"{fallback.__doc__}\n\n(B200: libflashoptim_b200 fo_step_host)"
        stepper.__wrapped__ = fallback
        return stepper

    new = {k: make(k) for k in orig}
    O.sgd_step, O.adamw_step, O.lion_step = new["sgd"], new["adamw"], new["lion"]
    O.STEP_FUNCTIONS.update(new)  # training.py imports the dict object itself
    return orig


def uninstall(flashopt_pkg, orig: dict) -> None:
    O = flashopt_pkg.optim
    O.sgd_step, O.adamw_step, O.lion_step = orig["sgd"], orig["adamw"], orig["lion"]
    O.STEP_FUNCTIONS.update(orig)
