"""ctypes wrapper around the C parity oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product
package.  Mirrors the reference's functional API
(/root/reference/pkg/src/flashopt/optim.py:187-261, formats.py:232-276,
quantize.py:109-158) on plain NumPy arrays: inputs are copied, the copy is
stepped in place by the C restatement, and errors are raised as ValueError
with the reference's message prefixes.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

ERR_GRAD_NONFINITE = 0x01
ERR_RHO_INVALID = 0x02
ERR_SPLIT_NONFINITE = 0x04
ERR_M_NONFINITE = 0x08
ERR_M_OVERFLOW = 0x10
ERR_V_NONFINITE = 0x20
ERR_V_NEGATIVE = 0x40
ERR_V_OVERFLOW = 0x80

OPT_TAGS = {"sgd": 0, "adamw": 1, "lion": 2}

# Reference messages (optim.py:183, formats.py:243,271, quantize.py:69,85,144).
MESSAGES = {
    ERR_GRAD_NONFINITE: "gradient-nonfinite: gradient contains NaN/Inf",
    ERR_RHO_INVALID: "invalid-correction-code: asymmetric minimum is forbidden",
    ERR_SPLIT_NONFINITE: "split-nonfinite: cannot split NaN/Inf master weights",
    ERR_M_NONFINITE: "quantize-nonfinite: state buffer contains NaN/Inf",
    ERR_M_OVERFLOW: "scale-overflow: group absmax exceeds FP16 range",
    ERR_V_NONFINITE: "quantize-nonfinite: state buffer contains NaN/Inf",
    ERR_V_NEGATIVE: "negative-variance: variance entries must be >= 0",
    ERR_V_OVERFLOW: "scale-overflow: group absmax exceeds FP16 range",
}

# Order in which the reference would raise (program order of each step).
PRECEDENCE = {
    "adamw": [ERR_GRAD_NONFINITE, ERR_RHO_INVALID, ERR_SPLIT_NONFINITE, ERR_M_NONFINITE,
              ERR_M_OVERFLOW, ERR_V_NONFINITE, ERR_V_NEGATIVE, ERR_V_OVERFLOW],
    "sgd": [ERR_GRAD_NONFINITE, ERR_M_NONFINITE, ERR_M_OVERFLOW, ERR_RHO_INVALID, ERR_SPLIT_NONFINITE],
    "lion": [ERR_GRAD_NONFINITE, ERR_RHO_INVALID, ERR_SPLIT_NONFINITE, ERR_M_NONFINITE, ERR_M_OVERFLOW],
}


def build() -> str:
    """Compile liboracle.so from oracle/flashopt_oracle.c (make)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class _Scalars(ctypes.Structure):
    _fields_ = [(k, ctypes.c_float) for k in
                ("lr", "wd", "eps", "b1", "omb1", "b2", "omb2", "mu", "bc1", "bc2")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, I32, U32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32
        L.fo_oracle_split.argtypes = [P, I64, I32, P, P]
        L.fo_oracle_split.restype = U32
        L.fo_oracle_reconstruct.argtypes = [P, P, I64, I32, P]
        L.fo_oracle_reconstruct.restype = U32
        L.fo_oracle_quantize_momentum.argtypes = [P, I64, I64, P, P]
        L.fo_oracle_quantize_momentum.restype = U32
        L.fo_oracle_dequantize_momentum.argtypes = [P, P, I64, I64, P]
        L.fo_oracle_dequantize_momentum.restype = None
        L.fo_oracle_quantize_variance.argtypes = [P, I64, I64, P, P]
        L.fo_oracle_quantize_variance.restype = U32
        L.fo_oracle_dequantize_variance.argtypes = [P, P, I64, I64, P]
        L.fo_oracle_dequantize_variance.restype = None
        L.fo_oracle_quantize_linear.argtypes = [P, I64, I64, I32, P, P]
        L.fo_oracle_quantize_linear.restype = U32
        L.fo_oracle_dequantize_linear.argtypes = [P, P, I64, I64, I32, P]
        L.fo_oracle_dequantize_linear.restype = None
        L.fo_oracle_make_scalars.argtypes = [I32, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_double, I64,
                                             ctypes.POINTER(_Scalars)]
        L.fo_oracle_make_scalars.restype = None
        L.fo_oracle_step.argtypes = [I32, P, P, I32, P, P, P, P, I32, P, I64, I64,
                                     ctypes.POINTER(_Scalars), I32]
        L.fo_oracle_step.restype = U32
        L.fo_oracle_max_threads.argtypes = []
        L.fo_oracle_max_threads.restype = I32
        L.fo_oracle_downcast_bf16.argtypes = [ctypes.c_float]
        L.fo_oracle_downcast_bf16.restype = ctypes.c_uint16
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


def raise_for(mask: int, optimizer: str) -> None:
    for bit in PRECEDENCE[optimizer]:
        if mask & bit:
            raise ValueError(MESSAGES[bit])


# --- codecs ---------------------------------------------------------------

def split(theta, width_bits: int = 8):
    theta = np.ascontiguousarray(theta, dtype=np.float32).ravel()
    lp = np.empty(theta.size, np.uint16)
    rho = np.empty(theta.size, np.int8 if width_bits == 8 else np.int16)
    err = lib().fo_oracle_split(_p(theta), theta.size, width_bits, _p(lp), _p(rho))
    if err:
        raise ValueError(MESSAGES[ERR_SPLIT_NONFINITE])
    return lp, rho


def reconstruct(lp, rho, width_bits: int = 8):
    lp = np.ascontiguousarray(lp, dtype=np.uint16).ravel()
    rho = np.ascontiguousarray(rho, dtype=np.int8 if width_bits == 8 else np.int16).ravel()
    out = np.empty(lp.size, np.float32)
    err = lib().fo_oracle_reconstruct(_p(lp), _p(rho), lp.size, width_bits, _p(out))
    if err:
        raise ValueError(MESSAGES[ERR_RHO_INVALID])
    return out


def _ngroups(n, G):
    return -(-n // G) if n else 0


def quantize_momentum(m, G: int = 32):
    m = np.ascontiguousarray(m, dtype=np.float32).ravel()
    codes = np.empty(m.size, np.int8)
    scales = np.empty(_ngroups(m.size, G), np.uint16)
    err = lib().fo_oracle_quantize_momentum(_p(m), m.size, G, _p(codes), _p(scales))
    if err:
        raise_for(err, "sgd")
    return codes, scales.view(np.float16)


def dequantize_momentum(codes, scales, G: int = 32):
    codes = np.ascontiguousarray(codes, dtype=np.int8).ravel()
    scales = np.ascontiguousarray(scales, dtype=np.float16).ravel().view(np.uint16)
    out = np.empty(codes.size, np.float32)
    lib().fo_oracle_dequantize_momentum(_p(codes), _p(scales), codes.size, G, _p(out))
    return out


def quantize_variance(v, G: int = 32):
    v = np.ascontiguousarray(v, dtype=np.float32).ravel()
    codes = np.empty(v.size, np.uint8)
    scales = np.empty(_ngroups(v.size, G), np.uint16)
    err = lib().fo_oracle_quantize_variance(_p(v), v.size, G, _p(codes), _p(scales))
    if err:
        raise_for(err, "adamw")
    return codes, scales.view(np.float16)


def dequantize_variance(codes, scales, G: int = 32):
    codes = np.ascontiguousarray(codes, dtype=np.uint8).ravel()
    scales = np.ascontiguousarray(scales, dtype=np.float16).ravel().view(np.uint16)
    out = np.empty(codes.size, np.float32)
    lib().fo_oracle_dequantize_variance(_p(codes), _p(scales), codes.size, G, _p(out))
    return out


# --- steps ------------------------------------------------------------------

@dataclass
class OracleState:
    """Plain-array flash state; field names follow the FLOP v1 records
    (checkpoint.py:111-123)."""

    lp: np.ndarray            # uint16 bf16 codes  ("weights.lp")
    rho: np.ndarray           # int8/int16         ("weights.rho")
    m_codes: np.ndarray       # int8               ("momentum.codes")
    m_scales: np.ndarray      # float16            ("momentum.scales")
    v_codes: np.ndarray | None = None   # uint8    ("variance.codes")
    v_scales: np.ndarray | None = None  # float16  ("variance.scales")
    t: int = 0
    group_size: int = 32
    variance_scheme: str = "companded"

    def copy(self) -> "OracleState":
        c = lambda a: None if a is None else a.copy()  # noqa: E731
        return OracleState(self.lp.copy(), self.rho.copy(), self.m_codes.copy(), self.m_scales.copy(),
                           c(self.v_codes), c(self.v_scales), self.t, self.group_size, self.variance_scheme)

    @property
    def width_bits(self) -> int:
        return 8 if self.rho.dtype == np.int8 else 16


def init_state(theta0, optimizer: str, G: int = 32) -> OracleState:
    """optim.py:143-161 init_flash_state."""
    lp, rho = split(theta0)
    n = lp.size
    ng = _ngroups(n, G)
    v_codes = np.zeros(n, np.uint8) if optimizer == "adamw" else None
    v_scales = np.zeros(ng, np.float16) if optimizer == "adamw" else None
    return OracleState(lp, rho, np.zeros(n, np.int8), np.zeros(ng, np.float16), v_codes, v_scales, 0, G)


def scalars(optimizer: str, t: int, lr: float, beta1: float = 0.9, beta2: float = 0.999,
            eps: float = 1e-8, weight_decay: float = 0.0, momentum: float = 0.9) -> _Scalars:
    s = _Scalars()
    lib().fo_oracle_make_scalars(OPT_TAGS[optimizer], lr, beta1, beta2, eps, weight_decay, momentum, t,
                                 ctypes.byref(s))
    return s


def step_inplace(optimizer: str, st: OracleState, grad: np.ndarray, nthreads: int = 1, **hp) -> int:
    """Step `st` in place; returns the error bitmask (no raise)."""
    grad = np.ascontiguousarray(grad, dtype=np.float32).ravel()
    if grad.size != st.lp.size:
        raise ValueError("gradient length does not match state")
    t = st.t + 1
    s = scalars(optimizer, t, **hp)
    vq = st.v_codes if optimizer == "adamw" else None
    vs = st.v_scales if optimizer == "adamw" else None
    err = lib().fo_oracle_step(
        OPT_TAGS[optimizer], _p(st.lp), _p(st.rho), st.width_bits, _p(st.m_codes),
        _p(st.m_scales.view(np.uint16)), None if vq is None else _p(vq),
        None if vs is None else _p(vs.view(np.uint16)), 0 if st.variance_scheme == "companded" else 1,
        _p(grad), st.lp.size, st.group_size, ctypes.byref(s), nthreads)
    st.t = t
    return int(err)


def step(optimizer: str, st: OracleState, grad: np.ndarray, nthreads: int = 1, **hp) -> OracleState:
    """Functional step with the reference's raise-before-return semantics."""
    out = st.copy()
    err = step_inplace(optimizer, out, grad, nthreads=nthreads, **hp)
    if err:
        raise_for(err, optimizer)
    return out


def max_threads() -> int:
    return int(lib().fo_oracle_max_threads())
