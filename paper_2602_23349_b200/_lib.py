"""ctypes binding of libflashoptim_b200.so (include/flashoptim_b200.h).

The shared library is built in-tree (paper_2602_23349_b200/csrc/Makefile,
driven by __graft_entry__.build()).  There is no fallback: if the library
is missing every entry point raises, so a GPU run can never silently take a
CPU or eager-PyTorch path.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FO_LIB_PATH") or os.path.join(_HERE, "libflashoptim_b200.so")
CSRC = os.path.join(_HERE, "csrc")

FO_OK = 0
FO_OPT_SGD, FO_OPT_ADAMW, FO_OPT_LION = 0, 1, 2
FO_GRAD_BF16, FO_GRAD_F32 = 0, 1
FO_VAR_COMPANDED, FO_VAR_LINEAR = 0, 1
FO_MAX_HPARAMS = 16
FO_MAX_PEERS = 7
OPT_TAGS = {"sgd": FO_OPT_SGD, "adamw": FO_OPT_ADAMW, "lion": FO_OPT_LION}

ERR_GRAD_NONFINITE = 0x01
ERR_RHO_INVALID = 0x02
ERR_SPLIT_NONFINITE = 0x04
ERR_M_NONFINITE = 0x08
ERR_M_OVERFLOW = 0x10
ERR_V_NONFINITE = 0x20
ERR_V_NEGATIVE = 0x40
ERR_V_OVERFLOW = 0x80


class fo_hparams(ctypes.Structure):
    _fields_ = [(k, ctypes.c_float) for k in
                ("lr", "wd", "eps", "b1", "omb1", "b2", "omb2", "mu", "bc1", "bc2", "rbc1", "rbc2")]


class fo_dev_scalars(ctypes.Structure):
    """include/flashoptim_b200.h: device-resident step counter, lr and bias table."""
    _fields_ = [("step", ctypes.c_void_p), ("lr", ctypes.c_void_p), ("bc_table", ctypes.c_void_p),
                ("bc_len", ctypes.c_int32), ("reserved", ctypes.c_int32), ("fix_bits", ctypes.c_void_p),
                ("fix_words", ctypes.c_int64), ("fix_count", ctypes.c_void_p)]


class fo_tensor(ctypes.Structure):
    _fields_ = [
        ("lp", ctypes.c_void_p),
        ("rho", ctypes.c_void_p),
        ("m_codes", ctypes.c_void_p),
        ("m_scales", ctypes.c_void_p),
        ("v_codes", ctypes.c_void_p),
        ("v_scales", ctypes.c_void_p),
        ("grad", ctypes.c_void_p),
        ("n", ctypes.c_int64),
        ("hp_index", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


# name -> (restype, argtypes); mirrors include/flashoptim_b200.h exactly.
_P, _I64, _I32, _U32, _D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double
SIGNATURES = {
    "fo_abi_version": (_U32, []),
    "fo_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "fo_error_message": (ctypes.c_char_p, [_U32, ctypes.c_int]),
    "fo_make_hparams": (None, [ctypes.c_int, _D, _D, _D, _D, _D, _D, _I64, ctypes.POINTER(fo_hparams)]),
    "fo_step_mt": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(fo_tensor), _I32, ctypes.POINTER(fo_hparams), _I32,
                                  ctypes.c_int, ctypes.c_int, _I32, ctypes.c_int, _P, _P]),
    "fo_adamw_step": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, ctypes.c_int, _I64, ctypes.POINTER(fo_hparams),
                                     _P, _P]),
    "fo_sgd_step": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.c_int, _I64, ctypes.POINTER(fo_hparams), _P, _P]),
    "fo_lion_step": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.c_int, _I64, ctypes.POINTER(fo_hparams), _P, _P]),
    "fo_split": (ctypes.c_int, [_P, _I64, _P, _P, ctypes.c_int, _P, _P]),
    "fo_reconstruct": (ctypes.c_int, [_P, _P, ctypes.c_int, _I64, _P, _P, _P]),
    "fo_quantize_momentum": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _P, _P]),
    "fo_dequantize_momentum": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P]),
    "fo_quantize_variance": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _P, _P]),
    "fo_dequantize_variance": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P]),
    "fo_selftest": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, _P, _P]),
    "fo_sweep": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_uint32, _P, _P]),
    "fo_step_host": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(fo_tensor), _I32, ctypes.POINTER(fo_hparams), _I32,
                                    ctypes.c_int, ctypes.c_int, _I32, ctypes.c_int, _I64, ctypes.POINTER(_U32)]),
    "fo_host_release": (None, []),
    "fo_fixup_stats": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.c_int]),
    "fo_reserve": (ctypes.c_int, [_P, _I64]),
    "fo_fused_tile_elems": (_I64, []),
    "fo_fix_words": (_I64, [ctypes.POINTER(fo_tensor), _I32]),
    "fo_step_mt_dev": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(fo_tensor), _I32, ctypes.POINTER(fo_hparams),
                                      ctypes.POINTER(fo_dev_scalars), ctypes.c_int, _P, _P]),
    "fo_bias_table": (ctypes.c_int, [_D, _D, _I32, _P, ctypes.POINTER(_I32)]),
    "fo_step_mt_peers": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(fo_tensor), _I32, ctypes.POINTER(fo_hparams),
                                        ctypes.c_int, ctypes.POINTER(_I64), _I32, _P, _P]),
    "fo_ipc_export": (ctypes.c_int, [_P, _P, ctypes.POINTER(_I64)]),
    "fo_ipc_open": (ctypes.c_int, [_P, _I64, ctypes.POINTER(ctypes.c_void_p)]),
    "fo_ipc_close": (ctypes.c_int, [_P, _I64]),
}

_lib = None


def build(verbose: bool = False) -> str:
    """Compile the CUDA library in-tree with nvcc (sm_100a)."""
    out = subprocess.run(["make", "-s", "-C", CSRC, "-j4"], capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"libflashoptim_b200 build failed:\n{out.stdout}\n{out.stderr}")
    return LIB_PATH


def lib() -> ctypes.CDLL:
    """Load the library (no fallback: raises if it is absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the FlashOptim step has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.fo_abi_version() != 2:
            raise RuntimeError("libflashoptim_b200 ABI version mismatch")
        _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status != FO_OK:
        msg = lib().fo_status_string(status).decode()
        raise RuntimeError(f"{what} failed: {msg} (status {status})")


def make_hparams(optimizer: str, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 weight_decay: float = 0.0, momentum: float = 0.9, t: int = 1) -> fo_hparams:
    hp = fo_hparams()
    lib().fo_make_hparams(OPT_TAGS[optimizer], lr, beta1, beta2, eps, weight_decay, momentum, int(t),
                          ctypes.byref(hp))
    return hp


def fixup_stats(stream: int | None = None, reset: bool = False) -> tuple[int, int]:
    """(slices re-run by fix-up launches, slices covered by fused launches)
    on `stream` (a cudaStream_t handle; default: torch's current stream)."""
    if stream is None:
        import torch

        stream = torch.cuda.current_stream().cuda_stream
    f, n = ctypes.c_uint64(0), ctypes.c_uint64(0)
    check(lib().fo_fixup_stats(stream, ctypes.byref(f), ctypes.byref(n), int(reset)), "fo_fixup_stats")
    return int(f.value), int(n.value)


def error_message(mask: int, optimizer: str) -> str:
    return lib().fo_error_message(mask, OPT_TAGS[optimizer]).decode()
