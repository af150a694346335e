"""Seeded synthetic FlashState / gradient generators shared by the tests,
the golden-vector script and bench.py's CPU legs.

A "random valid state" is what SURVEY.md §7.1 asks for: bf16 weight codes
with in-range corrections rho in [-127, 127], momentum codes in [-127, 127],
variance codes in [0, 255] and finite non-negative fp16 group scales, plus
bf16-representable gradients (the reference upcasts grads to f32,
optim.py:178-184).
"""

from __future__ import annotations

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round f32 to the nearest bf16 value (RNE), returned as f32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lower = u & np.uint32(0xFFFF)
    code = u >> np.uint32(16)
    code = code + ((lower > 0x8000) | ((lower == 0x8000) & ((code & 1) == 1)))
    return (code.astype(np.uint32) << np.uint32(16)).view(np.float32)


def bf16_codes(x: np.ndarray) -> np.ndarray:
    return (bf16_round(x).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def random_weights(rng: np.random.Generator, n: int, std: float = 0.02, wide_frac: float = 0.05) -> np.ndarray:
    """N(0, std^2) weights with a fraction spread over many binades (incl.
    subnormal-range magnitudes, exact zeros and binade bottoms)."""
    x = (rng.standard_normal(n) * std).astype(np.float32)
    k = int(n * wide_frac)
    if k:
        idx = rng.choice(n, size=k, replace=False)
        mag = 10.0 ** rng.uniform(-40, 3, size=k)
        x[idx] = (rng.standard_normal(k) * mag).astype(np.float32)
        z = idx[: max(1, k // 10)]
        x[z] = 0.0
        b = idx[k // 10: k // 5]
        x[b] = np.ldexp(np.sign(rng.standard_normal(b.size)), rng.integers(-130, 10, b.size)).astype(np.float32)
    return x


def random_fp16_scales(rng: np.random.Generator, ng: int, center: float, zero_frac: float = 0.02) -> np.ndarray:
    s = (np.abs(rng.standard_normal(ng)) * center * 10.0 ** rng.uniform(-2, 1, ng)).astype(np.float16)
    s[rng.random(ng) < zero_frac] = 0
    return s


def random_state(rng: np.random.Generator, n: int, optimizer: str, G: int = 32, lp=None, rho=None) -> dict:
    """Random valid FlashState arrays (FLOP v1 record names)."""
    ng = -(-n // G) if n else 0
    if lp is None:
        lp = bf16_codes(random_weights(rng, n))
    if rho is None:
        rho = rng.integers(-127, 128, n).astype(np.int8)
        rho[rng.random(n) < 0.05] = 0
    st = {
        "weights.lp": lp.astype(np.uint16),
        "weights.rho": rho,
        "momentum.codes": rng.integers(-127, 128, n).astype(np.int8),
        "momentum.scales": random_fp16_scales(rng, ng, 1e-3),
    }
    if optimizer == "adamw":
        st["variance.codes"] = rng.integers(0, 256, n).astype(np.uint8)
        st["variance.scales"] = random_fp16_scales(rng, ng, 1e-3)
    # all-zero groups: codes 0 with scale 0 (what init/zero grads produce)
    for key in ("momentum", "variance"):
        if f"{key}.scales" in st:
            zs = np.nonzero(st[f"{key}.scales"] == 0)[0]
            for g in zs:
                st[f"{key}.codes"][g * G:(g + 1) * G] = 0
    return st


def random_grad(rng: np.random.Generator, n: int, std: float = 1e-3, zero_frac: float = 0.01) -> np.ndarray:
    g = bf16_round((rng.standard_normal(n) * std).astype(np.float32))
    g[rng.random(n) < zero_frac] = 0.0
    return g


def random_hparams(rng: np.random.Generator, optimizer: str) -> dict:
    lr = float(10.0 ** rng.uniform(-5, -1))
    wd = float(rng.choice([0.0, 0.01, 0.1]))
    if optimizer == "adamw":
        return dict(lr=lr, beta1=0.9, beta2=float(rng.choice([0.95, 0.99, 0.999])), eps=1e-8, weight_decay=wd)
    if optimizer == "sgd":
        return dict(lr=lr, momentum=float(rng.choice([0.0, 0.9, 0.99])), weight_decay=wd)
    return dict(lr=lr, beta1=0.9, beta2=float(rng.choice([0.95, 0.99])), weight_decay=wd)
