"""Device self-checks of the fast exact primitives (csrc/fo_fast.cuh) against
the IEEE intrinsics they replace, through fo_selftest() in the C ABI.

These back the exactness arguments in DESIGN.md §4: every shortcut the fused
kernel takes (sqrt / reciprocal / Markstein quotients without range checks)
must agree bit for bit with sqrt.rn / rcp.rn / div.rn on its whole domain
(exhaustive) or on a large hash sample (for two-argument functions)."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu

U64_MAX = (1 << 64) - 1


def _run(mode: int, begin: int, count: int) -> tuple[int, int]:
    from paper_2602_23349_b200 import _lib

    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    out[1] = -1  # UINT64_MAX as the running min of failing indices
    _lib.check(_lib.lib().fo_selftest(mode, begin, count, out.data_ptr(), None), "fo_selftest")
    torch.cuda.synchronize()
    return int(out[0]), int(out[1]) & U64_MAX


def test_sqrt_exhaustive(cuda_dev):
    """sqrt_rn2 == sqrt.rn for +0 and every f32 in [2^-94, FLT_MAX]."""
    bad, first = _run(0, 0, 1 << 31)
    assert bad == 0, f"{bad} mismatches, first at bits {first:#x}"


def test_wide_sqrt_exhaustive(cuda_dev):
    """sqrt_rn2_wide == sqrt.rn for every f32 in [0, 2^64), subnormals included
    (the steady-state AdamW tile's variance root, no operand guard)."""
    bad, first = _run(7, 0, 0x5F800000)
    assert bad == 0, f"{bad} mismatches, first at bits {first:#x}"


def test_reciprocal_of_every_fp16_scale(cuda_dev):
    bad, first = _run(1, 0, 0x7C00)
    assert bad == 0, f"first failing fp16 bits {first:#x}"


def test_per_element_division_sampled(cuda_dev):
    """div_rn2 (per-element divisor) on 2^32 hash samples of its domain."""
    bad, first = _run(2, 0, 1 << 32)
    assert bad == 0, f"{bad} mismatches, first sample {first}"


def test_group_scale_division_sampled(cuda_dev):
    """m/s and r/s with s = every fp16 scale, 2^31 samples."""
    bad, first = _run(3, 0, 1 << 31)
    assert bad == 0, f"{bad} mismatches, first sample {first}"


def test_bias_correction_division_sampled(cuda_dev):
    """m/bc1, v/bc2 with host-side RN(1/bc), 2^30 samples of beta, t, a."""
    bad, first = _run(4, 0, 1 << 30)
    assert bad == 0, f"{bad} mismatches, first sample {first}"


def test_integer_reconstruct_exhaustive(cuda_dev):
    """The fused tile's integer reconstruct (fast::recon_bits + R(rho) LUT)
    against the IEEE restatement for every finite bf16 code x every rho;
    the two zero cases it gets wrong come out NaN or -0 (guard-tripping)."""
    bad, first = _run(6, 0, 1 << 24)
    assert bad == 0, f"{bad} mismatches, first at code {first >> 8:#06x} rho byte {first & 0xFF:#04x}"


def test_rcp_approx_error_bound(cuda_dev):
    """MUFU reciprocal: relative error < 2^-22 for every f32 in [1, 4) (the
    bound the approximate momentum coder's error budget uses; 1 + |m'|
    reaches just above 2)."""
    bad, first = _run(8, 0, 1 << 24)
    assert bad == 0, f"{bad} inputs over the bound, first mantissa {first:#x}"


def test_momentum_preimage_bound_sampled(cuda_dev):
    """mq_T (FO_MQ_APPROX) within 2^-12 of the reference's pre-rint momentum
    value, and its rint equal to the reference code away from half-integers:
    2^32 samples over every fp16 scale (quantize.py:109-122)."""
    bad, first = _run(9, 0, 1 << 32)
    assert bad == 0, f"{bad} violations, first sample {first}"
