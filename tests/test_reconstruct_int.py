"""CPU proof of the integer reconstruct used by the fused tile
(csrc/fo_fast.cuh recon_bits): for every finite bf16 code
and every correction code rho in [-127, 127],

    reconstruct(code, rho) == bits(code << 16) + R(rho) * (+1 | -1)

with R(rho) = rint_even(RN(rho/127) * 2^15) (signed like rho) and the sign
of the step taken from lp, except for lp = +-0 with rho of the other sign
(the sum is a NaN pattern) and (-0, rho = 0) (-0 instead of +0).  The
reference here is the C oracle (pinned to flashopt by test_oracle_golden.py,
formats.py:248-276)."""

from __future__ import annotations

import numpy as np

from oracle import oracle as O


def _recon_bits(lpbits: np.ndarray, r: int) -> np.ndarray:
    s = np.where((lpbits.view(np.int32) >> 30) < 0, -1, 1).astype(np.int64)  # (bits >> 30) | 1
    return ((lpbits.astype(np.int64) + r * s) & 0xFFFFFFFF).astype(np.uint32)


def test_integer_reconstruct_matches_oracle_everywhere():
    codes = np.arange(1 << 16, dtype=np.uint32)
    codes = codes[((codes >> 7) & 0xFF) != 0xFF]
    lpbits = codes << 16
    lp16 = codes.astype(np.uint16)
    f32 = np.float32
    for rho in range(-127, 128):
        r = int(np.rint(np.float32(np.float32(rho) / f32(127)) * f32(32768)))  # exact product, half-even
        got = _recon_bits(lpbits, r)
        ref = O.reconstruct(lp16, np.full(codes.size, rho, np.int8)).view(np.uint32)
        for i in np.nonzero(got != ref)[0]:
            c, g = int(codes[i]), int(got[i])
            zero_case = (c == 0x0000 and rho < 0) or (c == 0x8000 and rho >= 0)
            caught = (((g & 0x7F800000) == 0x7F800000) and (g & 0x7FFFFF) != 0) or g == 0x80000000
            assert zero_case and caught, f"code {c:#06x} rho {rho}: got {g:#010x} ref {int(ref[i]):#010x}"


def test_computed_R_equals_table():
    """FO_R_LUT=0 computes R(rho) with one FFMA2 instead of the table:
    float(rho) from the byte trick (rho + 128) | 0x4B000000 - (2^23 + 128),
    then RN(float(rho) * RN(32768/127) + 1.5 * 2^23) - 1.5 * 2^23.  The exact
    rho * 32768 / 127 is at least 0.5/127 from any half-integer, and the
    rounded constant moves it by < 0.002, so the single rounding lands on
    rint_even(RN(rho/127) * 2^15) for every int8 code."""
    f32 = np.float32
    c = f32(f32(32768) / f32(127))
    for rho in range(-128, 128):
        fx = np.uint32(0x4B000000 | ((rho + 128) & 0xFF)).view(np.float32)
        frho = f32(fx - f32(8388736.0))
        assert frho == rho
        if rho == -128:
            continue  # invalid code: the rho guard flags the slice
        t = np.float32(np.float64(frho) * np.float64(c) + 12582912.0)  # the FFMA: exact product + sum, one rounding
        r = int(t.view(np.uint32)) - 0x4B400000
        assert r == int(np.rint(f32(f32(rho) / f32(127)) * f32(32768))), rho
