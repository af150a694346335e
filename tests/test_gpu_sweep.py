"""GPU exhaustive FP32 sweep (fo_sweep, paper_2602_23349_b200/sweep.py) against
the reference's own sweep statistics (tests/golden/sweep_bf16.json, written by
tests/golden/make_sweep_golden.py running flashopt.sweep.exhaustive_sweep_multi
over all 510 blocks).  Counts, exact counts and maxima must match exactly;
float64 error sums only to summation-order rounding.  SURVEY.md §8f row 3;
PAPER.md:557 quotes 99.92% bitwise-exact reconstruction for bf16 + 16-bit
corrections."""

from __future__ import annotations

import json
import os

import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sweep_bf16.json")


def test_full_sweep_matches_reference(cuda_dev):
    from paper_2602_23349_b200 import sweep

    gold = json.load(open(GOLDEN))
    res = sweep.exhaustive_sweep_multi("bf16", sweep.SCHEMES)
    for s, g in gold.items():
        r = res[s]
        assert r.total_count == g["total_count"] == 510 << 23
        assert r.overflow_count == g["overflow_count"]
        assert r.exact_count == g["exact_count"], s
        assert r.normal_exact_count == g["normal_exact_count"], s
        assert r.nonzero_count == g["nonzero_count"]
        assert r.max_rel_err == g["max_rel_err"], s
        assert abs(r.mean_rel_err - g["mean_rel_err"]) <= 1e-9 * max(g["mean_rel_err"], 1e-30), s
        got = [[b.exponent, b.count, b.exact_count, b.max_rel_err] for b in r.buckets]
        want = [[b[0], b[1], b[2], b[4]] for b in g["buckets"]]
        assert got == want, s
        for b, gb in zip(r.buckets, g["buckets"]):
            assert abs(b.mean_rel_err - gb[3]) <= 1e-9 * max(gb[3], 1e-30)
    assert abs(res["ulp16"].exact_fraction - 0.9992) < 1e-4


def test_subset_blocks(cuda_dev):
    from paper_2602_23349_b200 import sweep

    r = sweep.exhaustive_sweep_multi("bf16", ("ulp8",), _blocks=[0, 127, 128, 255 + 127])["ulp8"]
    assert r.total_count == 4 << 23
    with pytest.raises(NotImplementedError):
        sweep.exhaustive_sweep_multi("fp16", ("ulp8",))
