"""Exhaustive FP32 reconstruction sweep on the GPU.

Mirror of the reference's sweep module (flashopt/sweep.py): every finite
FP32 bit pattern (both signs, 510 (sign, exponent-field) blocks of 2^23) is
pushed through a weight-compression scheme and compared with the original;
results aggregate into per-exponent buckets (count, bitwise-exact count,
mean and max relative error).  The per-block work (sweep.py:166-218
`_sweep_block`) runs in `fo_sweep` (csrc/fo_sweep.cu) with the same device
codec the generic step kernel uses; the bucket merge below restates
sweep.py:231-308.  The whole 4.28e9-pattern sweep takes well under a second
on a B200, against ~90 s for the reference on 8 CPU processes.

Counts, exact counts and maxima match the reference exactly
(tests/test_gpu_sweep.py against tests/golden/sweep_bf16.json, written by
the reference itself); float64 error sums differ only in summation order.

Only the BF16 format is implemented (the step's format); FP16 sweeps are
out of scope.
"""

from __future__ import annotations

import csv
import json
import time
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["SCHEMES", "SweepBucket", "SweepResult", "exhaustive_sweep", "exhaustive_sweep_multi",
           "write_buckets_csv", "write_summary_json"]

SCHEMES = ("ulp8", "ulp16", "none", "baseline")  # sweep.py:50, also fo_sweep's scheme bit order
_N_BLOCKS = 510
_BLOCK = 1 << 23
_N_BUCKETS = 258  # 0 zero, 1 subnormal, 2..256 exponent fields 1..255, 257 overflow
_ZERO, _SUBNORMAL, _OVERFLOW = 0, 1, 257


@dataclass
class SweepBucket:
    """Aggregate over all swept values sharing one FP32 exponent (sweep.py:60-72)."""

    exponent: int | str
    count: int
    exact_count: int
    mean_rel_err: float
    max_rel_err: float

    @property
    def exact_fraction(self) -> float:
        return self.exact_count / self.count if self.count else 0.0


@dataclass
class SweepResult:
    """Same fields and derived properties as sweep.py:75-129."""

    fmt: str
    scheme: str
    buckets: list
    total_count: int
    overflow_count: int
    exact_count: int
    rel_err_sum: float
    max_rel_err: float
    nonzero_count: int
    normal_count: int
    normal_exact_count: int
    elapsed_seconds: float
    workers: int

    @property
    def finite_downcast_count(self) -> int:
        return self.total_count - self.overflow_count

    @property
    def exact_fraction(self) -> float:
        return self.exact_count / self.finite_downcast_count

    @property
    def exact_fraction_normals_only(self) -> float:
        return self.normal_exact_count / self.normal_count

    @property
    def mean_rel_err(self) -> float:
        return self.rel_err_sum / self.nonzero_count

    def summary_dict(self) -> dict:
        return {"format": self.fmt, "scheme": self.scheme, "total_count": self.total_count,
                "finite_downcast_count": self.finite_downcast_count, "overflow_count": self.overflow_count,
                "exact_count": self.exact_count, "exact_fraction": self.exact_fraction,
                "exact_fraction_normals_only": self.exact_fraction_normals_only,
                "mean_rel_err": self.mean_rel_err, "max_rel_err": self.max_rel_err,
                "elapsed_seconds": self.elapsed_seconds, "workers": self.workers}


def _label(i: int):
    if i == _ZERO:
        return "zero"
    if i == _SUBNORMAL:
        return "subnormal"
    if i == _OVERFLOW:
        return "overflow"
    return i - 128  # exponent field i - 1, unbiased


def _fmt_name(fmt) -> str:
    name = fmt if isinstance(fmt, str) else getattr(fmt, "name", str(fmt))
    if name != "bf16":
        raise NotImplementedError("the GPU sweep implements the BF16 format only")
    return name


def exhaustive_sweep_multi(fmt="bf16", schemes=SCHEMES, workers=None, _blocks=None, device=None) -> dict:
    """Sweep all finite FP32 patterns (or the `_blocks` subset of the 510
    (sign, exponent) blocks) under each scheme; returns {scheme: SweepResult}."""
    import torch

    name = _fmt_name(fmt)
    for s in schemes:
        if s not in SCHEMES:
            raise ValueError(f"unknown sweep scheme: {s}")
    blocks = list(range(_N_BLOCKS)) if _blocks is None else sorted(set(int(b) for b in _blocks))
    mask = sum(1 << SCHEMES.index(s) for s in schemes)
    dev = torch.device(device or "cuda")
    t0 = time.perf_counter()
    recs = np.zeros((_N_BLOCKS, len(SCHEMES), 8), dtype=np.uint64)
    # contiguous runs of requested blocks, one launch each
    runs, i = [], 0
    while i < len(blocks):
        j = i
        while j + 1 < len(blocks) and blocks[j + 1] == blocks[j] + 1:
            j += 1
        runs.append((blocks[i], j - i + 1))
        i = j + 1
    for b0, nb in runs:
        out = torch.zeros(nb * len(SCHEMES) * 8, dtype=torch.int64, device=dev)
        _lib.check(_lib.lib().fo_sweep(b0, nb, mask, out.data_ptr(), None), "fo_sweep")
        recs[b0:b0 + nb] = out.cpu().numpy().view(np.uint64).reshape(nb, len(SCHEMES), 8)
    torch.cuda.synchronize(dev)
    elapsed = time.perf_counter() - t0

    results = {}
    for s in schemes:
        k = SCHEMES.index(s)
        counts = np.zeros(_N_BUCKETS, np.int64)
        exacts = np.zeros(_N_BUCKETS, np.int64)
        relsums = np.zeros(_N_BUCKETS, np.float64)
        relmaxs = np.zeros(_N_BUCKETS, np.float64)
        for b in blocks:
            r = recs[b, k]
            expf = b % 255
            bucket = _SUBNORMAL if expf == 0 else expf + 1
            counts[bucket] += int(r[0])
            exacts[bucket] += int(r[1])
            relsums[bucket] += float(r[5:6].view(np.float64)[0])
            relmaxs[bucket] = max(relmaxs[bucket], float(np.uint32(r[6]).view(np.float32)))
            counts[_OVERFLOW] += int(r[2])
            counts[_ZERO] += int(r[3])
            exacts[_ZERO] += int(r[4])
        buckets = []
        for i in range(_N_BUCKETS):
            if counts[i] == 0:
                continue
            nz = counts[i] if i not in (_ZERO, _OVERFLOW) else 0
            buckets.append(SweepBucket(_label(i), int(counts[i]), int(exacts[i]),
                                       float(relsums[i] / nz) if nz else 0.0, float(relmaxs[i])))
        normal = slice(2, _N_BUCKETS - 1)
        results[s] = SweepResult(
            fmt=name, scheme=s, buckets=buckets, total_count=int(counts.sum()),
            overflow_count=int(counts[_OVERFLOW]), exact_count=int(exacts.sum()),
            rel_err_sum=float(relsums.sum()), max_rel_err=float(relmaxs.max()),
            nonzero_count=int(counts[normal].sum() + counts[_SUBNORMAL]),
            normal_count=int(counts[normal].sum()), normal_exact_count=int(exacts[normal].sum()),
            elapsed_seconds=elapsed, workers=1)
        assert results[s].total_count == len(blocks) * _BLOCK
    return results


def exhaustive_sweep(fmt, scheme: str, workers=None) -> SweepResult:
    return exhaustive_sweep_multi(fmt, (scheme,), workers)[scheme]


def write_buckets_csv(result: SweepResult, path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["exponent", "count", "mean_rel_err", "max_rel_err", "exact_fraction"])
        for b in result.buckets:
            w.writerow([b.exponent, b.count, repr(b.mean_rel_err), repr(b.max_rel_err), repr(b.exact_fraction)])


def write_summary_json(results: dict, path) -> None:
    with open(path, "w") as fh:
        json.dump({s: r.summary_dict() for s, r in sorted(results.items())}, fh, indent=2, sort_keys=True)
        fh.write("\n")
