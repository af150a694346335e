"""Golden statistics of the reference's exhaustive FP32 sweep
(flashopt/sweep.py exhaustive_sweep_multi, BF16, all four schemes, all 510
(sign, exponent) blocks), run in the build container by importing the
reference from /root/reference.  Writes tests/golden/sweep_bf16.json:
per-scheme summary plus per-bucket count / exact_count / mean / max."""

import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
from flashopt.formats import BF16  # noqa: E402
from flashopt.sweep import SCHEMES, exhaustive_sweep_multi  # noqa: E402

t = time.time()
res = exhaustive_sweep_multi(BF16, SCHEMES, workers=int(os.environ.get("FLASHOPT_WORKERS", "8")))
out = {}
for s, r in res.items():
    d = r.summary_dict()
    d.pop("elapsed_seconds")
    d.pop("workers")
    d["buckets"] = [[b.exponent, b.count, b.exact_count, b.mean_rel_err, b.max_rel_err] for b in r.buckets]
    d["rel_err_sum"] = r.rel_err_sum
    d["nonzero_count"] = r.nonzero_count
    d["normal_count"] = r.normal_count
    d["normal_exact_count"] = r.normal_exact_count
    out[s] = d
here = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(here, "sweep_bf16.json"), "w") as f:
    json.dump(out, f, indent=0, sort_keys=True)
print("done in", time.time() - t, "s;", {s: out[s]["exact_fraction"] for s in out})
