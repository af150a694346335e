"""e2e (fo_step_host) throughput against the device slot size, on the
Llama-8B list: one JSON line per chunk size."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_23349_b200 import shapes as S  # noqa: E402
from paper_2602_23349_b200.flat import FlatStates  # noqa: E402
from paper_2602_23349_b200.optim import HP_TYPES  # noqa: E402

dev = torch.device("cuda:0")
sizes = [S.numel(s) for _, s in S.CONFIGS["llama31_8b"]()]
fl = FlatStates(sizes, "adamw", dev)
g = torch.empty(fl.total, dtype=torch.bfloat16, device=dev)
bench.init_random_state(fl, g, 5)
hp = HP_TYPES["adamw"](**bench.hparams_for("llama31_8b", "adamw"))
for ce in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "24,25,26,27").split(",")]:
    r = bench.host_e2e(fl, g, "adamw", hp, 1000, steps=2, warmup=1, chunk_elems=1 << ce)
    print(json.dumps({"chunk_log2": ce, "gparams_per_s": r["value"], "ms": r["ms_per_step"],
                      "frac_pcie": r["roofline"]["frac"]}), flush=True)
