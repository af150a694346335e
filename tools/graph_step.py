"""Host cost of the step on small lists: the same fused step launched from
Python per step (StepPlan.launch -> fo_step_mt) and replayed from a CUDA
graph of one step (same scalars: t >= the steady state, where the bias
corrections are 1), per BASELINE list.  Also the host time per launch call.
One JSON line per (config, optimizer, mode).

    python tools/graph_step.py [--steps 200]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def run(config: str, opt: str, steps: int) -> list:
    from paper_2602_23349_b200 import shapes as S
    from paper_2602_23349_b200.flat import FlatStates, StepPlan
    from paper_2602_23349_b200.optim import HP_TYPES

    dev = torch.device("cuda:0")
    sizes = [S.numel(s) for _, s in S.CONFIGS[config]()]
    fl = FlatStates(sizes, opt, dev)
    g = torch.empty(fl.total, dtype=torch.bfloat16, device=dev)
    bench.init_random_state(fl, g, 3)
    plan = StepPlan(opt, fl.states)
    plan.set_grads([g[o:o + n] for o, n in zip(fl.offsets, fl.sizes)])
    for st in fl.states:
        st.t = 1000
    hp = HP_TYPES[opt](**bench.hparams_for(config, opt))
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    s = torch.cuda.Stream(dev)
    out = []
    with torch.cuda.stream(s):
        sh = s.cuda_stream
        scal = [hp.scalars(1001)]

        def one():
            plan.launch(scal, err.data_ptr(), sh)

        for _ in range(5):
            one()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        a.record(s)
        for _ in range(steps):
            one()
        b.record(s)
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        out.append(dict(mode="launch", ms=ms, host_us_per_call=(h1 - h0) / steps * 1e6))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            one()
        for _ in range(5):
            graph.replay()
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        a.record(s)
        for _ in range(steps):
            graph.replay()
        b.record(s)
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        out.append(dict(mode="graph", ms=a.elapsed_time(b) / steps, host_us_per_call=(h1 - h0) / steps * 1e6))
    peak, _ = bench.peaks()
    n = fl.numel
    for o in out:
        o.update(config=config, optimizer=opt, params=n, gparams_per_s=n / (o["ms"] * 1e-3) / 1e9,
                 frac_of_measured_hbm=n * bench.BYTES_PER_PARAM[opt] / (o["ms"] * 1e-3) / 1e9 / peak,
                 device_errors=int(err.item()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    args = ap.parse_args()
    for cfg, opt in (("resnet50", "sgd"), ("resnet50", "lion"), ("gpt2_medium", "adamw")):
        for r in run(cfg, opt, args.steps):
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
