"""Step throughput of the reference's optional state layouts (SURVEY.md §8f
row 4): int16 corrections (N = 32767, formats.py:94-95), the linear-variance
ablation (quantize.py:161-185) and 2-byte-aligned views, next to the
default int8 / companded layout, on one BASELINE shapes list.  One JSON line
per variant.  FO_GENERIC=pergroup in the environment sends the non-default
layouts to the one-thread-per-group kernel instead of the group-32 kernel.

    python tools/bench_variants.py [--config gpt2_medium] [--optimizer adamw] [--steps 10]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def bytes_per_param(opt: str, rho_bits: int) -> float:
    return bench.BYTES_PER_PARAM[opt] + (2.0 if rho_bits == 16 else 0.0)  # rho read + written


def run(config: str, opt: str, variant: str, steps: int, warmup: int) -> dict:
    from paper_2602_23349_b200 import shapes as S
    from paper_2602_23349_b200.flat import FlatStates, StepPlan
    from paper_2602_23349_b200.optim import HP_TYPES

    dev = torch.device("cuda:0")
    sizes = [S.numel(s) for _, s in S.CONFIGS[config]()]
    rho_bits = 16 if variant == "int16" else 8
    scheme = "linear" if variant == "linear" else "companded"
    fl = FlatStates(sizes, opt, dev, rho_bits=rho_bits, variance_scheme=scheme)
    gflat = torch.empty(fl.total + 64, dtype=torch.bfloat16, device=dev)
    bench.init_random_state(fl, gflat[:fl.total], 7)
    shift = 1 if variant == "misaligned" else 0  # 2-byte aligned gradient views
    grads = [gflat[o + shift:o + shift + n] for o, n in zip(fl.offsets, fl.sizes)]
    plan = StepPlan(opt, fl.states)
    plan.set_grads(grads)
    for st in fl.states:
        st.t = 1000
    hp = HP_TYPES[opt](**bench.hparams_for(config, opt))
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    sh = torch.cuda.current_stream(dev).cuda_stream
    for _ in range(warmup):
        plan.launch([hp.scalars(fl.states[0].t + 1)], err.data_ptr(), sh)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        plan.launch([hp.scalars(fl.states[0].t + 1)], err.data_ptr(), sh)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    n = fl.numel
    bpp = bytes_per_param(opt, rho_bits)
    peak, _ = bench.peaks()
    # int16 corrections and linear variance take the fused kernel since round 2
    # (FO_FAST_LAYOUTS=0 keeps them on the exact kernels); misaligned views never do
    fused = variant == "default" or (variant in ("int16", "linear") and os.environ.get("FO_FAST_LAYOUTS") != "0")
    kernel = "step_ws_kernel" if fused else \
        ("step_generic_kernel" if os.environ.get("FO_GENERIC") == "pergroup" else "step_g32_kernel")
    return {"config": config, "optimizer": opt, "variant": variant, "kernel": kernel, "params": n,
            "ms_per_step": ms, "gparams_per_s": n / (ms * 1e-3) / 1e9, "bytes_per_param": bpp,
            "hbm_gbs": n * bpp / (ms * 1e-3) / 1e9, "frac_of_measured_hbm": n * bpp / (ms * 1e-3) / 1e9 / peak,
            "device_errors": int(err.item())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt2_medium")
    ap.add_argument("--optimizer", default="adamw")
    ap.add_argument("--variants", default="default,int16,linear,misaligned")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    for v in args.variants.split(","):
        if v == "linear" and args.optimizer != "adamw":
            continue
        print(json.dumps(run(args.config, args.optimizer, v, args.steps, args.warmup)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
