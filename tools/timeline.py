"""Kernel timeline without nsys (not installed in this image): torch.profiler
(CUPTI) around a few GPT-2-medium training steps with gradient release, and
around ZeRO-1 steps with the bucketed reduce-scatter started from backward
hooks (one rank, NCCL).  Writes a chrome trace (gzipped) and a JSON summary:
per stream, the busy time of our fused-step kernels and how much of it
overlaps kernels on other streams (backward / NCCL).

    python tools/timeline.py --out gpurun_out/timeline
"""
import argparse
import gzip
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402


def kernels_from_trace(path):
    with open(path) as f:
        tr = json.load(f)
    ev = [e for e in tr.get("traceEvents", []) if e.get("cat") == "kernel" and e.get("ph") == "X"]
    return [(e["name"], int(e["args"].get("stream", -1)), float(e["ts"]), float(e["ts"]) + float(e["dur"]))
            for e in ev]


def overlap_summary(kern, ours=("fo::",)):
    by_stream = {}
    for name, s, a, b in kern:
        by_stream.setdefault(s, []).append((a, b, name))
    out = {}
    for s, iv in by_stream.items():
        mine = [(a, b) for a, b, n in iv if any(n.startswith(o) or o in n for o in ours)]
        others = sorted((a, b) for s2, iv2 in by_stream.items() if s2 != s for a, b, _ in iv2)
        busy = sum(b - a for a, b in mine)
        ov = 0.0
        for a, b in mine:
            for c, d in others:
                if c >= b:
                    break
                if d > a:
                    ov += min(b, d) - max(a, c)
        out[str(s)] = {"kernels": len(iv), "fo_kernels": len(mine), "fo_busy_us": busy,
                       "fo_overlapped_by_other_streams_us": ov,
                       "names": sorted({n[:60] for _, _, n in iv})[:8]}
    return out


def release_trace(out_dir, steps=3):
    from bench_gpt2_train import make_model

    from paper_2602_23349_b200.release import GradientRelease
    from paper_2602_23349_b200.torch_optim import FlashAdamW

    model = make_model(torch.bfloat16)
    opt = FlashAdamW(list(model.parameters()), lr=6e-4, betas=(0.9, 0.95), weight_decay=0.1)
    rel = GradientRelease(opt)
    x = torch.randint(0, 50257, (8, 1024), device="cuda")
    for _ in range(2):
        model(input_ids=x, labels=x).loss.backward()
    torch.cuda.synchronize()
    path = os.path.join(out_dir, "release_trace.json")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            model(input_ids=x, labels=x).loss.backward()
        torch.cuda.synchronize()
    prof.export_chrome_trace(path)
    rel.check()
    return path, {"what": "GPT-2-medium bf16, batch 8 x 1024, FlashAdamW gradient release (bucketed, side stream)",
                  "steps": steps, "launch_calls": rel.launch_calls}


def zero_trace(out_dir, steps=3):
    import torch.distributed as dist

    from bench_gpt2_train import make_model

    from paper_2602_23349_b200 import optim as FO
    from paper_2602_23349_b200.zero import ZeroFlashOptimizer

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29577")
    dist.init_process_group("nccl", rank=0, world_size=1)
    model = make_model(torch.bfloat16)
    zo = ZeroFlashOptimizer(list(model.parameters()), "adamw", [FO.AdamHyperParams(lr=6e-4, beta2=0.95,
                                                                                    weight_decay=0.1)],
                            bucket_elems=1 << 25, overlap_grad_reduce=True)
    x = torch.randint(0, 50257, (8, 1024), device="cuda")

    def step():
        zo.zero_grad()
        model(input_ids=x, labels=x).loss.backward()
        zo.step()

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    path = os.path.join(out_dir, "zero_trace.json")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
    prof.export_chrome_trace(path)
    info = {"what": "GPT-2-medium bf16, ZeRO-1 on 1 NCCL rank, 32M-element buckets, reduce-scatter from grad hooks",
            "steps": steps, "buckets": len(zo.layout.buckets), "rs_launched_in_backward": zo.rs_launched_in_backward}
    zo.remove_hooks()
    dist.destroy_process_group()
    return path, info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/timeline")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    summary = {}
    for name, fn in (("release", release_trace), ("zero1", zero_trace)):
        path, info = fn(args.out)
        info["streams"] = overlap_summary(kernels_from_trace(path))
        summary[name] = info
        with open(path, "rb") as f, gzip.open(path + ".gz", "wb") as g:
            shutil.copyfileobj(f, g)
        os.remove(path)
    with open(os.path.join(args.out, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary)[:3000])


if __name__ == "__main__":
    main()
