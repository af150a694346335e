"""BASELINE.json config 5: GPT-2-medium training step with the fused
FlashAdamW step, deferred (optimizer.step() after backward) and with gradient
release (the step runs from backward hooks on a side stream), against
torch.optim.AdamW(fused=True) with fp32 master weights under bf16 autocast
(the usual mixed-precision recipe, 16 bytes/param of weights + states).
Also times a compressed FLOP v1 checkpoint save/load of the FlashAdamW state
and checks the reload bit for bit.

Random-init GPT-2-medium (HF layout: 24 layers, d=1024, 16 heads, tied
embeddings, 354.8M params), synthetic token batches (no dataset is
available offline), dropout off.  One JSON line per mode on stdout.

    python tools/bench_gpt2_train.py [--batch 8] [--seq 1024] [--steps 20] [--warmup 5]
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

HP = dict(lr=6e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)


def make_model(dtype, checkpointing: bool = False):
    from transformers import GPT2Config, GPT2LMHeadModel

    cfg = GPT2Config(n_layer=24, n_embd=1024, n_head=16, n_positions=1024, vocab_size=50257,
                     attn_pdrop=0.0, resid_pdrop=0.0, embd_pdrop=0.0, tie_word_embeddings=True)
    torch.manual_seed(0)
    m = GPT2LMHeadModel(cfg)
    m.config._attn_implementation = "sdpa"
    if checkpointing:
        m.gradient_checkpointing_enable()
    return m.to(device="cuda", dtype=dtype)


def run_mode(mode: str, args) -> dict:
    from paper_2602_23349_b200.release import GradientRelease
    from paper_2602_23349_b200.torch_optim import FlashAdamW

    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    fp32_master = mode == "torch_adamw_fp32"
    model = make_model(torch.float32 if fp32_master else torch.bfloat16, args.checkpointing)
    params = [p for p in model.parameters()]
    n_params = sum(p.numel() for p in params)
    release = None
    if mode == "torch_adamw_fp32":
        opt = torch.optim.AdamW(params, fused=True, **HP)
    else:
        opt = FlashAdamW(params, check_errors=False, **HP)
        if mode == "flash_release":
            release = GradientRelease(opt, timing=True)
    g = torch.Generator(device="cuda").manual_seed(1)
    batches = [torch.randint(0, 50257, (args.batch, args.seq), device="cuda", generator=g) for _ in range(4)]
    opt_ev = []
    boundary = []  # bytes allocated when backward has returned (the optimizer boundary)

    def step(i):
        x = batches[i % len(batches)]
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=fp32_master):
            loss = model(input_ids=x, labels=x).loss
        loss.backward()
        if i == 0 or len(boundary) < 2:
            torch.cuda.synchronize()
            boundary.append(torch.cuda.memory_allocated())
        if release is None:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            opt.step()
            b.record()
            opt_ev.append((a, b))
            opt.zero_grad(set_to_none=True)
        return loss

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    opt_ev.clear()
    if release is not None:
        release.side_stream_ms()  # drop the warm-up launches
    torch.cuda.reset_peak_memory_stats()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for i in range(args.steps):
        loss = step(i)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    if release is not None:
        release.check()
    elif mode != "torch_adamw_fp32":
        opt.raise_errors()
    opt_ms = sum(a.elapsed_time(b) for a, b in opt_ev) / len(opt_ev) if opt_ev else None
    peak = torch.cuda.max_memory_allocated()
    release_info = None
    if release is not None:
        opt_ms = release.side_stream_ms() / args.steps
        release_info = {"launch_calls_per_step": release.launch_calls / (args.warmup + args.steps),
                        "bucket_elems": release.bucket_elems,
                        "optimizer_ms_is": "side-stream device time of the fused launches (overlaps backward)"}
    # optimizer step alone, back to back on resident gradients: device time per
    # step (host enqueue cost overlaps), and the host cost of one step() call
    iso = None
    if release is None:
        x = batches[0]
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=fp32_master):
            model(input_ids=x, labels=x).loss.backward()
        for _ in range(3):
            opt.step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h = time.perf_counter()
        a.record()
        for _ in range(20):
            opt.step()
        b.record()
        host_ms = (time.perf_counter() - h) / 20 * 1e3
        torch.cuda.synchronize()
        dev_ms = a.elapsed_time(b) / 20
        iso = {"ms_per_step": dev_ms, "gparams_per_s": n_params / (dev_ms * 1e-3) / 1e9, "host_ms_per_call": host_ms}
        opt.zero_grad(set_to_none=True)
    state_bytes = 0
    for st in opt.state.values():
        for v in st.values():
            if isinstance(v, torch.Tensor):
                state_bytes += v.numel() * v.element_size()
    weight_bytes = sum(p.numel() * p.element_size() for p in params)
    # bytes held at the optimizer boundary beyond weights + optimizer state:
    # the gradients (2 B/param in bf16) in deferred mode, ~0 with release
    out = {
        "config": "gpt2_medium_train", "mode": mode, "params": n_params, "batch": args.batch, "seq": args.seq,
        "tokens_per_s": args.batch * args.seq / (ms * 1e-3), "ms_per_step": ms,
        "optimizer_step_ms": opt_ms,
        "optimizer_gparams_per_s": (n_params / (opt_ms * 1e-3) / 1e9) if opt_ms else None,
        "optimizer_step_back_to_back": iso,
        "peak_mem_gib": peak / 2**30,
        "allocated_at_optimizer_boundary_gib": boundary[-1] / 2**30,
        "boundary_minus_weights_and_state_bytes_per_param": None,
        "activation": "checkpointed" if args.checkpointing else "stored",
        "release": release_info,
        "weights_plus_state_bytes_per_param": (weight_bytes + state_bytes) / n_params,
        "final_loss": float(loss.item()),
        "data": "synthetic tokens, random init",
    }
    out["boundary_minus_weights_and_state_bytes_per_param"] = (boundary[-1] - weight_bytes - state_bytes) / n_params
    if mode == "flash":
        out["checkpoint"] = checkpoint_roundtrip(opt, params)
    if release is not None:
        release.remove()
    del opt, model, params
    return out


def checkpoint_roundtrip(opt, params) -> dict:
    """FLOP v1 save of every parameter's FlashAdamW state, reload into a
    fresh optimizer over fresh parameters, bitwise comparison."""
    from paper_2602_23349_b200.checkpoint import load_optimizer, save_optimizer
    from paper_2602_23349_b200.torch_optim import FlashAdamW

    d = tempfile.mkdtemp(prefix="fo_ckpt_")
    try:
        torch.cuda.synchronize()
        t = time.perf_counter()
        man = save_optimizer(opt, d)
        save_s = time.perf_counter() - t
        fresh = [torch.zeros_like(p) for p in params]
        opt2 = FlashAdamW(fresh, check_errors=False, **HP)
        torch.cuda.synchronize()
        t = time.perf_counter()
        load_optimizer(opt2, d)
        torch.cuda.synchronize()
        load_s = time.perf_counter() - t
        same = True
        for p, q in zip(params, fresh):
            same &= bool(torch.equal(p.data.view(torch.int16), q.data.view(torch.int16)))
            a, b = opt.state[p], opt2.state[q]
            for k in ("weights.rho", "momentum.codes", "variance.codes"):
                same &= bool(torch.equal(a[k], b[k]))
            for k in ("momentum.scales", "variance.scales"):
                same &= bool(torch.equal(a[k].view(torch.int16), b[k].view(torch.int16)))
            same &= int(a["step"]) == int(b["step"])
        n = sum(p.numel() for p in params)
        return {"files": len(man["params"]), "bytes": man["bytes"], "bytes_per_param": man["bytes"] / n,
                "save_s": save_s, "load_s": load_s, "bitwise_equal_after_reload": same,
                "format": "FLOP v1 per parameter (checkpoint.py), byte-identical to the reference writer"}
    finally:
        shutil.rmtree(d, ignore_errors=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--modes", default="flash,flash_release,torch_adamw_fp32")
    ap.add_argument("--checkpointing", action="store_true",
                    help="activation checkpointing (small activations, so gradients matter for the peak)")
    args = ap.parse_args()
    for mode in args.modes.split(","):
        print(json.dumps(run_mode(mode, args)), flush=True)


if __name__ == "__main__":
    main()
