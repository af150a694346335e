"""Randomised bitwise parity stress: the fused CUDA step against the C
oracle on random optimizers, sizes, states, gradient magnitude ranges
(down to subnormals), hyper-parameters across the fast ranges and beyond,
and step counters, for a wall-clock budget.  Prints one summary JSON line;
mismatching cases are written to gpurun_out/stress_fail_*.json.

    python tools/parity_stress.py [--seconds 240] [--seed 1] [--layouts]

--layouts also draws the optional layouts (int16 corrections, linear
variance) and training-like weights, which keep most slices on the fused
tile of those layouts.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import helpers as H  # noqa: E402
from devstate import from_device, mismatches, oracle_dict, oracle_state, to_device  # noqa: E402
from oracle import oracle as O  # noqa: E402


def pick_beta(rng):
    return float(rng.choice([0.0, 2.0 ** -29, 0.3, 0.9, 0.95, 0.99, 0.999, 1 - 2.0 ** -19]))


def random_case(rng, layouts=False):
    opt = str(rng.choice(["adamw", "sgd", "lion"]))
    rho_bits = int(rng.choice([8, 16])) if layouts else 8
    scheme = str(rng.choice(["companded", "linear"])) if (layouts and opt == "adamw") else "companded"
    training_like = bool(layouts and rng.random() < 0.5)
    n = int(rng.choice([int(rng.integers(1, 5000)), int(rng.integers(5000, 300000)), int(rng.integers(300000, 2000000))]))
    lr = float(10 ** rng.uniform(-8, 0.5))
    wd = float(rng.choice([0.0, 1e-4, 0.01, 0.1, 1.0]))
    if opt == "adamw":
        hp = dict(lr=lr, beta1=pick_beta(rng), beta2=pick_beta(rng), eps=float(10 ** rng.uniform(-30, 10)),
                  weight_decay=wd)
    elif opt == "sgd":
        hp = dict(lr=lr, momentum=pick_beta(rng), weight_decay=wd)
    else:
        hp = dict(lr=lr, beta1=pick_beta(rng), beta2=pick_beta(rng), weight_decay=wd)
    t = int(rng.choice([0, 1, int(rng.integers(2, 400)), int(rng.integers(400, 30000))]))
    lo, hi = sorted(rng.uniform(-149, 8, 2))
    inject = str(rng.choice(["none"] * 9 + ["nan", "inf", "huge", "rho"])) if rng.random() < 0.3 else "none"
    return dict(opt=opt, n=n, hp=hp, t=t, glo=float(lo), ghi=float(hi), zero_state=bool(rng.random() < 0.2),
                grad_f32=bool(rng.random() < 0.2), inject=inject, seed=int(rng.integers(0, 2 ** 31)),
                rho_bits=rho_bits, scheme=scheme, training_like=training_like)


def run_case(c, dev):
    from paper_2602_23349_b200 import optim as FO

    rng = np.random.default_rng(c["seed"])
    n, opt = c["n"], c["opt"]
    rho_bits, scheme = c.get("rho_bits", 8), c.get("scheme", "companded")
    lp = H.bf16_codes((rng.standard_normal(n) * 0.02).astype(np.float32)) if c.get("training_like") else None
    st = H.random_state(rng, n, opt, lp=lp)
    if rho_bits == 16:
        st["weights.rho"] = rng.integers(-32767, 32768, n).astype(np.int16)
    if c["zero_state"]:
        for k in st:
            if k not in ("weights.lp", "weights.rho"):
                st[k] = np.zeros_like(st[k])
    mag = 2.0 ** rng.uniform(c["glo"], c["ghi"], n)
    g = (np.sign(rng.standard_normal(n)) * mag).astype(np.float32)
    g[rng.random(n) < 0.01] = 0.0
    if not c["grad_f32"]:
        g = H.bf16_round(g)
    k = rng.integers(0, n, max(1, n // 100000))
    if c.get("inject") == "nan":
        g[k] = np.float32("nan")
    elif c.get("inject") == "inf":
        g[k] = np.float32("-inf")
    elif c.get("inject") == "huge":
        g[k] = np.float32(3e38)
    elif c.get("inject") == "rho":
        st["weights.rho"][k] = -128 if rho_bits == 8 else -32768
    ost = oracle_state(st, c["t"], 32, scheme)
    oerr = O.step_inplace(opt, ost, g, nthreads=8, **c["hp"])
    fs = to_device(st, c["t"], dev, 32, scheme)
    gd = torch.from_numpy(g).to(dev)
    if not c["grad_f32"]:
        gd = gd.bfloat16()
    try:
        FO.STEP_FUNCTIONS_INPLACE[opt](fs, gd, FO.HP_TYPES[opt](**c["hp"]))
        derr = ""
    except ValueError as e:
        derr = str(e)
    if oerr:
        return "error_both" if derr else "error_oracle_only"
    if derr:
        return "error_device_only"
    mm = mismatches(from_device(fs), oracle_dict(ost))
    return "ok" if all(v == 0 for v in mm.values()) else ("mismatch", mm)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--layouts", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + args.seconds
    counts, elems, fails = {}, 0, 0
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    while time.time() < t_end:
        c = random_case(rng, args.layouts)
        r = run_case(c, dev)
        key = r if isinstance(r, str) else r[0]
        counts[key] = counts.get(key, 0) + 1
        elems += c["n"]
        if key in ("mismatch", "error_oracle_only", "error_device_only"):
            fails += 1
            with open(os.path.join(ROOT, "gpurun_out", f"stress_fail_{fails}.json"), "w") as f:
                json.dump({"case": c, "result": r if isinstance(r, str) else r[1]}, f, default=str)
    print(json.dumps({"cases": sum(counts.values()), "elements": elems, "outcomes": counts, "failures": fails}))


if __name__ == "__main__":
    main()
