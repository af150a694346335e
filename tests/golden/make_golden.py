"""Generate tests/golden/*.npz from the live NumPy reference.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures travel with the repo; the GPU box and the CPU tests compare
against them without the reference.  Every case records the reference
inputs (FLOP v1 record names, gradient, hyper-parameters, step counter) and
the reference outputs (`out.<record>`), produced by
flashopt.optim.STEP_FUNCTIONS (optim.py:261) and the codecs of
flashopt.formats / flashopt.quantize.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import helpers as H  # noqa: E402
import refbridge as R  # noqa: E402


def step_cases():
    rng = np.random.default_rng(20260223)
    cases = []
    for opt in ("adamw", "sgd", "lion"):
        for n in (1, 33, 1000, 4133):
            for k in range(2):
                st = H.random_state(rng, n, opt)
                g = H.random_grad(rng, n, std=float(10 ** rng.uniform(-5, -1)))
                hp = H.random_hparams(rng, opt)
                t = int(rng.integers(0, 5000))
                cases.append((f"{opt}_n{n}_{k}", opt, st, g, hp, t))
    return cases


def main() -> None:
    if not R.available():
        raise SystemExit("reference not available")
    fo = R.flashopt()
    F, Q = fo.formats, fo.quantize
    index = {}
    # --- one fused step per case -------------------------------------------
    arrays = {}
    for name, opt, st, g, hp, t in step_cases():
        out = R.ref_step(opt, st, g, t, hp)
        for k, v in st.items():
            arrays[f"{name}/in.{k}"] = v
        for k, v in out.items():
            arrays[f"{name}/out.{k}"] = np.asarray(v)
        arrays[f"{name}/grad"] = g
        index[name] = {"optimizer": opt, "t": t, "hp": hp, "n": int(g.size)}
    np.savez_compressed(os.path.join(HERE, "steps.npz"), **arrays)
    # --- multi-step trajectories from init_flash_state ----------------------
    traj = {}
    rng = np.random.default_rng(7)
    for opt in ("adamw", "sgd", "lion"):
        n = 2048 + 5
        theta0 = H.random_weights(rng, n)
        fs = fo.optim.init_flash_state(theta0, opt)
        traj[f"{opt}/theta0"] = theta0
        hp = H.random_hparams(rng, opt)
        index[f"traj_{opt}"] = {"optimizer": opt, "hp": hp, "steps": 3}
        for s in range(3):
            g = H.random_grad(rng, n, std=1e-2)
            fs = fo.optim.STEP_FUNCTIONS[opt](fs, g, R.hp_object(opt, hp))
            traj[f"{opt}/grad{s}"] = g
            for k, v in R.from_ref_state(fs).items():
                traj[f"{opt}/step{s}.{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "trajectories.npz"), **traj)
    # --- codecs -------------------------------------------------------------
    rng = np.random.default_rng(11)
    u = rng.integers(0, 2**32, size=200_000, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    x = np.concatenate([x[np.isfinite(x)], H.random_weights(rng, 50_000),
                        np.array([0.0, -0.0, 1.00390625, 1.001953125, 70000.0, 3.3895314e38], np.float32)])
    lp, rho = F.split(x, F.BF16, F.INT8_CORRECTION)
    lp16, rho16 = F.split(x, F.BF16, F.INT16_CORRECTION)
    codes = np.repeat(np.arange(0, 65536, 97, dtype=np.uint32), 255).astype(np.uint16)
    rr = np.tile(np.arange(-127, 128, dtype=np.int16), codes.size // 255).astype(np.int8)
    rec = F.reconstruct(codes, rr, F.BF16, F.INT8_CORRECTION)
    m = (rng.standard_normal(40_003) * 10.0 ** rng.integers(-30, 4, 40_003)).astype(np.float32)
    qm = Q.quantize_momentum(m, Q.GroupSpec(32))
    qv = Q.quantize_variance(m * m, Q.GroupSpec(32))
    np.savez_compressed(
        os.path.join(HERE, "codecs.npz"),
        split_x=x, split_lp=lp, split_rho=rho, split_lp16=lp16, split_rho16=rho16,
        rec_lp=codes, rec_rho=rr, rec_out=rec,
        qm_x=m, qm_codes=qm.codes, qm_scales=qm.scales, qm_deq=Q.dequantize_momentum(qm),
        qv_x=m * m, qv_codes=qv.codes, qv_scales=qv.scales, qv_deq=Q.dequantize_variance(qv),
    )
    # --- FLOP v1 files written by the reference ------------------------------
    C = fo.checkpoint
    rng = np.random.default_rng(5)
    for opt, n in (("adamw", 1003), ("sgd", 64), ("lion", 33)):
        st = H.random_state(rng, n, opt)
        fs = R.to_ref_state(st, int(rng.integers(1, 1 << 40)))
        C.save_checkpoint(fs, os.path.join(HERE, f"ckpt_{opt}.flop"), optimizer=opt)
    st = H.random_state(rng, 100, "adamw")
    st["weights.rho"] = rng.integers(-32767, 32768, 100).astype(np.int16)
    C.save_checkpoint(R.to_ref_state(st, 9), os.path.join(HERE, "ckpt_adamw_rho16.flop"))
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
