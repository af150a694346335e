"""GPU: the CUDA step against vectors produced by the reference itself
(tests/golden/*.npz, made by tests/golden/make_golden.py) -- an anchor that
does not go through the C oracle."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

from devstate import bits, from_device, mismatches, to_device

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _index():
    with open(os.path.join(GOLD, "index.json")) as f:
        return json.load(f)


def test_steps_match_reference_vectors(cuda_dev):
    from paper_2602_23349_b200 import optim as FO

    idx = _index()
    z = np.load(os.path.join(GOLD, "steps.npz"))
    for name, meta in sorted(idx.items()):
        if name.startswith("traj_"):
            continue
        st = {k.split("/in.", 1)[1]: z[k] for k in z.files if k.startswith(f"{name}/in.")}
        ref = {k.split("/out.", 1)[1]: z[k] for k in z.files if k.startswith(f"{name}/out.")}
        fs = to_device(st, meta["t"], cuda_dev)
        opt = meta["optimizer"]
        FO.STEP_FUNCTIONS_INPLACE[opt](fs, torch.from_numpy(z[f"{name}/grad"]).to(cuda_dev).bfloat16(),
                                       FO.HP_TYPES[opt](**meta["hp"]))
        mm = mismatches(from_device(fs), ref)
        assert all(v == 0 for v in mm.values()), (name, mm)


def test_trajectories_from_init_match_reference(cuda_dev):
    from paper_2602_23349_b200 import optim as FO

    idx = _index()
    z = np.load(os.path.join(GOLD, "trajectories.npz"))
    for opt in ("adamw", "sgd", "lion"):
        meta = idx[f"traj_{opt}"]
        fs = FO.init_flash_state(torch.from_numpy(z[f"{opt}/theta0"]).to(cuda_dev), opt)
        hp = FO.HP_TYPES[opt](**meta["hp"])
        for s in range(meta["steps"]):
            FO.STEP_FUNCTIONS_INPLACE[opt](fs, torch.from_numpy(z[f"{opt}/grad{s}"]).to(cuda_dev).bfloat16(), hp)
            ref = {k.split(".", 1)[1]: z[k] for k in z.files if k.startswith(f"{opt}/step{s}.")}
            mm = mismatches(from_device(fs), ref)
            assert all(v == 0 for v in mm.values()), (opt, s, mm)


def test_codecs_match_reference_vectors(cuda_dev):
    from paper_2602_23349_b200 import formats as F
    from paper_2602_23349_b200 import quantize as Q

    z = np.load(os.path.join(GOLD, "codecs.npz"))
    x = torch.from_numpy(z["split_x"]).to(cuda_dev)
    lp, rho = F.split(x)
    assert np.array_equal(lp.view(torch.int16).cpu().numpy().view(np.uint16), z["split_lp"])
    assert np.array_equal(rho.cpu().numpy(), z["split_rho"])
    lp16, rho16 = F.split(x, F.INT16_CORRECTION)
    assert np.array_equal(rho16.cpu().numpy(), z["split_rho16"])
    rec = F.reconstruct(torch.from_numpy(z["rec_lp"].view(np.int16)).to(cuda_dev).view(torch.bfloat16),
                        torch.from_numpy(z["rec_rho"]).to(cuda_dev)).cpu().numpy()
    fin = np.isfinite(z["rec_out"])
    assert np.array_equal(bits(rec)[fin], bits(z["rec_out"])[fin])
    qm = Q.quantize_momentum(torch.from_numpy(z["qm_x"]).to(cuda_dev))
    assert np.array_equal(qm.codes.cpu().numpy(), z["qm_codes"])
    assert np.array_equal(bits(qm.scales.cpu().numpy()), bits(z["qm_scales"]))
    assert np.array_equal(bits(Q.dequantize_momentum(qm).cpu().numpy()), bits(z["qm_deq"]))
    qv = Q.quantize_variance(torch.from_numpy(z["qv_x"]).to(cuda_dev))
    assert np.array_equal(qv.codes.cpu().numpy(), z["qv_codes"])
    assert np.array_equal(bits(qv.scales.cpu().numpy()), bits(z["qv_scales"]))
    assert np.array_equal(bits(Q.dequantize_variance(qv).cpu().numpy()), bits(z["qv_deq"]))
