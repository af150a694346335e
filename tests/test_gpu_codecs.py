"""GPU codec parity: split / reconstruct / (de)quantize vs the C oracle."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import helpers as H

pytestmark = pytest.mark.gpu


def test_reconstruct_exhaustive_codes(cuda_dev, oracle_mod):
    """Every bf16 code x every valid int8 correction (16.7M pairs)."""
    from paper_2602_23349_b200 import formats as F

    codes = np.repeat(np.arange(65536, dtype=np.uint32), 255).astype(np.uint16)
    rho = np.tile(np.arange(-127, 128, dtype=np.int16), 65536).astype(np.int8)
    ref = oracle_mod.reconstruct(codes, rho)
    lp = torch.from_numpy(codes.view(np.int16)).to(cuda_dev).view(torch.bfloat16)
    got = F.reconstruct(lp, torch.from_numpy(rho).to(cuda_dev)).cpu().numpy()
    fin = np.isfinite(ref)
    assert np.array_equal(got.view(np.uint32)[fin], ref.view(np.uint32)[fin])
    assert np.array_equal(np.isinf(got), np.isinf(ref)) and np.array_equal(np.isnan(got), np.isnan(ref))


def test_split_random_bit_patterns(cuda_dev, oracle_mod):
    """2^24 random finite f32 bit patterns plus weight-like values."""
    from paper_2602_23349_b200 import formats as F

    rng = np.random.default_rng(0)
    u = rng.integers(0, 2**32, size=1 << 24, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    x = x[np.isfinite(x)]
    x = np.concatenate([x, H.random_weights(rng, 1 << 20), np.array([0.0, -0.0, 1.00390625, 1.001953125,
                                                                      3.3895314e38, -3.3895314e38], np.float32)])
    for bits in (8, 16):
        lp_ref, rho_ref = oracle_mod.split(x, bits)
        lp, rho = F.split(torch.from_numpy(x).to(cuda_dev), F.INT8_CORRECTION if bits == 8 else F.INT16_CORRECTION)
        assert np.array_equal(lp.view(torch.int16).cpu().numpy().view(np.uint16), lp_ref)
        assert np.array_equal(rho.cpu().numpy(), rho_ref)


def test_split_rejects_nonfinite(cuda_dev):
    from paper_2602_23349_b200 import formats as F

    with pytest.raises(ValueError, match="split-nonfinite"):
        F.split(torch.tensor([1.0, float("inf")], device=cuda_dev))


def test_known_answers(cuda_dev):
    """tests/test_formats.py:169-180, :222-246 known-answer vectors."""
    from paper_2602_23349_b200 import formats as F

    lp, rho = F.split(torch.tensor([1.00390625, 1.0, 1.001953125], device=cuda_dev))
    assert lp.float().tolist() == [1.0, 1.0, 1.0]
    assert rho.tolist() == [127, 0, 64]
    rec = F.reconstruct(torch.tensor([0x3F80, 0x3F80, 0x7F80], dtype=torch.int16, device=cuda_dev).view(
        torch.bfloat16), torch.tensor([127, 64, 93], dtype=torch.int8, device=cuda_dev)).cpu().numpy()
    assert rec[0] == np.float32(1.00390625)
    assert rec[1] == np.float32(1.0) + np.float32((np.float32(64) / np.float32(127)) * np.float32(2.0 ** -8))
    assert np.isposinf(rec[2])
    with pytest.raises(ValueError, match="invalid-correction-code"):
        F.reconstruct(torch.tensor([0x3F80], dtype=torch.int16, device=cuda_dev).view(torch.bfloat16),
                      torch.tensor([-128], dtype=torch.int8, device=cuda_dev))


@pytest.mark.parametrize("G", [4, 32, 33])
def test_quantize_roundtrip_vs_oracle(G, cuda_dev, oracle_mod):
    from paper_2602_23349_b200 import quantize as Q

    rng = np.random.default_rng(G)
    x = (rng.standard_normal(100_003) * 10.0 ** rng.integers(-30, 4, 100_003)).astype(np.float32)
    x[:64] = 0.0
    spec = Q.GroupSpec(G)
    qm = Q.quantize_momentum(torch.from_numpy(x).to(cuda_dev), spec)
    c_ref, s_ref = oracle_mod.quantize_momentum(x, G)
    assert np.array_equal(qm.codes.cpu().numpy(), c_ref)
    assert np.array_equal(qm.scales.cpu().numpy().view(np.uint16), s_ref.view(np.uint16))
    dm = Q.dequantize_momentum(qm).cpu().numpy()
    assert np.array_equal(dm.view(np.uint32), oracle_mod.dequantize_momentum(c_ref, s_ref, G).view(np.uint32))
    v = x * x
    qv = Q.quantize_variance(torch.from_numpy(v).to(cuda_dev), spec)
    c_ref, s_ref = oracle_mod.quantize_variance(v, G)
    assert np.array_equal(qv.codes.cpu().numpy(), c_ref)
    assert np.array_equal(qv.scales.cpu().numpy().view(np.uint16), s_ref.view(np.uint16))
    dv = Q.dequantize_variance(qv).cpu().numpy()
    assert np.array_equal(dv.view(np.uint32), oracle_mod.dequantize_variance(c_ref, s_ref, G).view(np.uint32))


def test_quantize_known_answers(cuda_dev):
    """tests/test_quantize.py:20-25, :80-86, :120-125, :167-171."""
    from paper_2602_23349_b200 import quantize as Q

    q = Q.quantize_momentum(torch.tensor([0.5, -1.0, 0.25, 0.0], device=cuda_dev), Q.GroupSpec(4))
    assert q.scales.tolist() == [1.0] and q.codes.tolist() == [85, -127, 51, 0]
    q = Q.quantize_variance(torch.tensor([4.0, 1.0, 0.25, 0.0], device=cuda_dev), Q.GroupSpec(4))
    assert q.scales.tolist() == [2.0] and q.codes.tolist() == [255, 128, 64, 0]
    q = Q.quantize_variance(torch.tensor([0.25, 0.01, 16.0, 4.0], device=cuda_dev), Q.GroupSpec(2))
    assert q.scales.tolist() == [0.5, 4.0]
    x = torch.ones(33, device=cuda_dev)
    x[32] = 0.25
    assert Q.quantize_momentum(x).scales.tolist() == [1.0, 0.25]
    with pytest.raises(ValueError, match="scale-overflow"):
        Q.quantize_momentum(torch.tensor([65505.0], device=cuda_dev), Q.GroupSpec(1))
    with pytest.raises(ValueError, match="quantize-nonfinite"):
        Q.quantize_momentum(torch.tensor([1.0, float("nan")], device=cuda_dev))


def test_scale_round_up_all_fp16_boundaries(cuda_dev, oracle_mod):
    """fp16 round-up scales at every fp16 value and its f32 neighbours."""
    from paper_2602_23349_b200 import quantize as Q

    h = np.arange(0, 0x7BFF + 1, dtype=np.uint16).view(np.float16).astype(np.float32)
    x = np.concatenate([h, np.nextafter(h, np.float32(np.inf)), np.nextafter(h, np.float32(0))])
    x = x[x <= 65504.0]
    q = Q.quantize_momentum(torch.from_numpy(x).to(cuda_dev), Q.GroupSpec(1))
    _, s_ref = oracle_mod.quantize_momentum(x, 1)
    assert np.array_equal(q.scales.cpu().numpy().view(np.uint16), s_ref.view(np.uint16))
