"""One tensor past 2^31 elements (64-bit offsets in every kernel path): a
FlashAdamW step over n = 2^31 + 777 elements on the device, checked against
the oracle on three 32-aligned windows -- the head, a window straddling
element 2^31, and the ragged tail (groups are independent, so a window
steps like a tensor of its own: SURVEY.md Appendix B probe 6).  ~15 GB of
HBM."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from devstate import mismatches, oracle_dict

pytestmark = pytest.mark.gpu

N = (1 << 31) + 777


def test_tensor_past_2_31_elements(cuda_dev, oracle_mod):
    from paper_2602_23349_b200 import optim as FO
    from paper_2602_23349_b200.formats import SplitTensor
    from paper_2602_23349_b200.quantize import GroupSpec, QuantizedState

    if torch.cuda.get_device_properties(cuda_dev).total_memory < 40 * 2**30:
        pytest.skip("needs ~15 GB of device memory")
    gen = torch.Generator(device=cuda_dev).manual_seed(31)
    ng = -(-N // 32)
    lp = (torch.randn(N, generator=gen, device=cuda_dev) * 0.02).to(torch.bfloat16)
    rho = torch.randint(-127, 128, (N,), generator=gen, device=cuda_dev, dtype=torch.int32).to(torch.int8)
    mq = torch.randint(-127, 128, (N,), generator=gen, device=cuda_dev, dtype=torch.int32).to(torch.int8)
    vq = torch.randint(0, 256, (N,), generator=gen, device=cuda_dev, dtype=torch.int32).to(torch.uint8)
    ms = (torch.rand(ng, generator=gen, device=cuda_dev) * 2e-3).half()
    vs = (torch.rand(ng, generator=gen, device=cuda_dev) * 2e-3).half()
    g = (torch.randn(N, generator=gen, device=cuda_dev) * 1e-3).to(torch.bfloat16)
    spec = GroupSpec(32)
    fs = FO.FlashState(SplitTensor(lp, rho), QuantizedState(mq, ms, spec, "momentum"),
                       QuantizedState(vq, vs, spec, "variance"), 500)
    windows = [(0, 1 << 20), ((1 << 31) - (1 << 19), (1 << 31) + (1 << 19)), (N - 100_000 + 7, N)]
    windows = [(a - a % 32, b) for a, b in windows]

    def grab(a, b):
        ga, gb = a // 32, -(-b // 32)
        return {"weights.lp": lp[a:b].view(torch.int16).cpu().numpy().view(np.uint16),
                "weights.rho": rho[a:b].cpu().numpy(), "momentum.codes": mq[a:b].cpu().numpy(),
                "momentum.scales": ms[ga:gb].cpu().numpy(), "variance.codes": vq[a:b].cpu().numpy(),
                "variance.scales": vs[ga:gb].cpu().numpy()}

    before = [grab(a, b) for a, b in windows]
    gwin = [g[a:b].float().cpu().numpy() for a, b in windows]
    hp = dict(lr=1e-5, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    FO.adamw_step_(fs, g, FO.AdamHyperParams(**hp))
    torch.cuda.synchronize()
    for (a, b), st0, gw in zip(windows, before, gwin):
        ost = oracle_mod.OracleState(st0["weights.lp"].copy(), st0["weights.rho"].copy(),
                                     st0["momentum.codes"].copy(), st0["momentum.scales"].copy(),
                                     st0["variance.codes"].copy(), st0["variance.scales"].copy(), 500)
        assert oracle_mod.step_inplace("adamw", ost, gw, **hp) == 0
        mm = mismatches(grab(a, b), oracle_dict(ost))
        assert all(v == 0 for v in mm.values()), ((a, b), mm)
