"""GPU: the three BASELINE.json parameter lists stepped by the product path
(flat.StepPlan, the fused multi-tensor launch) and checked against the C
oracle on 64 seeded windows of up to 2^20 elements spread over every tensor
of the list (interior windows and tensor tails), plus the fast-path share.
The same check runs inside bench.py after its timed region (`parity`)."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu

LISTS = [("resnet50", "sgd"), ("resnet50", "lion"), ("gpt2_medium", "adamw"), ("llama31_8b", "adamw")]


@pytest.mark.parametrize("config,opt", LISTS)
def test_list_windows_match_oracle(config, opt, cuda_dev, oracle_mod):
    import bench
    from paper_2602_23349_b200 import _lib
    from paper_2602_23349_b200 import shapes as S
    from paper_2602_23349_b200.flat import FlatStates, StepPlan
    from paper_2602_23349_b200.optim import HP_TYPES

    sizes = [S.numel(s) for _, s in S.CONFIGS[config]()]
    fl = FlatStates(sizes, opt, cuda_dev)
    grads_flat = torch.empty(fl.total, dtype=torch.bfloat16, device=cuda_dev)
    bench.init_random_state(fl, grads_flat, 4321)
    grads = [grads_flat[o:o + n] for o, n in zip(fl.offsets, fl.sizes)]
    plan = StepPlan(opt, fl.states)
    plan.set_grads(grads)
    for st in fl.states:
        st.t = 1000 if config == "llama31_8b" else 10  # steady state and early training instances
    hpd = bench.hparams_for(config, opt)
    hp = HP_TYPES[opt](**hpd)
    err = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
    sh = torch.cuda.current_stream().cuda_stream

    def one_step():
        plan.launch([hp.scalars(fl.states[0].t + 1)], err.data_ptr(), sh)

    one_step()  # a first step from the random state
    _lib.fixup_stats(sh, reset=True)
    wins = bench.choose_windows(fl.sizes, 64, 1 << 20, 7)
    res = bench.parity_check(fl.states, grads, wins, opt, hpd, one_step)
    flagged, slices = _lib.fixup_stats(sh, reset=True)
    assert int(err.item()) == 0
    assert res["windows"] == min(64, len(sizes))
    assert res["total_mismatches"] == 0, res
    assert slices > 0 and flagged <= 0.001 * slices, (flagged, slices)
    del fl, grads_flat, grads, plan
    torch.cuda.empty_cache()
