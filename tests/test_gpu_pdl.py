"""The fused kernel is a programmatic dependent launch (fo_step_impl.cuh,
launch_pdl / griddep_wait): its CTAs may be scheduled while the previous
kernel on the stream drains, and must touch no global memory before that
kernel's results are visible.  Here the kernel right before the step either
writes the gradients the step reads (read after write) or reads the weights
the step overwrites (write after read); a sleep kernel in front keeps the
launches queued, so the programmatic edge is the one in use.  Results must
equal the oracle bit for bit, as with a plain launch."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import helpers as H
from devstate import from_device, mismatches, oracle_dict, oracle_state, to_device

pytestmark = pytest.mark.gpu

OPTS = ["adamw", "sgd", "lion"]
N = 4 * 1024 * 1024 + 37


def _setup(opt, seed, dev):
    """State, gradient and hyper-parameters, plus a step launcher whose
    launch is the only work it queues (error word allocated up front, the
    stream's fix-up bitmap grown by one warm-up step on a copy)."""
    from paper_2602_23349_b200 import optim as FO
    from paper_2602_23349_b200._errors import DeviceErrors

    rng = np.random.default_rng(seed)
    st = H.random_state(rng, N, opt)
    g = H.random_grad(rng, N)
    hp = FO.HP_TYPES[opt](**H.random_hparams(rng, opt))
    err = DeviceErrors(dev)
    warm = to_device(st, 5, dev)
    FO.step_many(opt, [warm], [torch.zeros(N, dtype=torch.bfloat16, device=dev)], hp, errors=err)
    torch.cuda.synchronize()
    err.reset()
    torch.cuda.synchronize()

    def step(fs, grad):
        FO.step_many(opt, [fs], [grad], hp, errors=err)

    return st, g, hp, to_device(st, 5, dev), step, err


def _check(fs, st, g, hp, opt, oracle_mod, err):
    got = from_device(fs)
    assert err.mask() == 0
    ost = oracle_state(st, 5)
    assert oracle_mod.step_inplace(opt, ost, g, **vars(hp)) == 0
    mm = mismatches(got, oracle_dict(ost))
    assert not any(mm.values()), mm


@pytest.mark.parametrize("opt", OPTS)
def test_grads_written_by_the_previous_kernel(opt, cuda_dev, oracle_mod):
    st, g, hp, fs, step, err = _setup(opt, 401 + OPTS.index(opt), cuda_dev)
    src = torch.from_numpy(g).to(cuda_dev).to(torch.bfloat16)
    grad = torch.zeros_like(src)  # stale contents a racing step would read
    torch.cuda.synchronize()
    torch.cuda._sleep(20_000_000)  # the copy and the step queue behind this
    grad.copy_(src)  # the step's immediate predecessor writes its input
    step(fs, grad)
    _check(fs, st, g, hp, opt, oracle_mod, err)


@pytest.mark.parametrize("opt", OPTS)
def test_weights_read_by_the_previous_kernel(opt, cuda_dev, oracle_mod):
    st, g, hp, fs, step, err = _setup(opt, 501 + OPTS.index(opt), cuda_dev)
    grad = torch.from_numpy(g).to(cuda_dev).to(torch.bfloat16)
    lp = fs.weights.lp_values
    want = torch.sum(lp, dtype=torch.float32).item()  # the same reduction, stream idle
    torch.cuda.synchronize()
    torch.cuda._sleep(20_000_000)
    got_sum = torch.sum(lp, dtype=torch.float32)  # the step's immediate predecessor reads what it overwrites
    step(fs, grad)
    assert got_sum.item() == want
    _check(fs, st, g, hp, opt, oracle_mod, err)
