"""capturable=True: optimizer.step() captured into a CUDA graph and replayed
gives the same bytes as the eager optimizer stepping the same gradients
(fo_step_mt_dev: step counter, bias corrections and lr read from device
memory at run time; optim.py:208-258)."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu

SIZES = [1000, 32 * 1024 + 7, 8192 * 3 + 100, 77]


def _params(dev, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return [torch.nn.Parameter((torch.randn(n, generator=g) * 0.02).to(dev)) for n in SIZES]


def _make(cls, params, **kw):
    return cls(params, **kw)


def _state_bytes(opt, params):
    out = [p.data.view(torch.int16).clone() for p in params]
    for p in params:
        st = opt.state[p]
        for k in ("weights.rho", "momentum.codes", "momentum.scales", "variance.codes", "variance.scales"):
            if k in st:
                out.append(st[k].view(torch.uint8 if st[k].element_size() == 1 else torch.int16).clone())
    return out


def _same(a, b):
    return all(torch.equal(x, y) for x, y in zip(a, b))


CASES = [
    ("FlashAdamW", dict(lr=1e-3, betas=(0.5, 0.6), eps=1e-8, weight_decay=0.1)),  # bias corrections reach 1.0f at t ~ 40
    ("FlashAdamW", dict(lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)),
    ("FlashSGD", dict(lr=0.05, momentum=0.9, weight_decay=1e-4)),
    ("FlashLion", dict(lr=1e-4, betas=(0.9, 0.99), weight_decay=0.1)),
]


@pytest.mark.parametrize("name,kw", CASES)
def test_graph_replay_matches_eager(name, kw, cuda_dev):
    import paper_2602_23349_b200.torch_optim as P

    cls = getattr(P, name)
    pe, pc = _params(cuda_dev, 1), _params(cuda_dev, 1)
    eager = _make(cls, pe, **kw)
    cap = _make(cls, pc, capturable=True, **kw)
    static = [torch.zeros(n, dtype=torch.bfloat16, device=cuda_dev) for n in SIZES]
    for p, g in zip(pc, static):
        p.grad = g
    gen = torch.Generator(device=cuda_dev).manual_seed(7)

    def new_grads():
        return [(torch.randn(n, device=cuda_dev, generator=gen) * 1e-2).bfloat16() for n in SIZES]

    # warm-up steps on a side stream (torch's capture recipe), then capture one step
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            gs = new_grads()
            for x, g in zip(static, gs):
                x.copy_(g)
            cap.step()
            for p, g in zip(pe, gs):
                p.grad = g.clone()
            eager.step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    assert _same(_state_bytes(cap, pc), _state_bytes(eager, pe))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        cap.step()
    for it in range(45):
        gs = new_grads()
        for x, g in zip(static, gs):
            x.copy_(g)
        graph.replay()
        for p, g in zip(pe, gs):
            p.grad = g.clone()
        eager.step()
        torch.cuda.synchronize()
        assert _same(_state_bytes(cap, pc), _state_bytes(eager, pe)), it
    assert int(cap.state[pc[0]]["step"]) == int(eager.state[pe[0]]["step"]) == 48
    cap.raise_errors()


def test_device_lr_follows_schedule(cuda_dev):
    """A CUDA-tensor lr is read when the graph runs: a schedule written into it
    between replays matches the eager optimizer with the same float lr."""
    import paper_2602_23349_b200.torch_optim as P

    pe, pc = _params(cuda_dev, 2), _params(cuda_dev, 2)
    lr_t = torch.tensor(1e-3, dtype=torch.float32, device=cuda_dev)
    eager = P.FlashAdamW(pe, lr=1e-3, betas=(0.9, 0.95), weight_decay=0.1)
    cap = P.FlashAdamW(pc, lr=lr_t, betas=(0.9, 0.95), weight_decay=0.1, capturable=True)
    static = [torch.zeros(n, dtype=torch.bfloat16, device=cuda_dev) for n in SIZES]
    for p, g in zip(pc, static):
        p.grad = g
    gen = torch.Generator(device=cuda_dev).manual_seed(11)
    cap.step()  # warm-up (zero gradients) on both
    for p in pe:
        p.grad = torch.zeros_like(p, dtype=torch.bfloat16)
    eager.step()
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(graph, stream=s):
        cap.step()
    torch.cuda.current_stream().wait_stream(s)
    for it in range(10):
        lr = 1e-3 * (0.7 ** it)
        lr_t.fill_(lr)
        gs = [(torch.randn(n, device=cuda_dev, generator=gen) * 1e-2).bfloat16() for n in SIZES]
        for x, g in zip(static, gs):
            x.copy_(g)
        graph.replay()
        for grp in eager.param_groups:
            grp["lr"] = float(torch.tensor(lr, dtype=torch.float32))
        for p, g in zip(pe, gs):
            p.grad = g.clone()
        eager.step()
        torch.cuda.synchronize()
        assert _same(_state_bytes(cap, pc), _state_bytes(eager, pe)), it


def test_capturable_state_dict_round_trip(cuda_dev):
    import paper_2602_23349_b200.torch_optim as P

    pc = _params(cuda_dev, 3)
    cap = P.FlashAdamW(pc, lr=1e-3, capturable=True)
    for p in pc:
        p.grad = (torch.randn_like(p) * 1e-2).bfloat16()
    for _ in range(3):
        cap.step()
    sd = cap.state_dict()
    pc2 = [torch.nn.Parameter(p.detach().clone()) for p in pc]
    cap2 = P.FlashAdamW(pc2, lr=1e-3, capturable=True)
    cap2.load_state_dict(sd)
    assert int(cap2.state[pc2[0]]["step"]) == 3
    assert cap2.state[pc2[0]]["step"] is cap2.state[pc2[1]]["step"]  # one device counter per group
    for p, q in zip(pc, pc2):
        q.grad = p.grad.clone()
    cap.step()
    cap2.step()
    torch.cuda.synchronize()
    assert _same(_state_bytes(cap, pc), _state_bytes(cap2, pc2))


def test_capturable_flop_checkpoint_round_trip(cuda_dev, tmp_path):
    """checkpoint.save_optimizer / load_optimizer into a capturable optimizer:
    the loaded state gets one device counter per group and fresh launch
    tables, and steps on bitwise like the original."""
    import paper_2602_23349_b200.torch_optim as P
    from paper_2602_23349_b200 import checkpoint

    pc = _params(cuda_dev, 4)
    cap = P.FlashAdamW(pc, lr=1e-3, betas=(0.9, 0.95), capturable=True)
    for p in pc:
        p.grad = (torch.randn_like(p, dtype=torch.float32) * 1e-2).bfloat16()
    for _ in range(4):
        cap.step()
    checkpoint.save_optimizer(cap, str(tmp_path))
    pc2 = [torch.nn.Parameter(torch.zeros(n, device=cuda_dev)) for n in SIZES]
    cap2 = P.FlashAdamW(pc2, lr=1e-3, betas=(0.9, 0.95), capturable=True)
    checkpoint.load_optimizer(cap2, str(tmp_path))
    assert int(cap2.state[pc2[0]]["step"]) == 4
    assert cap2.state[pc2[0]]["step"] is cap2.state[pc2[-1]]["step"]
    for p, q in zip(pc, pc2):
        q.grad = p.grad.clone()
    cap.step()
    cap2.step()
    torch.cuda.synchronize()
    assert _same(_state_bytes(cap, pc), _state_bytes(cap2, pc2))


def test_release_refuses_capturable(cuda_dev):
    import paper_2602_23349_b200.torch_optim as P
    from paper_2602_23349_b200.release import GradientRelease

    opt = P.FlashSGD(_params(cuda_dev, 5), lr=0.1, capturable=True)
    with pytest.raises(ValueError, match="capturable"):
        GradientRelease(opt)
