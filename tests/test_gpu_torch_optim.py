"""GPU: torch.optim classes, state_dict, FLOP v1 optimizer checkpoints,
gradient release and the ZeRO-1 optimizer on one NCCL rank -- all bitwise
against the C oracle / each other."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import helpers as H
from devstate import bits, mismatches, oracle_dict

pytestmark = pytest.mark.gpu

OPTS = {"adamw": ("FlashAdamW", dict(lr=1e-3, betas=(0.9, 0.95), weight_decay=0.1),
                  dict(lr=1e-3, beta1=0.9, beta2=0.95, weight_decay=0.1)),
        "sgd": ("FlashSGD", dict(lr=0.05, momentum=0.9, weight_decay=1e-4),
                dict(lr=0.05, momentum=0.9, weight_decay=1e-4)),
        "lion": ("FlashLion", dict(lr=1e-4, betas=(0.9, 0.99), weight_decay=0.1),
                 dict(lr=1e-4, beta1=0.9, beta2=0.99, weight_decay=0.1))}


def _model(seed=0, dtype=torch.float32):
    torch.manual_seed(seed)
    m = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.GELU(), torch.nn.Linear(256, 64),
                            torch.nn.LayerNorm(64), torch.nn.Linear(64, 10))
    return m.to("cuda", dtype)


def _state_dict_np(opt, p) -> dict:
    st = opt.state[p]
    d = {"weights.lp": p.detach().reshape(-1).view(torch.int16).cpu().numpy().view(np.uint16),
         "weights.rho": st["weights.rho"].reshape(-1).cpu().numpy(),
         "momentum.codes": st["momentum.codes"].reshape(-1).cpu().numpy(),
         "momentum.scales": st["momentum.scales"].cpu().numpy()}
    if "variance.codes" in st:
        d["variance.codes"] = st["variance.codes"].reshape(-1).cpu().numpy()
        d["variance.scales"] = st["variance.scales"].cpu().numpy()
    return d


@pytest.mark.parametrize("name", ["adamw", "sgd", "lion"])
def test_torch_optimizer_matches_oracle(name, cuda_dev, oracle_mod):
    """fp32 model -> init_flash_state split -> 3 fused steps == oracle."""
    import paper_2602_23349_b200.torch_optim as TO

    cls, kw, okw = OPTS[name]
    model = _model()
    theta0 = [p.detach().reshape(-1).cpu().numpy().copy() for p in model.parameters()]
    opt = getattr(TO, cls)(model.parameters(), **kw)
    assert all(p.dtype == torch.bfloat16 for p in model.parameters())
    ost = [oracle_mod.init_state(t, name) for t in theta0]
    x = torch.randn(32, 64, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        opt.zero_grad()
        model(x).float().square().mean().backward()
        grads = [p.grad.detach().float().reshape(-1).cpu().numpy() for p in model.parameters()]
        opt.step()
        for st, g in zip(ost, grads):
            assert oracle_mod.step_inplace(name, st, g, **okw) == 0
    for p, st in zip(model.parameters(), ost):
        mm = mismatches(_state_dict_np(opt, p), oracle_dict(st))
        assert all(v == 0 for v in mm.values()), mm
        assert opt.state[p]["step"] == 3


def test_state_dict_roundtrip_is_bitwise(cuda_dev):
    import paper_2602_23349_b200.torch_optim as TO

    model = _model(1)
    opt = TO.FlashAdamW(model.parameters(), lr=1e-3)
    x = torch.randn(8, 64, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        opt.zero_grad()
        model(x).float().sum().backward()
        opt.step()
    sd = opt.state_dict()
    model2 = _model(2)
    with torch.no_grad():
        for a, b in zip(model2.parameters(), model.parameters()):
            a.data = b.detach().clone()
    opt2 = TO.FlashAdamW(model2.parameters(), lr=1e-3)
    opt2.load_state_dict(sd)
    for p, q in zip(model.parameters(), model2.parameters()):
        a, b = _state_dict_np(opt, p), _state_dict_np(opt2, q)
        assert all(np.array_equal(bits(a[k]), bits(b[k])) for k in a)
        assert opt2.state[q]["momentum.scales"].dtype == torch.float16
    # both continue identically
    for o, m in ((opt, model), (opt2, model2)):
        o.zero_grad()
        m(x).float().sum().backward()
        o.step()
    for p, q in zip(model.parameters(), model2.parameters()):
        assert torch.equal(p.view(torch.int16), q.view(torch.int16))


def test_optimizer_checkpoint_roundtrip(cuda_dev, tmp_path):
    import paper_2602_23349_b200.torch_optim as TO
    from paper_2602_23349_b200 import checkpoint as C

    model = _model(3)
    opt = TO.FlashLion(model.parameters(), lr=1e-4)
    x = torch.randn(8, 64, device="cuda", dtype=torch.bfloat16)
    opt.zero_grad()
    model(x).float().sum().backward()
    opt.step()
    man = C.save_optimizer(opt, tmp_path / "ck")
    assert man["optimizer"] == "lion" and len(man["params"]) == len(list(model.parameters()))
    model2 = _model(4)
    opt2 = TO.FlashLion(model2.parameters(), lr=1e-4)
    C.load_optimizer(opt2, tmp_path / "ck")
    for p, q in zip(model.parameters(), model2.parameters()):
        a, b = _state_dict_np(opt, p), _state_dict_np(opt2, q)
        assert all(np.array_equal(bits(a[k]), bits(b[k])) for k in a)
    assert C.inspect_checkpoint(tmp_path / "ck" / "00000.flop")["optimizer"] == "lion"


@pytest.mark.parametrize("name", ["adamw", "sgd", "lion"])
def test_gradient_release_equals_deferred_step(name, cuda_dev):
    """stepping from backward hooks == stepping after backward, bitwise."""
    import paper_2602_23349_b200.torch_optim as TO
    from paper_2602_23349_b200.release import GradientRelease

    cls, kw, _ = OPTS[name]
    ma, mb = _model(5), _model(5)
    oa = getattr(TO, cls)(ma.parameters(), **kw)
    ob = getattr(TO, cls)(mb.parameters(), **kw)
    rel = GradientRelease(ob)
    torch.manual_seed(7)
    xs = [torch.randn(16, 64, device="cuda", dtype=torch.bfloat16) for _ in range(4)]
    for x in xs:
        oa.zero_grad()
        ma(x).float().square().mean().backward()
        oa.step()
        mb(x).float().square().mean().backward()  # steps happen inside backward
        assert all(p.grad is None for p in mb.parameters())
    rel.check()
    assert rel.steps_launched == 4 * len(list(mb.parameters()))
    for p, q in zip(ma.parameters(), mb.parameters()):
        a, b = _state_dict_np(oa, p), _state_dict_np(ob, q)
        assert all(np.array_equal(bits(a[k]), bits(b[k])) for k in a), name


def test_gradient_release_with_tied_weights(cuda_dev):
    """GPT-2 style tied embedding / head: one parameter, one hook, one step."""
    import paper_2602_23349_b200.torch_optim as TO
    from paper_2602_23349_b200.release import GradientRelease

    def make():
        torch.manual_seed(11)
        emb = torch.nn.Embedding(100, 32).cuda()
        return emb

    ea, eb = make(), make()
    oa = TO.FlashAdamW(ea.parameters(), lr=1e-3)
    ob = TO.FlashAdamW(eb.parameters(), lr=1e-3)
    rel = GradientRelease(ob)
    ids = torch.randint(0, 100, (4, 7), device="cuda")
    for e, o in ((ea, oa), (eb, None)):
        h = e(ids)
        logits = h @ e.weight.t()  # tied head
        logits.float().logsumexp(-1).mean().backward()
        if o is not None:
            o.step()
    rel.check()
    assert rel.steps_launched == 1
    assert torch.equal(ea.weight.view(torch.int16), eb.weight.view(torch.int16))


def test_zero1_single_rank_nccl_matches_oracle(cuda_dev, oracle_mod):
    import os

    import torch.distributed as dist

    from paper_2602_23349_b200 import optim as FO
    from paper_2602_23349_b200.zero import ZeroFlashOptimizer

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        torch.manual_seed(0)
        params = [(torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16) for n in (1000, 4103, 33, 70000)]
        ost = []
        for p in params:
            lp = p.view(torch.int16).cpu().numpy().view(np.uint16).copy()
            n, ng = lp.size, -(-lp.size // 32)
            ost.append(oracle_mod.OracleState(lp, np.zeros(n, np.int8), np.zeros(n, np.int8), np.zeros(ng, np.float16),
                                              np.zeros(n, np.uint8), np.zeros(ng, np.float16), 0))
        hp = FO.AdamHyperParams(lr=1e-3, beta2=0.95, weight_decay=0.1)
        zo = ZeroFlashOptimizer(params, "adamw", [hp], reduce_op="sum")
        for s in range(3):
            zo.zero_grad()
            gs = [(torch.randn(p.numel(), device="cuda") * 1e-3).to(torch.bfloat16) for p in params]
            for p, g in zip(params, gs):
                p.grad.copy_(g)
            zo.step()
            for st, g in zip(ost, gs):
                assert oracle_mod.step_inplace("adamw", st, g.float().cpu().numpy(),
                                               lr=1e-3, beta2=0.95, weight_decay=0.1) == 0
        torch.cuda.synchronize()
        for p, st in zip(params, ost):
            assert np.array_equal(p.view(torch.int16).cpu().numpy().view(np.uint16), st.lp)
        # sharded checkpoint over NCCL: files byte-identical to the oracle state's, reload bit for bit
        import tempfile

        from paper_2602_23349_b200.checkpoint import save_checkpoint
        from paper_2602_23349_b200.host import HostFlashState

        with tempfile.TemporaryDirectory() as d:
            zo.save_checkpoint(d)
            for i, st in enumerate(ost):
                ref = os.path.join(d, f"ref{i}.flop")
                save_checkpoint(HostFlashState(st.lp, st.rho, st.m_codes, st.m_scales, st.v_codes, st.v_scales,
                                               st.t, 32), ref, "adamw")
                with open(ref, "rb") as f1, open(os.path.join(d, f"{i:05d}.flop"), "rb") as f2:
                    assert f1.read() == f2.read(), i
            fresh = [torch.zeros_like(p) for p in params]
            z2 = ZeroFlashOptimizer(fresh, "adamw", [hp], reduce_op="sum")
            z2.load_checkpoint(d)
            assert torch.equal(z2.flat_params.view(torch.int16), zo.flat_params.view(torch.int16))
            for a, b in zip(zo.states, z2.states):
                assert torch.equal(a.weights.corrections, b.weights.corrections)
                assert torch.equal(a.momentum.codes, b.momentum.codes)
                assert torch.equal(a.variance.codes, b.variance.codes)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["sync", "deferred", "off"])
def test_error_policies(mode, cuda_dev):
    """check_errors: "sync" raises inside the failing step; "deferred" (the
    default) never blocks and raises from a later step() or raise_errors();
    "off" only from raise_errors().  The message is the reference's."""
    import paper_2602_23349_b200.torch_optim as TO

    p = torch.nn.Parameter(torch.randn(4096, device="cuda", dtype=torch.bfloat16))
    opt = TO.FlashAdamW([p], lr=1e-3, check_errors=mode)
    p.grad = torch.full_like(p, float("nan"))
    if mode == "sync":
        with pytest.raises(ValueError, match="gradient-nonfinite"):
            opt.step()
        return
    opt.step()  # queued; nothing blocks
    p.grad = torch.zeros_like(p)
    if mode == "deferred":
        torch.cuda.synchronize()
        with pytest.raises(ValueError, match="gradient-nonfinite"):
            opt.step()
    else:
        opt.step()
        with pytest.raises(ValueError, match="gradient-nonfinite"):
            opt.raise_errors()
    opt.raise_errors()  # cleared after being reported


def test_default_step_does_not_sync(cuda_dev):
    """The default policy issues no blocking device-to-host read: a step is
    enqueued while the device is still busy with earlier work."""
    import paper_2602_23349_b200.torch_optim as TO

    p = torch.nn.Parameter(torch.randn(1 << 20, device="cuda", dtype=torch.bfloat16))
    opt = TO.FlashAdamW([p], lr=1e-3)
    p.grad = torch.randn_like(p) * 1e-3
    opt.step()
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)  # ~0.1 s of device work ahead of the step
    done = torch.cuda.Event()
    opt.step()
    done.record()
    assert not done.query()  # step() returned before the queued work finished
    torch.cuda.synchronize()
    opt.raise_errors()


def test_int16_checkpoint_layout_in_torch_optimizer(cuda_dev, oracle_mod, tmp_path):
    """A state loaded with int16 corrections (INT16_CORRECTION checkpoint) is
    stepped with the int16 layout; a group-size mismatch is refused."""
    import paper_2602_23349_b200.torch_optim as TO

    rng = np.random.default_rng(3)
    n = 5000
    st = H.random_state(rng, n, "adamw", rho=rng.integers(-32767, 32768, n).astype(np.int16))
    p = torch.nn.Parameter(torch.from_numpy(st["weights.lp"].view(np.int16)).cuda().view(torch.bfloat16))
    opt = TO.FlashAdamW([p], lr=1e-3, betas=(0.9, 0.95), weight_decay=0.1, check_errors=True)
    sd = opt.state_dict()
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    sd["state"][0].update({"weights.rho": T(st["weights.rho"]), "momentum.codes": T(st["momentum.codes"]),
                           "momentum.scales": T(st["momentum.scales"]).view(torch.int16),
                           "variance.codes": T(st["variance.codes"]),
                           "variance.scales": T(st["variance.scales"]).view(torch.int16), "step": 7})
    opt.load_state_dict(sd)
    g = H.random_grad(rng, n)
    p.grad = torch.from_numpy(g).cuda().to(torch.bfloat16)
    opt.step()
    from devstate import oracle_state

    ost = oracle_state(st, 7)
    assert oracle_mod.step_inplace("adamw", ost, g, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                                   weight_decay=0.1) == 0
    mm = mismatches(_state_dict_np(opt, p), oracle_dict(ost))
    assert all(v == 0 for v in mm.values()), mm
    opt2 = TO.FlashAdamW([torch.nn.Parameter(p.detach().clone())], lr=1e-3, group_size=64)
    with pytest.raises(ValueError, match="group size"):
        opt2.load_state_dict(opt.state_dict())


@pytest.mark.parametrize("name", ["adamw", "sgd", "lion"])
@pytest.mark.parametrize("bucket", [0, 5000, 1 << 22])
def test_gradient_release_matches_oracle(name, bucket, cuda_dev, oracle_mod):
    """Gradient release (steps launched from backward hooks, one fused launch
    per bucket) against the C oracle directly: fp32 init split, three
    backward passes, every parameter's state bitwise equal."""
    import paper_2602_23349_b200.torch_optim as TO
    from paper_2602_23349_b200.release import GradientRelease

    cls, kw, okw = OPTS[name]
    model = _model(9)
    theta0 = [p.detach().reshape(-1).cpu().numpy().copy() for p in model.parameters()]
    opt = getattr(TO, cls)(model.parameters(), **kw)
    params = list(model.parameters())
    index = {id(p): i for i, p in enumerate(params)}
    captured: dict = {}
    for p in params:  # registered before GradientRelease's hooks, so it sees each gradient first
        p.register_post_accumulate_grad_hook(
            lambda p: captured.__setitem__(index[id(p)], p.grad.detach().float().reshape(-1).cpu().numpy()))
    rel = GradientRelease(opt, bucket_elems=bucket, timing=True)
    ost = [oracle_mod.init_state(t, name) for t in theta0]
    torch.manual_seed(3)
    for _ in range(3):
        captured.clear()
        x = torch.randn(16, 64, device="cuda", dtype=torch.bfloat16)
        model(x).float().square().mean().backward()
        assert len(captured) == len(params)
        for i, st in enumerate(ost):
            assert oracle_mod.step_inplace(name, st, captured[i], **okw) == 0
    rel.check()
    assert rel.side_stream_ms() > 0
    if bucket == 1 << 22:
        assert rel.launch_calls == 3  # the whole model in one fused launch per backward
    elif bucket == 0:
        assert rel.launch_calls == 3 * len(params)
    for p, st in zip(params, ost):
        got = _state_dict_np(opt, p)
        mm = mismatches(got, oracle_dict(st))
        assert all(v == 0 for v in mm.values()), (name, mm)
