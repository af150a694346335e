"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of libflashoptim_b200.so on a few tensors,
with slices that trip the fast tile's guards (so the fix-up launch runs),
int16 corrections and linear variance on the fused kernel, the capturable
(device-scalar) instances, and the host streaming path with a group size
below 32.  Checks results
against the C oracle too, so a sanitizer run is also a parity run.

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import helpers as H  # noqa: E402
from devstate import from_device, mismatches, oracle_dict, oracle_state, to_device  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2602_23349_b200 import _lib, optim as FO  # noqa: E402
from paper_2602_23349_b200.host import HostFlashState, step_host  # noqa: E402

O.build()
dev = torch.device("cuda:0")
bad = 0
rng = np.random.default_rng(7)


def check(tag, got, ost):
    global bad
    mm = mismatches(got, oracle_dict(ost))
    if any(mm.values()):
        bad += 1
        print("MISMATCH", tag, mm)


for opt in ("adamw", "sgd", "lion"):
    hp = H.random_hparams(rng, opt)
    for n, G, rho_dt in ((20000 + 37, 32, np.int8), (9000, 32, np.int16), (5000, 64, np.int8)):
        st = H.random_state(rng, n, opt, G=G, rho=None if rho_dt == np.int8 else
                            rng.integers(-32767, 32768, n).astype(np.int16))
        g = H.random_grad(rng, n)
        fs = to_device(st, 5, dev, G)
        FO.STEP_FUNCTIONS_INPLACE[opt](fs, torch.from_numpy(g).to(dev).bfloat16(), FO.HP_TYPES[opt](**hp))
        ost = oracle_state(st, 5, G)
        assert O.step_inplace(opt, ost, g, **hp) == 0
        check(f"{opt} n={n} G={G} rho={rho_dt.__name__}", from_device(fs), ost)
    # host streaming path, G = 16, pieces straddling slots
    sts = [H.random_state(rng, n, opt, G=16) for n in (3000, 17, 5000)]
    gs = [H.random_grad(rng, n) for n in (3000, 17, 5000)]
    hs = [HostFlashState(s["weights.lp"].copy(), s["weights.rho"].copy(), s["momentum.codes"].copy(),
                         s["momentum.scales"].copy(), s.get("variance.codes", None) if opt != "adamw" else
                         s["variance.codes"].copy(), None if opt != "adamw" else s["variance.scales"].copy(), 2, 16)
          for s in sts]
    step_host(opt, hs, [(x.view(np.uint32) >> 16).astype(np.uint16) for x in gs], FO.HP_TYPES[opt](**hp),
              chunk_elems=2048)
    for s, h, g in zip(sts, hs, gs):
        ost = oracle_state(s, 2, 16)
        assert O.step_inplace(opt, ost, g, **hp) == 0
        d = {"weights.lp": h.lp, "weights.rho": h.rho, "momentum.codes": h.m_codes, "momentum.scales": h.m_scales}
        if opt == "adamw":
            d.update({"variance.codes": h.v_codes, "variance.scales": h.v_scales})
        check(f"host {opt} G=16", d, ost)
# linear variance on the fused kernel (int8 and int16 corrections)
for rho16 in (False, True):
    n = 12000 + 5
    st = H.random_state(rng, n, "adamw", rho=rng.integers(-32767, 32768, n).astype(np.int16) if rho16 else None)
    g = H.random_grad(rng, n)
    hp = H.random_hparams(rng, "adamw")
    fs = to_device(st, 5, dev, 32, "linear")
    FO.adamw_step_(fs, torch.from_numpy(g).to(dev).bfloat16(), FO.AdamHyperParams(**hp))
    ost = oracle_state(st, 5, 32, "linear")
    assert O.step_inplace("adamw", ost, g, **hp) == 0
    check(f"adamw linear rho16={rho16}", from_device(fs), ost)
# the capturable (device-scalar) kernels against the eager optimizer
import paper_2602_23349_b200.torch_optim as TO  # noqa: E402

for name in ("FlashAdamW", "FlashSGD", "FlashLion"):
    gen = torch.Generator().manual_seed(3)
    ps = [torch.nn.Parameter((torch.randn(n, generator=gen) * 0.02).to(dev)) for n in (5000, 70)]
    pe = [torch.nn.Parameter(p.detach().clone()) for p in ps]
    cap = getattr(TO, name)(ps, lr=1e-3, capturable=True)
    eag = getattr(TO, name)(pe, lr=1e-3)
    for _ in range(3):
        gs = [(torch.randn(p.numel(), generator=gen) * 1e-2).bfloat16().to(dev) for p in ps]
        for p, q, g in zip(ps, pe, gs):
            p.grad, q.grad = g.clone(), g.clone()
        cap.step()
        eag.step()
    torch.cuda.synchronize()
    for p, q in zip(ps, pe):
        if not torch.equal(p.data.view(torch.int16), q.data.view(torch.int16)):
            bad += 1
            print("MISMATCH capturable", name)
torch.cuda.synchronize()
f, s = _lib.fixup_stats(reset=True)
print(f"sanitize_driver: {bad} mismatching cases; fix-up slices {f} of {s}")
sys.exit(1 if bad else 0)
