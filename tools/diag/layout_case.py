"""Re-run one test_gpu_layouts case and print where the device and the
oracle differ (diagnostic)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
import helpers as H
from devstate import from_device, oracle_dict, oracle_state, to_device
from oracle import oracle as O
from paper_2602_23349_b200 import optim as FO, _lib

n, rb, scheme, seed = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
rng = np.random.default_rng(seed)
st = H.random_state(rng, n, "adamw")
if rb == 16:
    st["weights.rho"] = rng.integers(-32767, 32768, n).astype(np.int16)
g = H.random_grad(rng, n, std=float(10 ** rng.uniform(-5, -1)))
hp = H.random_hparams(rng, "adamw")
t = int(rng.integers(0, 3000))
dev = torch.device("cuda:0")
fs = to_device(st, t, dev, 32, scheme)
_lib.fixup_stats(reset=True)
FO.adamw_step_(fs, torch.from_numpy(g).to(dev).bfloat16(), FO.AdamHyperParams(**hp))
print("fixup (flagged, slices):", _lib.fixup_stats(reset=True))
got = from_device(fs)
ost = oracle_state(st, t, 32, scheme)
O.step_inplace("adamw", ost, g, **hp)
ref = oracle_dict(ost)
for k in got:
    d = np.nonzero(got[k] != ref[k])[0]
    if d.size:
        i = d[:4]
        print(k, "idx", i, "got", got[k][i], "ref", ref[k][i])
        j = i[0]
        print("  in: lp %04x rho %d m %d v %d g %r ms %r vs %r" % (st["weights.lp"][j], st["weights.rho"][j],
              st["momentum.codes"][j], st["variance.codes"][j], g[j], st["momentum.scales"][j // 32],
              st["variance.scales"][j // 32]), "out lp", got["weights.lp"][j], ref["weights.lp"][j])
