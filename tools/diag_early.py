"""Diagnostic: bit-identity of the N=1 fused update path, early (FC update in the conv backward's
extra CTAs) vs late (all in reduce_update), each run twice; per-tensor first differing step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1508_04186_b200 as D
from oracle import oracle as O
from tests.helpers import nets
from tests.test_gpu_parity_bf16 import smooth_theta, make

os.environ.pop("DQN_KEEP_GRAD", None)
dc, on, oc = nets(minibatch=32, replay_capacity=1000, precision=D.BF16, lr=1e-5)
theta0 = smooth_theta(on, 7)
tt = O.tensor_table(on)
res = {}
for mode in ("1", "1", "0", "0"):
    os.environ["DQN_EARLY_UPDATE"] = mode
    g, rp, _ = make(dc, on, theta0, 1000, 77)
    th = []
    for k in range(3):
        g.train(1)
        th.append(g.params(D.PARAMS_SERVER).copy())
    g.close()
    res.setdefault(mode, []).append(th)
for a, b, name in ((res["1"][0], res["1"][1], "early run-to-run"), (res["0"][0], res["0"][1], "late run-to-run"),
                   (res["1"][0], res["0"][0], "early vs late")):
    for k in range(3):
        diff = [i for i, (off, cnt) in enumerate(tt) if not np.array_equal(a[k][off:off + cnt], b[k][off:off + cnt])]
        print(name, "step", k, "differing tensors", diff)
