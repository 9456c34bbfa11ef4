"""Per-step gradient parity: oracle gradient evaluated at the GPU's own theta_k on
the GPU's sampled minibatch (isolates a wrong gradient from trajectory drift)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DQN_KEEP_GRAD", "1")
import paper_1508_04186_b200 as D  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.helpers import he_theta, nets, replay  # noqa: E402
from tools.diag_parity import table  # noqa: E402

prec = D.BF16 if "--bf16" in sys.argv else D.FP32
steps = 6
dc, on, oc = nets(minibatch=32, replay_capacity=1000, lr=2.5e-4, precision=prec)
theta0 = he_theta(on, 3)
if "--smooth" in sys.argv:  # every hidden pre-activation > 0: no ReLU kink near any unit
    tt = O.tensor_table(on)
    theta0 = np.abs(theta0)
    for i, (off, cnt) in enumerate(tt[:-2]):
        if i % 2 == 1:
            theta0[off:off + cnt] = 0.1
    # keep the output layer signed so targets and errors have both signs
    theta0[tt[-2][0]:] = he_theta(on, 3)[tt[-2][0]:]
rp, raw = replay(on, 1000, 1234)
g = D.DQN(dc, init_params=theta0)
g.push(*raw)
for k in range(steps):
    th = g.params(D.PARAMS_LOCAL).astype(np.float64)
    r_k = g.params(D.PARAMS_RMS).astype(np.float64)
    out = g.train(1, want_idx=True, want_loss=True)
    idx = out["idx"][0]
    y, _ = O.targets(on, theta0.astype(np.float64), rp.s_next[idx], rp.r[idx], rp.term[idx], oc.gamma)
    loss, gr = O.loss_grad(on, th, rp.s[idx], rp.a[idx], y)
    print(f"step {k}: loss gpu {out['loss'][0]:.7e} oracle {loss:.7e}  dup idx {len(idx) - len(set(idx.tolist()))}"
          f" term {int(rp.term[idx].sum())}")
    table(g.params(D.PARAMS_GRAD), gr, on, f"gradient at step {k}")
    th_next, _ = O.rmsprop(th, r_k, gr, oc.lr, oc.rms_decay, oc.rms_eps)
    gpu_next = g.params(D.PARAMS_SERVER)
    table(gpu_next - th, th_next - th, on, f"update at step {k} (oracle rule at the GPU state)")
# forward parity of the acting path at the final state
states = rp.s[:64]
q, am = g.q_values(states)
qo, amo = O.q_values(on, g.params(D.PARAMS_LOCAL).astype(np.float64), states)
print("q_values normwise", np.max(np.abs(q - qo)) / np.max(np.abs(qo)), "argmax agree", np.mean(am == amo))
