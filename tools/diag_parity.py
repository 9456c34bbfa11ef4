"""Per-tensor parity diagnostics of the GPU path vs the oracle (prints a table).

usage: python tools/diag_parity.py [--precision fp32|bf16] [--steps K] [--lr LR] [--b B]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DQN_KEEP_GRAD", "1")

import paper_1508_04186_b200 as D  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.helpers import he_theta, nets, replay  # noqa: E402


def table(x, y, net, title):
    names = []
    for i in range(len(net.convs)):
        names += [f"conv{i + 1}.W", f"conv{i + 1}.b"]
    for i in range(len(net.fcs)):
        names += [f"fc{i + 1}.W", f"fc{i + 1}.b"]
    names += ["out.W", "out.b"]
    print(f"--- {title}")
    for nm, (off, cnt) in zip(names, O.tensor_table(net)):
        yy, xx = np.asarray(y[off:off + cnt], np.float64), np.asarray(x[off:off + cnt], np.float64)
        den = max(np.max(np.abs(yy)), 1e-30)
        l2 = np.linalg.norm(xx - yy) / max(np.linalg.norm(yy), 1e-30)
        print(f"  {nm:8s} n={cnt:7d} |y|inf={den:.3e} normwise={np.max(np.abs(xx - yy)) / den:.3e} rel_l2={l2:.3e}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--lr", type=float, default=2.5e-4)
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--perturb", action="store_true")
    ap.add_argument("--every", action="store_true")
    a = ap.parse_args()
    prec = D.FP32 if a.precision == "fp32" else D.BF16
    dc, on, oc = nets(minibatch=a.b, replay_capacity=1000, lr=a.lr, precision=prec, rms_eps=a.eps)
    theta0 = he_theta(on, 3)
    rp, raw = replay(on, 1000, 1234)
    if a.perturb:
        # intrinsic sensitivity: the oracle against itself from theta0 perturbed at fp32 rounding level
        rng = np.random.default_rng(0)
        t64 = theta0.astype(np.float64)
        tp = t64 * (1.0 + 6e-8 * rng.standard_normal(t64.size))
        for k in [1, 2, 5, a.steps]:
            r0 = O.run(on, oc, 1000, [rp], t64, k)
            r1 = O.run(on, oc, 1000, [rp], tp, k)
            table(r1["theta"] - tp, r0["theta"] - t64, on, f"ORACLE perturbed: theta - theta0 after {k} steps")
        return
    g = D.DQN(dc, init_params=theta0)
    g.push(*raw)
    ks = list(range(1, a.steps + 1)) if a.every else [1, 2, 5, a.steps]
    done = 0
    for k in ks:
        g.train(k - done)
        done = k
        ref = O.run(on, oc, 1000, [rp], theta0.astype(np.float64), k, want_grad0=(k == 1))
        if k == 1:
            table(g.params(D.PARAMS_GRAD), ref["grad0"], on, "gradient of step 0")
        th = g.params(D.PARAMS_SERVER)
        table(th, ref["theta"], on, f"theta after {k} steps")
        table(th - theta0, ref["theta"] - theta0.astype(np.float64), on, f"theta - theta0 after {k} steps")


if __name__ == "__main__":
    main()
