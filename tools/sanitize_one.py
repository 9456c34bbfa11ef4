"""One small replica step of a config under compute-sanitizer (tools/sanitize.sh): the scaled net (generic
bf16 path) or the Mnih net, gated theta0, b = 32, two steps."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1508_04186_b200 as D  # noqa: E402
from tests.helpers import gated_theta, nets, replay  # noqa: E402

SCALED = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)
kw = SCALED if len(sys.argv) > 1 and sys.argv[1] == "scaled" else {}
prec = D.FP32 if len(sys.argv) > 2 and sys.argv[2] == "fp32" else D.BF16
dc, on, oc = nets(minibatch=32, replay_capacity=200, precision=prec, **kw)
g = D.DQN(dc, init_params=gated_theta(on, 3))
_, raw = replay(on, 200, 1)
g.push(*raw)
out = g.train(2, want_idx=True)
print("ok", out["idx"][0][:4], np.isfinite(g.params(D.PARAMS_SERVER)).all())
