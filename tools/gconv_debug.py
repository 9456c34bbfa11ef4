"""Step-by-step smoke of the generic bf16 conv path (scaled net) with progress prints and a traceback
dump if anything blocks (faulthandler)."""
import faulthandler
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(90, exit=True)
import paper_1508_04186_b200 as D  # noqa: E402
from tests.helpers import nets, replay, he_theta  # noqa: E402

SCALED = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)
t0 = time.time()
dc, on, oc = nets(minibatch=32, replay_capacity=300, precision=D.BF16, **SCALED)
print("config", time.time() - t0, flush=True)
g = D.DQN(dc, init_params=he_theta(on, 3))
print("created", time.time() - t0, flush=True)
rp, raw = replay(on, 300, 5)
g.push(*raw)
print("pushed", time.time() - t0, flush=True)
q, am = g.q_values(raw[0][:40])
print("q", q.shape, np.abs(q).max(), time.time() - t0, flush=True)
out = g.train(1)
print("train1", out["loss_mean"], time.time() - t0, flush=True)
out = g.train(5)
print("train5", out["loss_mean"], time.time() - t0, flush=True)
