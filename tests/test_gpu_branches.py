"""The generic path's graph branches change only where kernels run, not what they compute: the conv backward on
two streams (DQN_CONC_BWD) and the side branch of the head finish + non-conv update (DQN_SPLIT_UPDATE) give
bit-identical parameters, gradients and losses to the single-stream schedule (same kernels, same per-element
arithmetic, reductions in the same fixed order)."""
import os

import numpy as np
import pytest

import paper_1508_04186_b200 as D
from tests.helpers import gated_theta, nets, replay

pytestmark = pytest.mark.gpu
SCALED = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)


def run(conc_bwd, split_update, b):
    old = {k: os.environ.get(k) for k in ("DQN_CONC_BWD", "DQN_SPLIT_UPDATE")}
    os.environ["DQN_CONC_BWD"] = str(conc_bwd)
    os.environ["DQN_SPLIT_UPDATE"] = str(split_update)
    try:
        dc, on, _ = nets(minibatch=b, replay_capacity=600, precision=D.BF16, target_sync=2, lr=1e-5, rms_eps=1e-2,
                         **SCALED)
        g = D.DQN(dc, init_params=gated_theta(on, 3))
        _, raw = replay(on, 600, 5)
        g.push(*raw)
        out = g.train(4, want_idx=True, want_loss=True)
        th, gr = g.params(D.PARAMS_SERVER), g.params(D.PARAMS_GRAD)
        g.close()
        return out["idx"], out["loss"], th, gr
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("b", [32, 144, 512])
def test_graph_branches_are_bit_identical(b):
    ref = run(0, 0, b)
    for conc, split in ((1, 1), (1, 0), (0, 1)):
        got = run(conc, split, b)
        for x, y in zip(got, ref):
            assert np.array_equal(x, y), f"DQN_CONC_BWD={conc} DQN_SPLIT_UPDATE={split} differs at b={b}"
