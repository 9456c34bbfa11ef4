"""GPU parity of the asynchronous mode (DQN_ASYNC, BJ.configs[3]) against the
oracle's deterministic twin (O13: a fetch returns the server theta one round late) — the
server round runs on a second stream, overlapping the replica's next steps."""
import os

import numpy as np
import pytest

import paper_1508_04186_b200 as D
from oracle import oracle as O
from tests.helpers import he_theta, nets, per_tensor_rel, replay

pytestmark = pytest.mark.gpu
TINY_KW = dict(frames=3, height=17, width=13, convs=((5, 5, 2), (6, 3, 2)), fcs=(19,), n_actions=5)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available()
    yield


@pytest.mark.parametrize("n_push,n_fetch,C", [(1, 1, 2), (3, 3, 1), (2, 3, 2)])
def test_async_fp32_matches_lag1_twin(n_push, n_fetch, C):
    dc, on, oc = nets(minibatch=8, replay_capacity=64, n_push=n_push, n_fetch=n_fetch, target_sync=C, lr=2e-3,
                      sync_mode=D.ASYNC, **TINY_KW)
    oc.fetch_lag = 1
    theta0 = he_theta(on, 6)
    rp, raw = replay(on, 80, 12)
    g = D.DQN(dc, init_params=theta0)
    g.push(*raw)
    out = g.train(5, want_idx=True)
    out = g.train(7, want_idx=True)
    ref = O.run(on, oc, 64, [rp], theta0.astype(np.float64), 12)
    assert np.array_equal(out["idx"], ref["idx"][0, 5:])
    assert per_tensor_rel(g.params(D.PARAMS_SERVER), ref["theta"], on) < 1e-5
    assert np.array_equal(out["staleness"], ref["staleness"])
    assert out["generation"] == ref["n"]
    g.close()


def test_async_bf16_config3_shape_runs_and_tracks_staleness():
    """BJ.configs[3] per replica: Mnih net, b = 256, n_push = n_fetch = 10, async."""
    dc, on, oc = nets(minibatch=256, replay_capacity=2000, n_push=10, n_fetch=10, target_sync=1000,
                      precision=D.BF16, sync_mode=D.ASYNC)
    oc.fetch_lag = 1
    oc.n_push = oc.n_fetch = 10
    theta0 = he_theta(on, 2)
    rp, raw = replay(on, 2000, 3)
    g = D.DQN(dc, init_params=theta0)
    g.push(*raw)
    out = g.train(30, want_idx=True, want_loss=True)
    assert np.all(np.isfinite(out["loss"]))
    # rounds 0, 1, 2: staleness 0 for round 0's ten steps, 1 afterwards
    assert out["staleness"][0] == 10 and out["staleness"][1] == 20 and out["staleness"].sum() == 30
    assert out["generation"] == 3
    assert list(out["idx"][0][:4]) == [O.sample_index(dc.seed, 0, 0, j, 2000) for j in range(4)]
    g.close()
