"""GPU parity of the asynchronous modes (BJ.configs[3]) against the oracle.

* DQN_ASYNC_LAG1, the deterministic twin (O13): the server round runs on a second stream, and a fetch returns
  exactly the server theta one round late; equal to the oracle's fetch_lag = 1 run.
* DQN_ASYNC, Downpour's asynchrony: a fetch never waits, it takes the newest generation the
  comm stream has published (device flag), so which generation each step used depends on timing. The run
  reports that realised schedule (step_generation, A40) and the oracle replays it: given the schedule the
  result is exact (fp32 1e-5, bf16 2e-2 in the gated regime), and the staleness histogram is the oracle's.
  DQN_ASYNC_DELAY_US slows every server round down so that stale generations actually occur.
"""
import os

import numpy as np
import pytest

import paper_1508_04186_b200 as D
from oracle import oracle as O
from tests.helpers import delta_rel, gated_theta, he_theta, nets, per_tensor_rel, replay

pytestmark = pytest.mark.gpu
TINY_KW = dict(frames=3, height=17, width=13, convs=((5, 5, 2), (6, 3, 2)), fcs=(19,), n_actions=5)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available()
    yield


def fetch_schedule(step_gen, n_fetch):
    """per fetch f (at step f * n_fetch) the generation it returned, from the per-step generations"""
    return np.asarray(step_gen, np.int64)[::n_fetch]


@pytest.mark.parametrize("n_push,n_fetch,C", [(1, 1, 2), (3, 3, 1), (2, 3, 2)])
def test_async_lag1_twin_fp32(n_push, n_fetch, C):
    dc, on, oc = nets(minibatch=8, replay_capacity=64, n_push=n_push, n_fetch=n_fetch, target_sync=C, lr=2e-3,
                      sync_mode=D.ASYNC_LAG1, **TINY_KW)
    oc.fetch_lag = 1
    theta0 = he_theta(on, 6)
    rp, raw = replay(on, 80, 12)
    g = D.DQN(dc, init_params=theta0)
    g.push(*raw)
    g.train(5, want_idx=True)
    out = g.train(7, want_idx=True)
    ref = O.run(on, oc, 64, [rp], theta0.astype(np.float64), 12)
    assert np.array_equal(out["idx"], ref["idx"][0, 5:])
    assert per_tensor_rel(g.params(D.PARAMS_SERVER), ref["theta"], on) < 1e-5
    assert np.array_equal(out["staleness"], ref["staleness"])
    assert out["generation"] == ref["n"]
    g.close()


@pytest.mark.parametrize("n_push,n_fetch,C,delay_us", [(1, 1, 2, 0), (4, 1, 2, 0), (1, 1, 2, 300), (2, 1, 1, 300),
                                                      (3, 2, 2, 500)])
def test_async_free_running_fp32_equals_its_realised_schedule(n_push, n_fetch, C, delay_us):
    dc, on, oc = nets(minibatch=8, replay_capacity=64, n_push=n_push, n_fetch=n_fetch, target_sync=C, lr=2e-3,
                      sync_mode=D.ASYNC, **TINY_KW)
    theta0 = he_theta(on, 6)
    rp, raw = replay(on, 80, 12)
    os.environ["DQN_ASYNC_DELAY_US"] = str(delay_us)
    try:
        g = D.DQN(dc, init_params=theta0)
    finally:
        os.environ.pop("DQN_ASYNC_DELAY_US", None)
    g.push(*raw)
    steps = 24
    o1 = g.train(11, want_idx=True, want_generation=True)
    o2 = g.train(steps - 11, want_idx=True, want_generation=True)
    gen = np.concatenate([o1["step_generation"], o2["step_generation"]])
    # a step's generation was published before its fetch ran, and the push waits keep it within two rounds
    t = np.arange(steps)
    pushed = (t - t % n_fetch) // n_push  # rounds pushed when the step's fetch ran
    assert np.all(gen <= pushed) and np.all(gen >= pushed - 2) and np.all(np.diff(gen) >= 0)
    if delay_us == 0 and n_push >= 4:
        # a fetch takes the NEWEST published generation: two or more steps after a push its round (a few us
        # on this net) has long been published
        late = (t % n_push >= 2) & (t >= n_push)
        assert np.array_equal(gen[late], pushed[late])
    oc.fetch_gen = fetch_schedule(gen, n_fetch)[None, :]
    ref = O.run(on, oc, 64, [rp], theta0.astype(np.float64), steps)
    assert ref["rc"] == 0
    assert np.array_equal(np.concatenate([o1["idx"], o2["idx"]]), ref["idx"][0])
    th0 = theta0.astype(np.float64)
    assert delta_rel(g.params(D.PARAMS_SERVER), th0, ref["theta"], th0, on, ulps=ref["n"]) < 1e-5
    assert np.array_equal(o2["staleness"], ref["staleness"])
    assert o2["generation"] == ref["n"] == steps // n_push
    if delay_us >= 300:
        assert ref["staleness"][1:].sum() > 0  # the slow server made some steps stale
    g.close()


def test_async_bf16_config3_shape_gated():
    """BJ.configs[3] per replica (Mnih net, b = 256, n_push = n_fetch = 10, DQN_ASYNC) in the gated regime
    (A38): Delta theta of every tensor within 2e-2 of the oracle's replay of the realised schedule."""
    dc, on, oc = nets(minibatch=256, replay_capacity=2000, n_push=10, n_fetch=10, target_sync=1000,
                      precision=D.BF16, sync_mode=D.ASYNC, lr=1e-5, rms_eps=1e-2)
    theta0 = gated_theta(on, 2)
    rp, raw = replay(on, 2000, 3)
    g = D.DQN(dc, init_params=theta0)
    g.push(*raw)
    out = g.train(30, want_idx=True, want_loss=True, want_generation=True)
    assert np.all(np.isfinite(out["loss"]))
    assert out["staleness"].sum() == 30 and out["generation"] == 3
    oc.fetch_gen = fetch_schedule(out["step_generation"], 10)[None, :]
    ref = O.run(on, oc, 2000, [rp], theta0.astype(np.float64), 30)
    assert ref["rc"] == 0
    assert np.array_equal(out["idx"], ref["idx"][0])
    assert np.array_equal(out["staleness"], ref["staleness"])
    th0 = theta0.astype(np.float64)
    assert delta_rel(g.params(D.PARAMS_SERVER), th0, ref["theta"], th0, on, ulps=3) < 2e-2
    g.close()
