"""NEXT-3: on-GPU acting (dqn_collect) against the oracle's or_collect. Game logic, rendering,
eps-greedy draws and the Store are integer / byte work: bit-exact. The greedy branch is pinned with a
network whose Q is constant (zero weights, output biases [0, 1, 0, 0]: argmax 1 in every precision)."""
import numpy as np
import pytest

import paper_1508_04186_b200 as D
from oracle import oracle as O
from tests.helpers import he_theta, nets

pytestmark = pytest.mark.gpu
SEED = 0xACE


def make(precision=D.FP32, dedup=0, theta=None, b=16):
    dc, on, _ = nets(minibatch=b, replay_capacity=500, precision=precision, n_actions=4, replay_dedup=dedup)
    g = D.DQN(dc, init_params=he_theta(on, 3) if theta is None else theta)
    return g, dc, on


@pytest.mark.parametrize("precision", [D.FP32, D.BF16])
def test_random_policy_matches_oracle(precision):
    g, dc, on = make(precision)
    E, steps, n = 8, 60, 12
    out = g.collect(E, n, steps, 1.0, SEED, want_log=True)
    ref = O.collect(n, on.frames, on.height, E, steps, SEED, 1.0)
    assert np.array_equal(out["a"], ref["a"])
    assert np.array_equal(out["r"], ref["r"].astype(np.float32))
    assert np.array_equal(out["term"], ref["term"])
    assert np.array_equal(g.env_stacks(E), ref["stacks"])
    assert out["episodes"] == ref["episodes"].sum() and out["reward_sum"] == ref["r"].sum()
    assert out["env_steps"] == E * steps
    assert g.replay_size() == (E * steps, min(E * steps, dc.replay_capacity))
    g.close()


def test_greedy_branch_and_continuation():
    dc, on, _ = nets(minibatch=16, replay_capacity=500, n_actions=4)
    tt = O.tensor_table(on)
    theta = np.zeros(O.param_count(on), np.float32)
    ob_off, ob_cnt = tt[-1]
    theta[ob_off:ob_off + ob_cnt] = [0.0, 1.0, 0.0, 0.0]           # Q(s) = [0, 1, 0, 0] for every s
    g = D.DQN(dc, init_params=theta)
    E, n = 6, 12
    first = g.collect(E, n, 30, 0.25, SEED, want_log=True)
    second = g.collect(E, n, 20, 0.25, SEED, want_log=True)          # the games continue
    ref = O.collect(n, on.frames, on.height, E, 50, SEED, 0.25, greedy=np.ones((50, E), np.int32))
    assert np.array_equal(np.concatenate([first["a"], second["a"]]), ref["a"])
    assert np.array_equal(np.concatenate([first["r"], second["r"]]), ref["r"].astype(np.float32))
    assert np.array_equal(g.env_stacks(E), ref["stacks"])
    assert (ref["a"] == 1).mean() > 0.7                             # mostly the greedy action (eps = 0.25)
    g.close()


def test_collected_transitions_train_and_match_dedup():
    """The Store feeds training: the same collection with and without frame dedup gives the same replay,
    hence bit-identical training (the collector's s' is s shifted by one frame + the new frame)."""
    res = []
    for dedup in (0, 1):
        g, dc, on = make(D.BF16, dedup=dedup, b=32)
        g.collect(32, 12, 12, 1.0, SEED)
        out = g.train(3, want_idx=True)
        res.append((out["idx"], g.params(D.PARAMS_SERVER)))
        g.close()
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


def test_bad_arguments_are_rejected():
    g, dc, on = make()
    with pytest.raises(D.DqnError):
        g.collect(8, 5, 1, 1.0, SEED)                               # 84 % 5 != 0
    with pytest.raises(D.DqnError):
        g.collect(64, 12, 1, 1.0, SEED)                             # more games than the minibatch
    g.collect(4, 12, 2, 1.0, SEED)
    with pytest.raises(D.DqnError):
        g.collect(4, 12, 2, 1.0, SEED + 1)                          # the games persist: same seed required
    g.close()
    dc6, on6, _ = nets(minibatch=16, replay_capacity=100, n_actions=6)
    g6 = D.DQN(dc6, init_params=he_theta(on6, 3))
    with pytest.raises(D.DqnError):
        g6.collect(4, 12, 1, 1.0, SEED)                             # Snake has 4 actions
    g6.close()
