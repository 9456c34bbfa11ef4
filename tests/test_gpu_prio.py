"""Prioritized replay variant (NEXT-4; reading A41) on the GPU against oracle/prio.py, teacher-forced
step by step: from the leaf priorities the GPU holds before step T, the oracle's sum tree must have the GPU's
total bit for bit and draw the GPU's b slots exactly (every decision in fp32, same order); from the GPU's TD
errors of the step, the oracle's update must give the GPU's leaves after it exactly; stored transitions must
enter with the oracle's running max priority. The TD errors themselves are checked against the oracle's
forward on the drawn slots (step 0, theta0), so the forward really reads the drawn slots."""
import numpy as np
import pytest

import paper_1508_04186_b200 as D
import synth
from oracle import oracle as O
from oracle import prio as PR
from tests.helpers import he_theta, nets

pytestmark = pytest.mark.gpu
TINY_KW = dict(frames=3, height=17, width=13, convs=((5, 5, 2), (6, 3, 2)), fcs=(19,), n_actions=5)
SCALED = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)
CAP = 1500  # K = 3 levels above 32768 leaves; the second push wraps the ring


@pytest.mark.parametrize("precision,kw,alpha,b", [(D.FP32, TINY_KW, 1.0, 32), (D.FP32, TINY_KW, 0.5, 32),
                                                  (D.BF16, {}, 1.0, 32), (D.BF16, SCALED, 0.5, 32),
                                                  (D.FP32, TINY_KW, 0.5, 37), (D.BF16, {}, 1.0, 144)],
                         ids=["fp32-a1", "fp32-a05", "bf16-mnih-a1", "bf16-scaled-a05", "fp32-a05-b37",
                              "bf16-mnih-a1-b144"])
def test_prioritized_replay_teacher_forced(precision, kw, alpha, b):
    """b = 37 and 144: strata that are not a multiple of the 32-draw warp scan (a ragged last warp)."""
    eps = 1.0 if alpha == 1.0 else 0.01  # alpha = 1: every written priority exceeds the initial max (1)
    dc, on, _ = nets(minibatch=b, replay_capacity=CAP, precision=precision, target_sync=3, lr=1e-3,
                     replay_prio_alpha=alpha, replay_prio_eps=eps, **kw)
    theta0 = he_theta(on, 5)
    g = D.DQN(dc, init_params=theta0)
    K = PR.levels_for(CAP)
    data = synth.g_pong(1200, on.frames, on.height, on.width, on.n_actions, 21)
    g.push(*data)
    slots = [None] * CAP
    for i in range(1200):
        slots[i] = tuple(x[i] for x in data)
    leaves, total = g.priorities()
    assert np.all(leaves[:1200] == 1.0) and np.all(leaves[1200:] == 0.0) and total == 1200.0
    maxp = np.float32(1.0)
    for T in range(6):
        before, tot = g.priorities()
        lv = PR.build_tree(before, K)
        assert lv[-1][0] == np.float32(tot)  # the GPU's tree total is the oracle's butterfly sum, bit for bit
        out = g.train(1, want_idx=True, want_delta=True)
        idx, delta = out["idx"][0], out["delta"][0]
        assert np.array_equal(idx, PR.sample(lv, dc.seed, 0, T, dc.minibatch)), f"draws of step {T}"
        if T == 0:  # the forward read the drawn slots: delta against the oracle at theta0 (theta^ = theta0)
            s = np.stack([slots[i][0] for i in idx]); a = np.array([slots[i][1] for i in idx])
            r = np.array([slots[i][2] for i in idx]); sn = np.stack([slots[i][3] for i in idx])
            term = np.array([slots[i][4] for i in idx])
            q, _ = O.q_values(on, theta0.astype(np.float64), s)
            y, _ = O.targets(on, theta0.astype(np.float64), sn, r, term, dc.gamma)
            d_or = q[np.arange(len(a)), a] - y
            tol = 1e-4 if precision == D.FP32 else 2e-2
            assert np.max(np.abs(delta - d_or)) <= tol * max(1.0, np.max(np.abs(d_or)))
        after, _ = g.priorities()
        want, maxp = PR.update(before, maxp, idx, delta, alpha, eps)
        assert np.array_equal(after, want), f"leaf update of step {T}"
    # a second push wraps the ring: its slots enter with the running max priority
    more = synth.g_pong(600, on.frames, on.height, on.width, on.n_actions, 22)
    g.push(*more)
    leaves, total = g.priorities()
    stored = [(1200 + i) % CAP for i in range(600)]
    assert maxp > 1.0 or alpha != 1.0
    assert np.all(leaves[stored] == maxp)
    lv = PR.build_tree(leaves, K)
    assert lv[-1][0] == np.float32(total)
    out = g.train(1, want_idx=True)
    assert np.array_equal(out["idx"][0], PR.sample(lv, dc.seed, 0, 6, dc.minibatch))
    g.close()


def test_prioritized_replay_rejects_bad_alpha():
    dc, _, _ = nets(minibatch=8, replay_capacity=64, replay_prio_alpha=0.7, **TINY_KW)
    with pytest.raises(D.DqnError):
        D.DQN(dc)
