"""Frame-deduplicated replay (NEXT-4, dqn_config.replay_dedup): a slot stores F+1 frames and s' is
read as the window one frame later. On stacks where s' = s shifted by one frame + a new frame
(G-pong, P:59's sliding 4-frame history) every kernel reads the same bytes as with full stacks, so a
run must be bit-identical to the full-stack run; a push that breaks the shift property is rejected."""
import numpy as np
import pytest

import paper_1508_04186_b200 as D
import synth
from oracle import oracle as O
from tests.helpers import delta_rel, gated_theta, he_theta, nets

pytestmark = pytest.mark.gpu
TINY_KW = dict(frames=3, height=17, width=13, convs=((5, 5, 2), (6, 3, 2)), fcs=(19,), n_actions=5)
SCALED = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)


def run(dedup, precision, kw, steps=4, device_push=False):
    dc, on, _ = nets(minibatch=32, replay_capacity=150, precision=precision, target_sync=2, lr=1e-3,
                     replay_dedup=dedup, **kw)
    g = D.DQN(dc, init_params=he_theta(on, 3))
    data = synth.g_pong(200, on.frames, on.height, on.width, on.n_actions, 11)  # wraps the 150-slot ring
    if device_push:
        import torch
        data = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in data)
    g.push(*data)
    out = g.train(steps, want_idx=True)
    th = g.params(D.PARAMS_SERVER)
    q, _ = g.q_values(synth.g_pong(8, on.frames, on.height, on.width, on.n_actions, 12)[0])
    g.close()
    return out["idx"], th, q


@pytest.mark.parametrize("precision,kw", [(D.FP32, TINY_KW), (D.BF16, {}), (D.BF16, SCALED)],
                         ids=["fp32-tiny", "bf16-mnih", "bf16-scaled"])
def test_dedup_equals_full_stacks(precision, kw):
    i0, t0, q0 = run(0, precision, kw)
    i1, t1, q1 = run(1, precision, kw)
    assert np.array_equal(i0, i1)
    assert np.array_equal(t0, t1)
    assert np.array_equal(q0, q1)


def test_dedup_device_push_equals_host_push():
    i0, t0, _ = run(1, D.BF16, {}, device_push=False)
    i1, t1, _ = run(1, D.BF16, {}, device_push=True)
    assert np.array_equal(i0, i1) and np.array_equal(t0, t1)


@pytest.mark.parametrize("device_push", [False, True])
def test_dedup_rejects_unshifted_stacks(device_push):
    dc, on, _ = nets(minibatch=32, replay_capacity=100, precision=D.BF16, replay_dedup=1)
    g = D.DQN(dc, init_params=he_theta(on, 3))
    s, a, r, sn, t = synth.g_uniform(4, on.frames, on.height, on.width, on.n_actions, 5)  # independent s, s'
    data = (s, a, r, sn, t)
    if device_push:
        import torch
        data = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in data)
    with pytest.raises(D.DqnError) as e:
        g.push(*data)
    assert e.value.code == D.EINVAL
    assert g.replay_size() == (0, 0)  # nothing stored
    g.close()


@pytest.mark.parametrize("precision,kw", [(D.FP32, TINY_KW), (D.BF16, {})], ids=["fp32-tiny", "bf16-mnih"])
def test_dedup_matches_the_oracle(precision, kw):
    """The deduplicated replay against the oracle (which stores full stacks): the same transitions, so the
    same sampled slots (bit-exact) and theta after k steps within the path's bar (fp32 1e-5; bf16 in the gated
    regime, A38, 2e-2)."""
    steps = 4
    lr = 1e-3 if precision == D.FP32 else 1e-5
    eps = 1e-8 if precision == D.FP32 else 1e-2
    dc, on, oc = nets(minibatch=32, replay_capacity=150, precision=precision, target_sync=2, lr=lr, rms_eps=eps,
                      replay_dedup=1, **kw)
    th0 = he_theta(on, 3) if precision == D.FP32 else gated_theta(on, 3)
    data = synth.g_pong(200, on.frames, on.height, on.width, on.n_actions, 11)  # wraps the 150-slot ring
    g = D.DQN(dc, init_params=th0)
    g.push(*data)
    out = g.train(steps, want_idx=True)
    th = g.params(D.PARAMS_SERVER)
    g.close()
    s, a, r, sn, t = data
    ref = O.run(on, oc, 150, [O.Replay(s, a, r.astype(np.float64), sn, t)], th0.astype(np.float64), steps)
    assert np.array_equal(out["idx"], ref["idx"][0].astype(np.int32))
    tol = 1e-5 if precision == D.FP32 else 2e-2
    assert delta_rel(th, th0, ref["theta"], th0, on, ulps=steps) < tol
