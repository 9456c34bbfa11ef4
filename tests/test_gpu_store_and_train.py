"""dqn_store_and_train (Alg. 1's loop in one call): store transition i, then run step i.
It must equal k alternating dqn_push_transitions(1 item) + dqn_train_steps(1) calls bit for bit —
sampled indices (which see the replay size grow by one per step), losses and parameters — on the fp32
and bf16 paths, with host and device input buffers, including a replay that wraps around."""
import os

import numpy as np
import pytest

import paper_1508_04186_b200 as D
from tests.helpers import he_theta, nets, replay

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    yield


@pytest.mark.parametrize("prec,device_inputs,cap,b", [(D.FP32, False, 64, 8), (D.BF16, False, 64, 16),
                                                        (D.BF16, True, 64, 16), (D.BF16, False, 40, 16),
                                                        (D.BF16, False, 300, 256)])
def test_store_and_train_equals_alternating_calls(prec, device_inputs, cap, b):
    """b = 256: 256 image CTAs per group beside the forward's 14 Store CTAs; with 34-45 items in the replay
    nearly every step has draws of the slot being stored (they wait for the Store's release)."""
    import torch
    k, pre = 12, 33
    dc, on, _ = nets(minibatch=b, replay_capacity=cap, precision=prec, lr=1e-4)
    theta0 = he_theta(on, 5)
    _, raw = replay(on, pre + k, 9)
    head = tuple(x[:pre] for x in raw)
    tail = tuple(x[pre:] for x in raw)
    if device_inputs:
        tail = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in tail)

    g1 = D.DQN(dc, init_params=theta0)
    g1.push(*head)
    idx1, loss1 = [], []
    for i in range(k):
        g1.push(*(x[i:i + 1] for x in tail))
        o = g1.train(1, want_idx=True, want_loss=True)
        idx1.append(o["idx"][0])
        loss1.append(o["loss"][0])
    th1 = g1.params(D.PARAMS_SERVER)
    g1.close()

    g2 = D.DQN(dc, init_params=theta0)
    g2.push(*head)
    o = g2.train(k, want_idx=True, want_loss=True, store=tail)
    th2 = g2.params(D.PARAMS_SERVER)
    assert o["steps_done"] == k
    g2.close()

    assert np.array_equal(np.stack(idx1), o["idx"])
    assert np.array_equal(np.array(loss1, np.float32), o["loss"])
    assert np.array_equal(th1, th2)
    # the sampler saw the replay grow by one item per step (until it wraps at cap)
    sizes = [min(pre + i + 1, cap) for i in range(k)]
    assert all(int(o["idx"][i].max()) < sizes[i] for i in range(k))


def test_store_and_train_validates_before_running():
    dc, on, _ = nets(minibatch=8, replay_capacity=64, precision=D.FP32)
    g = D.DQN(dc, init_params=he_theta(on, 5))
    _, raw = replay(on, 4, 3)
    s, a, r, sn, t = raw
    a = a.copy()
    a[2] = on.n_actions  # out of range
    with pytest.raises(D.DqnError):
        g.train(4, store=(s, a, r, sn, t))
    assert g.replay_size() == (0, 0)  # nothing stored, nothing ran
    g.close()
