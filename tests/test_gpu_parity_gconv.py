"""bf16 tensor-core path for conv stacks other than Mnih-2013 (kernels_conv.cu), on the scaled net of
BASELINE.json configs[4] (conv32 8x8/4, conv64 4x4/2, conv64 3x3/1, fc512, 18 actions), against the fp64
oracle. Tolerances and the smooth regime as in test_gpu_parity_bf16 (A31); the gated-regime gradient,
k-step Delta theta, error-clip and refresh checks of this path are in test_gpu_parity_gated."""
import os

import numpy as np
import pytest

import paper_1508_04186_b200 as D
from oracle import oracle as O
from tests.helpers import near_tie_mask, nets, per_tensor_rel, replay
from tests.test_gpu_parity_bf16 import rel_l2_per_tensor, smooth_theta

pytestmark = pytest.mark.gpu
TOL = 2e-2
SCALED = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    yield


def make(dc, on, theta0, n_items, seed):
    rp, raw = replay(on, n_items, seed)
    g = D.DQN(dc, init_params=theta0)
    g.push(*raw)
    return g, rp, raw


def test_scaled_q_values():
    dc, on, oc = nets(minibatch=32, replay_capacity=300, precision=D.BF16, **SCALED)
    theta0 = smooth_theta(on, 3)
    g, rp, raw = make(dc, on, theta0, 300, 5)
    th = theta0.astype(np.float64)
    q, am = g.q_values(raw[0][:40])  # one chunk of 32 + a ragged tail of 8
    qo, amo = O.q_values(on, th, raw[0][:40])
    assert np.max(np.abs(q - qo)) / np.max(np.abs(qo)) < TOL
    ok = near_tie_mask(qo, TOL)
    assert np.array_equal(am[ok], amo[ok])
    g.close()


def test_scaled_one_step_gradient():
    dc, on, oc = nets(minibatch=32, replay_capacity=300, precision=D.BF16, **SCALED)
    theta0 = smooth_theta(on, 4)
    g, rp, raw = make(dc, on, theta0, 300, 6)
    th = theta0.astype(np.float64)
    assert O.min_abs_preact(on, th, raw[0][:32]) > 0.05
    out = g.train(1, want_idx=True, want_loss=True)
    ref = O.run(on, oc, 300, [rp], th, 1, want_grad0=True)
    assert np.array_equal(out["idx"], ref["idx"][0])
    assert abs(out["loss"][0] - ref["loss"][0, 0]) <= TOL * ref["loss"][0, 0]
    assert per_tensor_rel(g.params(D.PARAMS_GRAD), ref["grad0"], on) < TOL
    g.close()
