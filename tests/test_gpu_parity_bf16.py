"""GPU parity of the bf16 tensor-core path (DQN_BF16, tcgen05) against the fp64 oracle,
through the C ABI. Bar (BASELINE.json north_star): indices and argmax bit-exact
(argmax outside near-ties, A21), values within 2e-2.

bf16 rounds every operand to 8 significant bits, so a pre-activation within
~2^-8 of its scale from the ReLU kink may take the other branch of ReLU'(z)
than in fp64 (A30/A31). The kernels' arithmetic is therefore pinned at 2e-2
normwise per tensor in the "smooth" regime (every hidden pre-activation bounded
away from 0, so no unit can change branch), and in the default regime on the
quantities that are continuous (Q, loss, y) plus a relative-L2 gradient bound.
"""
import os

import numpy as np
import pytest

import paper_1508_04186_b200 as D
from oracle import oracle as O
from tests.helpers import delta_rel, gated_theta, he_theta, near_tie_mask, nets, per_tensor_rel, replay

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    yield


def smooth_theta(on, seed):
    """|He| weights and +0.1 biases on every hidden layer: all hidden pre-activations > 0.1."""
    th = he_theta(on, seed)
    tt = O.tensor_table(on)
    signed_out = th[tt[-2][0]:].copy()
    th = np.abs(th) * 0.5
    for i, (off, cnt) in enumerate(tt[:-2]):
        if i % 2 == 1:
            th[off:off + cnt] = 0.1
    th[tt[-2][0]:] = signed_out
    return th


def rel_l2_per_tensor(x, y, net):
    worst = 0.0
    for off, cnt in O.tensor_table(net):
        yy = np.asarray(y[off:off + cnt], np.float64)
        xx = np.asarray(x[off:off + cnt], np.float64)
        worst = max(worst, float(np.linalg.norm(xx - yy) / max(np.linalg.norm(yy), 1e-30)))
    return worst


def make(dc, on, theta0, n_items, seed):
    rp, raw = replay(on, n_items, seed)
    g = D.DQN(dc, init_params=theta0)
    g.push(*raw)
    return g, rp, raw


@pytest.mark.parametrize("b,fc", [(32, 256), (256, 256), (32, 128), (32, 512)])
def test_smooth_regime_gradient_and_q(b, fc):
    """fc 128 / 512: the model-size sweep points (tools/model_sweep.sh) on the same kernels."""
    dc, on, oc = nets(minibatch=b, replay_capacity=1000, precision=D.BF16, fcs=(fc,))
    theta0 = smooth_theta(on, 3)
    g, rp, raw = make(dc, on, theta0, 1000, 21)
    th = theta0.astype(np.float64)
    assert O.min_abs_preact(on, th, raw[0][:64]) > 0.05
    q, am = g.q_values(raw[0][:50])  # one chunk + ragged tail for b = 32
    qo, amo = O.q_values(on, th, raw[0][:50])
    assert np.max(np.abs(q - qo)) / np.max(np.abs(qo)) < TOL
    ok = near_tie_mask(qo, TOL)
    assert np.array_equal(am[ok], amo[ok])
    out = g.train(1, want_idx=True)
    ref = O.run(on, oc, 1000, [rp], th, 1, want_grad0=True)
    assert np.array_equal(out["idx"], ref["idx"][0])
    assert per_tensor_rel(g.params(D.PARAMS_GRAD), ref["grad0"], on) < TOL
    g.close()


def test_smooth_regime_ten_steps_teacher_forced():
    # a small alpha keeps theta inside the smooth regime for all 10 steps (checked below)
    dc, on, oc = nets(minibatch=32, replay_capacity=1000, precision=D.BF16, lr=1e-6)
    theta0 = smooth_theta(on, 5)
    g, rp, _ = make(dc, on, theta0, 1000, 1234)
    th0 = theta0.astype(np.float64)
    for k in range(10):
        th = g.params(D.PARAMS_LOCAL).astype(np.float64)
        out = g.train(1, want_idx=True, want_loss=True, want_argmax=True)
        idx = out["idx"][0]
        assert list(idx) == [O.sample_index(dc.seed, 0, k, j, 1000) for j in range(32)]
        y, am = O.targets(on, th0, rp.s_next[idx], rp.r[idx], rp.term[idx], oc.gamma)
        loss, grad = O.loss_grad(on, th, rp.s[idx], rp.a[idx], y)
        assert O.min_abs_preact(on, th, rp.s[idx]) > 0.05
        assert abs(out["loss"][0] - loss) <= TOL * loss
        assert per_tensor_rel(g.params(D.PARAMS_GRAD), grad, on) < TOL
        qn, _ = O.q_values(on, th0, rp.s_next[idx])
        ok = near_tie_mask(qn, TOL)
        assert np.array_equal(out["argmax"][0][ok], am[ok])
    g.close()


def test_default_regime_config0():
    """configs[0] with He init: continuous outputs at 2e-2; gradients (ReLU-branch sensitive) in rel-L2."""
    dc, on, oc = nets(minibatch=32, replay_capacity=1000, precision=D.BF16)
    theta0 = he_theta(on, 3)
    g, rp, raw = make(dc, on, theta0, 1000, 1234)
    th0 = theta0.astype(np.float64)
    q, _ = g.q_values(raw[0][:64])
    qo, _ = O.q_values(on, th0, raw[0][:64])
    assert np.max(np.abs(q - qo)) / np.max(np.abs(qo)) < TOL
    out = g.train(1, want_idx=True, want_loss=True)
    ref = O.run(on, oc, 1000, [rp], th0, 1, want_grad0=True)
    assert np.array_equal(out["idx"], ref["idx"][0])
    assert abs(out["loss"][0] - ref["loss"][0, 0]) <= TOL * ref["loss"][0, 0]
    assert rel_l2_per_tensor(g.params(D.PARAMS_GRAD), ref["grad0"], on) < 0.1
    out = g.train(9, want_idx=True)
    ref = O.run(on, oc, 1000, [rp], th0, 10)
    assert np.array_equal(out["idx"], ref["idx"][0, 1:])
    # parameters after k steps: test_gpu_parity_gated (A38); here units near their kink take either
    # branch in bf16 (A31), so the trajectories separate at the level of the gradient noise
    g.close()


def test_bf16_run_to_run_bit_identical():
    dc, on, _ = nets(minibatch=32, replay_capacity=300, precision=D.BF16)
    theta0 = he_theta(on, 4)
    res = []
    for _ in range(2):
        g, _, _ = make(dc, on, theta0, 300, 8)
        g.train(5)
        res.append(g.params(D.PARAMS_SERVER))
        g.close()
    assert np.array_equal(res[0], res[1])


def test_fused_reduce_update_path():
    """N = 1, n_push = 1 (the bench path): the conv partials' reduction runs inside the update kernel
    (reduce_update_kernel) and the FC / output-layer part of that update in extra CTAs of the conv backward
    launch (the early update). With DQN_EARLY_UPDATE=0 the same per-element arithmetic runs in
    reduce_update_kernel: the two runs are bit-identical, with keep_grad on or off, and Delta theta after
    5 steps matches the oracle within 2e-2 per tensor (gated regime, A38)."""
    dc, on, oc = nets(minibatch=32, replay_capacity=1000, precision=D.BF16, lr=1e-5, rms_eps=1e-2)
    theta0 = gated_theta(on, 7)
    res = {}
    for mode in ("early", "late", "nokeep"):
        if mode == "late":
            os.environ["DQN_EARLY_UPDATE"] = "0"
        try:
            cfg = dc if mode != "nokeep" else D.Config(**{**dc.__dict__, "keep_grad": 0})
            g, rp, _ = make(cfg, on, theta0, 1000, 77)
            g.train(5)
            res[mode] = (g.params(D.PARAMS_SERVER).astype(np.float64), g.params(D.PARAMS_LOCAL).astype(np.float64))
            g.close()
        finally:
            os.environ.pop("DQN_EARLY_UPDATE", None)
    for mode in ("late", "nokeep"):
        assert np.array_equal(res["early"][0], res[mode][0]) and np.array_equal(res["early"][1], res[mode][1])
    th, loc = res["early"]
    assert np.array_equal(th, loc)  # N = 1: the working copy is the server theta
    ref = O.run(on, oc, 1000, [rp], theta0.astype(np.float64), 5)
    th0 = theta0.astype(np.float64)
    assert delta_rel(th, th0, ref["theta"], th0, on, ulps=5) < TOL


def test_fig3_timing_fields():
    """dqn_step_stats carries the paper's Fig. 3 split from the last dqn_profile_steps: gradient
    time T, update time tau and communication, per replica step (-1 before any profile)."""
    dc, on, _ = nets(minibatch=32, replay_capacity=300, precision=D.BF16)
    g, _, _ = make(dc, on, he_theta(on, 4), 300, 8)
    out = g.train(2)
    assert out["grad_ms"] == -1.0 and out["update_ms"] == -1.0
    regions = g.profile(4)
    out = g.train(2)
    assert out["grad_ms"] > 0 and out["update_ms"] > 0 and out["comm_ms"] >= 0
    tot = sum(r["avg_us"] * r["steps"] for r in regions) / 4 / 1e3
    assert abs(out["grad_ms"] + out["update_ms"] + out["comm_ms"] - tot) <= 1e-6 + 1e-6 * tot
    g.close()
