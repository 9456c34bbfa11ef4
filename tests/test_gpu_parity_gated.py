"""bf16 tensor-core path against the fp64 oracle in the gated regime (A38), through the C ABI, on
the kernels bench.py times (keep_grad only adds a store of the pushed gradient in the update kernels).

In the gated regime (tests/helpers.gated_theta) half of every hidden layer's ReLU units are always off and
none is within 0.06 of its kink, so every ReLU mask (TD head dH, FC dX, conv dZ) is exercised and no bf16
rounding can flip a branch (A30/A31): the BASELINE.json north_star bar of 2e-2 applies to every tensor.

Parameters are compared as updates, Delta theta = theta_k - theta_0 per tensor (A29 on Delta theta). With
rms_eps = 1e-2 the RMSProp step alpha g / sqrt(r + eps) is a smooth function of g at these gradient scales,
so Delta theta inherits the gradient's precision; at eps = 1e-8 the first step is alpha sqrt(10) sign(g) and
one noise-level sign decides 2 alpha sqrt(10). The gated weights are small (|w| <= 0.04 / fan-in),
so multi-step runs use alpha = 1e-5: the weights then move by ~1 % per step and the gate holds (checked at the
end); the relative error of Delta theta does not depend on alpha."""
import numpy as np
import pytest

import paper_1508_04186_b200 as D
from oracle import oracle as O
from tests.helpers import bf16_rne, delta_rel, gated_theta_separated, near_tie_mask, nets, per_tensor_rel, replay

pytestmark = pytest.mark.gpu
TOL = 2e-2
GATE = 0.0599  # min |hidden pre-activation| the gated theta0 guarantees (bias 0.1 - margin 0.04)
SCALED = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    yield


def make(dc, on, n_items, seed, theta_seed, r_scale=1.0, out_std=0.5):
    theta0 = gated_theta_separated(on, theta_seed, out_std=out_std)
    rp, raw = replay(on, n_items, seed)
    if r_scale != 1.0:
        raw = (raw[0], raw[1], (raw[2] * r_scale).astype(np.float32), raw[3], raw[4])
        rp = O.Replay(raw[0], raw[1], raw[2].astype(np.float64), raw[3], raw[4])
    g = D.DQN(dc, init_params=theta0)
    g.push(*raw)
    return g, rp, raw, theta0.astype(np.float64)


CASES = [(dict(), 32), (dict(), 256), (dict(fcs=(128,)), 32), (dict(fcs=(512,)), 32), (dict(fcs=(2048,)), 32),
         (SCALED, 32), (SCALED, 512), (dict(SCALED, fcs=(1024,)), 32), (dict(SCALED, fcs=(2048,)), 64),
         (dict(), 16), (dict(), 80), (dict(), 144), (SCALED, 16), (SCALED, 144)]
IDS = ["mnih-b32", "mnih-b256", "mnih-fc128", "mnih-fc512", "mnih-fc2048", "scaled-b32", "scaled-b512",
       "scaled-fc1024", "scaled-fc2048",  # fc > 512: the FC backward on the K-pipelined GEMM (BJ.c5's sweep)
       # ragged minibatches: half a 32-sample head tile; 80 = 2.5 head tiles; 144 = one 128-row GEMM M tile plus
       # a 16-row tail (and the cluster-multicast TD head, b > 128)
       "mnih-b16", "mnih-b80", "mnih-b144", "scaled-b16", "scaled-b144"]


@pytest.mark.parametrize("kw,b", CASES, ids=IDS)
def test_gated_one_step(kw, b):
    """a1-a9 (+ a15): indices bit-exact, Q of a chunk plus a ragged tail, the loss and the gradient of every
    tensor within 2e-2 of the oracle (Alg. 1)."""
    cap = max(600, b + 88)
    dc, on, oc = nets(minibatch=b, replay_capacity=cap, precision=D.BF16, **kw)
    g, rp, raw, th0 = make(dc, on, cap, 21, 3)
    nq = b + 13 if b <= 64 else 45
    q, am = g.q_values(raw[0][:nq])
    qo, amo = O.q_values(on, th0, raw[0][:nq])
    assert np.max(np.abs(q - qo)) / np.max(np.abs(qo)) < TOL
    ok = near_tie_mask(qo, TOL)
    assert np.array_equal(am[ok], amo[ok])
    out = g.train(1, want_idx=True, want_loss=True, want_argmax=True)
    ref = O.run(on, oc, cap, [rp], th0, 1, want_grad0=True)
    idx = out["idx"][0]
    assert np.array_equal(idx, ref["idx"][0][0])
    assert O.min_abs_preact(on, th0, np.concatenate([rp.s[idx], rp.s_next[idx]])) >= GATE
    assert abs(out["loss"][0] - ref["loss"][0, 0]) <= TOL * ref["loss"][0, 0]
    qn, _ = O.q_values(on, th0, rp.s_next[idx])
    okn = near_tie_mask(qn, TOL)
    assert np.array_equal(out["argmax"][0][okn], ref["amax"][0, 0][okn])
    assert per_tensor_rel(g.params(D.PARAMS_GRAD), ref["grad0"], on) < TOL
    g.close()


@pytest.mark.parametrize("kw,steps", [(dict(), 10), (SCALED, 3)], ids=["mnih", "scaled"])
def test_gated_k_steps_delta_theta(kw, steps):
    """BASELINE.json configs[0]'s 10 SGD steps (scaled net: 3), free-running against the oracle's own
    trajectory, theta^ refreshed every C = 2 generations (a14): indices bit-exact, every step's loss and
    every tensor's Delta theta within 2e-2."""
    dc, on, oc = nets(minibatch=32, replay_capacity=1000, precision=D.BF16, lr=1e-5, rms_eps=1e-2, target_sync=2,
                      **kw)
    g, rp, _, th0 = make(dc, on, 1000, 1234, 5)
    out = g.train(steps, want_idx=True, want_loss=True)
    ref = O.run(on, oc, 1000, [rp], th0, steps)
    assert ref["rc"] == 0 and out["generation"] == ref["n"] == steps
    assert np.array_equal(out["idx"], ref["idx"][0])
    assert np.all(np.abs(out["loss"] - ref["loss"][0]) <= TOL * ref["loss"][0])
    th = g.params(D.PARAMS_SERVER)
    assert delta_rel(th, th0, ref["theta"], th0, on, ulps=steps) < TOL
    # r of Alg. 2 is quadratic in the gradients and free of theta's storage floor: 2 x the bar
    assert per_tensor_rel(g.params(D.PARAMS_RMS), ref["r"], on) < 2 * TOL
    assert np.array_equal(g.params(D.PARAMS_LOCAL), th)  # N = 1, n_fetch = 1: the working copy is theta
    assert O.min_abs_preact(on, ref["theta"], rp.s[:64]) >= 0.05  # still gated at the end
    g.close()


def test_gated_accumulate_n_push3():
    """a10: with n_push = 3 the pushed gradient is the sum of three steps' gradients at theta_0 (A8: no local
    update between pushes); after two rounds every tensor's Delta theta is within 2e-2."""
    dc, on, oc = nets(minibatch=32, replay_capacity=1000, precision=D.BF16, lr=1e-5, rms_eps=1e-2, n_push=3)
    g, rp, _, th0 = make(dc, on, 1000, 99, 6)
    out = g.train(3, want_idx=True)
    assert out["generation"] == 1
    acc = np.zeros_like(th0)
    for k in range(3):
        idx = out["idx"][k]
        y, _ = O.targets(on, th0, rp.s_next[idx], rp.r[idx], rp.term[idx], oc.gamma)
        acc += O.loss_grad(on, th0, rp.s[idx], rp.a[idx], y)[1]
    assert per_tensor_rel(g.params(D.PARAMS_GRAD), acc, on) < TOL
    g.train(3)
    ref = O.run(on, oc, 1000, [rp], th0, 6)
    assert delta_rel(g.params(D.PARAMS_SERVER), th0, ref["theta"], th0, on, ulps=2) < TOL
    assert per_tensor_rel(g.params(D.PARAMS_RMS), ref["r"], on) < 2 * TOL
    g.close()


@pytest.mark.parametrize("kw", [dict(), SCALED], ids=["mnih", "scaled"])
def test_gated_error_clip(kw):
    """a6 with err_clip = 1 (A3): small Q (output weights N(0, 0.1^2)) and rewards of +-4 give |delta| > 1 on
    the two thirds of the samples with r != 0 and |delta| < 1 on the rest; the clipped gradient matches the
    oracle's within 2e-2, and differs from the unclipped one (the test can fail)."""
    dc, on, oc = nets(minibatch=32, replay_capacity=500, precision=D.BF16, err_clip=1.0, **kw)
    g, rp, _, th0 = make(dc, on, 500, 31, 7, r_scale=4.0, out_std=0.1)
    out = g.train(1, want_idx=True)
    idx = out["idx"][0]
    y, _ = O.targets(on, th0, rp.s_next[idx], rp.r[idx], rp.term[idx], oc.gamma)
    q, _ = O.q_values(on, th0, rp.s[idx])
    delta = q[np.arange(32), rp.a[idx]] - y
    assert np.sum(np.abs(delta) > 1.0) >= 8 and np.sum(np.abs(delta) < 1.0) >= 4
    _, gc = O.loss_grad(on, th0, rp.s[idx], rp.a[idx], y, err_clip=1.0)
    _, gu = O.loss_grad(on, th0, rp.s[idx], rp.a[idx], y)
    assert per_tensor_rel(gu, gc, on) > 0.2
    assert per_tensor_rel(g.params(D.PARAMS_GRAD), gc, on) < TOL
    g.close()


@pytest.mark.parametrize("kw", [dict(), SCALED], ids=["mnih", "scaled"])
def test_target_refresh_and_bf16_working_copies(kw):
    """a14 (A10): after every step theta^ is bit-for-bit theta as of the last refresh (n - l >= C, C = 2),
    and both bf16 working copies the kernels read are the round-to-nearest-even bf16 of their fp32 theta."""
    dc, on, oc = nets(minibatch=32, replay_capacity=300, precision=D.BF16, lr=1e-2, target_sync=2, **kw)
    g, rp, _, th0 = make(dc, on, 300, 5, 8)
    hist = [g.params(D.PARAMS_LOCAL)]  # theta_n after n generations
    ell = 0
    for T in range(7):
        n = T  # N = 1, n_push = n_fetch = 1: the fetch at step T sees generation T
        if n - ell >= 2:
            ell = n
        g.train(1)
        hist.append(g.params(D.PARAMS_LOCAL))
        th_hat = g.params(D.PARAMS_TARGET)
        assert g.generation(D.PARAMS_TARGET) == ell
        assert np.array_equal(th_hat, hist[ell]), f"step {T}: theta^ is not theta_{ell}"
        assert np.array_equal(g.params(D.PARAMS_TARGET_BF16), bf16_rne(th_hat))
        assert np.array_equal(g.params(D.PARAMS_LOCAL_BF16), bf16_rne(hist[-1]))
    assert not np.array_equal(hist[2], hist[0]) and ell == 6
    g.close()
