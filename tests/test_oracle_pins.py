"""Pins of the fp64 oracle against things other than itself.

Every oracle function is checked here against a closed form, a worked example
(SPEC.md examples, cited), a library routine (scipy correlate, numpy matmul),
finite differences, brute force, or a published known-answer vector, so that a
dropped term, wrong sign/index or transposed operand fails at least one test.
"""
import math

import numpy as np
import pytest
from scipy import signal

from oracle import oracle as O
import synth

TINY = O.Net(frames=4, height=12, width=12, convs=((2, 4, 2), (3, 3, 1)), fcs=(4,), n_actions=3)


def he_theta(net, seed, scale=1.0):
    tt = O.tensor_table(net)
    stds = []
    for i, (off, cnt) in enumerate(tt):
        if i % 2 == 0:
            out_units = tt[i + 1][1]
            fan_in = cnt // out_units
            stds.append(scale * math.sqrt(2.0 / fan_in))
        else:
            stds.append(0.05 * scale)
    return synth.init_theta(tt, stds, seed).astype(np.float64)


# ---------------------------------------------------------------- shapes (O0)
def enumerate_params(convs, fcs, n_actions, F, H, W):
    total, c, h, w = 0, F, H, W
    for n, k, s in convs:
        for _ in range(n):            # one filter at a time: C*k*k weights + 1 bias
            total += c * k * k + 1
        c, h, w = n, (h - k) // s + 1, (w - k) // s + 1
    d = c * h * w
    for u in list(fcs) + [n_actions]:
        for _ in range(u):            # one unit at a time: D weights + 1 bias
            total += d + 1
        d = u
    return total


def test_param_count_mnih_and_scaled():
    # SURVEY §0 / BASELINE.md §2 values, checked by unit-by-unit enumeration
    assert O.param_count(O.MNIH) == 677686
    assert O.param_count(O.NATURE_SCALED) == 1693362
    for net in (O.MNIH, O.NATURE_SCALED, TINY):
        assert O.param_count(net) == enumerate_params(net.convs, net.fcs, net.n_actions, net.frames, net.height,
                                                      net.width)


def test_param_count_rejects_non_integer_conv_output():
    # S:65 "shape mismatch -> configuration error": (84-8)/3 is not an integer
    assert O.param_count(O.Net(convs=((16, 8, 3),))) == -1


def test_tensor_table_is_contiguous_w_then_b():
    tt = O.tensor_table(O.MNIH)
    assert [c for _, c in tt] == [16 * 4 * 64, 16, 32 * 16 * 16, 32, 256 * 2592, 256, 6 * 256, 6]
    off = 0
    for o, c in tt:
        assert o == off
        off += c


# ---------------------------------------------------------------- sampler (O3)
@pytest.mark.parametrize("ctr,key,expect", [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
])
def test_philox_known_answers(ctr, key, expect):
    # Random123 Philox4x32-10 known-answer vectors
    assert O.philox4x32_10(ctr, key) == expect


def test_sample_index_mapping_bruteforce():
    seed = 0x123456789ABCDEF
    for (rank, T, j, size) in [(0, 0, 0, 1000), (3, 2**33 + 5, 17, 1_000_000), (1, 7, 31, 1), (2, 9, 4, 3)]:
        x = O.philox4x32_10([j, T & 0xFFFFFFFF, T >> 32, rank], [seed & 0xFFFFFFFF, seed >> 32])
        u = (x[0] << 32) | x[1]
        assert O.sample_index(seed, rank, T, j, size) == (u * size) >> 64   # python big ints


def test_sample_index_size_one_is_zero():
    # S:163 size-1 buffer -> always the single entry
    assert all(O.sample_index(5, 0, T, j, 1) == 0 for T in range(20) for j in range(32))


def test_sample_index_uniform_chi_square():
    # S:164 chi-square goodness of fit at 0.01 over 1e5 draws
    size = 10
    counts = np.zeros(size)
    for T in range(3125):
        for j in range(32):
            counts[O.sample_index(0xD15EA5E, 0, T, j, size)] += 1
    n = counts.sum()
    chi2 = ((counts - n / size) ** 2 / (n / size)).sum()
    assert chi2 < 21.666  # chi2_{0.99}(9)


# ---------------------------------------------------------------- layers (O5)
def test_conv_zero_input_gives_bias():
    out = O.conv_forward(np.zeros((3, 9, 9)), np.random.default_rng(0).normal(size=(2, 3, 3, 3)),
                         np.array([0.5, -1.25]), 2)
    assert np.all(out[0] == 0.5) and np.all(out[1] == -1.25)


def test_conv_scalar_case():
    assert O.conv_forward(np.array([[[3.0]]]), np.array([[[[-2.0]]]]), np.array([0.25]), 1)[0, 0, 0] == -5.75


def test_conv_1x3x3_2x2_window_dot_products():
    x = np.arange(9, dtype=float).reshape(1, 3, 3)
    w = np.array([[[[1.0, 2.0], [3.0, 4.0]]]])
    out = O.conv_forward(x, w, np.zeros(1), 1)
    expect = [[0 * 1 + 1 * 2 + 3 * 3 + 4 * 4, 1 * 1 + 2 * 2 + 4 * 3 + 5 * 4],
              [3 * 1 + 4 * 2 + 6 * 3 + 7 * 4, 4 * 1 + 5 * 2 + 7 * 3 + 8 * 4]]
    assert np.array_equal(out[0], np.array(expect, float))


@pytest.mark.parametrize("C,H,N,k,s", [(4, 84, 16, 8, 4), (16, 20, 32, 4, 2), (3, 11, 5, 3, 1), (2, 13, 3, 5, 2)])
def test_conv_matches_scipy_correlate(C, H, N, k, s):
    rng = np.random.default_rng(C * 100 + k)
    x = rng.normal(size=(C, H, H))
    w = rng.normal(size=(N, C, k, k))
    b = rng.normal(size=N)
    out = O.conv_forward(x, w, b, s)
    for n in range(N):
        full = sum(signal.correlate(x[c], w[n, c], mode="valid") for c in range(C))
        ref = full[::s, ::s] + b[n]
        np.testing.assert_allclose(out[n], ref, rtol=1e-12, atol=1e-11)


def test_fc_examples():
    # S:76-78
    assert np.array_equal(O.fc_forward(np.array([1.0, 1.0]), np.array([[1.0, 2.0], [3.0, 4.0]]), np.zeros(2)),
                          np.array([3.0, 7.0]))
    x = np.array([0.3, -2.0, 5.0])
    assert np.array_equal(O.fc_forward(x, np.eye(3), np.zeros(3)), x)
    assert np.array_equal(O.fc_forward(np.zeros(3), np.ones((2, 3)), np.array([4.0, -1.0])), np.array([4.0, -1.0]))
    rng = np.random.default_rng(3)
    W, xx, bb = rng.normal(size=(7, 11)), rng.normal(size=11), rng.normal(size=7)
    np.testing.assert_allclose(O.fc_forward(xx, W, bb), W @ xx + bb, rtol=1e-13)


# ---------------------------------------------------------------- network (O4, O5)
def test_input_normalisation_exhaustive():
    # O4: x = u8/255 — a 1x1x1 state straight into a 1-unit linear output with weight 1
    net = O.Net(frames=1, height=1, width=1, convs=(), fcs=(), n_actions=1)
    theta = np.array([1.0, 0.0])
    states = np.arange(256, dtype=np.uint8).reshape(256, 1, 1, 1)
    q, _ = O.q_values(net, theta, states)
    assert np.array_equal(q[:, 0], np.arange(256) / 255.0)


def test_zero_weights_give_output_bias():
    # S:85 zero model -> zero Q; with only the output bias non-zero Q == that bias
    P = O.param_count(O.MNIH)
    theta = np.zeros(P)
    s = synth.g_uniform(1, 4, 84, 84, 6, 1)[0]
    q, _ = O.q_values(O.MNIH, theta, s)
    assert np.all(q == 0.0)
    theta[-6:] = [0.1, -0.2, 0.3, 0.4, -0.5, 0.6]
    q, am = O.q_values(O.MNIH, theta, s)
    assert np.array_equal(q[0], theta[-6:]) and am[0] == 5


def numpy_forward(net, theta, x):
    """Independent composition with library routines (scipy correlate, numpy matmul)."""
    tt = O.tensor_table(net)
    a = x
    t = 0
    c, h, w = net.frames, net.height, net.width
    for (n, k, s) in net.convs:
        W = theta[tt[t][0]:tt[t][0] + tt[t][1]].reshape(n, c, k, k)
        b = theta[tt[t + 1][0]:tt[t + 1][0] + n]
        z = np.stack([sum(signal.correlate(a[ci], W[ni, ci], mode="valid") for ci in range(c))[::s, ::s] + b[ni]
                      for ni in range(n)])
        a = np.maximum(z, 0.0)
        c, h, w = n, z.shape[1], z.shape[2]
        t += 2
    a = a.reshape(-1)
    units = list(net.fcs) + [net.n_actions]
    for i, u in enumerate(units):
        W = theta[tt[t][0]:tt[t][0] + tt[t][1]].reshape(u, -1)
        b = theta[tt[t + 1][0]:tt[t + 1][0] + u]
        z = W @ a + b
        a = np.maximum(z, 0.0) if i + 1 < len(units) else z
        t += 2
    return a


@pytest.mark.parametrize("net", [TINY, O.MNIH], ids=["tiny", "mnih"])
def test_forward_matches_library_composition(net):
    theta = he_theta(net, 11)
    s = synth.g_uniform(2, net.frames, net.height, net.width, net.n_actions, 5)[0]
    q, am = O.q_values(net, theta, s)
    for i in range(2):
        ref = numpy_forward(net, theta, s[i].astype(np.float64) / 255.0)
        np.testing.assert_allclose(q[i], ref, rtol=1e-11, atol=1e-12)
        assert am[i] == int(np.argmax(ref))


def test_min_abs_preact_matches_library_composition():
    theta = he_theta(TINY, 13)
    s = synth.g_uniform(3, 4, 12, 12, 3, 4)[0]
    ref = np.inf
    tt = O.tensor_table(TINY)
    for i in range(3):
        a, c, t = s[i] / 255.0, 4, 0
        for (n, k, st) in TINY.convs:
            W = theta[tt[t][0]:tt[t][0] + tt[t][1]].reshape(n, c, k, k)
            b = theta[tt[t + 1][0]:tt[t + 1][0] + n]
            z = np.stack([sum(signal.correlate(a[ci], W[ni, ci], mode="valid") for ci in range(c))[::st, ::st] + b[ni]
                          for ni in range(n)])
            ref = min(ref, np.min(np.abs(z)))
            a, c, t = np.maximum(z, 0), n, t + 2
        W = theta[tt[t][0]:tt[t][0] + tt[t][1]].reshape(4, -1)
        z = W @ a.ravel() + theta[tt[t + 1][0]:tt[t + 1][0] + 4]
        ref = min(ref, np.min(np.abs(z)))
    assert abs(O.min_abs_preact(TINY, theta, s) - ref) <= 1e-12 * max(ref, 1e-300) + 1e-15


def bias_only_net_theta(net, out_bias):
    theta = np.zeros(O.param_count(net))
    theta[-net.n_actions:] = out_bias
    return theta


def test_argmax_examples_and_ties():
    # [0.1,0.9,0.3,0.2] -> 1 ; tie [0.5,0.5] -> 0 (lowest index)
    net4 = O.Net(frames=1, height=2, width=2, convs=(), fcs=(), n_actions=4)
    s = np.zeros((1, 1, 2, 2), np.uint8)
    _, am = O.q_values(net4, bias_only_net_theta(net4, [0.1, 0.9, 0.3, 0.2]), s)
    assert am[0] == 1
    net2 = O.Net(frames=1, height=2, width=2, convs=(), fcs=(), n_actions=2)
    _, am = O.q_values(net2, bias_only_net_theta(net2, [0.5, 0.5]), s)
    assert am[0] == 0


def test_argmax_bruteforce_random():
    rng = np.random.default_rng(9)
    net = O.Net(frames=1, height=3, width=3, convs=(), fcs=(), n_actions=7)
    for _ in range(50):
        bias = rng.integers(-3, 3, size=7) / 2.0  # frequent ties
        _, am = O.q_values(net, bias_only_net_theta(net, bias), np.zeros((1, 1, 3, 3), np.uint8))
        best = max(range(7), key=lambda a: (bias[a], -a))
        assert am[0] == best


# ---------------------------------------------------------------- targets (O6)
def test_targets_hand_values():
    # terminal r=-1 -> -1 ; r=1, gamma=0.5, max Q^=2 -> 2.0 ; gamma=0 -> r
    net = O.Net(frames=1, height=2, width=2, convs=(), fcs=(), n_actions=3)
    th = bias_only_net_theta(net, [2.0, -1.0, 0.5])
    sn = np.zeros((3, 1, 2, 2), np.uint8)
    y, am = O.targets(net, th, sn, [-1.0, 1.0, 1.0], [1, 0, 0], 0.5)
    assert y[0] == -1.0 and y[1] == 2.0 and am[1] == 0
    y, _ = O.targets(net, th, sn, [-1.0, 1.0, 0.0], [0, 0, 0], 0.0)
    assert np.array_equal(y, [-1.0, 1.0, 0.0])


def test_terminal_target_independent_of_theta_hat():
    th1 = he_theta(TINY, 1)
    th2 = he_theta(TINY, 2) * 1e3
    sn = synth.g_uniform(4, 4, 12, 12, 3, 8)[3]
    y1, _ = O.targets(TINY, th1, sn, [0.5, -1, 1, 0], [1, 1, 1, 1], 0.99)
    y2, _ = O.targets(TINY, th2, sn, [0.5, -1, 1, 0], [1, 1, 1, 1], 0.99)
    assert np.array_equal(y1, [0.5, -1, 1, 0]) and np.array_equal(y2, y1)


def test_targets_bellman_against_forward():
    th = he_theta(TINY, 4)
    s, a, r, sn, term = synth.g_uniform(6, 4, 12, 12, 3, 21)
    term[:] = [0, 1, 0, 0, 1, 0]
    y, am = O.targets(TINY, th, sn, r, term, 0.9)
    for j in range(6):
        q = numpy_forward(TINY, th, sn[j] / 255.0)
        expect = r[j] if term[j] else r[j] + 0.9 * q.max()
        assert abs(y[j] - expect) < 1e-12
        assert am[j] == int(np.argmax(q))


# ---------------------------------------------------------------- gradient (O7)
def fd_loss(net, theta, x, a, y):
    Q = np.array([numpy_forward(net, theta, x[j]) for j in range(len(a))])
    return np.mean(0.5 * (Q[np.arange(len(a)), a] - y) ** 2)


def test_gradient_matches_central_finite_differences():
    # central FD, h = 1e-5, relative error < 1e-4, fp64
    net = TINY
    theta = he_theta(net, 31)
    rng = np.random.default_rng(5)
    b = 3
    x = rng.random((b, 4, 12, 12))
    a = np.array([0, 2, 1], np.int32)
    y = rng.normal(size=b)
    loss, g = O.loss_grad_x(net, theta, x, a, y)
    assert abs(loss - fd_loss(net, theta, x, a, y)) < 1e-12
    h = 1e-5
    fd = np.zeros_like(theta)
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        fd[i] = (fd_loss(net, tp, x, a, y) - fd_loss(net, tm, x, a, y)) / (2 * h)
    rel = np.abs(g - fd) / np.maximum(np.abs(fd), 1e-6)
    assert np.max(rel) < 1e-4, np.max(rel)
    assert np.max(np.abs(g)) > 1e-3  # the check is not vacuous


def test_zero_residual_gives_exactly_zero_gradient():
    # S:94 / S:109
    theta = he_theta(TINY, 7)
    s, a, _, _, _ = synth.g_uniform(4, 4, 12, 12, 3, 2)
    q, _ = O.q_values(TINY, theta, s)
    y = q[np.arange(4), a]
    loss, g = O.loss_grad(TINY, theta, s, a, y)
    assert loss == 0.0 and np.all(g == 0.0)


def test_b1_linear_closed_form():
    # Q = w.x (+b), grad_w = (w.x - y) x on the taken action only
    net = O.Net(frames=1, height=2, width=3, convs=(), fcs=(), n_actions=2)
    rng = np.random.default_rng(1)
    theta = rng.normal(size=O.param_count(net))
    s = rng.integers(0, 256, size=(1, 1, 2, 3), dtype=np.uint8)
    x = s.reshape(-1) / 255.0
    W, bb = theta[:12].reshape(2, 6), theta[12:]
    a, y = 1, 0.7
    _, g = O.loss_grad(net, theta, s, [a], [y])
    resid = W[a] @ x + bb[a] - y
    expect = np.zeros_like(theta)
    expect[6:12] = resid * x
    expect[13] = resid
    np.testing.assert_allclose(g, expect, rtol=1e-13, atol=1e-15)


def test_error_clip():
    # A3: |delta| < c leaves the gradient unchanged; beyond c it is clamped to c
    net = O.Net(frames=1, height=2, width=3, convs=(), fcs=(), n_actions=2)
    rng = np.random.default_rng(2)
    theta = rng.normal(size=O.param_count(net))
    s = rng.integers(0, 256, size=(1, 1, 2, 3), dtype=np.uint8)
    q, _ = O.q_values(net, theta, s)
    y_small, y_big = q[0, 0] - 0.3, q[0, 0] - 5.0
    _, g0 = O.loss_grad(net, theta, s, [0], [y_small])
    _, g1 = O.loss_grad(net, theta, s, [0], [y_small], err_clip=1.0)
    assert np.array_equal(g0, g1)
    _, g2 = O.loss_grad(net, theta, s, [0], [y_big])
    l3, g3 = O.loss_grad(net, theta, s, [0], [y_big], err_clip=1.0)
    np.testing.assert_allclose(g3, g2 / 5.0, rtol=1e-12, atol=1e-15)
    assert abs(l3 - 0.5 * 25.0) < 1e-9  # reported loss is the unclipped one (A27)


# ---------------------------------------------------------------- RMSProp (O9)
def test_rmsprop_hand_values():
    # r = 0, dtheta = 2, alpha = 0.1 -> r' = 0.4, step = 0.2/sqrt(0.4 + 1e-8) ~= 0.316227762
    th, r = O.rmsprop(np.array([1.0]), np.array([0.0]), np.array([2.0]), 0.1)
    assert abs(r[0] - 0.4) < 1e-15
    assert abs((1.0 - th[0]) - 0.316227762) < 1e-9
    # S:328 zero gradient: theta unchanged, r scaled by 0.9
    th, r = O.rmsprop(np.array([0.3, -2.0]), np.array([0.5, 2.0]), np.zeros(2), 0.1)
    assert np.array_equal(th, [0.3, -2.0]) and np.allclose(r, [0.45, 1.8], rtol=1e-15)


def test_rmsprop_r_updated_before_theta():
    # A5: theta uses the NEW r
    th, r = O.rmsprop(np.array([0.0]), np.array([4.0]), np.array([1.0]), 1.0, 0.9, 0.0)
    assert abs(r[0] - 3.7) < 1e-15 and abs(th[0] + 1.0 / math.sqrt(3.7)) < 1e-15


def test_gradient_does_not_depend_on_the_thread_count():
    """or_loss_grad sums the per-sample terms of P:123 in sample order whatever the number of OpenMP threads
    that computed them (bench.py's all-core cpu_baseline times the same arithmetic as the tests use)."""
    net = O.Net(frames=3, height=17, width=13, convs=((5, 5, 2), (6, 3, 2)), fcs=(19,), n_actions=5)
    tt = O.tensor_table(net)
    rng = np.random.default_rng(5)
    th = rng.normal(0, 0.3, O.param_count(net))
    s = rng.integers(0, 256, (37, 3, 17, 13), dtype=np.uint8)   # 2 blocks of 16 + a ragged 5
    a = rng.integers(0, 5, 37).astype(np.int32)
    y = rng.normal(0, 1, 37)
    n0 = O.threads()
    try:
        O.set_threads(1)
        l1, g1 = O.loss_grad(net, th, s, a, y)
        O.set_threads(0)
        lk, gk = O.loss_grad(net, th, s, a, y)
    finally:
        O.set_threads(n0)
    assert l1 == lk and np.array_equal(g1, gk)
    assert len(tt) == 8
