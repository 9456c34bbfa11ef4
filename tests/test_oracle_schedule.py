"""Pins of the oracle's replay + schedule (or_run: O2, O8-O12) against hand-built
serial loops over the individually pinned primitives.

The primitives (sampler, targets, gradient, RMSProp) are pinned in
test_oracle_pins.py; here the loops re-derive Alg. 1 / Alg. 2 step by step so a
wrong fetch/push/refresh order, a wrong accumulation or a wrong replay slot in
or_run fails.
"""
import numpy as np
import pytest

from oracle import oracle as O
import synth
from tests.test_oracle_pins import TINY, he_theta

CAP = 40


def make_replays(n_rep, n_push_each, seed, net=TINY):
    out = []
    for k in range(n_rep):
        s, a, r, sn, t = synth.g_uniform(n_push_each, net.frames, net.height, net.width, net.n_actions, seed + k)
        out.append(O.Replay(s, a, r.astype(np.float64), sn, t))
    return out


def ring_view(rp, cap):
    """last-N ring contents: push i -> slot i mod cap."""
    n = len(rp.a)
    slot_of = {}
    for i in range(n):
        slot_of[i % cap] = i
    size = min(n, cap)
    return [slot_of[sl] for sl in range(size)]


def serial_reference(cfg, replays, theta0, steps, cap, net=TINY, stale=None):
    """Alg. 1 x N + Alg. 2 written out: fetch every n_fetch (theta as it was fetch_lag rounds
    ago, O13), refresh when n-l >= C, accumulate, mean over N*n_push, one RMSProp per round."""
    N, b = cfg.n_replicas, cfg.minibatch
    history = [theta0.copy()]          # server theta after 0, 1, 2, ... rounds
    used = {}                          # (k, T) -> generation of the theta the gradient used
    theta = theta0.copy()
    r = np.zeros_like(theta)
    n = 0
    th_local = [theta0.copy() for _ in range(N)]
    th_hat = [theta0.copy() for _ in range(N)]
    n_loc = [0] * N
    ell = [0] * N
    acc = [np.zeros_like(theta) for _ in range(N)]
    views = [ring_view(rp, cap) for rp in replays]
    for T in range(steps):
        for k in range(N):
            if T % cfg.n_fetch == 0:
                m = max(n - cfg.fetch_lag, 0)
                if cfg.fetch_gen is not None:   # the realised schedule of an asynchronous run (A40)
                    m = int(cfg.fetch_gen[k][T // cfg.n_fetch])
                th_local[k] = history[m].copy()
                n_loc[k] = m
                if n_loc[k] - ell[k] >= cfg.target_sync:
                    th_hat[k] = th_local[k].copy()
                    ell[k] = n_loc[k]
            rp, view = replays[k], views[k]
            idx = [view[O.sample_index(cfg.seed, k, T, j, len(view))] for j in range(b)]
            y, _ = O.targets(net, th_hat[k], rp.s_next[idx], rp.r[idx], rp.term[idx], cfg.gamma)
            _, g = O.loss_grad(net, th_local[k], rp.s[idx], rp.a[idx], y, cfg.err_clip)
            acc[k] += g
            used[(k, T)] = n_loc[k]
        if (T + 1) % cfg.n_push == 0 and cfg.server_rule == 1:
            # Alg. 2 literally (A33): each worker's gradient (mean of its n_push) applied in rank order
            if stale is not None:
                for k in range(N):
                    for t in range(T + 1 - cfg.n_push, T + 1):
                        stale[min(n - used[(k, t)], 31)] += 1
            for k in range(N):
                theta, r = O.rmsprop(theta, r, acc[k] / cfg.n_push, cfg.lr, cfg.rms_decay, cfg.rms_eps)
                n += 1
                history.append(theta.copy())
            acc = [np.zeros_like(theta) for _ in range(N)]
        elif (T + 1) % cfg.n_push == 0:
            gbar = sum(acc) / (N * cfg.n_push)
            if stale is not None:
                for k in range(N):
                    for t in range(T + 1 - cfg.n_push, T + 1):
                        stale[min(n - used[(k, t)], 31)] += 1
            theta, r = O.rmsprop(theta, r, gbar, cfg.lr, cfg.rms_decay, cfg.rms_eps)
            n += 1
            history.append(theta.copy())
            acc = [np.zeros_like(theta) for _ in range(N)]
    return theta, r, n


@pytest.mark.parametrize("N,n_push,n_fetch,C", [
    (1, 1, 1, 10**9),   # serial DQN (Alg. 1 with a fixed target)
    (1, 1, 1, 1),       # C = 1: standard Q-learning targets
    (1, 1, 1, 2),
    (2, 1, 1, 3),       # Downpour deterministic, N = 2
    (3, 2, 1, 2),       # accumulate over 2 steps
    (2, 1, 3, 1),       # stale local model between fetches
    (2, 3, 2, 2),
])
def test_run_equals_serial_loop(N, n_push, n_fetch, C):
    cfg = O.TrainCfg(n_replicas=N, minibatch=3, n_push=n_push, n_fetch=n_fetch, target_sync=C, lr=1e-2,
                     gamma=0.9)
    replays = make_replays(N, 50, 100)  # 50 pushes into a 40-slot ring: wraps
    theta0 = he_theta(TINY, 3)
    steps = 6
    out = O.run(TINY, cfg, CAP, replays, theta0, steps)
    assert out["rc"] == 0
    th, r, n = serial_reference(cfg, replays, theta0, steps, CAP)
    assert out["n"] == n == steps // n_push
    np.testing.assert_allclose(out["theta"], th, rtol=0, atol=1e-13)
    np.testing.assert_allclose(out["r"], r, rtol=1e-12, atol=1e-18)


def test_n_replicas_equal_one_batch_of_N_b():
    # A7: with n_push = n_fetch = 1, N replicas == serial DQN with batch N*b on the
    # concatenation of the replicas' minibatches (to fp64 summation order)
    N, b = 3, 2
    cfg = O.TrainCfg(n_replicas=N, minibatch=b, lr=5e-3, gamma=0.95, target_sync=10**9)
    replays = make_replays(N, 30, 7)
    theta0 = he_theta(TINY, 5)
    out = O.run(TINY, cfg, CAP, replays, theta0, 2)
    theta, r = theta0.copy(), np.zeros_like(theta0)
    for T in range(2):
        S, A, Y = [], [], []
        for k in range(N):
            rp = replays[k]
            idx = [O.sample_index(cfg.seed, k, T, j, 30) for j in range(b)]
            y, _ = O.targets(TINY, theta0, rp.s_next[idx], rp.r[idx], rp.term[idx], cfg.gamma)
            S.append(rp.s[idx]); A.append(rp.a[idx]); Y.append(y)
        _, g = O.loss_grad(TINY, theta, np.concatenate(S), np.concatenate(A), np.concatenate(Y))
        theta, r = O.rmsprop(theta, r, g, cfg.lr)
    np.testing.assert_allclose(out["theta"], theta, rtol=0, atol=1e-12)


def test_targets_fixed_between_refreshes():
    # targets do not move with the live theta while theta^ is held; with
    # gamma = 0 the live-theta path cannot leak into y, so loss reveals r only.
    net = O.Net(frames=1, height=2, width=2, convs=(), fcs=(), n_actions=2)
    P = O.param_count(net)
    s = np.zeros((3, 1, 2, 2), np.uint8)
    rp = O.Replay(s, np.zeros(3, np.int32), np.array([1.0, 2.0, 3.0]), s, np.zeros(3, np.uint8))
    cfg = O.TrainCfg(minibatch=1, gamma=0.0, lr=0.0)
    out = O.run(net, cfg, 2, [rp], np.zeros(P), 8)
    # FIFO with capacity 2: slot 0 holds push 2 (r=3), slot 1 holds push 1 (r=2)
    r_of_slot = {0: 3.0, 1: 2.0}
    for T in range(8):
        sl = out["idx"][0, T, 0]
        assert out["loss"][0, T] == 0.5 * r_of_slot[sl] ** 2


def test_sampled_idx_follow_O3_and_ring_size():
    cfg = O.TrainCfg(n_replicas=2, minibatch=5, seed=77)
    replays = make_replays(2, 13, 3)
    out = O.run(TINY, cfg, CAP, replays, he_theta(TINY, 1), 3)
    for k in range(2):
        for T in range(3):
            assert list(out["idx"][k, T]) == [O.sample_index(77, k, T, j, 13) for j in range(5)]


def test_empty_replay_is_an_error():
    rp = O.Replay(np.zeros((0, 4, 12, 12), np.uint8), np.zeros(0, np.int32), np.zeros(0), np.zeros((0, 4, 12, 12),
                  np.uint8), np.zeros(0, np.uint8))
    out = O.run(TINY, O.TrainCfg(minibatch=2), CAP, [rp], he_theta(TINY, 1), 1)
    assert out["rc"] == -2


def test_nonfinite_reward_is_flagged_and_not_applied():
    replays = make_replays(1, 5, 9)
    replays[0].r[:] = np.inf
    theta0 = he_theta(TINY, 2)
    out = O.run(TINY, O.TrainCfg(minibatch=2), CAP, replays, theta0, 1)
    assert out["rc"] == -3
    moved = out["theta"] != theta0
    # every element whose mean gradient is non-finite keeps its value (A24)
    assert np.all(np.isfinite(out["theta"])) and not np.all(moved)


@pytest.mark.parametrize("N,n_push,n_fetch,lag", [(1, 1, 1, 1), (2, 2, 2, 1), (2, 3, 1, 2), (1, 2, 3, 1)])
def test_async_lag_twin_equals_serial_loop(N, n_push, n_fetch, lag):
    """O13: the asynchronous mode's deterministic twin — fetches land `lag` rounds late — and its
    staleness histogram (A25) against the written-out loop."""
    cfg = O.TrainCfg(n_replicas=N, minibatch=3, n_push=n_push, n_fetch=n_fetch, target_sync=2, lr=1e-2,
                     gamma=0.9, fetch_lag=lag)
    replays = make_replays(N, 50, 300)
    theta0 = he_theta(TINY, 4)
    steps = 7
    out = O.run(TINY, cfg, CAP, replays, theta0, steps)
    stale = np.zeros(32, np.int64)
    th, r, n = serial_reference(cfg, replays, theta0, steps, CAP, stale=stale)
    assert out["n"] == n
    np.testing.assert_allclose(out["theta"], th, rtol=0, atol=1e-13)
    assert np.array_equal(out["staleness"], stale)
    assert stale.sum() == N * n_push * (steps // n_push)


def test_lag1_one_step_rounds_have_staleness_one():
    # n_push = n_fetch = 1, lag 1: round 0 uses theta^(0) (staleness 0), every later round theta^(n-1)
    cfg = O.TrainCfg(n_replicas=1, minibatch=2, fetch_lag=1)
    out = O.run(TINY, cfg, CAP, make_replays(1, 30, 5), he_theta(TINY, 1), 6)
    assert out["staleness"][0] == 1 and out["staleness"][1] == 5 and out["staleness"].sum() == 6


@pytest.mark.parametrize("N,n_push,n_fetch,C,lag", [(2, 1, 1, 2, 0), (3, 2, 3, 1, 0), (2, 1, 1, 1, 1)])
def test_per_gradient_rule_equals_serial_loop(N, n_push, n_fetch, C, lag):
    """A33: server_rule = 1 applies every worker's gradient in turn (one RMSProp and n += 1 each)."""
    cfg = O.TrainCfg(n_replicas=N, minibatch=4, n_push=n_push, n_fetch=n_fetch, target_sync=C, lr=1e-2,
                     fetch_lag=lag, server_rule=1)
    reps = make_replays(N, 30, 71)
    th0 = he_theta(TINY, 5)
    ref = O.run(TINY, cfg, CAP, reps, th0, 6)
    th, r, n = serial_reference(cfg, reps, th0, 6, CAP)
    assert ref["n"] == n == N * (6 // n_push)
    assert np.allclose(ref["theta"], th, rtol=0, atol=1e-13)
    assert np.allclose(ref["r"], r, rtol=0, atol=1e-13)


def test_per_gradient_rule_with_one_worker_is_the_mean_rule():
    for n_push in (1, 2):
        base = O.TrainCfg(n_replicas=1, minibatch=4, n_push=n_push, target_sync=3, lr=1e-2)
        per = O.TrainCfg(n_replicas=1, minibatch=4, n_push=n_push, target_sync=3, lr=1e-2, server_rule=1)
        reps = make_replays(1, 30, 72)
        th0 = he_theta(TINY, 6)
        a, b = O.run(TINY, base, CAP, reps, th0, 6), O.run(TINY, per, CAP, reps, th0, 6)
        assert np.array_equal(a["theta"], b["theta"]) and a["n"] == b["n"]


def test_per_gradient_rule_two_equal_gradients_closed_form():
    """Two applications of the same gradient (Alg. 2 P:142-146 twice): r1 = .9 r + .1 g^2,
    th1 = th - a g / sqrt(r1 + eps), then r2, th2 from (th1, r1)."""
    g, th, r, a, eps = 0.3, 0.5, 0.2, 0.01, 1e-8
    r1 = 0.9 * r + 0.1 * g * g
    th1 = th - a * g / np.sqrt(r1 + eps)
    r2 = 0.9 * r1 + 0.1 * g * g
    th2 = th1 - a * g / np.sqrt(r2 + eps)
    t, rr = np.array([th]), np.array([r])
    for _ in range(2):
        t, rr = O.rmsprop(t, rr, np.array([g]), a, 0.9, eps)
    assert abs(t[0] - th2) < 1e-15 and abs(rr[0] - r2) < 1e-15


@pytest.mark.parametrize("N,n_push,n_fetch", [(1, 1, 1), (2, 2, 1), (2, 1, 3), (3, 2, 2)])
def test_realised_async_schedule_equals_serial_loop(N, n_push, n_fetch):
    """O13 generalised (A40): every fetch returns a generation chosen by the asynchronous run (any published
    one, here drawn at random from the last three); or_run with that schedule equals the written-out loop,
    and the fixed-lag schedules reproduce fetch_lag = 0 / 1 exactly."""
    steps = 9
    rng = np.random.default_rng(N * 100 + n_push * 10 + n_fetch)
    nf = -(-steps // n_fetch)
    gen_at = [(f * n_fetch) // n_push for f in range(nf)]   # server generation when fetch f happens (lock-step)
    fg = np.array([[max(g - int(rng.integers(0, 3)), 0) for g in gen_at] for _ in range(N)], np.int64)
    reps = make_replays(N, 60, 7)
    th0 = he_theta(TINY, 4)
    cfg = O.TrainCfg(n_replicas=N, minibatch=4, n_push=n_push, n_fetch=n_fetch, target_sync=2, lr=3e-3, gamma=0.9,
                     fetch_gen=fg)
    ref = serial_reference(cfg, reps, th0, steps, CAP)
    out = O.run(TINY, cfg, CAP, reps, th0, steps)
    assert out["rc"] == 0
    assert np.allclose(out["theta"], ref[0], rtol=0, atol=1e-12)
    for lag in (0, 1):
        fixed = np.array([[max(g - lag, 0) for g in gen_at] for _ in range(N)], np.int64)
        c1 = O.TrainCfg(**{**cfg.__dict__, "fetch_gen": fixed})
        c2 = O.TrainCfg(**{**cfg.__dict__, "fetch_gen": None, "fetch_lag": lag})
        assert np.array_equal(O.run(TINY, c1, CAP, reps, th0, steps)["theta"], O.run(TINY, c2, CAP, reps, th0, steps)["theta"])


@pytest.mark.parametrize("N,n_push", [(2, 2), (3, 1)])
def test_realised_async_schedule_per_gradient_rule_equals_serial_loop(N, n_push):
    """A33 + A40 (the asynchronous per-gradient mode): rounds publish only whole rounds (generations k N), every
    fetch takes one of the last three published; or_run equals the written-out loop."""
    steps = 8
    rng = np.random.default_rng(N * 10 + n_push)
    rounds_at = [T // n_push for T in range(steps)]      # rounds completed when fetch T happens (n_fetch = 1)
    fg = np.array([[max(r - int(rng.integers(0, 3)), 0) * N for r in rounds_at] for _ in range(N)], np.int64)
    reps = make_replays(N, 60, 9)
    th0 = he_theta(TINY, 5)
    cfg = O.TrainCfg(n_replicas=N, minibatch=4, n_push=n_push, n_fetch=1, target_sync=3, lr=3e-3, gamma=0.9,
                     fetch_gen=fg, server_rule=1)
    ref = serial_reference(cfg, reps, th0, steps, CAP)
    out = O.run(TINY, cfg, CAP, reps, th0, steps)
    assert out["rc"] == 0 and out["n"] == (steps // n_push) * N
    assert np.allclose(out["theta"], ref[0], rtol=0, atol=1e-12)


def test_realised_schedule_rejects_an_unpublished_generation():
    reps = make_replays(1, 30, 3)
    fg = np.array([[0, 5, 1]], np.int64)   # generation 5 does not exist at step 1
    cfg = O.TrainCfg(n_replicas=1, minibatch=2, fetch_gen=fg)
    assert O.run(TINY, cfg, CAP, reps, he_theta(TINY, 1), 3)["rc"] == -4
