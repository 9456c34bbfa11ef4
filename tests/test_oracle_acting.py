"""Pins of the oracle's acting side (NEXT-3): the Snake game of P:216 with the rule closures of SPEC
S:216-262 (readings A34-A36 in DESIGN.md), the eps-greedy behaviour policy and the collector
loop (Alg. 1). CPU only."""
import numpy as np
import pytest
from scipy import stats

from oracle import oracle as O

SEED = 0x5EED


def body(g):
    return [int(c) for c in g.body[:g.len]]


def test_reset_matches_spec_examples():
    n = 5
    g = O.snake_reset(n, SEED, 0, 7)
    assert g.len == 2 and g.dir == 1 and g.since == 0              # "starts with body length of two", heading right
    assert body(g) == [2 * n + 2, 2 * n + 1]                       # horizontal at the grid centre
    assert g.apple not in body(g) and 0 <= g.apple < n * n          # apple on a free cell
    h = O.snake_reset(n, SEED, 0, 7)
    assert body(h) == body(g) and h.apple == g.apple                 # same draw -> same state


def test_apple_is_uniform_over_free_cells():
    n = 5
    counts = np.zeros(n * n, np.int64)
    for t in range(20000):
        counts[O.snake_reset(n, SEED, 3, t).apple] += 1
    occupied = [2 * n + 2, 2 * n + 1]
    assert counts[occupied].sum() == 0
    free = np.delete(counts, occupied)
    assert stats.chisquare(free).pvalue > 0.01


def test_plain_move_reverse_and_wall():
    n = 6
    g = O.snake_reset(n, SEED, 0, 0)
    g.apple = 0                                                      # out of the way (top-left corner)
    r, term = O.snake_step(g, n, 3, SEED, 0, 1)                      # left = reverse of right: keeps moving right
    assert (r, term) == (0.0, False) and g.dir == 1
    assert body(g) == [3 * n + 4, 3 * n + 3] and g.since == 1        # head advanced, tail followed, length kept
    r, term = O.snake_step(g, n, 1, SEED, 0, 2)                      # to x = 5, the last column
    assert (r, term) == (0.0, False)
    before = body(g)
    r, term = O.snake_step(g, n, 1, SEED, 0, 3)                      # into the wall
    assert (r, term) == (-1.0, True) and body(g) == before           # death, state left unchanged


def test_eating_grows_and_scores():
    n = 6
    g = O.snake_reset(n, SEED, 0, 0)
    g.apple = 3 * n + 4                                              # right in front of the head
    r, term = O.snake_step(g, n, 1, SEED, 0, 1)
    assert (r, term) == (1.0, False)                                 # "ingesting an apple awards one point"
    assert g.len == 3 and body(g) == [3 * n + 4, 3 * n + 3, 3 * n + 2] and g.since == 0
    assert g.apple not in body(g)


def test_self_collision_is_death():
    n = 6
    g = O.snake_reset(n, SEED, 0, 0)
    # a length-5 snake: head (2,2) moving left, body (2,3) (3,3) (3,2) (3,1): turning down hits (3,2)
    cells = [2 * n + 2, 2 * n + 3, 3 * n + 3, 3 * n + 2, 3 * n + 1]
    g.len = len(cells)
    for i, c in enumerate(cells):
        g.body[i] = c
    g.dir = 3
    g.apple = 0
    r, term = O.snake_step(g, n, 2, SEED, 0, 1)
    assert (r, term) == (-1.0, True)                                 # "the agent loses one point"
    # moving into the tail cell is allowed: the tail moves away in the same step
    g2 = O.snake_reset(n, SEED, 0, 0)
    cells = [2 * n + 2, 2 * n + 3, 3 * n + 3, 3 * n + 2]             # head (2,2), tail (3,2) right below it
    g2.len = len(cells)
    for i, c in enumerate(cells):
        g2.body[i] = c
    g2.dir = 3
    g2.apple = 0
    r, term = O.snake_step(g2, n, 2, SEED, 0, 1)
    assert (r, term) == (0.0, False) and body(g2)[0] == 3 * n + 2


def test_step_cap_ends_the_episode_without_penalty():
    n = 4
    g = O.snake_reset(n, SEED, 0, 0)
    g.apple = 0
    g.since = 200 * n - 1
    g.body[0], g.body[1] = 2 * n + 2, 2 * n + 1
    r, term = O.snake_step(g, n, 0, SEED, 0, 1)                      # up into a free cell
    assert (r, term) == (0.0, True)


def test_render_values_and_counts():
    n, px = 5, 3
    g = O.snake_reset(n, SEED, 0, 1)
    f = O.snake_render(g, n, px)
    assert f.shape == (15, 15)
    assert set(np.unique(f)) <= {0, 128, 191, 255}
    assert (f == 191).sum() == px * px and (f == 128).sum() == px * px and (f == 255).sum() == px * px
    hy, hx = divmod(int(g.body[0]), n)
    assert (f[hy * px:(hy + 1) * px, hx * px:(hx + 1) * px] == 191).all()   # whole-cell replication


def test_eps_greedy():
    assert all(O.eps_greedy(SEED, 0, t, 0.0, 2) == 2 for t in range(200))   # eps = 0: the greedy action
    acts = np.array([O.eps_greedy(SEED, 1, t, 1.0, 0) for t in range(100000)])
    assert stats.chisquare(np.bincount(acts, minlength=4)).pvalue > 0.01    # eps = 1: uniform over 4 actions
    explore = np.mean([O.eps_greedy(SEED, 2, t, 0.3, 5) != 5 for t in range(20000)])
    assert abs(explore - 0.3) < 0.02                                          # P(explore) = eps
    assert O.eps_threshold(1.0) == 1 << 32 and O.eps_threshold(0.0) == 0


def test_collect_reward_accounting_and_stacks():
    n, F, H, E = 6, 4, 12, 8
    res = O.collect(n, F, H, E, 400, SEED, 1.0)
    r, term = res["r"], res["term"]
    for e in range(E):
        # per episode: score = apples - (1 if died); length = 2 + apples until the end (SPEC invariants)
        apples = 0
        for s in range(r.shape[0]):
            if r[s, e] == 1.0:
                apples += 1
            if term[s, e]:
                assert r[s, e] in (-1.0, 0.0, 1.0)
                apples = 0
        g = res["games"][e]
        assert g.len == 2 + apples                                      # the episode still running
    assert res["episodes"].sum() == term.sum()
    # every stack holds F frames of the current game; the newest is its render
    for e in range(E):
        assert np.array_equal(res["stacks"][e, -1], O.snake_render(res["games"][e], n, H // n))


def test_collect_continues_across_calls():
    n, F, H, E = 6, 4, 12, 3
    full = O.collect(n, F, H, E, 60, SEED, 1.0)
    part = O.collect(n, F, H, E, 25, SEED, 1.0)
    rest = O.collect(n, F, H, E, 35, SEED, 1.0, state=(part["games"], part["stacks"]), t0=25)
    assert np.array_equal(full["stacks"], rest["stacks"])
    assert np.array_equal(full["a"][25:], rest["a"]) and np.array_equal(full["r"][25:], rest["r"])


def test_random_policy_baseline_is_negative():
    # SPEC: on 5x5 the expected episode reward of the random policy is negative (death dominates)
    n, E = 5, 64
    res = O.collect(n, 1, 5, E, 2000, SEED, 1.0)
    ep = res["episodes"].sum()
    assert ep > 1000
    finished = res["r"][res["term"].astype(bool)]
    assert res["r"].sum() / ep < 0 and (finished == -1.0).mean() > 0.9
