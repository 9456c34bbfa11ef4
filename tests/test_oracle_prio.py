"""Pins of the prioritized-replay oracle (oracle/prio.py; reading A41 of P:99) against what mathematics fixes:
exact sums, fp64 sums, the inverse-CDF definition, stratification, the sampling distribution (chi-square), and
the update rule's special cases. CPU only."""
import math

import numpy as np
import pytest
from scipy import stats

from oracle import prio as PR

F32 = np.float32


def test_levels_for():
    assert PR.levels_for(1) == 1 and PR.levels_for(32) == 1 and PR.levels_for(33) == 2
    assert PR.levels_for(1000) == 2 and PR.levels_for(1024) == 2 and PR.levels_for(1025) == 3
    assert PR.levels_for(1_000_000) == 4


def test_butterfly_sum_exact_cases():
    # one-hot: the sum is the value itself wherever it sits (a wrong partner index would drop or double it)
    for k in range(32):
        c = np.zeros(32, F32)
        c[k] = F32(0.3)
        assert PR.butterfly_sum(c) == F32(0.3)
    # dyadic values: every partial sum is exact, so the sum is the exact total
    c = np.array([2.0 ** -(k % 7) for k in range(32)], F32)
    assert float(PR.butterfly_sum(c)) == sum(2.0 ** -(k % 7) for k in range(32))
    c = np.arange(32, dtype=F32)
    assert float(PR.butterfly_sum(c)) == 496.0


def test_butterfly_sum_close_to_fp64():
    rng = np.random.default_rng(1)
    for _ in range(50):
        c = rng.exponential(1.0, 32).astype(F32)
        exact = float(np.sum(c.astype(np.float64)))
        assert abs(float(PR.butterfly_sum(c)) - exact) <= 8 * np.finfo(F32).eps * exact


def test_tree_nodes_are_subtree_sums():
    rng = np.random.default_rng(2)
    leaves = rng.exponential(1.0, 1500).astype(F32)
    K = PR.levels_for(len(leaves))
    lv = PR.build_tree(leaves, K)
    assert [len(x) for x in lv] == [32 ** (K - l) for l in range(K + 1)]
    full = np.zeros(32 ** K)
    full[: len(leaves)] = leaves
    for l in range(1, K + 1):
        exact = full.reshape(-1, 32 ** l).sum(axis=1)
        assert np.allclose(lv[l].astype(np.float64), exact, rtol=1e-5, atol=0)
    # the vectorised level equals the written-out butterfly node by node
    for i in range(0, len(lv[1]), 7):
        assert lv[1][i] == PR.butterfly_sum(lv[0][32 * i: 32 * i + 32])


def test_descend_is_the_inverse_cdf():
    rng = np.random.default_rng(3)
    leaves = rng.exponential(1.0, 900).astype(F32)
    leaves[rng.random(900) < 0.2] = 0.0  # zero-priority slots are never taken
    K = PR.levels_for(len(leaves))
    lv = PR.build_tree(leaves, K)
    S = float(lv[-1][0])
    pre = np.concatenate([[0.0], np.cumsum(leaves.astype(np.float64))])
    tol = 1e-5 * S
    for t in np.linspace(0.0, S * (1 - 1e-7), 2000, dtype=np.float64):
        i = PR.descend(lv, F32(t))
        assert i < len(leaves) and leaves[i] > 0
        assert pre[i] - tol <= t <= pre[i + 1] + tol


def test_sample_is_stratified_and_monotone():
    rng = np.random.default_rng(4)
    leaves = rng.exponential(1.0, 700).astype(F32)
    lv = PR.build_tree(leaves, PR.levels_for(700))
    pre = np.concatenate([[0.0], np.cumsum(leaves.astype(np.float64))])
    S = pre[-1]
    for T in range(20):
        b = 16
        idx = PR.sample(lv, 0xABCDEF, 1, T, b)
        assert np.all(np.diff(idx) >= 0)  # targets increase with j and the descent is monotone
        for j, i in enumerate(idx):  # the leaf's mass interval meets stratum j
            assert pre[i] <= (j + 1) / b * S * (1 + 1e-6) and pre[i + 1] >= j / b * S * (1 - 1e-6)


def test_sampling_distribution_chi_square():
    p = np.array([1.0 + (k % 5) * 0.75 for k in range(40)], F32)
    lv = PR.build_tree(p, PR.levels_for(len(p)))
    b, steps = 4, 2500
    counts = np.zeros(len(p))
    for T in range(steps):
        for i in PR.sample(lv, 99, 0, T, b):
            counts[i] += 1
    expected = p.astype(np.float64) / p.sum() * b * steps
    chi2 = float(((counts - expected) ** 2 / expected).sum())
    # stratification makes the counts LESS dispersed than multinomial; a wrong distribution is far out
    assert stats.chi2.sf(chi2, len(p) - 1) > 1e-3


def test_uniform_u_range_and_uniformity():
    us = np.array([PR.uniform_u(5, 0, T, j) for T in range(200) for j in range(8)], np.float64)
    assert us.min() >= 0.0 and us.max() < 1.0
    assert stats.kstest(us, "uniform").pvalue > 1e-3


def test_leaf_priority_rule():
    assert PR.leaf_priority(-0.5, 1.0, 0.01) == F32(F32(0.5) + F32(0.01))
    assert PR.leaf_priority(0.5, 1.0, 0.01) == PR.leaf_priority(-0.5, 1.0, 0.01)
    assert PR.leaf_priority(0.23, 0.5, 0.02) == F32(math.sqrt(float(F32(F32(0.23) + F32(0.02)))))
    assert PR.leaf_priority(3.0, 0.5, 1.0) == F32(2.0)
    with pytest.raises(ValueError):
        PR.leaf_priority(1.0, 0.7, 0.0)


def test_update_duplicates_last_wins_and_maxp():
    leaves = np.ones(10, F32)
    out, m = PR.update(leaves, 1.0, [3, 5, 3], [2.0, 0.5, -4.0], 1.0, 0.0)
    assert out[3] == F32(4.0) and out[5] == F32(0.5) and m == F32(4.0)
    assert np.all(out[[0, 1, 2, 4, 6, 7, 8, 9]] == 1.0)
    out2 = PR.push(out, m, [7, 8])
    assert out2[7] == F32(4.0) and out2[8] == F32(4.0)
