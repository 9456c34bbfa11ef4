"""Oracle of the prioritized replay variant (NEXT-4; "A more sophisticated sampling strategy might
emphasize transitions from which we can learn the most, similar to prioritized sweeping").

TEST INFRASTRUCTURE ONLY: imported by tests/ (never by the product package, which never imports oracle/).

The paper names the idea and no rule, so the rule is DESIGN.md reading A41:
  * priority of a transition after it was sampled: p = (|delta| + eps_p)^alpha, alpha in {1, 1/2}
    (delta = Q(s, a; theta) - y, the unclipped TD error of the step that sampled it: "learn the most");
  * a stored transition enters with the largest priority written so far (1 initially), so it is sampled;
  * P(i) = p_i / sum_k p_k over the replay (alpha folded into p), drawn by stratified inverse-CDF sampling:
    sample j of step T targets t_j = ((j + u_j) / b) * S with S the total and u_j in [0, 1) a counter-based
    uniform (Philox word 2 of the sampler's counter (j, T, rank), A11), so the b draws of a step cover
    the b equal-mass strata of the distribution once each;
  * duplicates in one minibatch: the sample with the largest j writes the slot's priority.
Every integer decision (which leaf) is taken in fp32 on both sides, in the same order, so the GPU's and
this oracle's samples are bit-identical given the same leaf priorities:
  * a 32-ary sum tree: level 0 = leaves (32^K >= capacity, unused leaves 0), node i of level l + 1 = the
    butterfly sum of children 32 i .. 32 i + 31 of level l: v[k] <- v[k] + v[k ^ o] for o = 16, 8, 4, 2, 1
    (all in fp32), the node = v[0];
  * descent from the root: at a node with children c[0..31] and residual target t, scan k = 0..31 with a
    running fp32 prefix s: take the first k with c[k] > 0 and t < s + c[k]; if none (rounding), the last k
    with c[k] > 0; then t <- t - s (s = the prefix before k) and descend into child k.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from . import oracle as _or

F32 = np.float32
FAN = 32


def levels_for(capacity: int) -> int:
    """K: the number of 32-ary levels above the leaves, 32^K >= capacity (K >= 1)."""
    k, n = 1, FAN
    while n < capacity:
        n *= FAN
        k += 1
    return k


def butterfly_sum(c: np.ndarray) -> np.float32:
    """The fp32 butterfly sum of 32 values (v[k] <- v[k] + v[k ^ o], o = 16 .. 1), written out."""
    v = [F32(x) for x in c]
    assert len(v) == FAN
    o = 16
    while o >= 1:
        v = [F32(v[k] + v[k ^ o]) for k in range(FAN)]
        o //= 2
    return v[0]


def build_tree(leaves: np.ndarray, K: int) -> List[np.ndarray]:
    """levels[0] = the 32^K leaves (fp32), levels[l + 1][i] = butterfly_sum(levels[l][32 i : 32 i + 32])."""
    lv = [np.zeros(FAN ** K, F32)]
    lv[0][: len(leaves)] = np.asarray(leaves, F32)
    for l in range(K):
        prev = lv[l].reshape(-1, FAN)
        # the same butterfly as butterfly_sum, vectorised over the nodes of the level (per-element fp32 adds)
        v = prev.copy()
        o = 16
        while o >= 1:
            v = (v + v[:, np.arange(FAN) ^ o]).astype(F32)
            o //= 2
        lv.append(v[:, 0].copy())
    return lv


def uniform_u(seed: int, rank: int, T: int, j: int) -> np.float32:
    """u_j in [0, 1): the top 24 bits of Philox word 2 of counter (j, T_lo, T_hi, rank), key = seed (A11)."""
    o = _or.philox4x32_10([j & 0xFFFFFFFF, T & 0xFFFFFFFF, (T >> 32) & 0xFFFFFFFF, rank & 0xFFFFFFFF],
                          [seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF])
    return F32((o[2] >> 8) * (1.0 / 16777216.0))


def descend(lv: List[np.ndarray], t: np.float32) -> int:
    """The leaf the residual target t selects (module docstring's scan), from the root down."""
    K = len(lv) - 1
    node = 0
    t = F32(t)
    for l in range(K, 0, -1):
        c = lv[l - 1][node * FAN: node * FAN + FAN]
        s = F32(0.0)
        pick, pick_s = -1, F32(0.0)
        last, last_s = -1, F32(0.0)
        for k in range(FAN):
            ck = c[k]
            if ck > 0:
                if t < F32(s + ck):
                    pick, pick_s = k, s
                    break
                last, last_s = k, s
            s = F32(s + ck)
        if pick < 0:
            pick, pick_s = last, last_s
        if pick < 0:  # an all-zero node (only if the root is 0: nothing stored)
            pick, pick_s = 0, F32(0.0)
        t = F32(t - pick_s)
        node = node * FAN + pick
    return node


def sample(lv: List[np.ndarray], seed: int, rank: int, T: int, b: int) -> np.ndarray:
    """The b slots of step T: t_j = ((j + u_j) / b) * S in fp32 (S = the root), then descend."""
    S = lv[-1][0]
    q = F32(F32(S) / F32(b))
    out = np.zeros(b, np.int64)
    for j in range(b):
        t = F32(F32(F32(j) + uniform_u(seed, rank, T, j)) * q)
        out[j] = descend(lv, t)
    return out


def leaf_priority(delta: float, alpha: float, eps: float) -> np.float32:
    """p = (|delta| + eps)^alpha, alpha = 1: |delta| + eps; alpha = 1/2: its correctly rounded sqrt (fp32)."""
    x = F32(F32(abs(F32(delta))) + F32(eps))
    if alpha == 1.0:
        return x
    if alpha == 0.5:
        return F32(np.sqrt(x, dtype=F32))
    raise ValueError("alpha must be 1 or 0.5 (A41)")


def update(leaves: np.ndarray, maxp: float, idx, delta, alpha: float, eps: float) -> Tuple[np.ndarray, np.float32]:
    """After a step: the slot of sample j gets leaf_priority(delta_j); of duplicates the largest j wins;
    maxp <- max(maxp, the written priorities)."""
    out = np.asarray(leaves, F32).copy()
    m = F32(maxp)
    b = len(idx)
    for j in range(b):
        if any(int(idx[k]) == int(idx[j]) for k in range(j + 1, b)):
            continue  # a later sample of the same slot writes it
        p = leaf_priority(delta[j], alpha, eps)
        out[int(idx[j])] = p
        m = max(m, p)
    return out, F32(m)


def push(leaves: np.ndarray, maxp: float, slots) -> np.ndarray:
    """Stored transitions enter with the largest priority written so far."""
    out = np.asarray(leaves, F32).copy()
    for s in slots:
        out[int(s)] = F32(maxp)
    return out
