"""Shared test helpers: config pairs (GPU config <-> oracle net/cfg), He-scaled
theta0, replay generation, and the normwise per-tensor error metric of A29."""
import math

import numpy as np

import paper_1508_04186_b200 as D
import synth
from oracle import oracle as O


def nets(convs=((16, 8, 4), (32, 4, 2)), fcs=(256,), n_actions=6, frames=4, height=84, width=84, **kw):
    kw.setdefault("keep_grad", 1)  # the update kernels also store the pushed gradient (same kernels, DQN_PARAMS_GRAD)
    dc = D.Config(frames=frames, height=height, width=width, convs=convs, fcs=fcs, n_actions=n_actions, **kw)
    on = O.Net(frames=frames, height=height, width=width, convs=convs, fcs=fcs, n_actions=n_actions)
    oc = O.TrainCfg(n_replicas=1, minibatch=dc.minibatch, n_push=dc.n_push, n_fetch=dc.n_fetch,
                    target_sync=dc.target_sync, gamma=dc.gamma, lr=dc.lr, rms_decay=dc.rms_decay,
                    rms_eps=dc.rms_eps, err_clip=dc.err_clip, seed=dc.seed)
    return dc, on, oc


def he_theta(net, seed, bias_std=0.05):
    """theta0 with He-scaled weights so activations stay O(1) through the net."""
    tt = O.tensor_table(net)
    stds = []
    for i, (off, cnt) in enumerate(tt):
        if i % 2 == 0:
            fan_in = cnt // tt[i + 1][1]
            stds.append(math.sqrt(2.0 / fan_in))
        else:
            stds.append(bias_std)
    return synth.init_theta(tt, stds, seed)


def gated_theta(net, seed, margin=0.04, bias=0.1, out_std=0.5):
    """theta0 of the "gated" regime (A38): every hidden layer has mixed-sign weights with
    sum_i |w_i| * max|x_i| <= margin and biases +bias on a random half of its units, -bias on the other half,
    so every hidden pre-activation lies in [bias - margin, bias + margin] (units on) or [-bias - margin,
    -bias + margin] (units off) for EVERY input: half of the ReLU units are always off, none is within
    bias - margin of its kink, and no rounding can flip a branch. The on/off pattern is random, not by index
    parity, so a kernel that handles even and odd channels in different code paths cannot hide a missing mask
    behind it. The output layer is N(0, out_std^2) (biases N(0, 0.05^2))."""
    tt = O.tensor_table(net)
    rng = np.random.Generator(np.random.PCG64(seed))
    th = np.zeros(O.param_count(net), np.float32)
    n_layers = len(tt) // 2
    xmax = 1.0  # layer 1 reads u8 / 255 <= 1
    for l in range(n_layers):
        (wo, wc), (bo, bc) = tt[2 * l], tt[2 * l + 1]
        fan_in = wc // bc
        if l == n_layers - 1:
            th[wo:wo + wc] = rng.normal(0.0, out_std, wc)
            th[bo:bo + bc] = rng.normal(0.0, 0.05, bc)
            break
        c = margin / (fan_in * xmax)
        w = rng.uniform(0.25, 1.0, wc) * c * np.where(rng.random(wc) < 0.5, -1.0, 1.0)
        # float32 rounding of w can only move |w| by 2^-24 relative: the margin keeps ~1e-7 of slack
        th[wo:wo + wc] = w * (1.0 - 1e-6)
        on = np.zeros(bc, bool)
        on[rng.permutation(bc)[:bc // 2]] = True
        th[bo:bo + bc] = np.where(on, bias, -bias)
        xmax = bias + margin
    return th


def gated_theta_separated(net, seed, gap=0.05, **kw):
    """gated_theta of the first seed >= `seed` whose greedy action is well separated (A21): in the gated regime
    Q barely depends on the state, so every sample shares one top-2 gap; require it above `gap` * max|Q| for a
    blank state, a saturated one and a random one, so that argmax checks exclude no sample."""
    rng = np.random.default_rng(0)
    probes = np.stack([np.zeros((net.frames, net.height, net.width), np.uint8),
                       np.full((net.frames, net.height, net.width), 255, np.uint8),
                       rng.integers(0, 256, (net.frames, net.height, net.width), dtype=np.uint8)])
    for sd in range(seed, seed + 1000):
        th = gated_theta(net, sd, **kw)
        q, _ = O.q_values(net, th.astype(np.float64), probes)
        qs = np.sort(q, axis=1)
        if np.all(qs[:, -1] - qs[:, -2] > gap * np.max(np.abs(q), axis=1)):
            return th
    raise RuntimeError("no separated gated theta found")


def delta_rel(x, x0, y, y0, net, ulps=0):
    """max over tensors of ||(x - x0) - (y - y0)||_inf / ||y - y0||_inf: the per-tensor error of the
    update theta_k - theta_0 (A29 applied to Delta theta). Both sides store theta in fp32, so each step's
    result is rounded to an fp32 of its magnitude: `ulps` fp32 ulps of the tensor's largest |theta| (one per
    step) are the storage floor taken off the error first (A39). A tensor whose reference update
    is exactly zero must have a zero update too."""
    worst = 0.0
    for off, cnt in O.tensor_table(net):
        x0t = np.asarray(x0[off:off + cnt], np.float64)
        dx = np.asarray(x[off:off + cnt], np.float64) - x0t
        dy = np.asarray(y[off:off + cnt], np.float64) - np.asarray(y0[off:off + cnt], np.float64)
        den = np.max(np.abs(dy))
        mag = max(float(np.max(np.abs(x0t))), float(np.max(np.abs(np.asarray(y[off:off + cnt], np.float64)))))
        err = max(float(np.max(np.abs(dx - dy))) - ulps * 2.0 ** -23 * mag, 0.0)
        worst = max(worst, err / den if den > 0 else (0.0 if err == 0 else np.inf))
    return worst


def bf16_rne(x):
    """float32 -> bfloat16 (round to nearest even) -> float32, the conversion every bf16 copy of theta uses."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def replay(net, n, seed, kind="uniform"):
    gen = synth.g_uniform if kind == "uniform" else synth.g_pong
    s, a, r, sn, t = gen(n, net.frames, net.height, net.width, net.n_actions, seed)
    return O.Replay(s, a, r.astype(np.float64), sn, t), (s, a, r, sn, t)


def per_tensor_rel(x, y, net):
    """max over tensors of ||x - y||_inf / ||y||_inf (A29)."""
    worst = 0.0
    for off, cnt in O.tensor_table(net):
        yy = np.asarray(y[off:off + cnt], np.float64)
        xx = np.asarray(x[off:off + cnt], np.float64)
        den = np.max(np.abs(yy))
        if den == 0.0:
            den = 1.0
        worst = max(worst, float(np.max(np.abs(xx - yy)) / den))
    return worst


def near_tie_mask(q, rel):
    """True where the top-2 gap of a Q row exceeds rel * max|Q| (argmax must then agree, A21)."""
    qs = np.sort(q, axis=1)
    gap = qs[:, -1] - qs[:, -2] if q.shape[1] > 1 else np.full(q.shape[0], np.inf)
    scale = np.max(np.abs(q), axis=1)
    return gap > rel * np.maximum(scale, 1e-30)
