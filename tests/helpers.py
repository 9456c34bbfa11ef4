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
