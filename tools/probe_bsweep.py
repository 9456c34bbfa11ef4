"""Per-region device times of the bf16 Mnih step against the minibatch (one GPU): how the per-image kernels
scale past one wave of 148 SMs. usage: python tools/probe_bsweep.py [b ...]"""
import sys

import numpy as np

import paper_1508_04186_b200 as D
import synth

MNIH = dict(frames=4, height=84, width=84, convs=((16, 8, 4), (32, 4, 2)), fcs=(256,), n_actions=18)
for b in [int(x) for x in sys.argv[1:]] or [32, 64, 128, 144, 160, 256]:
    g = D.DQN(D.Config(**MNIH, minibatch=b, replay_capacity=20000, precision=D.BF16, target_sync=1000))
    g.push(*synth.g_pong(4000, 4, 84, 84, 18, 5))
    g.train(20)
    r = {x["name"]: round(x["avg_us"], 2) for x in g.profile(100)}
    print(b, r, flush=True)
    g.close()
