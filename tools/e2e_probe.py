"""Host-side cost of one e2e step (push 1 transition + train(1) + loss readback): Python binding vs
direct C-ABI calls, to see where the e2e time goes. Usage: python tools/e2e_probe.py"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_04186_b200 as D  # noqa: E402
import synth  # noqa: E402

cfg = D.Config(minibatch=32, replay_capacity=10000, precision=D.BF16, n_actions=6)
dqn = D.DQN(cfg)
s, a, r, sn, t = synth.g_pong(256, 4, 84, 84, 6, 1)
dqn.push(s, a, r, sn, t)
dqn.train(50)
ne = 300
hs = torch.from_numpy(s[:1].copy()).pin_memory()
hsn = torch.from_numpy(sn[:1].copy()).pin_memory()
ha = torch.zeros(1, dtype=torch.int32).pin_memory()
hr = torch.zeros(1, dtype=torch.float32).pin_memory()
ht = torch.zeros(1, dtype=torch.uint8).pin_memory()


def timed(fn, n=ne):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


L = D.lib()
st = D._Stats()
loss = np.zeros(1, np.float32)
st.loss_per_step = loss.ctypes.data
h = dqn._h
ps, pa, pr, pn, pt = hs.data_ptr(), ha.data_ptr(), hr.data_ptr(), hsn.data_ptr(), ht.data_ptr()
res = {
    "python push": timed(lambda: dqn.push(hs, ha, hr, hsn, ht)),
    "python train(1)": timed(lambda: dqn.train(1, want_loss=True)),
    "python push+train(1)": timed(lambda: (dqn.push(hs, ha, hr, hsn, ht), dqn.train(1, want_loss=True))),
    "C push": timed(lambda: L.dqn_push_transitions(h, 1, ps, pa, pr, pn, pt)),
    "C train(1)": timed(lambda: L.dqn_train_steps(h, 1, C.byref(st))),
    "C push+train(1)": timed(lambda: (L.dqn_push_transitions(h, 1, ps, pa, pr, pn, pt),
                                      L.dqn_train_steps(h, 1, C.byref(st)))),
    "C train(16) per step": timed(lambda: L.dqn_train_steps(h, 16, C.byref(st)), 50) / 16,
}
for k, v in res.items():
    print(f"{k:28s} {v:8.1f} us")
