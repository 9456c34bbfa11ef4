import sys; sys.path.insert(0, '.')
import torch, numpy as np
import paper_1508_04186_b200 as D, synth
cfg = D.Config(replay_capacity=100000)
g = D.DQN(cfg, stream=torch.cuda.current_stream().cuda_stream)
for n, seed in [(16, 5), (8192, 0x5EED), (300, 7), (8192, 0x5EED + 8192)]:
    s, a, r, sn, t = synth.g_pong_torch(n, 4, 84, 84, 6, seed, "cuda")
    print(n, a.dtype, a.min().item(), a.max().item(), r.dtype, torch.isfinite(r).all().item(), r.is_contiguous(), a.is_contiguous(), flush=True)
    try:
        g.push(s, a, r, sn, t); print("device push ok", flush=True)
    except Exception as e: print("device push", e, flush=True)
