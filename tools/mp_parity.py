"""Worker for the multi-GPU parity test (launched by torch.distributed.run, one rank per GPU).

Each rank is replica k of Alg. 1 and owner of shard k of Alg. 2: it pushes its own
seeded replay (independent per-worker histories), runs `steps` lock-step
replica steps through the C ABI (NCCL reduce-scatter push + all-gather fetch), and
rank 0 writes the gathered server theta, the generation and every rank's sampled
indices to --out (npz). The test compares that file with the oracle's N-replica run.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--n-push", type=int, default=1)
    ap.add_argument("--n-fetch", type=int, default=1)
    ap.add_argument("--target-sync", type=int, default=2)
    ap.add_argument("--b", type=int, default=16)
    ap.add_argument("--tiny", action="store_true")
    ap.add_argument("--scaled", action="store_true", help="BASELINE configs[4] net (generic bf16 conv path)")
    ap.add_argument("--smooth", action="store_true")
    ap.add_argument("--gated", action="store_true", help="gated-regime theta0 (tests/helpers.gated_theta, A38)")
    ap.add_argument("--eps", type=float, default=1e-8, help="RMSProp epsilon (A4)")
    ap.add_argument("--repeat", type=int, default=1, help="run the whole job this many times (bit identity)")
    ap.add_argument("--async-mode", action="store_true", help="DQN_ASYNC_LAG1 (the deterministic twin, O13)")
    ap.add_argument("--async-free", action="store_true", help="DQN_ASYNC (newest published generation, A40)")
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--server-rule", type=int, default=0, help="0 mean (A7), 1 per gradient (A33)")
    ap.add_argument("--store", type=int, default=0,
                    help="Alg. 1's loop: push 33 items, then this many store+step iterations, once as alternating "
                         "push(1) + train(1) calls and once as one dqn_store_and_train call (bit identity)")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1508_04186_b200 as D
    from tests.helpers import he_theta, nets, replay

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [D.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    kw = dict(frames=3, height=17, width=13, convs=((5, 5, 2), (6, 3, 2)), fcs=(19,), n_actions=5) if a.tiny else {}
    if a.scaled:
        kw = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)
    prec = D.FP32 if a.precision == "fp32" else D.BF16
    dc, on, oc = nets(minibatch=a.b, replay_capacity=200, n_push=a.n_push, n_fetch=a.n_fetch,
                      target_sync=a.target_sync, lr=a.lr, rms_eps=a.eps, precision=prec,
                      sync_mode=D.ASYNC_LAG1 if a.async_mode else D.ASYNC if a.async_free else D.DETERMINISTIC,
                      server_rule=a.server_rule, **kw)
    theta0 = he_theta(on, 3)
    if a.smooth:
        from tests.test_gpu_parity_bf16 import smooth_theta
        theta0 = smooth_theta(on, 3)
    if a.gated:
        from tests.helpers import gated_theta
        theta0 = gated_theta(on, 3)
    _, raw = replay(on, 250, 100 + rank)
    if a.store:
        store_mode(a, D, dc, theta0, raw, rank, world, obj[0], dist)
        return
    runs = []
    for _ in range(a.repeat):
        g = D.DQN(dc, rank=rank, world=world, nccl_id=obj[0] if not runs else None, init_params=theta0) \
            if not runs else None
        if g is None:  # a fresh communicator for every repetition
            o2 = [D.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(o2, src=0)
            g = D.DQN(dc, rank=rank, world=world, nccl_id=o2[0], init_params=theta0)
        g.push(*raw)
        out = g.train(a.steps, want_idx=True, want_generation=True)
        th = g.params(D.PARAMS_SERVER)        # collective
        rr = g.params(D.PARAMS_RMS)           # collective
        runs.append((th, rr))
        if len(runs) < a.repeat:
            g.close()
    idx = torch.from_numpy(out["idx"]).cuda()
    gathered = [torch.zeros_like(idx) for _ in range(world)]
    dist.all_gather(gathered, idx)
    gen = torch.from_numpy(out["step_generation"]).cuda()
    gens = [torch.zeros_like(gen) for _ in range(world)]
    dist.all_gather(gens, gen)
    if rank == 0:
        np.savez(a.out, theta=runs[0][0], r=runs[0][1], n=out["generation"],
                 idx=np.stack([x.cpu().numpy() for x in gathered]), staleness=out["staleness"],
                 step_generation=np.stack([x.cpu().numpy() for x in gens]),
                 identical=all(np.array_equal(t, runs[0][0]) and np.array_equal(r, runs[0][1]) for t, r in runs))
    g.close()
    dist.barrier()
    dist.destroy_process_group()


def store_mode(a, D, dc, theta0, raw, rank, world, nccl_id, dist):
    import torch
    head = tuple(x[:33] for x in raw)
    tail = tuple(x[33:33 + a.store] for x in raw)
    res = []
    for how in ("alternating", "store_and_train"):
        if how == "alternating":
            uid = nccl_id
        else:
            o2 = [D.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(o2, src=0)
            uid = o2[0]
        g = D.DQN(dc, rank=rank, world=world, nccl_id=uid, init_params=theta0)
        g.push(*head)
        if how == "alternating":
            idx, loss = [], []
            for i in range(a.store):
                g.push(*(x[i:i + 1] for x in tail))
                o = g.train(1, want_idx=True, want_loss=True)
                idx.append(o["idx"][0])
                loss.append(o["loss"][0])
            idx, loss = np.stack(idx), np.array(loss, np.float32)
        else:
            o = g.train(a.store, want_idx=True, want_loss=True, store=tail)
            idx, loss = o["idx"], o["loss"]
        th = g.params(D.PARAMS_SERVER)  # collective
        res.append((idx, loss, th))
        g.close()
    same = all(np.array_equal(x, y) for x, y in zip(res[0], res[1]))
    flag = torch.tensor([1 if same else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        np.savez(a.out, identical=bool(flag.item()), theta=res[1][2])
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
