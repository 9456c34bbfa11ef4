"""World-size-2 CPU (gloo) tests of the N > 1 host logic.

1. The sharded-parameter-server data flow the CUDA runtime implements (pad P to
   P_pad = ceil(P / 64N) * 64N, reduce-scatter the summed replica gradients so
   rank s owns [s*P_pad/N, (s+1)*P_pad/N), mean over N * n_push, RMSProp on the
   shard, all-gather the shards for the next fetch) reproduces the oracle's
   N-replica lock-step run (O9-O12), here with real torch.distributed
   collectives over gloo and the oracle's per-replica gradients.
2. bench.py's launcher contract under torch.distributed.run: rank 0 alone runs
   and prints the --impl reference JSON line, the other ranks exit 0.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import he_theta, nets, replay

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TINY_KW = dict(frames=3, height=17, width=13, convs=((5, 5, 2), (6, 3, 2)), fcs=(19,), n_actions=5)
STEPS, CAP, B = 4, 60, 4


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dc, on, oc = nets(minibatch=B, replay_capacity=CAP, lr=1e-2, target_sync=2, **TINY_KW)
    P = O.param_count(on)
    unit = 64 * world
    P_pad = (P + unit - 1) // unit * unit
    shard = P_pad // world
    theta_full = np.zeros(P_pad)
    theta_full[:P] = he_theta(on, 3)
    master = theta_full[rank * shard:(rank + 1) * shard].copy()
    r = np.zeros(shard)
    local = theta_full.copy()
    hat = theta_full.copy()
    n = ell = 0
    rp = replay(on, 80, 100 + rank)[0]
    ring = [(i % CAP, i) for i in range(80)]
    slot_item = {}
    for sl, i in ring:
        slot_item[sl] = i
    for T in range(STEPS):
        # fetch: all-gather of the owners' shards (a13), then refresh (O11)
        parts = [torch.zeros(shard, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(master))
        local = torch.cat(parts).numpy()
        if n - ell >= oc.target_sync:
            hat, ell = local.copy(), n
        idx = [slot_item[O.sample_index(oc.seed, rank, T, j, CAP)] for j in range(B)]
        y, _ = O.targets(on, hat[:P], rp.s_next[idx], rp.r[idx], rp.term[idx], oc.gamma)
        _, g = O.loss_grad(on, local[:P], rp.s[idx], rp.a[idx], y)
        G = np.zeros(P_pad)
        G[:P] = g
        # push: reduce-scatter (sum) to the shard owners (a11), mean, RMSProp on the shard (a12)
        red = torch.from_numpy(G)
        dist.all_reduce(red)
        gbar = red.numpy()[rank * shard:(rank + 1) * shard] / (world * 1)
        master, r = O.rmsprop(master, r, gbar, oc.lr, oc.rms_decay, oc.rms_eps)
        n += 1
    parts = [torch.zeros(shard, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(master))
    if rank == 0:
        np.save(out, torch.cat(parts).numpy()[:P])
    dist.destroy_process_group()


def test_sharded_server_dataflow_matches_oracle(tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "theta.npy")
    mp.start_processes(_worker, args=(2, 29533, out), nprocs=2, start_method="spawn", join=True)
    dc, on, oc = nets(minibatch=B, replay_capacity=CAP, lr=1e-2, target_sync=2, **TINY_KW)
    oc.n_replicas = 2
    reps = [replay(on, 80, 100 + k)[0] for k in range(2)]
    ref = O.run(on, oc, CAP, reps, he_theta(on, 3).astype(np.float64), STEPS)
    np.testing.assert_allclose(np.load(out), ref["theta"], rtol=0, atol=1e-12)


def test_bench_reference_arm_under_torchrun():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29541", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--impl", "reference", "--steps", "2", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
