"""Multi-GPU parity (BASELINE.json configs[2]): N replicas, each owning 1/N of the
parameter server, NCCL reduce-scatter push + all-gather fetch, deterministic
schedule, against the oracle's N-replica lock-step run (O9-O12, A7)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import delta_rel, gated_theta, he_theta, nets, per_tensor_rel, replay

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TINY_KW = dict(frames=3, height=17, width=13, convs=((5, 5, 2), (6, 3, 2)), fcs=(19,), n_actions=5)


def n_gpus():
    import torch
    return torch.cuda.device_count()


def run_ranks(world, tmp_path, *extra, env=None, tag="mp"):
    out = str(tmp_path / f"{tag}.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "tools", "mp_parity.py"),
           "--out", out, *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=None if env is None else {**os.environ, **env})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("n_push,n_fetch,C", [(1, 1, 2), (2, 3, 1)])
def test_two_replicas_fp32_match_oracle(tmp_path, n_push, n_fetch, C):
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    res = run_ranks(2, tmp_path, "--tiny", "--n-push", str(n_push), "--n-fetch", str(n_fetch), "--target-sync",
                    str(C), "--steps", "6")
    dc, on, oc = nets(minibatch=16, replay_capacity=200, n_push=n_push, n_fetch=n_fetch, target_sync=C, lr=1e-3,
                      **TINY_KW)
    oc.n_replicas = 2
    reps = [replay(on, 250, 100 + k)[0] for k in range(2)]
    th0 = he_theta(on, 3).astype(np.float64)
    ref = O.run(on, oc, 200, reps, th0, 6)
    assert int(res["n"]) == ref["n"]
    assert np.array_equal(res["idx"], ref["idx"].astype(np.int32))
    assert delta_rel(res["theta"], th0, ref["theta"], th0, on, ulps=ref["n"]) < 1e-5
    assert per_tensor_rel(res["r"], ref["r"], on) < 2e-5


def _bf16_case(tmp_path, world, scaled=False, n_push=1, n_fetch=1, extra=()):
    """bf16 at N = world in the gated regime (A38): Delta theta of every tensor within 2e-2 of the oracle's
    N-replica mean-gradient RMSProp (and r within 4e-2, quadratic in the gradients)."""
    kw = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18) if scaled else {}
    args = ["--precision", "bf16", "--b", "32", "--steps", "4", "--gated", "--lr", "1e-5", "--eps", "1e-2",
            "--n-push", str(n_push), "--n-fetch", str(n_fetch), *extra] + (["--scaled"] if scaled else [])
    res = run_ranks(world, tmp_path, *args)
    dc, on, oc = nets(minibatch=32, replay_capacity=200, lr=1e-5, rms_eps=1e-2, target_sync=2, n_push=n_push,
                      n_fetch=n_fetch, **kw)
    oc.n_replicas = world
    reps = [replay(on, 250, 100 + k)[0] for k in range(world)]
    th0 = gated_theta(on, 3).astype(np.float64)
    ref = O.run(on, oc, 200, reps, th0, 4)
    assert int(res["n"]) == ref["n"]
    assert np.array_equal(res["idx"], ref["idx"].astype(np.int32))
    assert delta_rel(res["theta"], th0, ref["theta"], th0, on, ulps=ref["n"]) < 2e-2
    assert per_tensor_rel(res["r"], ref["r"], on) < 4e-2
    return res


def test_two_replicas_bf16_mnih(tmp_path):
    """BASELINE.json configs[2] at N = 2: the fused server round (NEXT-1) on the bf16 Mnih kernels."""
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    _bf16_case(tmp_path, 2)


def test_two_replicas_bf16_nccl_path_bit_identical(tmp_path):
    """n_fetch = 2: push = NCCL reduce-scatter, fetch = NCCL all-gather of the bf16 working copy (a11, a13);
    two runs on fresh communicators are bit-identical (SURVEY §8(e) determinism, NCCL_ALGO/PROTO pinned)."""
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    res = _bf16_case(tmp_path, 2, n_push=2, n_fetch=2, extra=("--repeat", "2"))
    assert bool(res["identical"])


def test_two_replicas_fused_round_bit_identical(tmp_path):
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    res = _bf16_case(tmp_path, 2, extra=("--repeat", "2"))
    assert bool(res["identical"])


def test_two_replicas_async_fp32_match_lag1_twin(tmp_path):
    """DQN_ASYNC at N = 2: the reduce-scatter / update / all-gather round overlaps the next steps on
    the comm stream; the result equals the oracle's lag-1 twin (O13)."""
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    res = run_ranks(2, tmp_path, "--tiny", "--n-push", "2", "--n-fetch", "2", "--target-sync", "1", "--steps", "8",
                    "--async-mode")
    dc, on, oc = nets(minibatch=16, replay_capacity=200, n_push=2, n_fetch=2, target_sync=1, lr=1e-3, **TINY_KW)
    oc.n_replicas = 2
    oc.fetch_lag = 1
    reps = [replay(on, 250, 100 + k)[0] for k in range(2)]
    th0 = he_theta(on, 3).astype(np.float64)
    ref = O.run(on, oc, 200, reps, th0, 8)
    assert int(res["n"]) == ref["n"]
    assert np.array_equal(res["idx"], ref["idx"].astype(np.int32))
    assert delta_rel(res["theta"], th0, ref["theta"], th0, on, ulps=ref["n"]) < 1e-5
    # rank 0's histogram counts its own replica steps; the oracle's counts both replicas
    assert np.array_equal(res["staleness"] * 2, ref["staleness"])


def test_two_replicas_async_free_running_equals_realised_schedule(tmp_path):
    """DQN_ASYNC at N = 2 (Downpour's asynchrony, A40): each replica fetches the newest generation its comm
    stream has published; the oracle replays both replicas' realised schedules exactly."""
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    res = run_ranks(2, tmp_path, "--tiny", "--n-push", "2", "--n-fetch", "1", "--target-sync", "2", "--steps", "10",
                    "--async-free", env={"DQN_ASYNC_DELAY_US": "200"})
    dc, on, oc = nets(minibatch=16, replay_capacity=200, n_push=2, n_fetch=1, target_sync=2, lr=1e-3, **TINY_KW)
    oc.n_replicas = 2
    oc.fetch_gen = res["step_generation"]  # n_fetch = 1: one fetch per step
    reps = [replay(on, 250, 100 + k)[0] for k in range(2)]
    th0 = he_theta(on, 3).astype(np.float64)
    ref = O.run(on, oc, 200, reps, th0, 10)
    assert ref["rc"] == 0 and int(res["n"]) == ref["n"] == 5
    assert np.array_equal(res["idx"], ref["idx"].astype(np.int32))
    assert delta_rel(res["theta"], th0, ref["theta"], th0, on, ulps=ref["n"]) < 1e-5


@pytest.mark.parametrize("mode", ["--async-free", "--async-mode"])
def test_two_replicas_async_per_gradient_rule(tmp_path, mode):
    """NEXT-2 in the asynchronous modes (A33 + A40): the round's reduce-scatter becomes an all-to-all into each
    owner's inbox and the owner applies worker 0's gradient, then worker 1's (n += 2 per round), while the
    replicas keep stepping; the oracle (server_rule = 1) replays the realised schedule (free-running) or the
    lag-one-round twin. Staleness counts generations: multiples of N here."""
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    env = {"DQN_ASYNC_DELAY_US": "200"} if mode == "--async-free" else None
    res = run_ranks(2, tmp_path, "--tiny", "--n-push", "2", "--n-fetch", "1", "--target-sync", "3", "--steps", "10",
                    mode, "--server-rule", "1", env=env)
    dc, on, oc = nets(minibatch=16, replay_capacity=200, n_push=2, n_fetch=1, target_sync=3, lr=1e-3, **TINY_KW)
    oc.n_replicas = 2
    oc.server_rule = 1
    oc.fetch_gen = res["step_generation"]  # n_fetch = 1: one fetch per step
    assert np.all(res["step_generation"] % 2 == 0)  # only whole rounds are published
    reps = [replay(on, 250, 100 + k)[0] for k in range(2)]
    th0 = he_theta(on, 3).astype(np.float64)
    ref = O.run(on, oc, 200, reps, th0, 10)
    assert ref["rc"] == 0 and int(res["n"]) == ref["n"] == 10
    assert np.array_equal(res["idx"], ref["idx"].astype(np.int32))
    assert delta_rel(res["theta"], th0, ref["theta"], th0, on, ulps=ref["n"]) < 1e-5


@pytest.mark.parametrize("world", [4, 8])
def test_many_replicas_fp32_match_oracle(tmp_path, world):
    """N = 4 / 8 (skipped on smaller boxes): the fused server round (NEXT-1) with every rank owning
    1/N of theta, against the oracle's N-replica lock-step run."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    res = run_ranks(world, tmp_path, "--tiny", "--n-push", "1", "--n-fetch", "1", "--target-sync", "2", "--steps", "5")
    dc, on, oc = nets(minibatch=16, replay_capacity=200, target_sync=2, lr=1e-3, **TINY_KW)
    oc.n_replicas = world
    reps = [replay(on, 250, 100 + k)[0] for k in range(world)]
    th0 = he_theta(on, 3).astype(np.float64)
    ref = O.run(on, oc, 200, reps, th0, 5)
    assert int(res["n"]) == ref["n"]
    assert np.array_equal(res["idx"], ref["idx"].astype(np.int32))
    assert delta_rel(res["theta"], th0, ref["theta"], th0, on, ulps=ref["n"]) < 1e-5


@pytest.mark.parametrize("world", [4, 8])
def test_many_replicas_bf16_mnih(tmp_path, world):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    _bf16_case(tmp_path, world)


def test_two_replicas_bf16_scaled_generic_path(tmp_path):
    """The generic bf16 conv path (scaled net, BASELINE.json configs[4]) at N = 2 with the fused server round."""
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    _bf16_case(tmp_path, 2, scaled=True)


@pytest.mark.parametrize("n_push", [1, 2])
def test_two_replicas_per_gradient_rule(tmp_path, n_push):
    """DQN_SERVER_PER_GRADIENT (A33, Alg. 2 literally): the fused server round applies worker 0's then
    worker 1's gradient, one RMSProp and n += 1 each; against the oracle's server_rule = 1 run."""
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    res = run_ranks(2, tmp_path, "--tiny", "--n-push", str(n_push), "--n-fetch", "1", "--target-sync", "3",
                    "--steps", "6", "--server-rule", "1")
    dc, on, oc = nets(minibatch=16, replay_capacity=200, n_push=n_push, target_sync=3, lr=1e-3, **TINY_KW)
    oc.n_replicas = 2
    oc.server_rule = 1
    reps = [replay(on, 250, 100 + k)[0] for k in range(2)]
    th0 = he_theta(on, 3).astype(np.float64)
    ref = O.run(on, oc, 200, reps, th0, 6)
    assert int(res["n"]) == ref["n"] == 2 * (6 // n_push)
    assert np.array_equal(res["idx"], ref["idx"].astype(np.int32))
    assert delta_rel(res["theta"], th0, ref["theta"], th0, on, ulps=ref["n"]) < 1e-5


@pytest.mark.parametrize("env", [{}, {"DQN_STORE_IN_FWD": "0"}], ids=["store-in-forward", "store-kernel"])
def test_two_replicas_store_and_train_equals_alternating_calls(tmp_path, env):
    """Alg. 1's loop at N = 2 on the bf16 Mnih path with the fused server round: one dqn_store_and_train call
    equals alternating push(1) + train(1) calls bit for bit on every rank (indices, losses, server theta)."""
    if n_gpus() < 2:
        pytest.skip("needs 2 GPUs")
    res = run_ranks(2, tmp_path, "--precision", "bf16", "--b", "32", "--store", "10", "--lr", "1e-4", env=env,
                    tag="store")
    assert bool(res["identical"])
