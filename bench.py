"""bench.py — DQN transitions/sec trained on B200 (BASELINE.json metric).

One "step" = one replica step of Alg. 1 (sample b transitions from the on-GPU
replay, forward s with theta and s' with theta^, TD target, backward) plus the
parameter-server round of Alg. 2 it triggers (push = reduce-scatter, RMSProp
shard update, fetch = all-gather), i.e. every row of SURVEY.md §8(a).

N = 1 : BASELINE.json configs[1] — 1 replica, Mnih-2013 net, b = 32, replay of
        1M transitions on the GPU, target net refreshed every C = 1000 steps.
N > 1 : configs[2] — Downpour with the sharded parameter server, b = 32 per
        replica, n_push = n_fetch = 1 deterministic schedule (weak scaling).

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
       (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MNIH = dict(convs=((16, 8, 4), (32, 4, 2)), fcs=(256,), n_actions=6)
SCALED = dict(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)
# BASELINE.json configs[0..4]; C = target refresh period, async = DQN_ASYNC (lag-1 staleness mode)
CONFIGS = {
    "c1": dict(idx=0, net=MNIH, b=32, replay=1000, n_push=1, n_fetch=1, C=2**62, async_=False),
    "c2": dict(idx=1, net=MNIH, b=32, replay=1_000_000, n_push=1, n_fetch=1, C=1000, async_=False),
    "c3": dict(idx=2, net=MNIH, b=32, replay=1_000_000, n_push=1, n_fetch=1, C=1000, async_=False),
    "c4": dict(idx=3, net=MNIH, b=256, replay=1_000_000, n_push=10, n_fetch=10, C=1000, async_=True),
    "c5": dict(idx=4, net=SCALED, b=512, replay=1_000_000, n_push=1, n_fetch=1, C=1000, async_=False),
}
for _c in CONFIGS.values():
    _c["async"] = _c.pop("async_")


def net_name(net):
    conv = ", ".join(f"conv{f} {k}x{k}/{s}" for f, k, s in net["convs"])
    return f"{conv}, fc{net['fcs'][0]}, {net['n_actions']} actions"
METRIC = "DQN transitions/sec trained (device-timed, max over ranks) at 1/2/4/8 B200"
UNIT = "transitions/s"
FP32_ALU_PEAK_TFLOPS = 2 * 128 * 148 * 1.965e9 / 1e12  # FFMA lanes x SMs x clocks.max.sm


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(hbm=d.get("hbm_gbs", 6650.0), bf16=d.get("bf16_tflops", 1590.0),
                    bf16_sus=d.get("bf16_tflops_sustained", 1400.0), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


def region_work(name: str, b: int, net=MNIH, world: int = 1, dtype: str = "bf16"):
    """Algorithmic FLOPs and HBM bytes of one step region. Convolutions:
    forward on s (theta) and s' (theta^), backward dW for every layer and dX for every layer but the first;
    FC likewise. Activations are `dtype` (bf16: 2 B, f32: 4 B); the replay slots are u8 (the 56,448 B of s and
    s' per transition of a2); gradients are fp32. The shard update moves 22 B per parameter (read theta, r, G;
    write theta, r and the bf16 theta; 20 B on the fp32 path). The fused server round (N = world
    > 1) moves, per rank and owned parameter, N fp32 gradient reads (N - 1 over NVLink), theta and r read and
    written, bf16 theta stored to N replicas (6N + 16 B)."""
    F, H, W = 4, 84, 84
    state = F * H * W
    e = 2 if dtype == "bf16" else 4
    upd = 22 if dtype == "bf16" else 20
    layers, c, h = [], F, H
    for (n, k, s) in net["convs"]:
        ho = (h - k) // s + 1
        layers.append(dict(C=c, N=n, k=k, HoWo=ho * ho, in_elems=c * h * h))
        c, h = n, ho
    D, Hfc, A = c * h * h, net["fcs"][0], net["n_actions"]
    macs = lambda L: L["HoWo"] * L["N"] * L["C"] * L["k"] ** 2  # noqa: E731
    P = sum(L["N"] * (L["C"] * L["k"] ** 2 + 1) for L in layers) + Hfc * (D + 1) + A * (Hfc + 1)
    conv_params = sum(L["N"] * (L["C"] * L["k"] ** 2 + 1) for L in layers)
    w = {}
    for i, L in enumerate(layers):
        in_b = b * (state if i == 0 else L["in_elems"] * e)  # u8 slots for layer 1
        out_b = b * L["N"] * L["HoWo"] * e
        w[f"conv{i + 1}_fwd"] = (2 * 2 * b * macs(L), 2 * in_b + 2 * out_b)
        w[f"conv{i + 1}_bwd"] = ((2 if i else 1) * 2 * b * macs(L), in_b + out_b + (in_b if i else 0))
    w["fc1_fwd"] = (2 * 2 * b * D * Hfc, 2 * b * D * e + 2 * D * Hfc * e + 2 * b * Hfc * 4)
    w["head_td"] = w["head_sample"] = (2 * 2 * b * Hfc * A, 2 * b * Hfc * 4 + 2 * A * (Hfc + 1) * 4)
    w["fc1_bwd"] = (4 * b * D * Hfc, b * Hfc * e + 2 * b * D * e + D * Hfc * e + D * Hfc * 4)
    w["rmsprop_update"] = (0, P * upd)
    w["reduce_update"] = (0, conv_params * upd + b * conv_params * 4)  # + the per-image conv partials
    w["sample"] = (0, b * 4)
    shard = -(-P // (64 * world)) * 64
    w["server_round_fused"] = (0, shard * (6 * world + 16))
    # fused regions of the bf16 tensor-core path
    w["conv_fwd"] = tuple(sum(w[f"conv{i + 1}_fwd"][q] for i in range(len(layers))) for q in range(2))
    w["conv_bwd"] = tuple(sum(w[f"conv{i + 1}_bwd"][q] for i in range(len(layers))) for q in range(2))
    w["fc1_bwd_head_finish"] = w["fc1_bwd"]
    w["_P"] = (P, conv_params)
    return w.get(name, (0, 0))


def param_count_of(net=MNIH) -> int:
    return region_work("_P", 1, net)[0]


REGION_KERNELS = {"conv_fwd": ["fwd_conv_bf16_kernel"], "fc1_fwd": ["tc_gemm_kernel"],
                  "head_sample": ["head_sample_kernel"], "fc1_bwd_head_finish": ["tc_pair_kernel"],
                  "conv_bwd": ["bwd_conv_bf16_kernel", "bwd_reduce_kernel"], "rmsprop_update": ["rmsprop_kernel"],
                  "reduce_update": ["reduce_update_kernel"]}


def conv_param_count(net=MNIH) -> int:
    c, n_params = 4, 0
    for (n, k, s) in net["convs"]:
        n_params += n * (c * k * k + 1)
        c = n
    return n_params


def region_traffic(name: str, dtype: str, net=MNIH):
    """DRAM bytes (read + write) of one step's launches of a region's kernels, from the committed `ncu --set
    full` captures of this round (profiles/r2_traffic.json, tools/traffic_json.py): per kernel on the Mnih
    path, per region on the generic path (the scaled net); None when not captured."""
    p = os.path.join(ROOT, "profiles", "r2_traffic.json")
    if dtype != "bf16" or not os.path.exists(p):
        return None
    with open(p) as f:
        t = json.load(f)
    if net == MNIH and name in REGION_KERNELS:
        ks = [k for k in REGION_KERNELS[name] if k in t["mnih"]]  # the kernels of the region that ran in the capture
        return sum((t["mnih"][k]["dram_read_MB"] + t["mnih"][k]["dram_write_MB"]) * 1e6 for k in ks) if ks else None
    if net == SCALED and name in t["scaled"]["regions"]:
        return t["scaled"]["regions"][name]["bytes"]
    return None


def roofline(regions, b, net, world, dtype, profile_steps):
    """the dominant step region's algorithmic work over its measured mean duration (CUDA events
    around it inside the replayed step graph), against BOTH the tensor and the HBM peak; `bound` / `frac`
    are the binding one (the larger of flops / tensor peak and bytes / HBM peak). `step` is the same for the
    whole step (every region's work over the sum of the region times)."""
    pk = peaks()
    P, conv_params = param_count_of(net), conv_param_count(net)
    names = {r["name"] for r in regions}
    # N = 1 bf16 Mnih path: the conv backward launch also runs the early RMSProp update of the non-conv
    # parameters (22 B/param)
    early = (dtype == "bf16" and world == 1 and "reduce_update" in names and b + 32 <= 148
             and os.environ.get("DQN_EARLY_UPDATE", "1") != "0")

    def work(name):
        f, by = region_work(name, b, net, world, dtype)
        if early and name == "conv_bwd":
            by += (P - conv_params) * 22
        return f, by

    full = [r for r in regions if r["steps"] >= profile_steps // 2]
    step_us = sum(r["avg_us"] for r in full)
    top = max(regions, key=lambda r: r["avg_us"])
    tpk = pk["bf16_sus"] if dtype == "bf16" else FP32_ALU_PEAK_TFLOPS
    tunit_bound = "tensor" if dtype == "bf16" else "alu"

    def fracs(f, by, us):
        t = {"achieved": f / (us * 1e-6) / 1e12, "peak": tpk, "unit": "TFLOP/s"}
        t["frac"] = t["achieved"] / t["peak"]
        h = {"achieved": by / (us * 1e-6) / 1e9, "peak": pk["hbm"], "unit": "GB/s"}
        h["frac"] = h["achieved"] / h["peak"]
        return t, h

    flops, byts = work(top["name"])
    t, h = fracs(flops, byts, top["avg_us"])
    bind_hbm = byts / (pk["hbm"] * 1e9) > flops / (tpk * 1e12)
    roof = dict(h if bind_hbm else t)
    roof["bound"] = "hbm" if bind_hbm else tunit_bound
    roof["traffic"] = region_traffic(top["name"], dtype, dict(net, fcs=tuple(net["fcs"])))
    roof.update(kernel=top["name"], avg_us=top["avg_us"], algorithmic_flops=flops, algorithmic_bytes=byts,
                share_of_step=top["avg_us"] / step_us if step_us else None, tensor=t, hbm=h)
    sf = sum(work(r["name"])[0] for r in full)
    sb = sum(work(r["name"])[1] for r in full)
    st, sh = fracs(sf, sb, step_us)
    roof["step"] = {"us": step_us, "flops": sf, "bytes": sb, "tensor_frac": st["frac"], "hbm_frac": sh["frac"]}
    roof["peak_source"] = (f"{pk['src']} MEASURED_PEAKS.json: bf16_tflops_sustained (tensor), hbm_gbs (hbm)"
                           if dtype == "bf16" else "derived: 148 SMs x 128 FFMA lanes x 2 x 1.965 GHz (alu); "
                           f"{pk['src']} MEASURED_PEAKS.json hbm_gbs (hbm)")
    if top["name"] == "server_round_fused":
        roof["note"] = ("the fused server round (N > 1) is bound by cross-GPU flag latency (two barriers, "
                        "DESIGN.md §6a), not by its bytes")
    elif early and top["name"] == "conv_bwd":
        roof["note"] = "conv backward + the early RMSProp update of the non-conv parameters in one launch"
    return roof


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_rate(O, net, rp, theta0, b, budget_s):
    """transitions/s of the oracle's replica step (O.run: sample, targets with theta^, gradient, RMSProp) on a
    bounded sample: as many steps of minibatch b as fit the time budget."""
    cfg = O.TrainCfg(minibatch=b, target_sync=1000)
    t0 = time.perf_counter()
    O.run(net, cfg, len(rp.a), [rp], theta0, 1)
    one = time.perf_counter() - t0
    steps = max(1, int(budget_s / max(one, 1e-3)))
    t0 = time.perf_counter()
    O.run(net, cfg, len(rp.a), [rp], theta0, steps)
    dt = time.perf_counter() - t0
    return steps * b / dt, steps, dt


def cpu_baseline(budget_s: float = 15.0, b: int = 32):
    """The oracle as it stands (fp64; per-sample gradient terms on all host cores with OpenMP, summed in sample
    order), on a bounded sample of the workload; plus the same on one thread."""
    import numpy as np

    import synth
    from oracle import oracle as O

    net = O.Net(**MNIH)
    s, a, r, sn, t = synth.g_pong(1000, 4, 84, 84, 6, 0x5EED)
    rp = O.Replay(s, a, r.astype(np.float64), sn, t)
    theta0 = synth.init_theta(O.tensor_table(net), [0.01] * 8, 7).astype(np.float64)
    n0 = O.threads()
    O.set_threads(0)
    cores = O.threads()
    v, steps, dt = _oracle_rate(O, net, rp, theta0, b, budget_s)
    O.set_threads(1)
    v1, steps1, _ = _oracle_rate(O, net, rp, theta0, b, budget_s / 3)
    O.set_threads(n0)
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "nproc": os.cpu_count(),
            "sample": f"{steps} replica steps of b={b} (Mnih net, replay 1k G-pong instead of 1M), fp64, "
                      f"{cores} OpenMP threads over the minibatch samples",
            "single_thread": {"value": v1, "cores": 1, "sample": f"{steps1} replica steps, 1 thread"}}


def run_reference(args, world, rank):
    """--impl reference: the fp64 oracle timed on the host cores (rank 0 only), all cores."""
    if rank != 0:
        return
    import numpy as np

    import synth
    from oracle import oracle as O

    net = O.Net(**MNIH)
    b_full = 32
    s, a, r, sn, t = synth.g_pong(1000, 4, 84, 84, 6, 0x5EED)
    rp = O.Replay(s, a, r.astype(np.float64), sn, t)
    theta0 = synth.init_theta(O.tensor_table(net), [0.01] * 8, 7).astype(np.float64)
    O.set_threads(0)
    cores = O.threads()
    # each step: a bounded sample of the replica step (b_s of the 32 transitions) so K + W steps take ~2 min
    t0 = time.perf_counter()
    O.run(net, O.TrainCfg(minibatch=min(16, b_full), target_sync=1000), 1000, [rp], theta0, 1)
    per_tr = (time.perf_counter() - t0) / min(16, b_full)
    total = max(1, args.steps + args.warmup)
    b_s = int(max(1, min(b_full, 120.0 / (per_tr * total))))
    cfg = O.TrainCfg(minibatch=b_s, target_sync=1000)
    O.run(net, cfg, 1000, [rp], theta0, args.warmup)
    t0 = time.perf_counter()
    O.run(net, cfg, 1000, [rp], theta0, args.steps)
    dt = time.perf_counter() - t0
    v = args.steps * b_s / dt
    sample = (f"{args.steps} oracle replica steps of b={b_s} (of b={b_full}), Mnih net, replay 1k G-pong "
              f"(of 1M), fp64, {cores} OpenMP threads over the minibatch samples")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "BASELINE.json configs[1]" if world == 1 else "BASELINE.json configs[2]",
                       "minibatch": b_full, "replay": 1_000_000, "net": "Mnih-2013"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="auto", choices=["auto", "fp32", "bf16"])
    ap.add_argument("--replay", type=int, default=None, help="replay capacity per replica (default: the config's)")
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="BASELINE.json config (default: c2 at N = 1, c3 at N > 1)")
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--e2e-chunk", type=int, default=50, help="Alg. 1 iterations per dqn_store_and_train call (e2e)")
    ap.add_argument("--profile-steps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-acting", dest="acting", action="store_false",
                    help="skip the on-GPU acting measurement (NEXT-3)")
    ap.add_argument("--fc", type=int, default=None,
                    help="override the hidden FC width of the config's net (model-size sweep, SURVEY §8(d) BJ.c5)")
    ap.add_argument("--dedup", action="store_true",
                    help="frame-deduplicated replay (F+1 frames per slot; G-pong stacks slide by one frame)")
    ap.add_argument("--prio-alpha", type=float, default=0.0,
                    help="prioritized replay variant (NEXT-4, A41): alpha in {1, 0.5}; 0 = uniform (default)")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import numpy as np
    import torch

    import paper_1508_04186_b200 as D
    import synth

    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()  # the context's stream: data generation, the library and the events share it
    torch.cuda.set_stream(stream)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [D.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    else:
        dist = None
        nccl_id = None

    def barrier():
        if dist is not None:
            dist.barrier()

    ck = args.config or ("c2" if world == 1 else "c3")
    C = CONFIGS[ck]
    if args.replay is None:
        args.replay = C["replay"]
    prec = {"fp32": D.FP32, "bf16": D.BF16}.get(args.precision)
    b = C["b"]
    net = C["net"] if args.fc is None else dict(C["net"], fcs=(args.fc,))
    cfg = None
    for p in ([prec] if prec is not None else [D.BF16, D.FP32]):
        cfg = D.Config(**net, minibatch=b, replay_capacity=args.replay, target_sync=C["C"], precision=p,
                       lr=2.5e-4, gamma=0.99, n_push=C["n_push"], n_fetch=C["n_fetch"],
                       sync_mode=D.ASYNC if C["async"] else D.DETERMINISTIC, replay_dedup=int(args.dedup),
                       replay_prio_alpha=args.prio_alpha, replay_prio_eps=0.01 if args.prio_alpha else 0.0)
        try:
            dqn = D.DQN(cfg, rank=rank, world=world, nccl_id=nccl_id, stream=stream.cuda_stream)
            break
        except D.DqnError as e:
            if prec is not None or p == D.FP32 or e.code != D.EINVAL:
                raise
    dtype = "bf16" if cfg.precision == D.BF16 else "f32"

    # ---- prefill the replay memory with G-pong transitions generated on the GPU
    t0 = time.time()
    chunk = 8192
    done = 0
    while done < args.replay:
        n = min(chunk, args.replay - done)
        s, a, r, sn, t = synth.g_pong_torch(n, 4, 84, 84, net["n_actions"], 0x5EED + 1000 * rank + done, "cuda")
        dqn.push(s, a, r, sn, t)
        done += n
    del s, a, r, sn, t
    torch.cuda.synchronize()
    prefill_s = time.time() - t0

    # ---- warm-up (captures the step graphs)
    dqn.train(args.warmup)
    torch.cuda.synchronize()
    barrier()

    # ---- timed region: K steps in one dqn_train_steps call. The library records CUDA events on its stream
    # right before the first step graph launch and right after the last one (stats.device_ms), so the
    # call's closing host sync and counter readback stay outside; the bracket below is barrier + sync.
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        out = dqn.train(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms_bracket = ev0.elapsed_time(ev1)
    ms = float(out["device_ms"])
    launches = out["kernel_launches"]
    if dist is not None:
        tt = torch.tensor([ms, ms_bracket], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, ms_bracket = float(tt[0].item()), float(tt[1].item())
    value = world * b * args.steps / (ms / 1e3)

    # ---- e2e: through the public API with host buffers; per step push the step's new experience
    # (Alg. 1: one Store per iteration) from pinned host memory, run the step, read the loss back
    ne = args.e2e_steps
    gp = synth.g_pong(ne + 3, 4, 84, 84, 6, 99 + rank)  # s' = s shifted by one frame + a new frame
    hs = torch.from_numpy(gp[0]).pin_memory()
    hsn = torch.from_numpy(gp[3]).pin_memory()
    ha = torch.zeros(ne, dtype=torch.int32).pin_memory()
    hr = torch.zeros(ne, dtype=torch.float32).pin_memory()
    ht = torch.zeros(ne, dtype=torch.uint8).pin_memory()
    for i in range(min(3, ne)):  # untimed warm-up of both host-push paths
        dqn.push(hs[i:i + 1], ha[i:i + 1], hr[i:i + 1], hsn[i:i + 1], ht[i:i + 1])
        dqn.train(1, want_loss=True)
        if not C["async"]:
            dqn.train(1, want_loss=True, store=(hs[i:i + 1], ha[i:i + 1], hr[i:i + 1], hsn[i:i + 1], ht[i:i + 1]))

    def timed(fn):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        if dist is not None:
            tt = torch.tensor([t], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    # (1) Alg. 1's loop through dqn_store_and_train, `chunk` iterations per call: every iteration stores
    # its new experience (H2D from pinned host memory) and runs one step; every step's loss comes back
    ch = max(1, args.e2e_chunk)

    def loop_store_and_train():
        for i0 in range(0, ne, ch):
            m = min(ch, ne - i0)
            sl = slice(i0, i0 + m)
            dqn.train(m, want_loss=True, store=(hs[sl], ha[sl], hr[sl], hsn[sl], ht[sl]))

    # (2) one push call and one train call (with its host sync) per step
    def loop_sync_per_step():
        for i in range(ne):
            dqn.push(hs[i:i + 1], ha[i:i + 1], hr[i:i + 1], hsn[i:i + 1], ht[i:i + 1])
            dqn.train(1, want_loss=True)

    ems1 = timed(loop_sync_per_step)
    ems = ems1 if C["async"] else timed(loop_store_and_train)  # store_and_train is the deterministic schedule's
    h2d = 2 * 4 * 84 * 84 + 4 + 4 + 1
    e2e = {"value": world * b * ne / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": 4 + 48 / ch, "steps": ne,
           "what": (f"Alg. 1 loop through dqn_store_and_train, {ch} iterations per call: per step the new experience "
                    "H2D from pinned host memory, its Store, one replica step, its loss D2H; one host sync per call")
           if not C["async"] else "DQN_ASYNC: as sync_per_step (dqn_store_and_train needs the deterministic schedule)",
           "sync_per_step": {"value": world * b * ne / (ems1 / 1e3), "d2h_bytes_per_step": 4 + 48,
                             "what": "per step: dqn_push_transitions(1, pinned host) + dqn_train_steps(1) "
                                     "(host sync) + loss/counters D2H"}}

    # ---- NEXT-3 acting: on-GPU Snake games, eps-greedy on Q from the forward, Store into the replay
    acting = None
    if args.acting and world == 1:
        acfg = D.Config(**dict(MNIH, n_actions=4), minibatch=256, replay_capacity=100_000, precision=cfg.precision)
        ag = D.DQN(acfg, stream=stream.cuda_stream)
        ag.collect(256, 12, 3, 0.1, 0xACE)  # creates the games; warm-up
        ares = ag.collect(256, 12, 100, 0.1, 0xACE)
        acting = {"env_steps_per_s": ares["env_steps"] / (ares["device_ms"] / 1e3), "n_envs": 256, "steps": 100,
                  "epsilon": 0.1, "game": "Snake 12x12 rendered 84x84 (P:216, SPEC closures)",
                  "what": "per step: Q forward of 256 stacks, eps-greedy, game step + render, Store into the replay"}
        ag.close()

    # ---- per-region device times (CUDA events inside the replayed step graph)
    regions = dqn.profile(args.profile_steps) if args.profile_steps > 0 else []
    roof = roofline(regions, b, net, world, dtype, args.profile_steps) if regions else None

    if rank != 0:
        dqn.close()
        if dist is not None:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "timing": {"device_ms": ms, "bracket_ms": ms_bracket,
                   "what": "device_ms: CUDA events the library records on its stream around the K steps' graph "
                           "launches (max over ranks); bracket_ms: events around the whole dqn_train_steps call "
                           "(includes its closing counter readback and host sync)"},
        "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": {"workload": f"BASELINE.json configs[{C['idx']}]" + (f", FC width {args.fc} (model-size sweep)"
                                                                      if args.fc is not None else ""),
                   "net": net_name(net), "minibatch_per_replica": b,
                   "replay_per_replica": args.replay, "replay_dedup": bool(args.dedup),
                   "replay_sampling": (f"prioritized, alpha {args.prio_alpha} (A41)" if args.prio_alpha else "uniform"),
                   "target_sync_C": C["C"] if C["C"] < 2**40 else None,
                   "n_push": C["n_push"], "n_fetch": C["n_fetch"],
                   "sync_mode": "async (a fetch takes the newest published generation)" if C["async"] else "deterministic",
                   "parallelism": f"dp{world} + sharded parameter server", "gamma": 0.99,
                   "l2": f"inputs larger than L2: each step gathers {b} random s and s' slots of a "
                         f"{args.replay * 56454 / 1e9:.1f} GB replay from HBM (bf16 path: the step's forward "
                         "bulk-prefetches the next step's slots into L2; the counter-based sampler knows them)",
                   "prefill_s": round(prefill_s, 1)},
        "gpu_launches": launches,
        "staleness_hist": [int(x) for x in out["staleness"][:8]] if C["async"] else None,
        "clocks": clk.summary(),
        "e2e": e2e,
        "acting": acting,
        "roofline": roof,
        "regions_us": {r["name"]: round(r["avg_us"], 2) for r in regions},
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)
    dqn.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
