"""Markdown table of a model-size sweep (tools/model_sweep.sh JSON lines): P, transitions/s, µs/step, and the
per-step gradient time T (forward + backward regions), update / server-round time tau (Fig. 3's lines)."""
import json
import sys

UPD = ("rmsprop_update", "reduce_update", "server_round_fused", "push_reduce_scatter", "fetch_all_gather")
print("| net | N | transitions/s | µs/step | T: gradient regions µs | tau (+comm): update/round regions µs | T / tau |")
print("|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    d = json.loads(line)
    reg = d.get("regions_us", {})
    tau = sum(v for k, v in reg.items() if k in UPD)
    T = sum(v for k, v in reg.items() if k not in UPD)
    print(f"| {d['config']['net']} | {d['n_gpus']} | {d['value'] / 1e3:.0f} K | {d['ms_per_step'] * 1e3:.1f} | "
          f"{T:.1f} | {tau:.1f} | {T / tau if tau else float('nan'):.1f} |")
