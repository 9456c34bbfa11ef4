"""profiles/r2_summary.md: the round-2 evidence in one page, generated from the committed files under profiles/
(bench lines, launch lists, ncu summaries, traffic, sweep, GPU test log, mutation check).

usage: python tools/r2_summary.py > profiles/r2_summary.md
"""
import csv
import json
import os

P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")


def line(name):
    with open(os.path.join(P, f"r2_bench_{name}.json")) as f:
        return json.loads([l for l in f if l.startswith("{")][0])


def fmt(v):
    return f"{v / 1e6:.2f} M" if v >= 1e6 else f"{v / 1e3:.0f} K"


rows = [("n1", "BJ.configs[1]: Mnih, b = 32, 1M-slot replay, C = 1000", 1),
        ("n1_20", "the same at the driver's 20 steps", 1),
        ("c1", "BJ.configs[0]: replay 1 k", 1),
        ("n2", "BJ.configs[2]: fused server round", 2),
        ("n4", "BJ.configs[2]: fused server round", 4),
        ("c4", "BJ.configs[3]: Mnih, b = 256, async n_push = n_fetch = 10", 1),
        ("c4_n4", "BJ.configs[3]", 4),
        ("c5", "BJ.configs[4]: scaled net, b = 512", 1),
        ("c5_n2", "BJ.configs[4], fused round", 2),
        ("c5_n4", "BJ.configs[4], fused round", 4),
        ("c2_prio", "BJ.configs[1] + prioritized replay (A41)", 1)]
print("# Round 2 profiles — B200 (sm_100a)\n")
print("The numbers come from `gpurun` boxes at the end of the round. `tools/final_r2.sh` on one 4-GPU box produced the")
print("reference arm, the sweep, and the ncu launch lists and captures. Every ncu pass ran after the same command had")
print("exited 0 without ncu. Lines whose code changed afterwards were re-measured on later boxes:")
print("* BJ.configs[2] (`tools/final_r2_round.sh`, then `tools/final_r2_multi.sh`);")
print("* BJ.configs[3] and the GPU suite (`tools/final_r2_last.sh`);")
print("* BJ.configs[1] at N = 1 and a 2-GPU suite (`tools/final_r2_n1.sh`).")
print("Clocks: see each line's `clocks` (1965 MHz, no throttle reason).\n")
print("## Bench lines (`bench.py`, device-timed, max over ranks)\n")
print("| file | workload | N | transitions/s | µs/step | e2e | dominant region | bound, fraction | step tensor / HBM |")
print("|---|---|---|---|---|---|---|---|---|")
base = {}
for name, what, n in rows:
    try:
        d = line(name)
    except (OSError, IndexError):
        continue
    r = d.get("roofline") or {}
    st = r.get("step") or {}
    frac = f"{r.get('bound')} {100 * (r.get('frac') or 0):.1f} %" if r else "—"
    stf = f"{100 * st.get('tensor_frac', 0):.1f} % / {100 * st.get('hbm_frac', 0):.1f} %" if st else "—"
    print(f"| `r2_bench_{name}.json` | {what} | {n} | **{fmt(d['value'])}** | {d['ms_per_step'] * 1e3:.1f} | "
          f"{fmt(d['e2e']['value'])} | {r.get('kernel', '—')} ({r.get('avg_us', 0):.1f} µs) | {frac} | {stf} |")
ref = line("ref")
cb = line("n1").get("cpu_baseline") or {}
print(f"\nReference arm (`r2_bench_ref.json`, the fp64 oracle as the reference, {ref['cpu_baseline']['cores']} threads): "
      f"{ref['value']:.0f} tr/s. `cpu_baseline` of the N = 1 line: {cb.get('value', 0):.0f} tr/s on "
      f"{cb.get('cores')} threads ({(cb.get('single_thread') or {}).get('value', 0):.0f} on one), {cb.get('cpu_model', '')}.\n")
for tag, title in (("c2", "BJ.configs[1] (Mnih path)"), ("c5", "BJ.configs[4] (generic path)")):
    print(f"## Launch list, {title} (`r2_{tag}_launches_summary.txt`: per launch, serialised, cold caches)\n")
    print("```")
    with open(os.path.join(P, f"r2_{tag}_launches_summary.txt")) as f:
        print("".join(l for l in f.readlines()[:24]).rstrip())
    print("```\n")
    print(f"## `ncu --set full`, one step of {title} (`r2_{tag}_ncu_full_summary.csv`)\n")
    rr = list(csv.reader(open(os.path.join(P, f"r2_{tag}_ncu_full_summary.csv"))))
    print("| " + " | ".join(rr[0]) + " |")
    print("|" + "---|" * len(rr[0]))
    for r in rr[1:]:
        print("| " + " | ".join(r) + " |")
    print()
t = json.load(open(os.path.join(P, "r2_traffic.json")))
print("## DRAM traffic per step region (`r2_traffic.json`, from the captures above; the bench's `roofline.traffic`)\n")
print("| region (generic path) | launches | ncu µs | DRAM MB |")
print("|---|---|---|---|")
for k, v in t["scaled"]["regions"].items():
    print(f"| {k} | {v['launches']} | {v['ncu_us']:.1f} | {v['bytes'] / 1e6:.1f} |")
print("\n## Model-size sweep (`r2_sweep.md`, SURVEY §8(d) BJ.c5)\n")
print(open(os.path.join(P, "r2_sweep.md")).read().rstrip())
log = open(os.path.join(P, "r2_pytest_gpu.log")).read().splitlines()
print("\n## GPU tests and mutation check\n")
print(f"`r2_pytest_gpu.log` (4-GPU box, `-rA`): {[l for l in log if 'passed' in l][-1].strip()}. "
      f"`r2_mutations.txt`: {open(os.path.join(P, 'r2_mutations.txt')).read().splitlines()[-1].strip()}. "
      f"Smoke (`r2_smoke.log`): {'; '.join(l.strip() for l in open(os.path.join(P, 'r2_smoke.log')) if l.startswith('smoke'))}.")
print(f"\nStep timeline of the N = 1 Mnih step (`r2_trace_step.txt`, CTA 0 globaltimer stamps, 256 ns resolution).")
