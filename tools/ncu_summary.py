"""Summaries of an `ncu --set full` capture for profiles/: per-kernel table (markdown) and the per-launch DRAM
traffic JSON bench.py reads for roofline.traffic.
usage: ncu -i full.ncu-rep --page raw --csv --metrics <M> > raw.csv; python tools/ncu_summary.py raw.csv traffic.json"""
import csv
import json
import sys
from collections import defaultdict

M = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__grid_size",
     "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
     "lts__t_sector_hit_rate.pct", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
     "sm__warps_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def main(raw, out_json):
    rows = list(csv.reader(open(raw)))
    hdr, units = rows[0], rows[1]
    col = {m: hdr.index(m) for m in M if m in hdr}
    acc = defaultdict(lambda: defaultdict(list))
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        k = r[hdr.index("Kernel Name")].split("(")[0]
        for m, i in col.items():
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            acc[k][m].append(v * SCALE.get(units[i], 1.0))
    mean = lambda xs: sum(xs) / len(xs) if xs else float("nan")  # noqa: E731
    traffic = {}
    print("| kernel | launches | grid × block | regs | dyn smem KB | duration µs | DRAM read MB | DRAM write MB | "
          "warps active % | tc-pipe % | L2 hit % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for k, d in sorted(acc.items(), key=lambda kv: -mean(kv[1]["gpu__time_duration.sum"])):
        g = lambda m: mean(d.get(m, []))  # noqa: E731
        print(f"| {k} | {len(d['gpu__time_duration.sum'])} | {g('launch__grid_size'):.0f} × {g('launch__block_size'):.0f} | "
              f"{g('launch__registers_per_thread'):.0f} | {g('launch__shared_mem_per_block_dynamic'):.1f} | "
              f"{g('gpu__time_duration.sum'):.2f} | {g('dram__bytes_read.sum'):.2f} | {g('dram__bytes_write.sum'):.2f} | "
              f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{g('sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active'):.2f} | {g('lts__t_sector_hit_rate.pct'):.1f} |")
        traffic[k] = {"dram_read_MB": g("dram__bytes_read.sum"), "dram_write_MB": g("dram__bytes_write.sum"),
                      "ncu_us": g("gpu__time_duration.sum")}
    if out_json:
        json.dump(traffic, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
