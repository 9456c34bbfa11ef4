"""Per-launch summary of an ncu --set full report exported with `ncu -i X --page raw --csv`: time, DRAM bytes,
tensor-pipe and memory-throughput percentages. usage: python tools/ncu_summary.py raw.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units, rows = rows[0], rows[1], rows[2:]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3,
         "msecond": 1e3}


def val(d, k):
    i = h.index(k)
    v = d[i].replace(",", "")
    return float(v) * SCALE.get(units[i], 1.0)


cols = [("us", "gpu__time_duration.sum"), ("dram_rd_MB", "dram__bytes_read.sum"),
        ("dram_wr_MB", "dram__bytes_write.sum"),
        ("tensor_pipe_%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("bf16_ops_%", "sm__ops_path_tensor_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed"),
        ("mem_%", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")]
print("kernel,grid," + ",".join(c[0] for c in cols))
for r in rows:
    d = dict(zip(h, r))
    out = []
    for name, k in cols:
        if k not in h:
            out.append("")
            continue
        v = val(r, k)
        if name.endswith("_MB"):
            v /= 1e6
        out.append(f"{v:.2f}")
    print(f'{d["Kernel Name"].split("(")[0][:32]},"{d["Grid Size"]}",' + ",".join(out))
