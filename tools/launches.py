"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].replace("void ", "")[:48]
    v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
    agg.setdefault(k, []).append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'mean_us':>9s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:48s} {len(v):8d} {sum(v) / len(v):9.2f} {sum(v) / tot:7.1%}")
