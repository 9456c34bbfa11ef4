"""Summarise an ncu --csv launch list by (kernel, grid): mean us per launch and launches."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr, rows = rows[0], rows[1:]
ki, gi, vi, ui = hdr.index("Kernel Name"), hdr.index("Grid Size"), hdr.index("Metric Value"), hdr.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows:
    d[(r[ki].split("(")[0].replace("void ", ""), r[gi])].append(float(r[vi]) * (1e-3 if r[ui] == "ns" else 1.0))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k[0][:30]:30s} {k[1]:16s} n={len(v):4d} mean={sum(v) / len(v):8.2f} us share={sum(v) / tot:6.1%}")
