"""Top SASS lines by warp-stall samples from `ncu -i rep --page source --csv` (stdin)."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
top = int(sys.argv[1]) if len(sys.argv) > 1 else 25
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        name = rows[i][1][:90]
        hdr = rows[i + 1]
        si = hdr.index("Warp Stall Sampling (All Samples)")
        data = []
        j = i + 2
        while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
            try:
                data.append((int(rows[j][si]), rows[j][1].strip()[:100]))
            except (ValueError, IndexError):
                pass
            j += 1
        tot = sum(d[0] for d in data) or 1
        print(f"== {name}  samples={tot}")
        for n, src in sorted(data, reverse=True)[:top]:
            print(f"  {n / tot:6.1%}  {src}")
        i = j
    else:
        i += 1
