"""profiles/r2_traffic.json from the round's `ncu --set full` captures (exported with
`ncu -i X.ncu-rep --page raw --csv`): DRAM bytes (read + write) per launch of every kernel of one step, keyed
the way bench.py's roofline looks them up.

  mnih   : per kernel name (every launch of the Mnih path's kernels is one per step)
  scaled : per bench region of the generic path (one step's launches in order, attributed to the region whose
           kernels they are; the side-branch head finish and FC update are not in a main-stream region)

usage: python tools/traffic_json.py mnih_raw.csv scaled_raw.csv > profiles/r2_traffic.json
"""
import csv
import json
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    rows = list(csv.reader(open(path)))
    h, units, rows = rows[0], rows[1], rows[2:]
    ri, wi, ti = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("gpu__time_duration.sum")
    out = []
    for r in rows:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("dqn::", "").split("<")[0]
        rd = float(r[ri].replace(",", "")) * SCALE[units[ri]]
        wr = float(r[wi].replace(",", "")) * SCALE[units[wi]]
        us = float(r[ti].replace(",", "")) * (1e-3 if units[ti] in ("ns", "nsecond") else 1.0)
        out.append(dict(kernel=name, grid=r[h.index("Grid Size")], dram_read_MB=rd / 1e6, dram_write_MB=wr / 1e6,
                        ncu_us=us))
    return out


def mnih(path):
    t = {}
    for l in launches(path):
        t.setdefault(l["kernel"], dict(dram_read_MB=l["dram_read_MB"], dram_write_MB=l["dram_write_MB"],
                                       ncu_us=l["ncu_us"]))
    return t


def scaled(path):
    ls = launches(path)
    starts = [i for i, l in enumerate(ls) if l["kernel"] == "gather_s2d_kernel"]
    i0 = starts[0]
    # one step from a gather to the next; with a single gather in the capture, the launches before it are the
    # previous step's tail and complete the cycle (the capture holds at least one step's worth of launches)
    if len(starts) > 1:
        step = ls[i0:starts[1]]
    else:  # the capture's last launches repeat its first ones (the next step began): count them once
        names = [l["kernel"] for l in ls]
        k = max((k for k in range(i0 + 1) if names[:k] == names[len(names) - k:]), default=0)
        step = ls[i0:] + ls[k:i0]
    reg = {}
    seen_head = False
    tg = 0
    for l in step:
        k = l["kernel"]
        if k in ("gather_s2d_kernel",) or (k == "tconv_kernel" and not seen_head):
            r = "conv_fwd"
        elif k == "tgemm_kernel":
            r = "fc1_fwd" if tg == 0 else "fc1_bwd_head_finish"
            tg += 1
        elif k.startswith("head_sample"):
            r = "head_sample"
            seen_head = True
        elif k == "chw_to_hwc_kernel":
            r = "fc1_bwd_head_finish"
        elif k in ("twgrad_kernel", "gconv_wreduce_kernel") or (k == "tconv_kernel" and seen_head):
            r = "conv_bwd"
        else:
            continue  # gpack (before the gather) and the side branch (head finish, the FC update)
        e = reg.setdefault(r, dict(bytes=0.0, launches=0, ncu_us=0.0))
        e["bytes"] += (l["dram_read_MB"] + l["dram_write_MB"]) * 1e6
        e["launches"] += 1
        e["ncu_us"] += l["ncu_us"]
    return dict(regions=reg, step_launches=[l["kernel"] for l in step])


if __name__ == "__main__":
    print(json.dumps({"source": "ncu --set full --clock-control none (cold caches per launch), round 2",
                      "mnih": mnih(sys.argv[1]), "scaled": scaled(sys.argv[2])}, indent=1))
