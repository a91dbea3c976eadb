"""Per-kernel DRAM traffic of one cycle from an ncu launch list.

    python tools/traffic.py launches.csv WORKLOAD TOP [profiles/traffic.json]

The launch list must carry dram__bytes_read.sum and dram__bytes_write.sum
(tools/gpu_full.sh); the last complete 3D cycle (k3_top* ... k3_up_cell of
level TOP) is named the way bench.py names kernels (k3_down_L6, ...), and
traffic.json[WORKLOAD][name] = read + write bytes of that launch.
"""
import collections
import csv
import json
import os
import sys

path, workload, top = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                        "traffic.json")
rows = list(csv.reader(open(path)))
hdr = None
launches = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = d["ID"]
    e = launches.setdefault(key, {"name": d["Kernel Name"]})
    unit = d.get("Metric Unit", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
             "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(unit, 1)
    e[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * scale
seq = list(launches.values())
def base(name):
    return name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]


starts = [k for k, e in enumerate(seq) if base(e["name"]).startswith("k3_top")]
assert starts, "no 3D cycle in the launch list"
res = {}
cur = up = None
for e in seq[starts[-2] if len(starts) > 1 else starts[-1]:]:
    fn = base(e["name"])
    b = e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
    if fn.startswith("k3_top") or fn == "k3_ffp":
        if res.get(f"k3_down_L{top}") is not None and cur is not None:
            break
        cur = top
        name = f"k3_down_L{top}"
    elif fn.startswith("k3_smooth") or fn in ("k3_smr", "k3_smc"):
        name = f"k3_smooth_L{cur}"
    elif fn == "k3_down_c":
        cur -= 1
        name = f"k3_down_L{cur}"
    elif fn == "k3_chain":
        name = "k3_chain"
        up = cur
    elif fn.startswith("k3_up"):
        name = f"k3_up_L{up}"
        up += 1
    else:
        continue
    res[name] = b
data = json.load(open(out)) if os.path.exists(out) else {}
data[workload] = res
json.dump(data, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
