"""Per-kernel DRAM traffic from an ncu launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum): average bytes and time per launch.

python tools/traffic_summary.py launches.csv [out.json]
"""
import csv
import json
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui, idi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                       h.index("Metric Unit"), h.index("ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}
per = defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    names[r[idi]] = r[ki]
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    k = names[i].split("(")[0].replace("void ", "")[:60]
    a = agg[k]
    a[0] += 1
    a[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[2] += m.get("gpu__time_duration.sum", 0)
out = {k: {"launches": n, "dram_bytes_per_launch": round(b / n), "us_per_launch": round(1e6 * t / n, 2)}
       for k, (n, b, t) in sorted(agg.items(), key=lambda x: -x[1][2])}
print(json.dumps(out, indent=1))
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
