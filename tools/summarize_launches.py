"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki][:90]
        v = float(r[vi].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
allt = sum(tot.values())
unit = hdr[hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
print(f"total {allt/1e3:.1f} us over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v/1e3:10.1f} us {100*v/allt:5.1f}%  n={cnt[k]:5d}  avg={v/cnt[k]/1e3:8.2f} us  {k}")
