"""Stall samples of an ncu --set full capture aggregated per CUDA source line, with the top
stall reasons of each line:  python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg, why, line, fname = {}, {}, None, ""
for r in rows[rows.index(hdr) + 1:]:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) <= i_s or r[0] == "Line No":
        continue
    if r[0]:
        line = (f"{fname}:{r[0]}", r[1].strip()[:64])
    if r[i_s].isdigit() and line:
        agg[line] = agg.get(line, 0) + int(r[i_s])
        w = why.setdefault(line, {})
        for i, h in reasons:
            if r[i].isdigit():
                w[h] = w.get(h, 0) + int(r[i])
tot = sum(agg.values())
print(f"{tot} samples")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    rs = sorted(why[k].items(), key=lambda x: -x[1])[:3]
    print(f"{v:6d} {100 * v / tot:5.1f}%  {k[0]:26s} {k[1]:64s} " +
          " ".join(f"{h[6:]}={n}" for h, n in rs if n))
