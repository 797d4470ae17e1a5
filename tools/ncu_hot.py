"""Summarise an ncu SASS source page (csv) -> hottest instructions and stall mix.
usage: ncu -i X.ncu-rep --page source --csv --print-source=sass > s.csv; python tools/ncu_hot.py s.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = []
for r in rows[2:]:  # first kernel section only
    if r and r[0] == "Kernel Name":
        break
    data.append(r)
ix = {h: i for i, h in enumerate(hdr)}
samp = ix["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[samp] or 0) for r in data)
agg = {s: sum(int(r[ix[s]] or 0) for r in data) for s in stalls}
print(f"total samples {tot}")
for s, v in sorted(agg.items(), key=lambda x: -x[1])[:8]:
    print(f"  {s:28s} {100.0 * v / max(tot, 1):5.1f}%")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
order = sorted(range(len(data)), key=lambda i: -int(data[i][samp] or 0))[:N]
for i in sorted(order):
    r = data[i]
    top = sorted(((int(r[ix[s]] or 0), s) for s in stalls), reverse=True)[:2]
    print(f"{i:6d} {100.0 * int(r[samp]) / tot:5.1f}%  {r[1].strip()[:60]:60s} {top[0][1]}:{top[0][0]} {top[1][1]}:{top[1][0]}")
