"""Aggregate an ncu source page exported with --print-source=sass,cuda by CUDA
source line: stall samples, instructions executed and the top stall reasons.
usage: ncu -i X.ncu-rep -k regex:K --page source --csv --print-source=sass,cuda > m.csv
       python tools/ncu_lines.py m.csv [N] [--by inst|samples]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
by = 1 if "inst" in sys.argv else 0
f, hdr, ix, cur = None, None, {}, None
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(hdr)}
        continue
    if not r[0]:
        continue
    cur = (f, int(r[0]))
    src[cur] = r[1]
    num = lambda i: int(r[i]) if i < len(r) and r[i].isdigit() else 0
    agg[cur][0] += num(4)
    agg[cur][1] += num(7)
    for h in hdr:
        if h.startswith("stall_") and "Not Issued" not in h and num(ix[h]):
            agg[cur][2][h[6:]] += num(ix[h])
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts}  warp-instructions {ti}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][by])[:N]:
    print(f"{k[0]:14s}{k[1]:5d} smp {100 * v[0] / ts:5.1f}% inst {100 * v[1] / ti:5.1f}%  "
          f"{src[k].strip()[:64]:64s} {dict(v[2].most_common(2))}")
