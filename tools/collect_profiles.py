"""Copy one gpu_profile.sh capture (gpurun_out/*_<V>*) into profiles/: the launch lists
(one text table), ncu --set full summaries, traffic.json (dram read + write per launch),
bench lines, smoke log, step timeline.  usage: python tools/collect_profiles.py v16"""
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys

V = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
KEY = {"select_kernel": "select_kernel", "token_reg_kernel": "token_cluster_kernel",
       "token_cluster_kernel": "token_cluster_kernel", "attend_kernel": "attend_kernel",
       "attend_mla_kernel": "attend_kernel"}
WL = {"c3": "c3-qwen3-32b-96k-b32", "c2": "c2-qwen3-8b-48k-b16", "c4": "c4-glm47flash-mla-64k-b32"}

out = []
for c in ("c3", "c2", "c4"):
    f = os.path.join(G, f"launches_{c}_{V}.csv")
    if not os.path.exists(f):
        continue
    lines = open(f).read().splitlines()
    i = next(k for k, line in enumerate(lines) if line.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[i:]))))
    h = rows[0]
    iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    recs = {}
    for r in rows[1:]:
        recs.setdefault((int(r[iid]), r[ik]), {})[r[im]] = r[iv].replace(",", "")
    out.append(f"# {c}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
               f"smsp__inst_executed.sum --clock-control none -k regex:'qq_kernel|select|token|attend' -s 8 -c 8 "
               f"python bench.py --config {c} --steps 2 --warmup 3 (cold cache, serialised: compare shares)")
    for (k, name), m in sorted(recs.items()):
        out.append(f"{c} {k:3d} {name[:60]:60s} time_ns={float(m['gpu__time_duration.sum']):.0f} "
                   f"dram_read={float(m['dram__bytes_read.sum']):.0f} dram_write={float(m['dram__bytes_write.sum']):.0f} "
                   f"inst={float(m['smsp__inst_executed.sum']):.0f}")
open(os.path.join(P, f"r01_launches_{V}.txt"), "w").write("\n".join(out) + "\n")


def traffic(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, v = rows[0], rows[1], rows[-1]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def get(k):
        i = h.index(k)
        return float(v[i].replace(",", "")) * mult.get(units[i], 1)
    return get("dram__bytes_read.sum") + get("dram__bytes_write.sum")


tpath = os.path.join(P, "traffic.json")
tr = json.load(open(tpath)) if os.path.exists(tpath) else {}
for rep in sorted(glob.glob(os.path.join(G, f"full_*_{V}.ncu-rep"))):
    base = os.path.basename(rep)[len("full_"):-len(".ncu-rep")]  # <kernel>_<cfg>_<V>
    kern, cfg = base[: -len(V) - 1].rsplit("_", 1)
    with open(os.path.join(P, f"r01_ncu_{base}.txt"), "w") as f:
        f.write(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                               capture_output=True, text=True).stdout)
    tr.setdefault(WL[cfg], {})[KEY[kern]] = traffic(rep)
json.dump(tr, open(tpath, "w"), indent=1)
for c in ("c3", "c2", "c4"):
    src = os.path.join(G, f"bench_{c}_{V}.json")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(P, f"r01_bench_{c}_{V}.json"))
for src, dst in ((f"bench_ref_{V}.json", f"r01_bench_reference_c3_{V}.json"), (f"smoke_{V}.log", f"r01_smoke_{V}.log"),
                 (f"timeline_{V}.txt", f"r01_timeline_{V}.txt")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
print(json.dumps(tr, indent=1))
