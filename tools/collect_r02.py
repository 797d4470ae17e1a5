"""Round-2 evidence: gpurun_out/r02* of tools/gpu_profile_r02.sh -> profiles/ (launch lists, ncu --set full
summaries with tensor-pipe utilisation and the top warp-stall reasons, traffic.json, bench lines, smoke,
timeline).   usage: python tools/collect_r02.py v1"""
import csv
import glob
import io
import json
import os
import re
import shutil
import subprocess
import sys

V = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.environ.get("TLS_PROFILES_OUT", os.path.join(ROOT, "profiles"))
WL = {"c3": "c3-qwen3-32b-96k-b32", "c2": "c2-qwen3-8b-48k-b16", "c4": "c4-glm47flash-mla-64k-b32"}
SLOT = {"select_kernel": "select_kernel", "token_reg_kernel": "token_cluster_kernel", "token_pair_kernel": "token_pair_kernel", "token_pair_nt_kernel": "token_pair_nt_kernel",
        "token_cluster_kernel": "token_cluster_kernel", "attend_kernel": "attend_kernel",
        "attend_mla_kernel": "attend_kernel", "qq_kernel": "qq_kernel"}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__cluster_dim_x", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]

# ---- launch lists
out = []
for c in ("c3", "c2", "c4"):
    f = os.path.join(G, f"r02launch_{c}_{V}.csv")
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
open(os.path.join(P, f"r02_launches_{V}.txt"), "w").write("\n".join(out) + "\n")

# ---- ncu --set full summaries
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
traffic = {}
for f in sorted(glob.glob(os.path.join(G, f"r02full_*_{V}.ncu-rep"))):
    m = re.match(r"r02full_(.+)_(c\d)_" + V, os.path.basename(f)[:-8])
    kern, cfg = m.group(1), m.group(2)
    txt = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        continue
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    lines = [f"# ncu --set full --clock-control none --import-source on -k regex:^{kern} -s 3 -c 1 "
             f"python tools/profile_step.py --config {cfg} --steps 3  (one launch, {WL[cfg]})"]
    for k in KEYS:
        if k in d:
            lines.append(f"{k:70s} {d[k]} {u[k]}")
    tens = [k for k in h if "tensor" in k and ("pct" in k or k.endswith(".sum")) and d.get(k, "") not in ("", "n/a")]
    for k in tens[:12]:
        lines.append(f"{k:70s} {d[k]} {u[k]}")
    stalls = []
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(d[k].replace(",", "")), k))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    lines.append("top warp-stall reasons (warps stalled per issue-active cycle):")
    for val, k in stalls[:8]:
        lines.append(f"   {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {val:.3f}")
    open(os.path.join(P, f"r02_ncu_{kern}_{cfg}_{V}.txt"), "w").write("\n".join(lines) + "\n")
    try:
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * mult.get(u["dram__bytes_read.sum"], 1)
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * mult.get(u["dram__bytes_write.sum"], 1)
        traffic.setdefault(WL[cfg], {})[SLOT.get(kern, kern)] = rd + wr
    except (KeyError, ValueError):
        pass
old = {}
tp = os.path.join(P, "traffic.json")
if os.path.exists(tp):
    old = json.load(open(tp))
for w, ks in traffic.items():
    old.setdefault(w, {}).update(ks)
json.dump(old, open(tp, "w"), indent=1)

# ---- bench lines, smoke, timeline
for c in ("c3", "c2", "c4"):
    f = os.path.join(G, f"r02bench_{c}_{V}.json")
    if os.path.exists(f):
        shutil.copy(f, os.path.join(P, f"r02_bench_{c}_{V}.json"))
for src, dst in ((f"r02smoke_{V}.log", f"r02_smoke_{V}.log"), (f"r02timeline_{V}.txt", f"r02_timeline_{V}.txt"),
                 (f"r02k2stamps_{V}.txt", f"r02_k2stamps_{V}.txt")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
print("collected", V)
