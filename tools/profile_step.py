"""Run a few steps of one call (decode / select / attend) for ncu capture:
    ncu --set full -k regex:tls_decode -s 3 -c 1 -o prof python tools/profile_step.py --what decode
Not a bench line (numbers under a profiler are never reported)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--what", default="decode", choices=["decode", "select", "attend", "all"])
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--batch", type=int, default=0)
args = ap.parse_args()
w = W.CONFIGS[args.config]
if args.batch:
    w = w.with_(batch=args.batch)
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
sel = tls.select(cfg, queries[0], inputs["seq_lens"], idx)
whats = ["select", "attend", "decode"] if args.what == "all" else [args.what]
for i in range(args.steps):
    for wh in whats:
        if wh == "decode":
            tls.decode(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
        elif wh == "select":
            tls.select(cfg, queries[i % 8], inputs["seq_lens"], idx, out=sel)
        else:
            tls.sparse_attend(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"], sel[1], sel[2])
torch.cuda.synchronize()
print("done")
