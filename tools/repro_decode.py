"""Diagnostic: run tls_decode on a (possibly reduced) config and synchronise."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

name = sys.argv[1]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else None
what = sys.argv[3] if len(sys.argv) > 3 else "decode"
w = W.CONFIGS[name]
if batch:
    w = w.with_(batch=batch)
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
for i in range(3):
    if what == "decode":
        tls.decode(cfg, queries[i], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    else:
        sel = tls.select(cfg, queries[i], inputs["seq_lens"], idx)
        tls.sparse_attend(cfg, queries[i], inputs["k_cache"], inputs["v_cache"], sel[1], sel[2])
    torch.cuda.synchronize()
    print("step", i, "ok", flush=True)
