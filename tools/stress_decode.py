"""Diagnostic: run many decode steps (with L2 flushes) and synchronise each."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
w = W.CONFIGS[name]
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(steps):
    flush.fill_(1)
    tls.select(cfg, queries[i % 8], inputs["seq_lens"], idx)
    tls.decode(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    torch.cuda.synchronize()
print(name, "stress ok", steps, flush=True)
