"""Diagnostic: phase stamps of attend_mla_tc_kernel (TLS_DEBUG_BUF) at C4: per CTA, us from its start.
python tools/mla_tc_timeline.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

os.environ.setdefault("TLS_MLA_TC", "1")
w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
buf = torch.zeros(65536 * 32, dtype=torch.int64, device="cuda")
for it in range(4):
    if it == 3:
        buf.zero_()
        os.environ["TLS_DEBUG_BUF"] = hex(buf.data_ptr())
    tls.decode(cfg, queries[it % 8], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    torch.cuda.synchronize()
os.environ.pop("TLS_DEBUG_BUF", None)
d = buf[65536 * 24: 65536 * 24 + 32 * 512].view(512, 32).cpu().numpy().astype(np.int64)
d = d[d[:, 0] > 0]
t0 = d[:, 0].min()
names = {0: "start", 1: "prologue done", 18: "epilogue done", 19: "merge start", 20: "end"}
for c in range(4):
    names.update({3 + 4 * c: f"c{c} S done", 4 + 4 * c: f"c{c} P written"})
print(f"{len(d)} CTAs; us since the first CTA start: p10 / p50 / p90")
for i in sorted(names):
    col = d[:, i]
    ok = col > 0
    if ok.any():
        v = (col[ok] - t0) / 1e3
        print(f"  {names[i]:18s} {np.percentile(v, 10):7.1f} {np.percentile(v, 50):7.1f} {np.percentile(v, 90):7.1f}")
