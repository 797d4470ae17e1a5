"""Diagnostic: per-phase latency of the token-select kernel (globaltimer stamps)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = W.CONFIGS[name]
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
cs = tls.cluster_size(cfg, 0)
buf = torch.zeros((w.batch * w.num_kv_heads * cs, 8), dtype=torch.int64, device="cuda")
lib = tls.load()
for it in range(3):
    lib.tls_debug_phase_timing(buf.data_ptr() if it == 2 else None)
    tls.select(cfg, queries[it], inputs["seq_lens"], idx)
torch.cuda.synchronize()
lib.tls_debug_phase_timing(None)
t = buf.cpu().double()
if cs > 1:
    t = t.view(-1, cs, 8)[:, 0, :]  # rank 0 runs every phase
t0 = t[:, 0].min()
names = ["q gather + block top-k", "stats pass (ring)", "stats merge", "keys pass (ring)", "key exchange", "top-k_t + emit", "-"]
d = (t[:, 1:] - t[:, :-1]) / 1e3
print(f"{name}: cs={cs} ctas={t.shape[0]} kernel span {(t[:, 7].max() - t0) / 1e3:.1f} us; "
      f"CTA lifetime median {((t[:, 7] - t[:, 0]) / 1e3).median():.1f} us")
for i, nm in enumerate(names):
    print(f"  {nm:14s} median {d[:, i].median():7.2f} us  p90 {d[:, i].quantile(0.9):7.2f} us")
starts = ((t[:, 0] - t0) / 1e3).sort().values
print("  CTA start times (us) quantiles:", [round(float(starts[int(q * (len(starts) - 1))]), 1) for q in (0, .25, .5, .75, 1)])
