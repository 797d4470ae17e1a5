"""Diagnostic: per-phase timeline of the fused step kernel (step.cu) from its
%globaltimer stamps (TLS_DEBUG_BUF): for every CTA, phase boundaries
start | a1 | a2 | a3 staged | a3 keys | a4 | a5 | merge end.  Prints phase
durations (percentiles over CTAs) and the CTA start/end spread.  Not a bench line."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = W.CONFIGS[name]
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
nc = tls.cluster_size(cfg, 2)
pairs = w.batch * w.num_kv_heads
buf = torch.zeros(65536 * 8 + pairs * nc * 2, dtype=torch.int64, device="cuda")
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(4):
    if it == 3:
        os.environ["TLS_DEBUG_BUF"] = hex(buf.data_ptr())
    flush_buf.fill_(1)
    ev[0].record()
    tls.decode(cfg, queries[it], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    ev[1].record()
    torch.cuda.synchronize()
    if it == 3:
        del os.environ["TLS_DEBUG_BUF"]
t = buf[: pairs * nc * 8].view(pairs, nc, 8).cpu().numpy().astype(np.float64)
x = buf[65536 * 8:].view(pairs, nc, 2).cpu().numpy().astype(np.float64)
t0 = t[:, :, 0].min()
t = (t - t0) / 1e3  # us
x = (x - t0) / 1e3
for nm, a, bcol, col in (("a2 wait for siblings (1st barrier)", 1, 0, 0), ("a4 wait for siblings (1st barrier)", 4, 1, 0)):
    dlt = (x[:, :, bcol] - t[:, :, a]).ravel()
    print(f"  {nm:36s}" + "  ".join(f"{np.percentile(dlt, p):6.1f}" for p in (0, 10, 50, 90, 100)))
print(f"{w.name}: pairs={pairs} nc={nc} step (event, with stamps) {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us")
names = ["a1 (stream+gemv)", "a2 (top-k_b)", "a3 stage wait", "a3 compute", "a4 (top-k_t)", "a5 attention", "a5 merge"]
pct = [0, 10, 50, 90, 100]
print("  phase (us per CTA)        " + "  ".join(f"p{p:<5d}" for p in pct))
for i, nm in enumerate(names):
    dlt = (t[:, :, i + 1] - t[:, :, i]).ravel()
    print(f"  {nm:24s}" + "  ".join(f"{np.percentile(dlt, p):6.1f}" for p in pct))
life = (t[:, :, 7] - t[:, :, 0]).ravel()
print(f"  {'CTA lifetime':24s}" + "  ".join(f"{np.percentile(life, p):6.1f}" for p in pct))
st = t[:, 0, 0]
en = t[:, 0, 7]
print(f"  cluster start us: " + " ".join(f"{np.percentile(st, p):.1f}" for p in pct))
print(f"  cluster end us:   " + " ".join(f"{np.percentile(en, p):.1f}" for p in pct))
# concurrency: clusters alive at sampled times
ts = np.linspace(0, en.max(), 12)
print("  clusters alive at t:", " ".join(f"{x:.0f}:{int(((st <= x) & (en > x)).sum())}" for x in ts))
