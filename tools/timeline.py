"""Diagnostic: one overlapped decode step as a per-pair timeline from the
%globaltimer stamps (TLS_DEBUG_BUF): select worker (a2) start/end, token
cluster (a3) start/end, attention CTA (a4+a5) start/prologue end/end, as
percentiles over pairs, relative to the earliest select stamp.  Not a bench line."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = W.CONFIGS[name]
if len(sys.argv) > 2:
    w = w.with_(batch=int(sys.argv[2]))
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
buf = torch.zeros(4 * 65536 * 8, dtype=torch.int64, device="cuda")
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
os.environ.pop("TLS_DEBUG_BUF")
pairs = w.batch * w.num_kv_heads
sel = buf[: pairs * 16].view(pairs, 16).cpu().double() / 1e3
k2 = buf[65536 * 16: 65536 * 16 + pairs * 64].view(pairs, 8, 8).cpu().double() / 1e3
k3 = buf[65536 * 24: 65536 * 24 + pairs * 8].view(pairs, 8).cpu().double() / 1e3
t0 = sel[:, 6].min()


def q(x):
    x = x[(x > -1e8) & (x < 1e8)].sort().values
    n = len(x)
    if n == 0:
        return "   (no stamps)"
    return " ".join(f"{float(x[min(n - 1, int(f * n))]):6.1f}" for f in (0.0, 0.1, 0.5, 0.9, 1.0))


k2v = k2[:, :, 0] > 0
k2s = torch.where(k2v, k2[:, :, 0], torch.full_like(k2[:, :, 0], 1e18)).min(1).values
k2e = torch.where(k2v, k2[:, :, 6], torch.full_like(k2[:, :, 6], -1e18)).max(1).values
print(f"{w.name} pairs={pairs}; step with debug stamps {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us (event)")
print("  us rel. first select stamp:      min    p10    med    p90    max")
print(f"  select last-tile CTA start   {q(sel[:, 6] - t0)}")
print(f"  select worker start          {q(sel[:, 0] - t0)}")
print(f"  select worker end            {q(sel[:, 2] - t0)}")
print(f"  K2 first CTA start           {q(k2s - t0)}")
print(f"  K2 last CTA end              {q(k2e - t0)}")
print(f"  K3 start                     {q(k3[:, 0] - t0)}")
print(f"  K3 prologue end              {q(k3[:, 4] - t0)}")
print(f"  K3 end                       {q(k3[:, 5] - t0)}")
print(f"  K2 start - worker end        {q(k2s - sel[:, 2])}")
print(f"  K2 duration                  {q(k2e - k2s)}")
print(f"  K3 start - K2 end            {q(k3[:, 0] - k2e)}")
print(f"  K3 duration                  {q(k3[:, 5] - k3[:, 0])}")
