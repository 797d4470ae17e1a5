"""Diagnostic: per-phase latency of the token-cluster kernel (K2) and of K3's
selection prologue, from %globaltimer stamps (TLS_DEBUG_BUF)."""
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
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), os.environ.get("TLS_PATTERN", "outlier"))
os.environ["TLS_FUSED_MODE"] = "1"
buf = torch.zeros(4 * 65536 * 8, dtype=torch.int64, device="cuda")
for it in range(3):
    if it == 2:
        os.environ["TLS_DEBUG_BUF"] = hex(buf.data_ptr())
    tls.decode(cfg, queries[it], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    torch.cuda.synchronize()
os.environ.pop("TLS_DEBUG_BUF")
pairs = w.batch * w.num_kv_heads
k2 = buf[65536 * 16: 65536 * 16 + pairs * 8 * 8].view(pairs, 8, 8).cpu().double()
k3 = buf[65536 * 24: 65536 * 24 + pairs * 8].view(pairs, 8).cpu().double()
t0 = k2[:, :, 0][k2[:, :, 0] > 0].min()
def med(x):
    x = x[x == x]
    return float(x.median()) / 1e3 if len(x) else float("nan")
valid = k2[:, :, 0] > 0
d = (k2[:, :, 1:7] - k2[:, :, 0:6])[valid]
print(f"{name}: K2 span {(k2[:, :, 6][valid].max() - t0) / 1e3:.1f} us; CTA lifetime median {med(k2[:, :, 6][valid] - k2[:, :, 0][valid]):.1f} us")
for i, nm in enumerate(["setup (cand, q, TMA issue)", "wait staged index", "pass 1 stats", "cluster sync", "merge + pass 2 keys", "cluster wait"]):
    print(f"  K2 {nm:28s} median {med(d[:, i]):6.2f} us")
k3t0 = k3[:, 0].min()
print(f"K3 wait->start after its K2 (per pair) median {med(k3[:, 0] - k2[:, :, 6].max(1).values):.1f} us")
print(f"K3 start (rel. K2 start) median {(k3[:, 0] - t0).median() / 1e3:.1f} us, K3 span {(k3[:, 5].max() - k3t0) / 1e3:.1f} us")
print(f"  K3 select: to classification end median {med(k3[:, 6] - k3[:, 2]):6.2f} us, rank+scan+emit {med(k3[:, 3] - k3[:, 6]):6.2f} us;"
      f" boundary-bin keys median {float(k3[:, 7].median()):.0f} max {float(k3[:, 7].max()):.0f}")
cyc = buf[65536 * 28: 65536 * 28 + pairs * 8].view(pairs, 8).cpu().double()
print("  K3 select cycles (cumulative, median): " + ", ".join(
    f"{nm} {float(cyc[:, i].median()):.0f}" for i, nm in enumerate(["hist scan", "search+load", "classify", "rank", "scan", "emit"])))
for i, nm in enumerate(["load keys+hist (TMA)", "-", "select + emit", "padding + sync", "attention"]):
    print(f"  K3 {nm:28s} median {med(k3[:, i + 1] - k3[:, i]):6.2f} us")
