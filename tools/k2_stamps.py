"""Diagnostic: per-CTA phase breakdown of the token kernel (a3) from its %globaltimer stamps (TLS_DEBUG_BUF):
0 start, 1 copies issued (after the hand-off wait), 2 staged data landed, 3 CTA stats merged, 4 cluster sync,
5 keys + histogram written, 6 end.  Percentiles over CTAs (chunks < 8).  Not a bench line."""
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
buf = torch.zeros(4 * 65536 * 8, dtype=torch.int64, device="cuda")
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    if it == 3:
        os.environ["TLS_DEBUG_BUF"] = hex(buf.data_ptr())
    flush_buf.fill_(1)
    tls.decode(cfg, queries[it], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    torch.cuda.synchronize()
os.environ.pop("TLS_DEBUG_BUF")
pairs = w.batch * w.num_kv_heads
k2 = buf[65536 * 16: 65536 * 16 + pairs * 64].view(pairs * 8, 8).cpu().double() / 1e3
k2 = k2[k2[:, 0] > 0]
form = tls.cluster_size(cfg, 5)
names = (["wait+issue", "pass1 (warp 0)", "pass1 all warps", "lz merge", "pass2 keys+hist", "end"] if form in (1, 4, 5) else
         ["wait+issue", "landed", "pass1+CTA merge", "cluster sync", "pass2 keys+hist", "end"])
print(f"{w.name}: form {form}, {k2.shape[0]} token CTAs, per-phase us:      min    p10    med    p90    max")
for i in range(6):
    x = (k2[:, i + 1] - k2[:, i]).sort().values
    n = len(x)
    print(f"  {names[i]:22s}" + " ".join(f"{float(x[min(n - 1, int(f * n))]):6.2f}" for f in (0, .1, .5, .9, 1)))
if form in (1, 4):
    x = (k2[:, 7] - k2[:, 0]).sort().values
    n = len(x)
    print(f"  {'  of which hand-off+ids':22s}" + " ".join(f"{float(x[min(n - 1, int(f * n))]):6.2f}" for f in (0, .1, .5, .9, 1)))
x = (k2[:, 6] - k2[:, 0]).sort().values
n = len(x)
print(f"  {'total':22s}" + " ".join(f"{float(x[min(n - 1, int(f * n))]):6.2f}" for f in (0, .1, .5, .9, 1)))
# the attention kernel's a4 prologue (K3 stamps at 65536*24 + pair*8: 0 start, 2 keys landed, 3 selected,
# 4 prologue end, 5 attention end)
k3 = buf[65536 * 24: 65536 * 24 + pairs * 8].view(pairs, 8).cpu().double() / 1e3
k3 = k3[k3[:, 0] > 0]
print(f"{w.name}: {k3.shape[0]} attention CTAs (rank 0), per-phase us:   min    p10    med    p90    max")
for nm, a, b in (("hand-off+keys landed", 0, 2), ("top-k_t select", 2, 3), ("emit", 3, 4), ("attention", 4, 5)):
    x = (k3[:, b] - k3[:, a]).sort().values
    n = len(x)
    print(f"  {nm:22s}" + " ".join(f"{float(x[min(n - 1, int(f * n))]):6.2f}" for f in (0, .1, .5, .9, 1)))
# inside hist_topk_select: clock64 cycles since the function's start at its checkpoints (per pair, rank-0 CTA:
# dbg + 65536*4 of the K3 base), and the boundary-bin size (K3 stamp slot 7)
cyc = buf[65536 * 24 + 65536 * 4: 65536 * 24 + 65536 * 4 + pairs * 8].view(pairs, 8)[:, :6].cpu().double()
cyc = cyc[cyc[:, 5] > 0]
if cyc.shape[0]:
    med = cyc.median(0).values.tolist()
    print(f"{w.name}: hist_topk_select median cycles at (boundary bin, interval, boundary keys gathered, threshold, "
          f"positions, emitted): {[int(x) for x in med]}")
nbk = buf[65536 * 24: 65536 * 24 + pairs * 8].view(pairs, 8)[:, 7].cpu().double()
nbk = nbk.sort().values
print(f"{w.name}: boundary-bin keys per pair: min {int(nbk[0])} median {int(nbk[len(nbk) // 2])} max {int(nbk[-1])}")
