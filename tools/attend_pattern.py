"""Diagnostic: the standalone attention kernel (tls_sparse_attend, a5 only) at C3 over three token-id patterns --
the selection of a real decode step (scattered within 128 blocks), 1024 random tokens, and 1024 contiguous tokens --
to separate the kernel's limits from the gather's DRAM access pattern.  Device time per call, L2 flushed.
Not a bench line."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
bids, tids, nt, ts = tls.select(cfg, queries[0], inputs["seq_lens"], idx)
kt = w.top_tokens
g = torch.Generator(device="cpu").manual_seed(0)
n = inputs["seq_lens"].long().cpu()
rand = torch.stack([torch.stack([torch.randperm(int(n[b]), generator=g)[:kt].sort().values for _ in range(w.num_kv_heads)])
                    for b in range(w.batch)]).int().cuda()
cont = torch.stack([torch.stack([torch.arange(kt) + (int(n[b]) - kt) // 2 for _ in range(w.num_kv_heads)])
                    for b in range(w.batch)]).int().cuda()
full = torch.full_like(nt, kt)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
row = (w.d_k + w.d_v) * 2 if w.layout == "gqa" else w.d_k * 2
for name, ids, cnt in (("selected", tids, nt), ("random", rand, full), ("contiguous", cont, full)):
    ts_ = []
    for it in range(23):
        flush.fill_(1)
        ev[0].record()
        tls.sparse_attend(cfg, queries[0], inputs["k_cache"], inputs["v_cache"], ids, cnt)
        ev[1].record()
        torch.cuda.synchronize()
        if it >= 3:
            ts_.append(ev[0].elapsed_time(ev[1]) * 1e3)
    us = sorted(ts_)[len(ts_) // 2]
    byts = int(cnt.sum()) * row
    print(f"{w.name} {name:10s}: {us:7.1f} us  {byts / us / 1e3:7.0f} GB/s  ({byts / 1e6:.0f} MB of K/V rows)")
