"""Diagnostic: device time of tls_select, tls_sparse_attend and the fused
tls_decode for one workload (L2 flushed before each call).  Not a bench line."""
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
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--cs", default="")
args = ap.parse_args()
w = W.CONFIGS[args.config]
for cs in (args.cs.split(",") if args.cs else [""]):
    if cs:
        os.environ["TLS_CLUSTER"] = cs
    dev = torch.device("cuda")
    cfg, inputs, idx, queries = bench.build_state(w, 0, dev, "outlier")
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    st = torch.cuda.current_stream()
    sel = tls.select(cfg, queries[0], inputs["seq_lens"], idx)
    sc_out = torch.empty((w.batch, w.num_kv_heads, cfg.num_blocks), dtype=torch.float32, device=dev)
    fns = {
        "scores": lambda i: tls.block_scores(cfg, queries[i % 8], inputs["seq_lens"], idx, out=sc_out),
        "select": lambda i: tls.select(cfg, queries[i % 8], inputs["seq_lens"], idx, out=sel),
        "attend": lambda i: tls.sparse_attend(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"], sel[1], sel[2]),
        "decode": lambda i: tls.decode(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx),
    }
    nbytes = bench.algorithmic_bytes_per_pair(w) * w.batch * w.num_kv_heads
    for k, f in fns.items():
        t = bench.time_steps(f, args.steps, 5, flush, st)
        ms = sorted(t)[len(t) // 2]
        print(f"{w.name} cs={tls.cluster_size(cfg, 2)} {k:7s} median {ms*1e3:9.1f} us"
              + (f"  ({nbytes / ms / 1e6:.0f} GB/s algorithmic)" if k == "decode" else ""))
    del inputs, idx
    torch.cuda.empty_cache()
