"""Diagnostic: is the GQA attention kernel memory- or issue-bound?  Times
tls_sparse_attend at C3 over (a) the real selection, (b) the same number of
tokens all pointing at one row (K/V L2-resident), (c) a contiguous token range
(sequential rows).  Not a bench line."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dev = torch.device("cuda")
cfg, inputs, idx, queries = bench.build_state(w, 0, dev, "outlier")
sel = tls.select(cfg, queries[0], inputs["seq_lens"], idx)
tids, nt = sel[1], sel[2]
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
variants = {"selected": tids, "one_row": torch.zeros_like(tids),
            "contiguous": torch.arange(w.top_tokens, dtype=torch.int32, device=dev).expand_as(tids).contiguous()}
for k, t in variants.items():
    ts = bench.time_steps(lambda i: tls.sparse_attend(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"], t, nt),
                          50, 5, lambda: flush_buf.fill_(1), st)
    print(f"{w.name} attend {k:10s} median {sorted(ts)[25] * 1e3:7.1f} us", flush=True)
