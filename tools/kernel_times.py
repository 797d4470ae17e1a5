"""Diagnostic: live per-kernel device time (library events around each launch)
of tls_decode for a workload at several batch sizes.  Not a bench line."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
batches = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [W.CONFIGS[name].batch]
dev = torch.device("cuda")
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for bsz in batches:
    w = W.CONFIGS[name].with_(batch=bsz)
    cfg, inputs, idx, queries = bench.build_state(w, 0, dev, "outlier")
    f = lambda i: tls.decode(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)  # noqa
    steps = 100
    tls.timing_enable(steps + 10)
    t = bench.time_steps(f, steps, 10, lambda: flush_buf.fill_(1), torch.cuda.current_stream(),
                         on_timed_start=tls.timing_read)
    ms, calls = tls.timing_read()
    tls.timing_enable(0)
    parts = "  ".join(f"{k.replace('_kernel', '')} {v / calls * 1e3:6.1f}" for k, v in ms.items())
    print(f"{w.name} batch={bsz} pairs={bsz * w.num_kv_heads}: step {sorted(t)[len(t) // 2] * 1e3:6.1f} us | {parts}",
          flush=True)
    del inputs, idx
    torch.cuda.empty_cache()
