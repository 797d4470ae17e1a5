"""Context: device time per decode step vs the selection budgets (K_t in {512, 1024, 2048}; K_b in
{64, 128, 256}) and the input pattern (uniform / outlier / peaked), L2 flushed, PDL-overlapped
tls_decode.  Not a bench line.  usage: python tools/budget_sweep.py [c3,c2]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3", "c2"]
dev = torch.device("cuda")
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
clocks = bench.ClockSampler(0)  # SM clock / throttle reasons during each record's timed region
clocks.start()
for name in names:
    base = W.CONFIGS[name]
    for pattern in ("outlier", "uniform", "peaked"):
        cfg0, inputs, idx, queries = bench.build_state(base, 0, dev, pattern)
        for kb, kt in ((128, 512), (128, 1024), (128, 2048), (64, 1024), (256, 1024)):
            if pattern != "outlier" and (kb, kt) != (128, 1024):
                continue
            cfg = tls.TLSConfig(**{**base.config_kwargs(), "top_blocks": kb, "top_tokens": kt})
            t_rec0 = __import__("time").time()
            try:
                ts = bench.time_steps(lambda i: tls.decode(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"],
                                                           inputs["seq_lens"], idx), 50, 5, lambda: flush_buf.fill_(1), st)
                t = sorted(ts)[len(ts) // 2] * 1e3
                rec = {"workload": base.name, "pattern": pattern, "top_blocks": kb, "top_tokens": kt, "us_per_step": t,
                       "tokens_per_s": base.batch / (t * 1e-6)}
            except Exception as e:  # noqa: BLE001
                rec = {"workload": base.name, "pattern": pattern, "top_blocks": kb, "top_tokens": kt,
                       "error": f"{type(e).__name__}: {e}"[:160]}
            rec["clocks"] = clocks.summary(t_rec0, __import__("time").time())
            print(json.dumps(rec), flush=True)
        del inputs, idx, queries
        torch.cuda.empty_cache()
