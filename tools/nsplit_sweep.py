"""Diagnostic: device time of one tls_decode step vs the sub-batch pipeline
depth TLS_NSPLIT (L2 flushed before each step).  Also checks that every split
gives bit-identical outputs and selections.  Not a bench line."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

if len(sys.argv) > 3 and sys.argv[3] == "noprio":
    os.environ["TLS_NOPRIO"] = "1"
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3"]
splits = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4, 6, 8]
dev = torch.device("cuda")
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for name in names:
    w = W.CONFIGS[name]
    cfg, inputs, idx, queries = bench.build_state(w, 0, dev, "outlier")
    st = torch.cuda.current_stream()
    ref = None
    nbytes = bench.algorithmic_bytes_per_pair(w) * w.batch * w.num_kv_heads
    for ns in splits:
        os.environ["TLS_NSPLIT"] = str(ns)
        f = lambda i: tls.decode(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)  # noqa
        r = f(0)
        torch.cuda.synchronize()
        if ref is None:
            ref = [x.clone() for x in r if x is not None]
        else:
            got = [x for x in r if x is not None]
            # selections are per pair -> identical; outputs may differ by rounding when the
            # attention cluster size (chosen from the sub-batch's pair count) changes
            same = all(torch.equal(a, b) for a, b in zip(ref[2:], got[2:]))
            dout = (ref[0].float() - got[0].float()).abs().max().item()
            assert same, f"split {ns}: selections differ from split 1"
            print(f"  split {ns}: selections identical, max|dout| = {dout:.2e}")
        t = bench.time_steps(f, 200, 10, lambda: flush_buf.fill_(1), st)
        ms = sorted(t)[len(t) // 2]
        # the same step captured in a CUDA graph (host launch cost removed)
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        s2.wait_stream(st)
        with torch.cuda.stream(s2):
            f(0)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s2):
                f(0)
        torch.cuda.synchronize()
        tg = bench.time_steps(lambda i: g.replay(), 200, 10, lambda: flush_buf.fill_(1), st)
        mg = sorted(tg)[len(tg) // 2]
        print(f"{w.name} nsplit={ns} median {ms * 1e3:8.1f} us  {nbytes / ms / 1e6:7.0f} GB/s | graph {mg * 1e3:8.1f} us "
              f"{nbytes / mg / 1e6:7.0f} GB/s", flush=True)
    del inputs, idx
    torch.cuda.empty_cache()

# one chain alone at each sub-batch size (what a perfectly overlapped split would cost per chain)
for name in names:
    w0 = W.CONFIGS[name]
    for ns in splits:
        os.environ["TLS_NSPLIT"] = "1"
        w = w0.with_(batch=max(1, w0.batch // ns))
        cfg, inputs, idx, queries = bench.build_state(w, 0, dev, "outlier")
        f = lambda i: tls.decode(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)  # noqa
        t = bench.time_steps(f, 100, 10, lambda: flush_buf.fill_(1), torch.cuda.current_stream())
        print(f"{w.name} batch={w.batch} alone: median {sorted(t)[len(t) // 2] * 1e3:8.1f} us", flush=True)
        del inputs, idx
        torch.cuda.empty_cache()
