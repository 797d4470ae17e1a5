"""KV-offload engine measurement (C5): the K/V caches
in pinned host memory, the index on the GPU, a drifting query (q_{t+1} = q_t + eps
* noise), one select + cache_fetch + attend step per decode step.  Reports
device time per step (CUDA events, L2 flushed), rows fetched per step (the
PCIe / C2C traffic of the zero-copy gather), and the resident tls_decode time on
the same inputs.  Not a bench.py line.

With --mode block: the asynchronous block-granular engine (AsyncOffloadDecoder:
one-step lag S_t = TokenSelect(q_t, M_{t-1}), M_t's missing blocks fetched on a
side stream under the attention), timed on the main stream, against the resident
lag-mode tls_decode on the same inputs.

usage: python tools/offload_bench.py [--batch 64] [--steps 20] [--eps 0.05] [--mode token|block]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--eps", type=float, default=0.05)
ap.add_argument("--mode", default="token", choices=["token", "block"])
ap.add_argument("--layers", type=int, default=1, help="block mode: layers per token step (one cache each)")
args = ap.parse_args()
w = W.CONFIGS["c5"].with_(batch=args.batch)
dev = torch.device("cuda")
cfg, inputs, idx, queries = bench.build_state(w, 0, dev, "outlier")
t0 = time.time()
k_host = tls.host_kv(inputs["k_cache"])
v_host = tls.host_kv(inputs["v_cache"])
pin_s = time.time() - t0
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
g = torch.Generator(device=dev).manual_seed(11)
q = queries[0].clone()
qs = []
for _ in range(args.steps + 1):
    qs.append(q.clone())
    q = (q.float() + args.eps * torch.randn(q.shape, generator=g, device=dev)).to(q.dtype)
st = torch.cuda.current_stream()
clocks = bench.ClockSampler(0)  # SM clock / throttle reasons during the timed region (recorded with the numbers)
clocks.start()
t_rec0 = time.time()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
misses = []
row = 2 * w.d_k * 2  # K + V bytes per token (bf16)
pairs = w.batch * w.num_kv_heads
if args.mode == "token":
    cache = tls.alloc_token_cache(cfg, cfg.top_tokens, dev)
    tls.offload_decode(cfg, qs[0], k_host, v_host, inputs["seq_lens"], idx, cache)  # warm: the first step fetches all
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush_buf.fill_(1)
        ev[i][0].record(st)
        res = tls.offload_decode(cfg, qs[i + 1], k_host, v_host, inputs["seq_lens"], idx, cache)
        ev[i][1].record(st)
        misses.append(res[7])
    torch.cuda.synchronize()
    t_off = sorted(a.elapsed_time(b) for a, b in ev)[args.steps // 2] * 1e3
    mean_miss = float(torch.stack(misses).float().mean())
    t_res = sorted(bench.time_steps(lambda i: tls.decode(cfg, qs[1 + i % args.steps], inputs["k_cache"],
                                                          inputs["v_cache"], inputs["seq_lens"], idx), args.steps, 3,
                                    lambda: flush_buf.fill_(1), st))[args.steps // 2] * 1e3
    rec = {"workload": w.name, "mode": "token cache, synchronous fetch", "batch": w.batch, "context": w.context,
           "eps": args.eps, "steps": args.steps, "offload_us_per_step": t_off, "resident_decode_us_per_step": t_res,
           "mean_misses_per_pair_per_step": mean_miss, "top_tokens": w.top_tokens,
           "hit_rate": 1.0 - mean_miss / w.top_tokens, "fetched_bytes_per_step": mean_miss * pairs * row}
else:
    L = args.layers  # every layer reads the same host KV and index through its own GPU block cache
    engs = [tls.AsyncOffloadDecoder(cfg, k_host, v_host, inputs["seq_lens"], idx) for _ in range(L)]
    for e in engs:
        e.step(qs[0])  # first step: synchronous, fetches every block of M_0
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush_buf.fill_(1)
        ev[i][0].record(st)
        for e in engs:  # layer l's update overlaps layers l+1.. of this step
            e.step(qs[i + 1])
        ev[i][1].record(st)
        misses.append(torch.stack([e.last_miss for e in engs]))
    torch.cuda.synchronize()
    t_off = sorted(a.elapsed_time(b) for a, b in ev)[args.steps // 2] * 1e3 / L
    mean_miss = float(torch.stack(misses).float().mean())
    # resident reference: the same lag-mode steps (guide = the previous step's M) with the KV in HBM
    guides = [None]
    for i in range(args.steps + 1):
        guides.append(tls.decode(cfg, qs[i], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx,
                                 guide_block_ids=guides[-1])[2].clone())
    t_res = sorted(bench.time_steps(lambda i: tls.decode(cfg, qs[1 + i % args.steps], inputs["k_cache"],
                                                          inputs["v_cache"], inputs["seq_lens"], idx,
                                                          guide_block_ids=guides[1 + i % args.steps]),
                                    args.steps, 3, lambda: flush_buf.fill_(1), st))[args.steps // 2] * 1e3
    rec = {"workload": w.name, "mode": "block cache, asynchronous fetch (one-step lag, side stream)",
           "layers": L, "batch": w.batch, "context": w.context, "eps": args.eps, "steps": args.steps,
           "offload_us_per_layer_step": t_off, "resident_lag_decode_us_per_step": t_res,
           "mean_blocks_fetched_per_pair_per_step": mean_miss, "top_blocks": w.top_blocks,
           "block_hit_rate": 1.0 - mean_miss / w.top_blocks,
           "fetched_bytes_per_layer_step": mean_miss * pairs * w.block_size * row,
           "gpu_cache_bytes_per_layer": int(engs[0].cache.k_slots.numel() * 2 * 2)}
rec.update(host_kv_bytes=int(k_host.numel() * 2 + v_host.numel() * 2), pin_seconds=pin_s,
           clocks=clocks.summary(t_rec0, time.time()))
print(json.dumps(rec), flush=True)
