"""Context for the paper's operator speedups:
device time of one TLS decode step vs a dense decode over the full context, on the
same synthetic workload, L2 flushed before each call.  Not a bench line.

Comparison operators of the paper, same inputs (tests/test_gpu_compare_ops.py checks both
against the oracle):
  quest -- ops.quest_decode: block selection only (a1, a2 by tls_block_scores / tls_block_topk), attention over
           every token of the K_b selected blocks (tls_expand_blocks, tls_sparse_attend);
  ds    -- ops.ds_decode: token selection only, every block a candidate (tls_block_iota, tls_token_stats,
           tls_token_keys, tls_topk_rows -- the CUDA-core kernels of the sequence split -- tls_sparse_attend).
Every record carries the SM clock sampled during its timings.
Dense baselines: GQA -- flash_attn.flash_attn_with_kvcache (the library's FA2 decode
kernel; the KV cache is re-laid out to [B, S, Hkv, D] once, untimed); MLA (d_k 576,
beyond flash_attn's head dims) -- this repo's attention kernel over every token.

usage: python tools/compare_dense.py [c3,c2,c4,pb-gqa,pb-mla] > profiles/r01_compare_dense.json
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

EXTRA = {  # the paper's kernel-benchmark shape at its largest point: batch 8, 128k
    "pb-gqa": W.CONFIGS["c2"].with_(name="pb-gqa-128k-b8", batch=8, context=131072, max_seq_len=131072),
    "pb-mla": W.CONFIGS["c4"].with_(name="pb-mla-128k-b8", batch=8, context=131072, max_seq_len=131072),
}


def med(ts):
    return sorted(ts)[len(ts) // 2]


def main():
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3", "c2", "c4"]
    dev = torch.device("cuda")
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    st = torch.cuda.current_stream()
    res = []
    clocks = bench.ClockSampler(0)
    clocks.start()
    for name in names:
        t_rec0 = __import__("time").time()
        w = EXTRA.get(name) or W.CONFIGS[name]
        cfg, inputs, idx, queries = bench.build_state(w, 0, dev, "outlier")
        q = queries[0]
        t_tls = med(bench.time_steps(lambda i: tls.decode(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"],
                                                           inputs["seq_lens"], idx), 50, 5, flush, st))
        rec = {"workload": w.name, "tls_us": t_tls * 1e3, "context": w.context, "batch": w.batch, "layout": w.layout}
        for tag, fn in (("quest", tls.quest_decode), ("ds", tls.ds_decode)):
            try:
                t_v = med(bench.time_steps(lambda i: fn(cfg, queries[i % 8], inputs["k_cache"], inputs["v_cache"],
                                                        inputs["seq_lens"], idx), 20, 3, flush, st))
                rec.update({f"{tag}_us": t_v * 1e3, f"tls_speedup_vs_{tag}": t_v / t_tls})
            except Exception as e:  # noqa: BLE001
                rec[f"{tag}_error"] = f"{type(e).__name__}: {e}"[:200]
        if w.layout == "gqa":
            try:
                from flash_attn import flash_attn_with_kvcache
                kc = inputs["k_cache"].transpose(1, 2).contiguous()  # [B, S, Hkv, D]
                vc = inputs["v_cache"].transpose(1, 2).contiguous()
                qf = q.unsqueeze(1).contiguous()  # [B, 1, Hq, D]
                sl = inputs["seq_lens"]
                t_fa = med(bench.time_steps(lambda i: flash_attn_with_kvcache(qf, kc, vc, cache_seqlens=sl,
                                                                              softmax_scale=w.scale), 50, 5, flush, st))
                rec.update(dense="flash_attn_with_kvcache (FA2)", dense_us=t_fa * 1e3, speedup=t_fa / t_tls)
                del kc, vc
            except Exception as e:  # noqa: BLE001
                rec.update(dense_error=f"{type(e).__name__}: {e}"[:200])
        else:
            n = w.context
            dcfg = tls.TLSConfig(**{**w.config_kwargs(), "top_tokens": n, "top_blocks": cfg.num_blocks})
            tids = torch.arange(n, dtype=torch.int32, device=dev).view(1, 1, n).expand(w.batch, w.num_kv_heads, n).contiguous()
            ntok = inputs["seq_lens"].view(w.batch, 1).expand(w.batch, w.num_kv_heads).contiguous().to(torch.int32)
            try:
                t_d = med(bench.time_steps(lambda i: tls.sparse_attend(dcfg, queries[i % 8], inputs["k_cache"], None,
                                                                       tids, ntok), 20, 3, flush, st))
                rec.update(dense="this repo's attention kernel over every token", dense_us=t_d * 1e3, speedup=t_d / t_tls)
            except Exception as e:  # noqa: BLE001
                rec.update(dense_error=f"{type(e).__name__}: {e}"[:200])
        rec["clocks"] = clocks.summary(t_rec0, __import__("time").time())
        print(json.dumps(rec), flush=True)
        res.append(rec)
        del inputs, idx, queries
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
    # (the clock sampler thread is a daemon; nvidia-smi exits with the process)
