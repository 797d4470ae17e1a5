"""Experiment: decode the batch as sub-batches on 2 CUDA streams (pairs are
independent, so the result is identical) to overlap issue-bound token scoring of
one sub-batch with the HBM-bound kernels of another.  Device time per step."""
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
dev = torch.device("cuda")
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def sub(t, lo, hi):
    return t[lo:hi]


def make_parts(splits):
    bounds = [round(w.batch * i / sum(splits) * 1.0) for i in range(len(splits) + 1)]
    acc = 0
    bounds = [0]
    for s_ in splits:
        acc += s_
        bounds.append(round(w.batch * acc / sum(splits)))
    parts = []
    for i in range(len(splits)):
        lo, hi = bounds[i], bounds[i + 1]
        c = tls.TLSConfig(**{**w.with_(batch=hi - lo).config_kwargs()})
        ix = tls.TLSIndex(idx.block_minmax[lo:hi], idx.codes[lo:hi], idx.scale_zero[lo:hi], idx.channels)
        parts.append((c, lo, hi, ix, torch.cuda.Stream(dev)))
    return parts


main = torch.cuda.current_stream(dev)
for splits in ([1], [1, 1], [1, 2], [1, 1, 1, 1]):
    parts = make_parts(splits)

    def step(i):
        ev = torch.cuda.Event()
        ev.record(main)
        done = []
        for c, lo, hi, ix, st in parts:
            st.wait_event(ev)
            with torch.cuda.stream(st):
                vc = inputs["v_cache"][lo:hi] if inputs["v_cache"] is not None else None
                tls.decode(c, queries[i % 8][lo:hi], inputs["k_cache"][lo:hi], vc, inputs["seq_lens"][lo:hi], ix)
                e2 = torch.cuda.Event()
                e2.record(st)
                done.append(e2)
        for e2 in done:
            main.wait_event(e2)

    t = bench.time_steps(step, 50, 5, lambda: flush_buf.fill_(1), main)
    ms = sorted(t)[len(t) // 2]
    print(f"{name} splits={splits}: median {ms * 1e3:.1f} us/step")
