"""One small decode step of each kernel family, for compute-sanitizer (tests/test_gpu_sanitizer.py):
C1 (fp32 GQA, the generic attention path), a bf16 GQA G=8 case (select_kernel, token_reg_kernel, the mma.sync
attention with a 2-CTA split), a bf16 MLA case (token_cluster_kernel, attend_mla_kernel), the index build,
the calibration and the sequence-split kernels.  Not a bench line."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import ops, seqsplit as SS, workloads as W  # noqa: E402

CASES = [
    W.CONFIGS["c1"],
    W.Workload("san-gqa8", 2, 16, 2, 128, 128, 3000, top_blocks=16, top_tokens=256),
    W.Workload("san-mla", 1, 16, 1, 576, 512, 2100, d_c=128, top_blocks=8, top_tokens=128, layout="mla",
               sm_scale=1.0 / math.sqrt(192.0)),
]
for w in CASES:
    inputs = W.make_inputs(w, seed=1, device="cuda", ragged=True)
    cfg = tls.TLSConfig(**w.config_kwargs())
    q_cal, k_cal = W.calibration_sample(w, inputs, seed=1)
    channels, _ = tls.calibrate_channels(cfg, q_cal, k_cal)
    idx = tls.alloc_index(cfg, channels)
    tls.build_index(cfg, inputs["k_cache"], inputs["seq_lens"], idx)
    for _ in range(2):  # the second call runs on the workspace state the first one left
        tls.decode(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    if w.layout == "gqa" and w.dtype == torch.bfloat16:
        os.environ["TLS_CLUSTER"] = "2"
        tls.decode(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
        os.environ.pop("TLS_CLUSTER")
        states = []
        for t0, L in SS.split_ranges(cfg.max_seq_len, cfg.block_size, 2):
            import dataclasses

            c = dataclasses.replace(cfg, max_seq_len=L)
            kc = inputs["k_cache"][:, :, t0:t0 + L].contiguous()
            vc = inputs["v_cache"][:, :, t0:t0 + L].contiguous()
            ix = ops.alloc_index(c, channels)
            ops.build_index(c, kc, SS.local_seq_lens(inputs["seq_lens"], t0, L), ix)
            states.append(SS.RankState(cfg=c, index=ix, k_cache=kc, v_cache=vc, t0=t0))
        SS.run_ranks(states, inputs["q"], inputs["seq_lens"])
    torch.cuda.synchronize()
print("sanitize cases done")
