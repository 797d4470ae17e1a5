"""Diagnostic: the persistent step kernel against the kernel chain (TLS_NO_PSTEP) on one small case."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402
from tests import test_gpu_parity as T  # noqa: E402

w = W.Workload("smoke-gqa", 2, 16, 2, 128, 128, 3000, top_blocks=16, top_tokens=256)
cfg, inputs, idx = T.setup_case(w, seed=0, pattern="peaked")
mode = os.environ.get("MODE", "both")
res = tls.decode(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
torch.cuda.synchronize()
print("pstep mode", tls.select_mode(cfg))
os.environ["TLS_NO_PSTEP"] = "1"
ref = tls.decode(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
torch.cuda.synchronize()
print("chain mode", tls.select_mode(cfg))
names = ["out", "lse", "block_ids", "token_ids", "num_tokens", "token_scores"]
for n_, a, b in zip(names, res, ref):
    if a is None:
        continue
    if a.dtype in (torch.int32,):
        bad = (a != b).nonzero()
        print(n_, "mismatches", bad.shape[0], a.flatten()[:20].tolist(), b.flatten()[:20].tolist())
    else:
        print(n_, "maxdiff", (a.float() - b.float()).abs().max().item())
