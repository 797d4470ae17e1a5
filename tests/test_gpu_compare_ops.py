"""The paper's comparison operators (P:395 baselines, P:413 efficiency) on the GPU, checked
against the fp64 oracle with the parity suite's rules:

* Quest (block level only, ops.quest_decode): M_t = the oracle's top-k_b by s_i (near-tie rule,
  strict fp32 tier clean), the attended token set = every token of the GPU's M_t (exact), and the output the
  oracle's attention over that set (bf16 / fp32 tolerance).
* DS (token level only, ops.ds_decode): every block a candidate (k_b = m): S_t = the oracle's top-k_t of
  alpha~ over the whole context (near-tie rule), ln alpha~ of the selection, and the output.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from oracle import tls_oracle as O
from tests import parity as P
from tests import test_gpu_parity as T

pytestmark = pytest.mark.gpu

tls = pytest.importorskip("paper_2604_07815_b200")
from paper_2604_07815_b200 import workloads as W  # noqa: E402

CASES = {
    "gqa8": W.Workload("cmp-gqa8", 2, 16, 2, 128, 128, 9000, top_blocks=16, top_tokens=512),
    "gqa4_fp32": W.Workload("cmp-fp32", 2, 8, 2, 64, 64, 3000, top_blocks=8, top_tokens=200, dtype=torch.float32),
    "mla": W.Workload("cmp-mla", 1, 16, 1, 576, 512, 5000, d_c=128, top_blocks=8, top_tokens=256, layout="mla",
                      sm_scale=1.0 / math.sqrt(192.0)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_quest_matches_oracle(name):
    w = CASES[name]
    cfg, inputs, idx = T.setup_case(w, seed=13, pattern="peaked")
    out, lse, bids, tids, nt = tls.quest_decode(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"],
                                                inputs["seq_lens"], idx)
    torch.cuda.synchronize()
    G = w.num_q_heads // w.num_kv_heads
    for b in range(w.batch):
        n = int(inputs["seq_lens"][b])
        for g in range(w.num_kv_heads):
            q, keys, values = P.pair_slices(w, inputs, b, g)
            kmax, kmin = O.block_summaries(keys, w.block_size)
            s = O.block_scores(q, kmax, kmin)
            kb = min(w.top_blocks, len(s))
            gb = bids[b, g].cpu().numpy()
            P.check_ids_layout(gb, kb)
            gb = gb[:kb]
            _, bad = P.near_tie_mismatches(s, O.topk_ids(s, w.top_blocks), gb, kb, T.STRICT_BLOCK[w.layout])
            assert not bad, (b, g, bad)
            cand = O.candidate_tokens(gb, n, w.block_size)  # every token of M_t (P:137's J)
            k = int(nt[b, g])
            assert k == len(cand) and np.array_equal(tids[b, g, :k].cpu().numpy(), cand)
            assert (tids[b, g, k:] == -1).all()
            o_ref, l_ref = O.sparse_attention(q, keys, values, cand, w.scale)
            P.compare_output(P.to64(out[b, g * G:(g + 1) * G]), o_ref, w.dtype, f"quest {b},{g}")
            np.testing.assert_allclose(P.to64(lse[b, g * G:(g + 1) * G]), l_ref, rtol=0, atol=1e-3)


@pytest.mark.parametrize("name", list(CASES))
def test_ds_matches_oracle(name):
    w = CASES[name]
    cfg, inputs, idx = T.setup_case(w, seed=14, pattern="peaked")
    out, lse, tids, nt, lk = tls.ds_decode(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"],
                                           inputs["seq_lens"], idx)
    torch.cuda.synchronize()
    G = w.num_q_heads // w.num_kv_heads
    prm = O.TLSParams(block_size=w.block_size, top_blocks=10 ** 9, top_tokens=w.top_tokens, sm_scale=w.scale)
    near = 0
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            q, keys, values = P.pair_slices(w, inputs, b, g)
            ch = idx.channels[g].cpu().numpy()
            ref = O.tls_pair(q, keys, values, ch, prm)  # k_b >= m: every block a candidate (U4)
            cand = ref["candidates"]
            assert len(cand) == keys.shape[0]
            k = int(nt[b, g])
            assert k == len(ref["token_ids"])
            gt = tids[b, g, :k].cpu().numpy()
            pos_o, pos_g = np.searchsorted(cand, ref["token_ids"]), np.searchsorted(cand, gt)
            assert np.array_equal(cand[pos_g], gt)
            exc, bad = P.near_tie_mismatches(ref["alpha"], pos_o, pos_g, k, P.NORTH_STAR_REL)
            assert not bad, (b, g, len(bad))
            _, bad = P.near_tie_mismatches(ref["alpha"], pos_o, pos_g, k, T.STRICT_TOKEN)
            assert not bad, (b, g, len(bad))
            near += len(exc)
            np.testing.assert_allclose(lk[b, g, :k].cpu().numpy(), np.log(ref["alpha"][pos_g]), rtol=0, atol=2e-3)
            o_ref, _ = O.sparse_attention(q, keys, values, gt, w.scale)
            P.compare_output(P.to64(out[b, g * G:(g + 1) * G]), o_ref, w.dtype, f"ds {b},{g}")
    print(f"{name}: DS near-ties {near}")
