"""GPU parity of the sequence-split decode (paper_2604_07815_b200/seqsplit.py) through the
C ABI (tls_block_scores, tls_block_topk, tls_topk_rows, tls_select_range, tls_token_stats, tls_token_keys,
tls_sparse_attend, tls_attn_merge): P ranks simulated in one process on one GPU (the all_gathers served in
lockstep), each rank holding a block-aligned slice of the KV cache and an index built over it.  Checked
against the fp64 oracle's UNSPLIT decode of each pair with the parity suite's rules (block and token sets
identical up to near-ties, strict fp32 tier clean; attention on the GPU's ids within the bf16 / fp32
tolerance), plus the generic top-k kernel against brute force with planted ties."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest
import torch

from oracle import tls_oracle as O
from tests import parity as P
from tests import test_gpu_parity as T

pytestmark = pytest.mark.gpu

tls = pytest.importorskip("paper_2604_07815_b200")
from paper_2604_07815_b200 import ops  # noqa: E402
from paper_2604_07815_b200 import seqsplit as SS  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

CASES = {
    "gqa8": W.Workload("ss-gqa8", 2, 16, 2, 128, 128, 20000, top_blocks=32, top_tokens=512),
    "gqa4_fp32": W.Workload("ss-fp32", 2, 8, 2, 128, 128, 7000, top_blocks=16, top_tokens=300, dtype=torch.float32),
    "mla": W.Workload("ss-mla", 2, 16, 1, 576, 512, 9000, d_c=128, top_blocks=16, top_tokens=256, layout="mla",
                      sm_scale=1 / 192 ** 0.5),
}


def rank_states(w, cfg, inputs, channels, Pn):
    states = []
    for t0, L in SS.split_ranges(cfg.max_seq_len, cfg.block_size, Pn):
        c = dataclasses.replace(cfg, max_seq_len=L)
        if w.layout == "mla":
            kc = inputs["k_cache"][:, t0:t0 + L].contiguous()
            vc = None
        else:
            kc = inputs["k_cache"][:, :, t0:t0 + L].contiguous()
            vc = inputs["v_cache"][:, :, t0:t0 + L].contiguous()
        idx = ops.alloc_index(c, channels)
        ops.build_index(c, kc, SS.local_seq_lens(inputs["seq_lens"], t0, L), idx)
        states.append(SS.RankState(cfg=c, index=idx, k_cache=kc, v_cache=vc, t0=t0))
    return states


def check_against_oracle(w, inputs, channels, res):
    out, lse, m_glob, s_glob, n_glob = res
    G = w.num_q_heads // w.num_kv_heads
    near = {"block": 0, "token": 0}
    for b in range(w.batch):
        n = int(inputs["seq_lens"][b])
        for g in range(w.num_kv_heads):
            q, keys, values = P.pair_slices(w, inputs, b, g)
            ch = channels[g].cpu().numpy()
            kmax, kmin = O.block_summaries(keys, w.block_size)
            s = O.block_scores(q, kmax, kmin)
            kb = min(w.top_blocks, len(s))
            gb = m_glob[b, g].cpu().numpy()
            P.check_ids_layout(gb, kb)
            gb = gb[:kb]
            exc, bad = P.near_tie_mismatches(s, O.topk_ids(s, w.top_blocks), gb, kb, P.NORTH_STAR_REL)
            assert not bad, (b, g, bad)
            _, bad = P.near_tie_mismatches(s, O.topk_ids(s, w.top_blocks), gb, kb, T.STRICT_BLOCK[w.layout])
            assert not bad, (b, g, bad)
            near["block"] += len(exc)
            codes, scale, zero = O.quantize_keys(keys[:, ch])
            cand = O.candidate_tokens(gb, n, w.block_size)
            alpha = O.approx_scores(q, ch, codes, scale, zero, cand, w.scale)
            ot = O.select_tokens(alpha, cand, w.top_tokens)
            nt = int(n_glob[b, g])
            assert nt == min(w.top_tokens, len(cand))
            gt = s_glob[b, g].cpu().numpy()
            P.check_ids_layout(gt, nt)
            gt = gt[:nt]
            pos_o, pos_g = np.searchsorted(cand, ot), np.searchsorted(cand, gt)
            assert np.array_equal(cand[pos_g], gt)
            exc, bad = P.near_tie_mismatches(alpha, pos_o, pos_g, nt, P.NORTH_STAR_REL)
            assert not bad, (b, g, len(bad))
            _, bad = P.near_tie_mismatches(alpha, pos_o, pos_g, nt, T.STRICT_TOKEN)
            assert not bad, (b, g, len(bad))
            near["token"] += len(exc)
            o_ref, l_ref = O.sparse_attention(q, keys, values, gt, w.scale)
            P.compare_output(P.to64(out[b, g * G:(g + 1) * G]), o_ref, w.dtype, f"seqsplit pair {b},{g}")
            np.testing.assert_allclose(P.to64(lse[b, g * G:(g + 1) * G]), l_ref, rtol=0, atol=1e-3)
    return near


@pytest.mark.parametrize("name,Pn", [("gqa8", 2), ("gqa8", 3), ("gqa4_fp32", 4), ("mla", 2)])
def test_seqsplit_matches_unsplit_oracle(name, Pn):
    w = CASES[name]
    cfg, inputs, idx_full = T.setup_case(w, seed=3, pattern="peaked")
    res = SS.run_ranks(rank_states(w, cfg, inputs, idx_full.channels, Pn), inputs["q"], inputs["seq_lens"])
    torch.cuda.synchronize()
    for r in res[1:]:  # every rank holds the same result
        for a, b in zip(r, res[0]):
            assert torch.equal(a, b)
    print(name, Pn, check_against_oracle(w, inputs, idx_full.channels, res[0]))


def test_topk_rows_brute_force_with_ties():
    g = torch.Generator().manual_seed(11)
    for rows, n, k in [(5, 1000, 37), (3, 64, 64), (2, 3000, 1), (4, 257, 300)]:
        keys = torch.randint(0, 20, (rows, n), generator=g).float() / 4  # many exact ties
        ids = torch.arange(n, dtype=torch.int32).repeat(rows, 1) * 3 + 5
        ids[:, ::7] = -1  # empty entries
        ok, oi, cnt = ops.topk_rows(keys.cuda(), ids.cuda(), k)
        for r in range(rows):
            v = ids[r] >= 0
            vk, vi = keys[r][v].double().numpy(), ids[r][v].numpy()
            order = np.lexsort((vi, -vk))[:k]
            ref = np.sort(vi[order])
            assert int(cnt[r]) == len(ref)
            assert np.array_equal(oi[r, : len(ref)].cpu().numpy(), ref)
            assert (oi[r, len(ref):] == -1).all()
            np.testing.assert_array_equal(ok[r, : len(ref)].cpu().numpy(), keys[r].numpy()[(ref - 5) // 3])


def test_select_range_and_attn_merge():
    ids = torch.tensor([[0, 3, 64, 65, 200, -1], [1, 2, 3, -1, -1, -1]], dtype=torch.int32).cuda()
    out, cnt = ops.select_range(ids, 3, 100)
    assert out.tolist() == [[0, 61, 62, -1, -1, -1], [0, -1, -1, -1, -1, -1]] and cnt.tolist() == [3, 1]
    cfg = ops.TLSConfig(batch=1, num_q_heads=2, num_kv_heads=1, d_k=64, d_v=64, max_seq_len=64, dtype=torch.float32)
    po = torch.randn(3, 1, 2, 64).cuda()
    pl = torch.tensor([[[0.5, -float("inf")]], [[1.5, 2.0]], [[-float("inf"), -float("inf")]]]).cuda()
    o, l = ops.attn_merge(cfg, po, pl)
    w0 = torch.softmax(torch.tensor([0.5, 1.5]), 0)
    torch.testing.assert_close(o[0, 0].cpu(), (w0[0] * po[0, 0, 0] + w0[1] * po[1, 0, 0]).cpu(), rtol=0, atol=1e-5)
    torch.testing.assert_close(o[0, 1].cpu(), po[1, 0, 1].cpu(), rtol=0, atol=1e-6)
    assert abs(float(l[0, 0]) - float(torch.logsumexp(torch.tensor([0.5, 1.5]), 0))) < 1e-5
