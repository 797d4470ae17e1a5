"""Multi-step decode loops against the fp64 oracle:

* f2, incremental append (tls_build_index(start_token = n)): every step writes the new token's K/V row,
  extends its sequence by one and rebuilds the index from that token on; the whole index of every pair is
  then compared bit for bit with the oracle's index of the grown cache (O2 block summaries, O5 quantiser), and
  the step's decode is checked against the oracle with the parity suite's rules.
* f1, the asynchronous offload engine (AsyncOffloadDecoder: block cache, one-step lag): at every
  step S_t must equal the oracle's TokenSelect(q_t, M_{t-1}) on the GPU's previous block set (lag mode,
  P:373), the output the oracle's attention over S_t, M_t the oracle's top-k_b (near-tie rule), and the
  blocks fetched must equal the oracle-side ledger of the engine's residency rule: the cache keeps
  C_t = M_{t-2} u M_{t-1} (capacity 2 k_b), so T_t = M_t \\ C_t -- never more than the paper's M_t \\ M_{t-1}
  (P:378).  Three query streams: stationary (T_t empty after the first step), alternating between two
  queries (empty from the third step: C_t holds both block sets) and a drifting random walk.
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

APPEND = {
    "gqa": W.Workload("a-gqa", 2, 16, 2, 128, 128, 3000, top_blocks=12, top_tokens=256, max_seq_len=3100),
    "mla": W.Workload("a-mla", 2, 16, 1, 576, 512, 2000, d_c=128, top_blocks=8, top_tokens=200, layout="mla",
                      sm_scale=1.0 / math.sqrt(192.0), max_seq_len=2100),
}


def check_index_against_oracle(w, inputs, idx, b, g):
    n = int(inputs["seq_lens"][b])
    _, keys, _ = P.pair_slices(w, inputs, b, g)
    kmax, kmin = O.block_summaries(keys, w.block_size)
    m = kmax.shape[0]
    bm = P.to64(idx.block_minmax[b, g, :m])
    assert np.array_equal(bm[:, 0], kmax) and np.array_equal(bm[:, 1], kmin), (b, g, n)
    ch = idx.channels[g].cpu().numpy()
    codes, scale, zero = O.quantize_keys(keys[:, ch])
    packed = idx.codes[b, g, :n].cpu().numpy()
    got = np.stack([packed & 0xF, packed >> 4], axis=-1).reshape(n, w.d_c)
    assert np.array_equal(got, codes), (b, g, n)
    sz = idx.scale_zero[b, g, :n].cpu().numpy()
    assert np.array_equal(sz[:, 0], scale) and np.array_equal(sz[:, 1], zero), (b, g, n)


@pytest.mark.parametrize("name", list(APPEND))
def test_append_decode_loop_matches_oracle(name):
    w = APPEND[name]
    cfg, inputs, idx = T.setup_case(w, seed=21, ragged=True)
    g = torch.Generator(device="cuda").manual_seed(5)
    mla = w.layout == "mla"
    for step in range(70):  # crosses at least one block boundary for every sequence
        # the new token of every sequence: K (and V) rows at position n, then the index from n on
        for b in range(w.batch):
            n = int(inputs["seq_lens"][b])
            if mla:
                inputs["k_cache"][b, n] = torch.randn(w.d_k, generator=g, device="cuda").to(w.dtype)
            else:
                inputs["k_cache"][b, :, n] = torch.randn(w.num_kv_heads, w.d_k, generator=g, device="cuda").to(w.dtype)
                inputs["v_cache"][b, :, n] = torch.randn(w.num_kv_heads, w.d_v, generator=g, device="cuda").to(w.dtype)
        start = int(inputs["seq_lens"].min())
        inputs["seq_lens"] += 1
        tls.build_index(cfg, inputs["k_cache"], inputs["seq_lens"], idx, start_token=start)
        if step % 23 == 0 or step == 69:
            torch.cuda.synchronize()
            for b in range(w.batch):
                for h in range(w.num_kv_heads):
                    check_index_against_oracle(w, inputs, idx, b, h)
            inputs["q"] = torch.randn(inputs["q"].shape, generator=g, device="cuda").to(w.dtype)
            res = T.run_decode(cfg, inputs, idx)
            torch.cuda.synchronize()
            stats = {"block_near_ties": 0, "token_near_ties": 0}
            for b in range(w.batch):
                for h in range(w.num_kv_heads):
                    T.check_pair(w, cfg, inputs, idx, res, b, h, stats)


OFFLOAD = W.Workload("f-gqa", 2, 16, 2, 128, 128, 8000, top_blocks=16, top_tokens=256)


def query_stream(kind, q0, steps, gen):
    qs = [q0]
    q1 = torch.randn(q0.shape, generator=gen, device=q0.device).to(q0.dtype)
    for t in range(1, steps):
        if kind == "stationary":
            qs.append(q0)
        elif kind == "alternating":
            qs.append(q1 if t % 2 else q0)
        else:  # drifting: a random walk of the query (S:527's drifting workload; eps = 0.3 per step here so that
            # M_t moves by a few blocks per step on these small caches)
            qs.append((qs[-1].float() + 0.3 * torch.randn(q0.shape, generator=gen, device=q0.device)).to(q0.dtype))
    return qs


@pytest.mark.parametrize("kind", ["stationary", "alternating", "drifting"])
def test_async_offload_steps_match_oracle_and_ledger(kind):
    w = OFFLOAD
    cfg, inputs, idx = T.setup_case(w, seed=31, pattern="peaked")
    k_host = tls.host_kv(inputs["k_cache"])
    v_host = tls.host_kv(inputs["v_cache"])
    eng = tls.AsyncOffloadDecoder(cfg, k_host, v_host, inputs["seq_lens"], idx)
    gen = torch.Generator(device="cuda").manual_seed(9)
    G = w.num_q_heads // w.num_kv_heads
    prm = P.params(w)
    hist = []  # the GPU's M_t per step, per pair
    fetched, paper = [], []
    for t, q in enumerate(query_stream(kind, inputs["q"], 6, gen)):
        res = eng.step(q)
        torch.cuda.synchronize()
        miss = eng.last_miss.cpu().numpy() if t > 0 else None
        mt = {}
        for b in range(w.batch):
            n = int(inputs["seq_lens"][b])
            for g in range(w.num_kv_heads):
                qg = P.to64(q[b, g * G:(g + 1) * G])
                keys = P.to64(inputs["k_cache"][b, g, :n])
                values = P.to64(inputs["v_cache"][b, g, :n])
                ch = idx.channels[g].cpu().numpy()
                gb = res[2][b, g].cpu().numpy()
                gb = gb[gb >= 0]
                mt[(b, g)] = set(int(x) for x in gb)
                # M_t: the oracle's top-k_b up to near-ties
                kmax, kmin = O.block_summaries(keys, w.block_size)
                s = O.block_scores(qg, kmax, kmin)
                _, bad = P.near_tie_mismatches(s, O.topk_ids(s, w.top_blocks), gb, len(gb), P.NORTH_STAR_REL)
                assert not bad, (t, b, g, bad)
                # S_t = TokenSelect(q_t, M_{t-1}) on the GPU's previous block set (step 0: M_0 itself)
                guide = np.asarray(sorted(hist[-1][(b, g)] if hist else mt[(b, g)]), dtype=np.int64)
                ref = O.tls_pair(qg, keys, values, ch, prm, guide_block_ids=guide)
                nt = int(res[4][b, g])
                gt = res[3][b, g, :nt].cpu().numpy()
                cand = ref["candidates"]
                assert nt == len(ref["token_ids"])
                pos_o, pos_g = np.searchsorted(cand, ref["token_ids"]), np.searchsorted(cand, gt)
                assert np.array_equal(cand[pos_g], gt), (t, b, g)
                _, bad = P.near_tie_mismatches(ref["alpha"], pos_o, pos_g, nt, T.STRICT_TOKEN)
                assert not bad, (t, b, g, len(bad))
                o_ref, _ = O.sparse_attention(qg, keys, values, gt, w.scale)
                P.compare_output(P.to64(res[0][b, g * G:(g + 1) * G]), o_ref, w.dtype, f"offload step {t}")
                # the transfer ledger: fetched = M_t \ (M_{t-1} u M_{t-2})
                if t > 0:
                    resident = hist[-1][(b, g)] | (hist[-2][(b, g)] if len(hist) > 1 else set())
                    assert int(miss[b, g]) == len(mt[(b, g)] - resident), (t, b, g)
                    fetched.append(int(miss[b, g]))
                    paper.append(len(mt[(b, g)] - hist[-1][(b, g)]))
        hist.append(mt)
    print(f"{kind}: blocks fetched per pair-step {np.mean(fetched):.2f} (paper's M_t minus M_t-1: {np.mean(paper):.2f})")
    if kind == "stationary":
        assert sum(fetched) == 0
    if kind == "alternating":
        assert sum(fetched[2 * w.batch * w.num_kv_heads:]) == 0  # from step 3 on both block sets are resident
    if kind == "drifting":
        assert sum(paper) > 0  # the walk does move M_t
    assert all(f <= p for f, p in zip(fetched, paper))
