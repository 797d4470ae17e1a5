"""GPU parity of the CUDA path (libtls.so through the C ABI) against the fp64
oracle on the same seeded inputs (north star (a)/(b)).

Sizes: small cases the oracle finishes in seconds that still span several
tiles / blocks and a ragged tail, every layout (MHA, GQA G=4/8, MLA) and dtype
(bf16, fp32), every cluster size, the degenerate budgets, lag mode, and the
full BASELINE.json sizes on sampled pairs in the launch configuration bench.py
times.
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest
import torch

from oracle import tls_oracle as O
from tests import parity as P

pytestmark = pytest.mark.gpu

tls = pytest.importorskip("paper_2604_07815_b200")
from paper_2604_07815_b200 import workloads as W  # noqa: E402

DEV = "cuda"

SMALL = {
    "c1": W.CONFIGS["c1"],
    "gqa4": W.Workload("t-gqa4", 3, 16, 4, 128, 128, 5000, top_blocks=16, top_tokens=256),
    "gqa8": W.Workload("t-gqa8", 2, 16, 2, 128, 128, 8192, top_blocks=32, top_tokens=512),
    "mha": W.Workload("t-mha", 2, 4, 4, 64, 64, 3000, top_blocks=8, top_tokens=128),
    "mla": W.Workload("t-mla", 2, 16, 1, 576, 512, 4133, d_c=128, top_blocks=16, top_tokens=256, layout="mla",
                      sm_scale=1.0 / math.sqrt(192.0)),
    # even max_seq_len: the token kernel's one-cluster-per-pair form (token_pair_nt_kernel) applies
    "mla_even": W.Workload("t-mla-even", 2, 16, 1, 576, 512, 4133, max_seq_len=4134, d_c=128, top_blocks=16,
                           top_tokens=256, layout="mla", sm_scale=1.0 / math.sqrt(192.0)),
    "fp32_dc64_g8": W.Workload("t-fp32-dc64", 2, 16, 2, 128, 128, 3100, d_c=64, top_blocks=12, top_tokens=200,
                               dtype=torch.float32),
    "b128": W.Workload("t-b128", 2, 8, 2, 128, 128, 6000, block_size=128, top_blocks=10, top_tokens=300),
}

# strict-tier tolerances (fp32 forward-error bound of the GPU arithmetic; U16)
STRICT_BLOCK = {"gqa": 2e-5, "mla": 1e-4}
STRICT_TOKEN = 1e-4


def setup_case(w, seed=0, pattern="outlier", ragged=True):
    inputs = W.make_inputs(w, seed=seed, pattern=pattern, device=DEV, ragged=ragged)
    q_cal, k_cal = W.calibration_sample(w, inputs, seed=seed, pattern=pattern)
    channels = P.oracle_channels(w, q_cal, k_cal).to(DEV)
    cfg = tls.TLSConfig(**w.config_kwargs())
    idx = tls.alloc_index(cfg, channels)
    tls.build_index(cfg, inputs["k_cache"], inputs["seq_lens"], idx)
    return cfg, inputs, idx


def check_pair(w, cfg, inputs, idx, res, b, g, stats):
    out, lse, bids, tids, ntok, tsc = res
    G = w.num_q_heads // w.num_kv_heads
    n = int(inputs["seq_lens"][b].item())
    q, keys, values = P.pair_slices(w, inputs, b, g)
    ch = idx.channels[g].cpu().numpy()
    prm = P.params(w)
    # ---- block stage ----
    kmax, kmin = O.block_summaries(keys, w.block_size)
    s = O.block_scores(q, kmax, kmin)
    m = len(s)
    ob = O.topk_ids(s, w.top_blocks)
    gb = bids[b, g].cpu().numpy()
    kb = min(w.top_blocks, m)
    P.check_ids_layout(gb, kb)
    gb = gb[:kb]
    exc, bad = P.near_tie_mismatches(s, ob, gb, kb, P.NORTH_STAR_REL)
    assert not bad, f"pair {b},{g}: block mismatches beyond the near-tie band: {bad}"
    exc_s, bad_s = P.near_tie_mismatches(s, ob, gb, kb, STRICT_BLOCK[w.layout if w.layout == 'mla' else 'gqa'])
    assert not bad_s, f"pair {b},{g}: block mismatches beyond the strict fp32 band: {bad_s}"
    stats["block_near_ties"] += len(exc)
    # ---- token stage on the GPU's candidate blocks ----
    codes, scale, zero = O.quantize_keys(keys[:, ch])
    cand = O.candidate_tokens(gb, n, w.block_size)
    alpha = O.approx_scores(q, ch, codes, scale, zero, cand, w.scale)
    ot = O.select_tokens(alpha, cand, w.top_tokens)
    nt = int(ntok[b, g].item())
    assert nt == min(w.top_tokens, len(cand))
    gt = tids[b, g].cpu().numpy()
    P.check_ids_layout(gt, nt)
    gt = gt[:nt]
    pos_o = np.searchsorted(cand, ot)
    pos_g = np.searchsorted(cand, gt)
    assert np.array_equal(cand[pos_g], gt), "GPU token outside the candidate blocks"
    exc, bad = P.near_tie_mismatches(alpha, pos_o, pos_g, nt, P.NORTH_STAR_REL)
    assert not bad, f"pair {b},{g}: token mismatches beyond the near-tie band: {len(bad)}"
    exc_s, bad_s = P.near_tie_mismatches(alpha, pos_o, pos_g, nt, STRICT_TOKEN)
    assert not bad_s, f"pair {b},{g}: token mismatches beyond the strict band: {len(bad_s)}"
    stats["token_near_ties"] += len(exc)
    # token scores = ln alpha~ of the selected tokens
    ts = tsc[b, g].cpu().numpy()[:nt]
    np.testing.assert_allclose(ts, np.log(alpha[pos_g]), rtol=0, atol=2e-3)
    # ---- attention on the GPU's ids (reading U17) ----
    o_ref, l_ref = O.sparse_attention(q, keys, values, gt, w.scale)
    o_gpu = P.to64(out[b, g * G:(g + 1) * G])
    P.compare_output(o_gpu, o_ref, w.dtype, f"pair {b},{g} out")
    np.testing.assert_allclose(P.to64(lse[b, g * G:(g + 1) * G]), l_ref, rtol=0, atol=1e-3)
    # end to end against the oracle's own ids (reported; equal when no flip)
    if len(exc) == 0 and set(ot) == set(gt):
        o_e2e, _ = O.sparse_attention(q, keys, values, ot, w.scale)
        P.compare_output(o_gpu, o_e2e, w.dtype, f"pair {b},{g} e2e")


def run_decode(cfg, inputs, idx, guide=None):
    return tls.decode(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx,
                      guide_block_ids=guide)


@pytest.mark.parametrize("name", list(SMALL))
def test_decode_parity_small(name):
    w = SMALL[name]
    cfg, inputs, idx = setup_case(w)
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            check_pair(w, cfg, inputs, idx, res, b, g, stats)
    print(f"{name}: near-ties {stats}")


@pytest.mark.parametrize("cs", [1, 2, 4, 8, 16])
def test_every_cluster_size(cs, monkeypatch):
    monkeypatch.setenv("TLS_CLUSTER", str(cs))
    w = SMALL["gqa4"]
    cfg, inputs, idx = setup_case(w, seed=1, pattern="peaked")
    assert tls.cluster_size(cfg, 2) == cs
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            check_pair(w, cfg, inputs, idx, res, b, g, stats)


@pytest.mark.parametrize("name", ["gqa4", "mla", "c1"])
def test_build_index_bit_exact(name):
    w = SMALL[name]
    cfg, inputs, idx = setup_case(w)
    torch.cuda.synchronize()
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            n = int(inputs["seq_lens"][b].item())
            _, keys, _ = P.pair_slices(w, inputs, b, g)
            kmax, kmin = O.block_summaries(keys, w.block_size)
            m = kmax.shape[0]
            bm = P.to64(idx.block_minmax[b, g, :m])
            assert np.array_equal(bm[:, 0], kmax) and np.array_equal(bm[:, 1], kmin)
            ch = idx.channels[g].cpu().numpy()
            codes, scale, zero = O.quantize_keys(keys[:, ch])
            packed = idx.codes[b, g, :n].cpu().numpy()
            lo, hi = packed & 0xF, packed >> 4
            got = np.stack([lo, hi], axis=-1).reshape(n, w.d_c)
            assert np.array_equal(got, codes), "INT4 codes differ"
            sz = idx.scale_zero[b, g, :n].cpu().numpy()
            assert np.array_equal(sz[:, 0], scale) and np.array_equal(sz[:, 1], zero)


def test_incremental_append_matches_full_build():
    w = SMALL["gqa4"]
    cfg, inputs, idx = setup_case(w, ragged=False)
    full = [t.clone() for t in (idx.block_minmax, idx.codes, idx.scale_zero)]
    # rebuild only from token 3000 on after corrupting that tail
    start = 3000
    sb = start // w.block_size
    idx.block_minmax[:, :, sb:].fill_(0)
    idx.codes[:, :, sb * w.block_size:].fill_(0)
    idx.scale_zero[:, :, sb * w.block_size:].fill_(0)
    tls.build_index(cfg, inputs["k_cache"], inputs["seq_lens"], idx, start_token=start)
    torch.cuda.synchronize()
    assert torch.equal(idx.block_minmax, full[0])
    assert torch.equal(idx.codes, full[1])
    assert torch.equal(idx.scale_zero, full[2])


@pytest.mark.parametrize("name", ["gqa8", "mla", "c1"])
def test_calibration_matches_oracle(name):
    w = SMALL[name]
    inputs = W.make_inputs(w, seed=3, pattern="outlier", device=DEV)
    q_cal, k_cal = W.calibration_sample(w, inputs, seed=3)
    cfg = tls.TLSConfig(**w.config_kwargs())
    ch, sc = tls.calibrate_channels(cfg, q_cal, k_cal)
    torch.cuda.synchronize()
    G = w.num_q_heads // w.num_kv_heads
    for g in range(w.num_kv_heads):
        och, osc = O.calibrate_channels(P.to64(q_cal)[:, g * G:(g + 1) * G], P.to64(k_cal)[g], w.d_c)
        assert np.array_equal(ch[g].cpu().numpy(), och)
        assert np.array_equal(sc[g].cpu().numpy(), osc.astype(np.float32))


@pytest.mark.parametrize("name", ["gqa4", "mla", "c1"])
def test_degenerate_budget_is_dense_attention(name):
    base = SMALL[name]
    w = base.with_(top_blocks=10_000, top_tokens=base.S)
    cfg, inputs, idx = setup_case(w)
    out, lse, bids, tids, ntok, _ = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    G = w.num_q_heads // w.num_kv_heads
    for b in range(w.batch):
        n = int(inputs["seq_lens"][b].item())
        for g in range(w.num_kv_heads):
            assert int(ntok[b, g]) == n
            assert np.array_equal(tids[b, g, :n].cpu().numpy(), np.arange(n))
            q, keys, values = P.pair_slices(w, inputs, b, g)
            o_ref, l_ref = O.dense_attention(q, keys, values, w.scale)
            P.compare_output(P.to64(out[b, g * G:(g + 1) * G]), o_ref, w.dtype, "dense")
            np.testing.assert_allclose(P.to64(lse[b, g * G:(g + 1) * G]), l_ref, rtol=0, atol=1e-3)


def test_lag_mode_uses_guide_blocks():
    w = SMALL["gqa4"]
    cfg, inputs, idx = setup_case(w, seed=5)
    gen = torch.Generator().manual_seed(5)
    guide = torch.full((w.batch, w.num_kv_heads, w.top_blocks), -1, dtype=torch.int32)
    for b in range(w.batch):
        m = (int(inputs["seq_lens"][b]) + w.block_size - 1) // w.block_size
        for g in range(w.num_kv_heads):
            k = int(torch.randint(1, w.top_blocks + 1, (1,), generator=gen))
            ids = torch.randperm(m, generator=gen)[:k].sort().values
            guide[b, g, : len(ids)] = ids.to(torch.int32)
    guide = guide.to(DEV)
    out, lse, bids, tids, ntok, tsc = run_decode(cfg, inputs, idx, guide=guide)
    torch.cuda.synchronize()
    G = w.num_q_heads // w.num_kv_heads
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            q, keys, values = P.pair_slices(w, inputs, b, g)
            gd = guide[b, g].cpu().numpy()
            r = O.tls_pair(q, keys, values, idx.channels[g].cpu().numpy(), P.params(w), guide_block_ids=gd)
            nt = int(ntok[b, g])
            assert nt == min(w.top_tokens, len(r["candidates"]))
            gt = tids[b, g, :nt].cpu().numpy()
            cand = r["candidates"]
            exc, bad = P.near_tie_mismatches(r["alpha"], np.searchsorted(cand, r["token_ids"]),
                                             np.searchsorted(cand, gt), nt, STRICT_TOKEN)
            assert not bad
            o_ref, _ = O.sparse_attention(q, keys, values, gt, w.scale)
            P.compare_output(P.to64(out[b, g * G:(g + 1) * G]), o_ref, w.dtype, "lag")


@pytest.mark.parametrize("name", ["gqa8", "mla"])
def test_separate_calls_equal_fused(name):
    w = SMALL[name]
    cfg, inputs, idx = setup_case(w, seed=2)
    fused = run_decode(cfg, inputs, idx)
    bids, tids, ntok, tsc = tls.select(cfg, inputs["q"], inputs["seq_lens"], idx)
    out, lse = tls.sparse_attend(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"], tids, ntok)
    torch.cuda.synchronize()
    assert torch.equal(bids, fused[2]) and torch.equal(tids, fused[3]) and torch.equal(ntok, fused[4])
    assert torch.equal(tsc, fused[5])
    if tls.select_mode(cfg) == 3:
        # the fused step attends in its own kernel (nc-way split, DSMEM merge), tls_sparse_attend in the
        # attention kernel (its own split): the same sum in a different order
        torch.testing.assert_close(out.float(), fused[0].float(), rtol=0, atol=2e-2)
        torch.testing.assert_close(lse, fused[1], rtol=0, atol=1e-4)
    else:
        torch.testing.assert_close(out.float(), fused[0].float(), rtol=0, atol=1e-6)
        torch.testing.assert_close(lse, fused[1], rtol=0, atol=1e-6)


def test_edge_single_token_and_k1():
    w = W.Workload("t-edge", 3, 8, 2, 128, 128, 700, top_blocks=1, top_tokens=1)
    inputs = W.make_inputs(w, seed=9, device=DEV, seq_lens=[1, 65, 700])
    q_cal, k_cal = W.calibration_sample(w, inputs, seed=9)
    channels = P.oracle_channels(w, q_cal, k_cal).to(DEV)
    cfg = tls.TLSConfig(**w.config_kwargs())
    idx = tls.alloc_index(cfg, channels)
    tls.build_index(cfg, inputs["k_cache"], inputs["seq_lens"], idx)
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            check_pair(w, cfg, inputs, idx, res, b, g, stats)


@pytest.mark.parametrize("form", ["2", "1", "4", "cluster"])
def test_empty_and_partial_sequences_every_token_form(form, monkeypatch):
    """A batch with an empty sequence (n = 0: no candidate, no selected token, output 0 / lse -inf), one shorter than a
    block and one ending mid-block, through every token-kernel form (the pair forms mask the partial last block's
    rows; the empty pair stages nothing)."""
    monkeypatch.setenv("TLS_K2_FORM", form)
    w = W.Workload("t-empty", 4, 16, 2, 128, 128, 2000, top_blocks=8, top_tokens=200)
    inputs = W.make_inputs(w, seed=13, device=DEV, seq_lens=[1999, 0, 40, 1217])  # (calibration reads sequence 0)
    q_cal, k_cal = W.calibration_sample(w, inputs, seed=13)
    channels = P.oracle_channels(w, q_cal, k_cal).to(DEV)
    cfg = tls.TLSConfig(**w.config_kwargs())
    idx = tls.alloc_index(cfg, channels)
    tls.build_index(cfg, inputs["k_cache"], inputs["seq_lens"], idx)
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    out, lse, bids, tids, ntok, tsc = res
    assert int(ntok[1].max()) == 0 and bool((tids[1] == -1).all()) and bool((bids[1] == -1).all())
    assert bool(torch.isfinite(out[1].float()).all()) and float(out[1].float().abs().max()) == 0.0
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in (0, 2, 3):
        for g in range(w.num_kv_heads):
            check_pair(w, cfg, inputs, idx, res, b, g, stats)


def test_errors_are_reported():
    w = SMALL["gqa4"]
    cfg, inputs, idx = setup_case(w)
    bad = tls.TLSConfig(**{**w.config_kwargs(), "d_c": 48})
    with pytest.raises(tls.TLSError, match="UNSUPPORTED"):
        tls.select(bad, inputs["q"], inputs["seq_lens"], idx)
    bad = tls.TLSConfig(**{**w.config_kwargs(), "num_kv_heads": 3})
    with pytest.raises((tls.TLSError, ValueError)):
        tls.select(bad, inputs["q"], inputs["seq_lens"], idx)


# ---- full BASELINE.json sizes, sampled pairs, bench launch configuration ----
N_FULL_PAIRS = 16


def sampled_pairs(w, n, seed):
    """n distinct (b, g) pairs: the first and the last pair plus a seeded sample of the rest."""
    allp = [(b, g) for b in range(w.batch) for g in range(w.num_kv_heads)]
    if len(allp) <= n:
        return allp
    rng = np.random.default_rng(seed)
    mid = rng.choice(np.arange(1, len(allp) - 1), size=n - 2, replace=False)
    return [allp[0]] + [allp[i] for i in sorted(mid)] + [allp[-1]]


def run_full(w, pattern, seed=0, n_pairs=N_FULL_PAIRS):
    inputs = W.make_inputs(w, seed=seed, pattern=pattern, device=DEV)
    q_cal, k_cal = W.calibration_sample(w, inputs, seed=seed, pattern=pattern)
    channels = P.oracle_channels(w, q_cal, k_cal).to(DEV)
    cfg = tls.TLSConfig(**w.config_kwargs())
    idx = tls.alloc_index(cfg, channels)
    tls.build_index(cfg, inputs["k_cache"], inputs["seq_lens"], idx)
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    pairs = sampled_pairs(w, n_pairs, seed + 101)
    for b, g in pairs:
        check_pair(w, cfg, inputs, idx, res, b, g, stats)
    print(f"{w.name} {pattern}: {len(pairs)} pairs, near-ties {stats}")
    del inputs, idx, res
    torch.cuda.empty_cache()
    return stats


@pytest.mark.slow
@pytest.mark.parametrize("pattern", ["outlier", "uniform", "peaked"])
@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_full_size_sampled_pairs(name, pattern):
    """BASELINE.json's C2/C3/C4 at full size in the launch configuration bench.py times (one tls_decode over the
    whole batch), 16 sampled pairs per case checked element by element against the oracle: the bench's own
    `outlier` pattern, `uniform` (flat alpha~: the widest top-k_t boundary) and `peaked`."""
    run_full(W.CONFIGS[name], pattern)


@pytest.mark.slow
@pytest.mark.parametrize("kb,kt", [(128, 512), (128, 2048), (256, 1024), (64, 1024)])
def test_budgets_c3_shape(kb, kt):
    """The paper's budgets (k_b = 128 blocks, k_t in {512, 1024, 2048}) and k_b in {64, 256} on the C3
    per-pair shape (Qwen3-32B, 96k context; batch 2 = 16 pairs, every pair checked)."""
    w = W.CONFIGS["c3"].with_(batch=2, top_blocks=kb, top_tokens=kt)
    run_full(w, "outlier", seed=2, n_pairs=16)
    run_full(w, "uniform", seed=3, n_pairs=16)


@pytest.mark.parametrize("name", ["gqa4", "mla", "c1"])
def test_block_scores_match_direct_form(name):
    """tls_block_scores vs the oracle's direct Quest form O3, fp32 bound."""
    w = SMALL[name]
    cfg, inputs, idx = setup_case(w, seed=6)
    sc = tls.block_scores(cfg, inputs["q"], inputs["seq_lens"], idx)
    torch.cuda.synchronize()
    G = w.num_q_heads // w.num_kv_heads
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            q, keys, _ = P.pair_slices(w, inputs, b, g)
            kmax, kmin = O.block_summaries(keys, w.block_size)
            ref = O.block_scores(q, kmax, kmin)
            got = sc[b, g, : len(ref)].double().cpu().numpy()
            bound = 2e-6 * (np.abs(q).sum() * np.maximum(np.abs(kmax), np.abs(kmin)).max(axis=1) + 1.0)
            assert np.all(np.abs(got - ref) <= bound)


def test_kernel_timing_hook_records_every_launch():
    """tls_timing_enable/read: one record per select/decode call, 4 slots, and
    recording does not change the results."""
    for name in ("gqa8", "mla"):  # the fused step kernel (one slot) and the kernel chain (three slots)
        check_timing_hook(SMALL[name])


def check_timing_hook(w):
    cfg, inputs, idx = setup_case(w, seed=3)
    ref = run_decode(cfg, inputs, idx)
    tls.timing_enable(2)
    try:
        res = run_decode(cfg, inputs, idx)
        tls.select(cfg, inputs["q"], inputs["seq_lens"], idx)
        run_decode(cfg, inputs, idx)  # more calls than reserved: events created on demand
        ms, calls = tls.timing_read(cfg)
        assert calls == 3
        assert set(ms) == set(tls.kernel_names(cfg)) and all(v > 0 for v in ms.values())
        ms2, calls2 = tls.timing_read(cfg)
        assert calls2 == 0 and all(v == 0 for v in ms2.values())
    finally:
        tls.timing_enable(0)
    run_decode(cfg, inputs, idx)
    assert tls.timing_read()[1] == 0  # disabled: nothing recorded
    torch.cuda.synchronize()
    for a, b in zip(ref, res):
        assert torch.equal(a, b)


@pytest.mark.parametrize("name", ["gqa8", "mla", "c1"])
def test_repeated_calls_and_launch_modes_agree(name, monkeypatch):
    """The pair-completion protocol across calls: select_kernel's workers wait
    for the score sentinel and restore it, and the token / attention kernels
    wait for per-pair ready flags (epoch per call) under PDL.  Ten back-to-back
    calls on one workspace, the same calls without PDL, and a fresh
    (tls_workspace_init) workspace must all give bit-identical results; a
    different query in between must not leak into the next call."""
    w = SMALL[name]
    cfg, inputs, idx = setup_case(w, seed=4)
    ref = run_decode(cfg, inputs, idx)
    q2 = inputs["q"].flip(0).contiguous()
    for i in range(10):
        res = run_decode(cfg, inputs, idx) if i % 2 == 0 else tls.decode(
            cfg, q2, inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
        if i % 2 == 0:
            torch.cuda.synchronize()
            for a, b in zip(ref, res):
                assert a is None and b is None or torch.equal(a, b)
    monkeypatch.setenv("TLS_NO_PDL", "1")
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    for a, b in zip(ref, res):
        assert a is None and b is None or torch.equal(a, b)


def test_sub_batch_pipeline_and_tile_size_agree(monkeypatch):
    """TLS_NSPLIT (sub-batch chains on internal streams) and TLS_TILE_KB (block
    rows per scoring CTA) change only scheduling: selections identical, outputs
    equal up to the attention split-K rounding."""
    w = SMALL["gqa4"]
    cfg, inputs, idx = setup_case(w, seed=5)
    ref = run_decode(cfg, inputs, idx)
    for env in ({"TLS_NSPLIT": "3"}, {"TLS_TILE_KB": "8"}, {"TLS_TILE_KB": "16", "TLS_NSPLIT": "2"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        res = run_decode(cfg, inputs, idx)
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(zip(ref[2:], res[2:])):
            assert torch.equal(a, b), (env, i, (a != b).sum().item(), a.flatten()[:8], b.flatten()[:8])
        torch.testing.assert_close(res[0].float(), ref[0].float(), rtol=0, atol=2e-2)
        for k in env:
            monkeypatch.delenv(k)


@pytest.mark.parametrize("pattern", ["all_equal", "four_values"])
def test_block_topk_exact_ties(pattern):
    """a2 with exactly tied block scores (ties -> lower block id, U2): blocks repeat so the k_b-th score
    falls inside a large tie group (or every score is equal), m = 1200 blocks (the one-pass register select).
    Expected = stable order by (-score, id) of the same library's block scores (tls_block_scores)."""
    w = W.Workload("ties", 2, 8, 2, 128, 128, 64 * 1200, top_blocks=128, top_tokens=256)
    cfg, inputs, idx = setup_case(w, seed=3, ragged=False)
    k = inputs["k_cache"]
    B = w.block_size
    period = 1 if pattern == "all_equal" else 4
    blocks = k.view(w.batch, w.num_kv_heads, -1, B, w.d_k)
    src = blocks[:, :, :period].clone()
    reps = blocks.shape[2] // period
    blocks.copy_(src.repeat(1, 1, reps, 1, 1))
    tls.build_index(cfg, k, inputs["seq_lens"], idx)
    sc = tls.block_scores(cfg, inputs["q"], inputs["seq_lens"], idx)
    bids = tls.select(cfg, inputs["q"], inputs["seq_lens"], idx)[0]
    torch.cuda.synchronize()
    m = blocks.shape[2]
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            s = sc[b, g, :m].double().cpu().numpy()
            order = np.lexsort((np.arange(m), -s))  # by -score, then id
            exp = np.sort(order[: w.top_blocks])
            assert np.array_equal(bids[b, g].cpu().numpy(), exp), (pattern, b, g)


@pytest.mark.parametrize("period", [1, 12])
def test_token_topk_exact_ties(period):
    """a4 with exactly tied ranking keys (ties -> lower token id, U2): token t of every pair repeats the
    content of token t mod period, so every block scores the same (M_t = the first k_b blocks) and the candidates
    form `period` groups of bitwise-equal keys.  S_t must be whole groups plus the lowest-id prefix of at most one
    group (period 12: a 683-key boundary group, the register select; period 1: one 8192-key group, the fallback)."""
    w = W.Workload("tties", 1, 8, 2, 128, 128, 64 * 256, top_blocks=128, top_tokens=1024)
    cfg, inputs, idx = setup_case(w, seed=4, ragged=False)
    k, v = inputs["k_cache"], inputs["v_cache"]
    S = k.shape[2]
    src = torch.arange(S, device=k.device) % period
    k.copy_(k[:, :, src])
    v.copy_(v[:, :, src])
    tls.build_index(cfg, k, inputs["seq_lens"], idx)
    out, lse, bids, tids, nt, ts = tls.decode(cfg, inputs["q"], k, v, inputs["seq_lens"], idx)
    torch.cuda.synchronize()
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            assert torch.equal(bids[b, g].cpu(), torch.arange(w.top_blocks, dtype=torch.int32))
            n = int(nt[b, g])
            assert n == w.top_tokens
            sel = tids[b, g, :n].cpu().numpy()
            assert np.all(np.diff(sel) > 0)  # ascending, distinct
            cand = np.arange(w.top_blocks * w.block_size)
            partial = 0
            for grp in range(period):
                members = cand[cand % period == grp]
                chosen = np.intersect1d(sel, members)
                if 0 < len(chosen) < len(members):
                    partial += 1
                    assert np.array_equal(chosen, members[: len(chosen)]), (period, grp)  # lowest ids first
            assert partial <= 1


def test_mla_attention_large_selection_uses_small_chunks():
    """MLA attention over K_t = n = 131072 selected tokens (a5): the CTA's selected-token list leaves no room
    for the 64-token double-buffered staging, so the plan falls back to 32-token chunks (3 stages); the output must
    still equal dense attention (torch fp32 reference of the same definition, within the bf16 tolerance)."""
    w = W.Workload("mla-big", 1, 32, 1, 576, 512, 131072, d_c=128, top_blocks=2048, top_tokens=131072, layout="mla",
                   sm_scale=1.0 / math.sqrt(192.0))
    cfg = tls.TLSConfig(**w.config_kwargs())
    assert tls.cluster_size(cfg, 3) == 32 and tls.cluster_size(cfg, 4) == 2  # the mma.sync 32-token fallback runs
    small = tls.TLSConfig(**SMALL["mla"].config_kwargs())
    assert tls.cluster_size(small, 4) == 2 and tls.cluster_size(small, 3) == 64  # MLA: mma.sync by default
    g = torch.Generator(device=DEV).manual_seed(11)
    q = torch.randn((1, 32, 576), generator=g, device=DEV).to(torch.bfloat16)
    k = torch.randn((1, w.context, 576), generator=g, device=DEV).to(torch.bfloat16)
    tids = torch.arange(w.context, dtype=torch.int32, device=DEV).view(1, 1, -1).contiguous()
    nt = torch.full((1, 1), w.context, dtype=torch.int32, device=DEV)
    out, lse = tls.sparse_attend(cfg, q, k, None, tids, nt)
    s = (q[0].float() @ k[0].float().T) * w.scale
    ref = torch.softmax(s, dim=-1) @ k[0, :, :512].float()
    torch.cuda.synchronize()
    torch.testing.assert_close(out[0].float(), ref, rtol=0, atol=2e-2)
    torch.testing.assert_close(lse[0], torch.logsumexp(s, dim=-1), rtol=0, atol=1e-2)


@pytest.mark.parametrize("name", ["gqa4", "gqa8"])
def test_streaming_select_experiment(name, monkeypatch):
    """The opt-in streaming a1 + a2 kernel (TLS_STREAM_SEL=1, fused.cu stream_select_kernel: one streamer CTA
    per SM, warp-specialised TMA ring, a2 markers) selects the same blocks and tokens as the oracle."""
    monkeypatch.setenv("TLS_STREAM_SEL", "1")
    w = SMALL[name]
    cfg, inputs, idx = setup_case(w, seed=6)
    for _ in range(3):  # repeated calls: the ticket / exit counters and per-SM words reset themselves
        res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            check_pair(w, cfg, inputs, idx, res, b, g, stats)


@pytest.mark.parametrize("case", ["small", "dense", "c4"])
def test_mla_tcgen05_attention(case, monkeypatch):
    """The MLA attention on the 5th-generation tensor cores (TLS_MLA_TC=1, attend.cu attend_mla_tc_kernel:
    tcgen05.mma with TMEM accumulators, S^T = K Q^T and O^T += V^T P^T from one core-matrix copy of each 64-token
    chunk) against the oracle: the decode of small MLA cases, the degenerate budget (= dense attention),
    and BASELINE.json's C4 at full size on sampled pairs."""
    monkeypatch.setenv("TLS_MLA_TC", "1")
    if case == "c4":
        run_full(W.CONFIGS["c4"], "outlier", seed=5, n_pairs=8)
        return
    w = SMALL["mla"] if case == "small" else SMALL["mla"].with_(top_blocks=10 ** 4, top_tokens=10 ** 5)
    cfg, inputs, idx = setup_case(w, seed=8)
    assert tls.cluster_size(cfg, 4) == 3  # the tcgen05 plan runs
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            check_pair(w, cfg, inputs, idx, res, b, g, stats)


@pytest.mark.parametrize("name", ["gqa4", "gqa8", "c1", "fp32_dc64_g8", "b128", "mha"])
@pytest.mark.parametrize("form", ["pair4", "pair2", "pair1", "cluster"])
def test_token_kernel_forms(name, form, monkeypatch):
    """Both forms of the token-scoring kernel (a3) against the oracle: one 1024-thread CTA per pair holding the
    whole candidate index (the default where G <= 8 and it fits shared memory), and the cluster of chunk CTAs
    (TLS_K2_FORM=cluster; the only form for MLA / G > 8)."""
    monkeypatch.setenv("TLS_K2_FORM", {"pair4": "4", "pair2": "2", "pair1": "1", "cluster": "cluster"}[form])
    w = SMALL[name]
    cfg, inputs, idx = setup_case(w, seed=5, pattern="uniform")
    assert tls.cluster_size(cfg, 5) == {"pair4": 5, "pair2": 4, "pair1": 1}.get(form, 2)
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            check_pair(w, cfg, inputs, idx, res, b, g, stats)


@pytest.mark.parametrize("name", ["mla", "g16", "g12"])
@pytest.mark.parametrize("form", ["auto", "cluster"])
def test_token_kernel_nt_forms(name, form, monkeypatch):
    """G > 8 (MLA's 32 heads, GQA groups of 16 / 12): token_pair_nt_kernel (a cluster of 256-thread CTAs per pair,
    logits in TMEM, softmax statistics by a second TMEM pass) against the oracle, and the cluster form."""
    if form == "cluster":
        monkeypatch.setenv("TLS_K2_FORM", "cluster")
    w = {"mla": SMALL["mla_even"],  # even S: the pair form's 16-byte scale/zero rows
         "g16": W.Workload("t-g16", 2, 32, 2, 128, 128, 6000, top_blocks=24, top_tokens=400),
         "g12": W.Workload("t-g12", 2, 24, 2, 128, 128, 5000, top_blocks=16, top_tokens=300)}[name]
    cfg, inputs, idx = setup_case(w, seed=7, pattern="outlier")
    assert (tls.cluster_size(cfg, 5) == 6) == (form == "auto")
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            check_pair(w, cfg, inputs, idx, res, b, g, stats)


@pytest.mark.parametrize("name,every,form", [("gqa8", 16, "auto"), ("mla", 16, "auto"), ("gqa8", 1000, "auto"),
                                             ("mla", 700, "auto"), ("gqa8", 16, "cluster"), ("gqa8", 1000, "cluster"),
                                             ("gqa8", 16, "1"), ("gqa8", 1000, "1"), ("mla_even", 16, "auto"),
                                             ("mla_even", 700, "auto")])
def test_sink_tokens_wide_logit_span(name, every, form, monkeypatch):
    """Reading U20: attention-sink-like keys (tokens aligned with the group's queries so strongly that the
    logits of the pair span > 200 nats) must not collapse the other candidates' ranking keys: alpha~ of an ordinary
    token is then ~e^-200 of a sink's, below fp32's range as a value, but its ln alpha~ is representable and the
    top-k_t among the ordinary tokens must still follow the oracle's order."""
    if form != "auto":
        monkeypatch.setenv("TLS_K2_FORM", form)
    w = SMALL[name]
    inputs = W.make_inputs(w, seed=17, pattern="uniform", device=DEV, ragged=False)
    G = w.num_q_heads // w.num_kv_heads
    g = torch.Generator(device="cpu").manual_seed(17)
    for b in range(w.batch):
        for kh in range(w.num_kv_heads):
            qbar = inputs["q"][b, kh * G:(kh + 1) * G].float().mean(0)
            u = qbar / qbar.norm()
            # every=16: one sink in every 16-token tile, so that every warp of the token kernel holds sinks and
            # ordinary tokens together (log-domain keys); every=700/1000: most warps hold no sink, their keys carry
            # the ~200-nat offset to lz in the per-warp factor r_w.  k_t exceeds the number of candidate sinks, so
            # the boundary falls among the others
            n_b = int(inputs["seq_lens"][b])
            for t in range(5, n_b, every):
                # logit boost ~ 40 * |q_h . u| * sqrt(d) * sm_scale: >= ~200 nats above the rest
                if w.layout == "mla":
                    inputs["k_cache"][b, t] = (inputs["k_cache"][b, t].float() + 40.0 * u * math.sqrt(w.d_k)).to(w.dtype)
                else:
                    inputs["k_cache"][b, kh, t] = (inputs["k_cache"][b, kh, t].float() + 40.0 * u * math.sqrt(w.d_k)).to(w.dtype)
    q_cal, k_cal = W.calibration_sample(w, inputs, seed=17)
    channels = P.oracle_channels(w, q_cal, k_cal).to(DEV)
    cfg = tls.TLSConfig(**w.config_kwargs())
    idx = tls.alloc_index(cfg, channels)
    tls.build_index(cfg, inputs["k_cache"], inputs["seq_lens"], idx)
    res = run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in range(w.batch):
        for kh in range(w.num_kv_heads):
            check_pair(w, cfg, inputs, idx, res, b, kh, stats)
