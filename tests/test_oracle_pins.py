"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names the pin kind of SURVEY §8(c) / DESIGN.md §3: closed forms,
hand cases (tests/golden/hand_cases.json), brute force on tiny inputs, the
paper's own alternative formula (GEMM form P:104-118), a textbook/library
routine (torch fp64 scaled_dot_product_attention), invariants and the
quantiser's error bound.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch

from oracle import tls_oracle as O

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")))


# ---------------------------------------------------------------- hand cases
@pytest.mark.parametrize("case", GOLDEN["block_summaries"])
def test_hand_block_summaries(case):
    kmax, kmin = O.block_summaries(np.array(case["keys"], float), case["block_size"])
    np.testing.assert_array_equal(kmax, case["kmax"])
    np.testing.assert_array_equal(kmin, case["kmin"])


@pytest.mark.parametrize("case", GOLDEN["block_scores"])
def test_hand_block_scores(case):
    s = O.block_scores(np.array(case["q"], float), np.array(case["kmax"], float), np.array(case["kmin"], float))
    np.testing.assert_array_equal(s, case["scores"])


@pytest.mark.parametrize("case", GOLDEN["topk"])
def test_hand_topk(case):
    np.testing.assert_array_equal(O.topk_ids(np.array(case["scores"], float), case["k"]), case["ids"])


@pytest.mark.parametrize("case", GOLDEN["quantize"])
def test_hand_quantize(case):
    codes, scale, zero = O.quantize_keys(np.array([case["row"]], np.float32))
    np.testing.assert_array_equal(codes[0], case["codes"])
    if "scale" in case:
        assert scale[0] == np.float32(case["scale"])
    else:
        a, b = case["scale_f32_of"].split("/")
        assert scale[0] == np.float32(float(a)) / np.float32(float(b))
    assert zero[0] == np.float32(case["zero"])


@pytest.mark.parametrize("case", GOLDEN["approx_scores"])
def test_hand_approx_scores(case):
    keys = np.array(case["keys"], float)  # small non-negative integers: code = key, scale 1, zero 0
    codes = keys.astype(np.uint8)
    n, d = keys.shape
    alpha = O.approx_scores(
        np.array(case["q"], float), np.arange(d), codes, np.ones(n, np.float32), np.zeros(n, np.float32),
        np.arange(n), case["sm_scale"],
    )
    np.testing.assert_allclose(alpha, case["alpha"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("case", GOLDEN["calibrate"])
def test_hand_calibrate(case):
    ch, s = O.calibrate_channels(np.array(case["q_cal"], float), np.array(case["k_cal"], float), case["d_c"])
    np.testing.assert_array_equal(s, case["scores"])
    np.testing.assert_array_equal(ch, case["channels"])


@pytest.mark.parametrize("case", GOLDEN["attention"])
def test_hand_attention(case):
    out, lse = O.sparse_attention(
        np.array(case["q"], float), np.array(case["keys"], float), np.array(case["values"], float),
        np.array(case["ids"]), case["sm_scale"],
    )
    np.testing.assert_allclose(out, case["out"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(lse, case["lse"], rtol=0, atol=1e-14)


# ------------------------------------------------ T1: GEMM identity
def test_gemm_form_equals_direct_form():
    """≥1000 random instances: direct Quest score == the paper's GEMM form
     == the head-collapsed GEMV form used on the GPU
    (Q± = sum_h max/min(q_h, 0); linearity of sum_h)."""
    rng = np.random.default_rng(1)
    count = 0
    for G in (1, 4, 5, 8, 32):
        for d in (8, 128, 576):
            for m in (4, 64):
                reps = 1000 // 30 + 1
                for _ in range(reps):
                    q = rng.standard_normal((G, d))
                    keys = rng.standard_normal((m * 4, d))
                    kmax, kmin = O.block_summaries(keys, 4)
                    direct = O.block_scores(q, kmax, kmin)
                    gemm = O.block_scores_gemm_form(q, kmax, kmin)
                    qp = np.maximum(q, 0).sum(0)
                    qm = np.minimum(q, 0).sum(0)
                    gemv = kmax @ qp + kmin @ qm
                    scale = np.abs(direct).max() + 1e-300
                    assert np.max(np.abs(direct - gemm)) <= 1e-12 * scale
                    assert np.max(np.abs(direct - gemv)) <= 1e-12 * scale
                    count += 1
    assert count >= 1000


def test_max_identity_closed_form():
    """max(q a, q b) = max(q,0) a + min(q,0) b whenever a >= b (the identity behind P:110)."""
    rng = np.random.default_rng(2)
    q = rng.standard_normal(100000)
    a = rng.standard_normal(100000)
    b = a - np.abs(rng.standard_normal(100000))
    lhs = np.maximum(q * a, q * b)
    rhs = np.maximum(q, 0) * a + np.minimum(q, 0) * b
    np.testing.assert_array_equal(lhs, rhs)


# ----------------------------------------------- brute force on tiny inputs
def _scan_summaries(keys, B):
    n, d = keys.shape
    m = -(-n // B)
    kmax = np.full((m, d), -np.inf)
    kmin = np.full((m, d), np.inf)
    for j in range(n):
        for c in range(d):
            kmax[j // B, c] = max(kmax[j // B, c], keys[j, c])
            kmin[j // B, c] = min(kmin[j // B, c], keys[j, c])
    return kmax, kmin


@pytest.mark.parametrize("n,B", [(7, 4), (64, 16), (100, 64), (5, 1), (33, 32)])
def test_summaries_match_scan(n, B):
    rng = np.random.default_rng(n * 100 + B)
    keys = rng.standard_normal((n, 6))
    kmax, kmin = O.block_summaries(keys, B)
    smax, smin = _scan_summaries(keys, B)
    np.testing.assert_array_equal(kmax, smax)
    np.testing.assert_array_equal(kmin, smin)


def _is_valid_topk(scores, k, ids):
    """Pairwise characterisation of 'top-k, ties -> lower index' (U2/U4)."""
    sel = set(int(i) for i in ids)
    if len(sel) != len(ids) or len(ids) != min(k, len(scores)):
        return False
    if list(ids) != sorted(ids):
        return False
    for i in sel:
        for j in range(len(scores)):
            if j in sel:
                continue
            if not (scores[i] > scores[j] or (scores[i] == scores[j] and i < j)):
                return False
    return True


def test_topk_bruteforce_with_ties():
    rng = np.random.default_rng(3)
    for trial in range(400):
        n = int(rng.integers(1, 12))
        scores = rng.integers(0, 4, size=n).astype(float)  # many planted ties
        k = int(rng.integers(0, 14))
        ids = O.topk_ids(scores, k)
        assert _is_valid_topk(scores, k, ids), (scores, k, ids)
        # exhaustive: the unique valid subset is the one returned
        valid = [c for c in itertools.combinations(range(n), min(k, n)) if _is_valid_topk(scores, k, list(c))]
        assert valid == [tuple(ids)]


def test_block_selection_bruteforce():
    """O3+O4 on tiny inputs vs per-token loops: every block score from loops, then
    the exhaustive pairwise check of the selected set."""
    rng = np.random.default_rng(4)
    for B in (4, 16, 64):
        for _ in range(10):
            n = int(rng.integers(1, 512))
            G, d = int(rng.integers(1, 5)), 8
            q = rng.standard_normal((G, d))
            keys = rng.standard_normal((n, d))
            kb = int(rng.integers(1, 12))
            ids, s = O.select_blocks(q, *O.block_summaries(keys, B), kb)
            m = -(-n // B)
            loop = np.zeros(m)
            for i in range(m):
                blk = keys[i * B : (i + 1) * B]
                for h in range(G):
                    for c in range(d):
                        loop[i] += max(q[h, c] * blk[:, c].max(), q[h, c] * blk[:, c].min())
            np.testing.assert_allclose(s, loop, rtol=1e-12, atol=1e-12)
            assert _is_valid_topk(s, kb, ids)


def test_token_selection_bruteforce():
    """O6-O10 on tiny inputs: alpha~ from explicit per-head loops, selection
    checked exhaustively."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        n, B, d, d_c, G = int(rng.integers(8, 200)), 8, 16, 4, int(rng.integers(1, 5))
        keys = rng.standard_normal((n, d)).astype(np.float32)
        q = rng.standard_normal((G, d))
        channels = np.sort(rng.choice(d, d_c, replace=False))
        codes, scale, zero = O.quantize_keys(keys[:, channels])
        blocks = np.sort(rng.choice(-(-n // B), min(3, -(-n // B)), replace=False))
        cand = O.candidate_tokens(blocks, n, B)
        sm = 0.25
        alpha = O.approx_scores(q, channels, codes, scale, zero, cand, sm)
        ref = np.zeros(len(cand))
        for h in range(G):
            logit = [sm * sum(q[h, channels[c]] * (float(zero[j]) + float(scale[j]) * int(codes[j, c])) for c in range(d_c)) for j in cand]
            e = np.exp(np.array(logit) - max(logit))
            ref += e / e.sum() / G
        np.testing.assert_allclose(alpha, ref, rtol=1e-12, atol=1e-15)
        kt = int(rng.integers(1, 40))
        tok = O.select_tokens(alpha, cand, kt)
        pos = np.searchsorted(cand, tok)
        assert _is_valid_topk(alpha, kt, list(pos))
        # candidate confinement: every selected token lies in a selected block
        assert all((t // B) in set(blocks.tolist()) for t in tok)


# ------------------------------------------------------- T6 upper bound
def test_block_score_upper_bounds_member_logits():
    """G=1: q.k_j <= s_i for every token j of block i (brute force)."""
    rng = np.random.default_rng(6)
    for _ in range(50):
        n, B, d = 200, 16, 12
        keys = rng.standard_normal((n, d))
        q = rng.standard_normal((1, d))
        s = O.block_scores(q, *O.block_summaries(keys, B))
        for j in range(n):
            assert q[0] @ keys[j] <= s[j // B] + 1e-12


def test_selection_shift_invariance():
    rng = np.random.default_rng(7)
    for _ in range(50):
        s = rng.standard_normal(100)
        np.testing.assert_array_equal(O.topk_ids(s, 10), O.topk_ids(s + 7.25, 10))


# ------------------------------------------------ T5 quantiser error bound
def test_quantiser_error_bound_1e5_rows():
    """|k~ - x| <= scale/2 on >= 1e5 rows; the bound holds up to
    the fp32 rounding of the quotient (relative 2^-23 on the code)."""
    rng = np.random.default_rng(8)
    rows = (rng.standard_normal((100000, 32)) * rng.uniform(0.01, 100, size=(100000, 1))).astype(np.float32)
    # make the values bf16-exact like the cache
    rows = torch.from_numpy(rows).to(torch.bfloat16).float().numpy()
    codes, scale, zero = O.quantize_keys(rows)
    deq = O.dequantize(codes, scale, zero)
    err = np.abs(deq - rows.astype(np.float64))
    bound = scale.astype(np.float64)[:, None] * (0.5 + 16 * 2.0**-23)
    assert np.all(err <= bound)
    assert codes.max() <= 15
    # each row uses both ends of the grid unless constant
    nz = scale > 0
    assert np.all(codes[nz].min(axis=1) == 0) and np.all(codes[nz].max(axis=1) == 15)


def test_quantiser_constant_rows():
    rows = np.full((10, 8), 1.5, np.float32)
    codes, scale, zero = O.quantize_keys(rows)
    assert np.all(scale == 0) and np.all(codes == 0) and np.all(zero == np.float32(1.5))


# ------------------------------------------------------------ T7 invariants
def test_alpha_invariant_to_sm_scale_when_g1():
    rng = np.random.default_rng(9)
    keys = rng.standard_normal((300, 16)).astype(np.float32)
    q = rng.standard_normal((1, 16))
    ch = np.arange(0, 16, 2)
    codes, scale, zero = O.quantize_keys(keys[:, ch])
    cand = np.arange(300)
    sel = [O.select_tokens(O.approx_scores(q, ch, codes, scale, zero, cand, sm), cand, 37) for sm in (1.0, 0.25, 1 / np.sqrt(8))]
    np.testing.assert_array_equal(sel[0], sel[1])
    np.testing.assert_array_equal(sel[0], sel[2])


def test_identity_channels_on_grid_keys_give_exact_attention_weights():
    """d_c = d, C = identity, keys on the quantisation grid -> alpha~ equals the
    head-mean of the exact attention weights softmax(q K^T * sm_scale),
    computed here with torch.softmax."""
    rng = np.random.default_rng(10)
    n, d, G = 257, 8, 3
    codes = rng.integers(0, 16, size=(n, d))
    codes[:, 0] = 0
    codes[:, 1] = 15  # every row spans the full grid
    sc = 2.0 ** rng.integers(-3, 2, size=n)
    z = rng.integers(-8, 8, size=n) * 0.5
    keys = (z[:, None] + sc[:, None] * codes).astype(np.float32)
    q = rng.standard_normal((G, d))
    c2, s2, z2 = O.quantize_keys(keys)
    np.testing.assert_array_equal(c2, codes)
    alpha = O.approx_scores(q, np.arange(d), c2, s2, z2, np.arange(n), 0.3)
    w = torch.softmax(torch.tensor(q) @ torch.tensor(keys, dtype=torch.float64).T * 0.3, dim=-1).mean(0).numpy()
    np.testing.assert_allclose(alpha, w, rtol=1e-12, atol=1e-16)


def test_alpha_is_a_distribution():
    rng = np.random.default_rng(11)
    keys = rng.standard_normal((500, 32)).astype(np.float32)
    codes, scale, zero = O.quantize_keys(keys[:, :8])
    alpha = O.approx_scores(rng.standard_normal((4, 32)), np.arange(8), codes, scale, zero, np.arange(100, 400), 0.1)
    assert abs(alpha.sum() - 1) < 1e-12 and np.all(alpha > 0)


# ----------------------------------------------- T3 degenerate budget
def _sdpa(q, keys, values, sm):
    qt = torch.tensor(q, dtype=torch.float64)[None, :, None, :]  # [1, G, 1, d]
    kt = torch.tensor(keys, dtype=torch.float64)[None, None].expand(1, q.shape[0], -1, -1)
    vt = torch.tensor(values, dtype=torch.float64)[None, None].expand(1, q.shape[0], -1, -1)
    return torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, scale=sm)[0, :, 0].numpy()


def _hand_loop_attention(q, keys, values, sm):
    out = np.zeros((q.shape[0], values.shape[1]))
    for h in range(q.shape[0]):
        logits = [sm * float(np.dot(q[h], keys[j])) for j in range(keys.shape[0])]
        mx = max(logits)
        w = [np.exp(x - mx) for x in logits]
        z = sum(w)
        for j in range(keys.shape[0]):
            out[h] += w[j] / z * values[j]
    return out


@pytest.mark.parametrize("layout,G,d_k,d_v", [("mha", 1, 32, 32), ("gqa", 4, 64, 64), ("mla", 8, 72, 64)])
def test_degenerate_budget_equals_dense_attention(layout, G, d_k, d_v):
    """K_b >= m and K_t >= n -> the whole pipeline is dense attention,
    checked against torch's fp64 SDPA and a hand loop, over 50 seeds."""
    for seed in range(50):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(1, 200))
        keys = rng.standard_normal((n, d_k)).astype(np.float32)
        values = keys[:, :d_v] if layout == "mla" else rng.standard_normal((n, d_v))
        q = rng.standard_normal((G, d_k))
        ch = np.sort(rng.choice(d_k, 8, replace=False))
        p = O.TLSParams(block_size=16, top_blocks=10**6, top_tokens=10**6, sm_scale=1 / np.sqrt(d_k))
        r = O.tls_pair(q, keys, values, ch, p)
        np.testing.assert_array_equal(r["token_ids"], np.arange(n))
        ref = _sdpa(q, keys, values, p.sm_scale)
        np.testing.assert_allclose(r["out"], ref, rtol=0, atol=1e-12)
        if seed < 5:
            np.testing.assert_allclose(r["out"], _hand_loop_attention(q, keys, values, p.sm_scale), atol=1e-12)
        lse_ref = np.log(np.exp(q @ keys.astype(np.float64).T * p.sm_scale).sum(1))
        np.testing.assert_allclose(r["lse"], lse_ref, rtol=1e-12)


def test_sparse_attention_equals_gather_then_sdpa():
    rng = np.random.default_rng(12)
    keys = rng.standard_normal((512, 32))
    values = rng.standard_normal((512, 16))
    q = rng.standard_normal((4, 32))
    ids = np.sort(rng.choice(512, 64, replace=False))
    out, _ = O.sparse_attention(q, keys, values, ids, 0.2)
    np.testing.assert_allclose(out, _sdpa(q, keys[ids], values[ids], 0.2), atol=1e-12)


# -------------------------------------------------------- T8 invariants
def test_attention_convexity_and_permutation_equivariance():
    rng = np.random.default_rng(13)
    keys = rng.standard_normal((300, 16))
    values = rng.standard_normal((300, 8))
    q = rng.standard_normal((2, 16))
    ids = np.sort(rng.choice(300, 50, replace=False))
    out, lse = O.sparse_attention(q, keys, values, ids, 0.3)
    lo, hi = values[ids].min(0), values[ids].max(0)
    assert np.all(out >= lo - 1e-12) and np.all(out <= hi + 1e-12)
    perm = rng.permutation(300)
    inv = np.argsort(perm)
    out2, lse2 = O.sparse_attention(q, keys[perm], values[perm], inv[ids], 0.3)
    np.testing.assert_allclose(out2, out, atol=1e-13)
    np.testing.assert_allclose(lse2, lse, atol=1e-13)


# --------------------------------------------- T9 MLA absorption
def test_mla_absorbed_equals_explicit_multihead():
    """Absorbed MLA (one shared latent KV head: K row = [c_j; k_rope_j],
    V row = c_j = K[:, :d_v], q_abs_h = [W_UK_h^T q_nope_h; q_rope_h]) followed
    by W_UV_h equals explicit per-head MLA with up-projected K/V."""
    rng = np.random.default_rng(14)
    H, d_lat, d_rope, d_nope, d_vh, n = 4, 32, 8, 16, 12, 90
    c = rng.standard_normal((n, d_lat))
    kr = rng.standard_normal((n, d_rope))
    W_UK = rng.standard_normal((H, d_nope, d_lat)) / np.sqrt(d_lat)
    W_UV = rng.standard_normal((H, d_vh, d_lat)) / np.sqrt(d_lat)
    q_nope = rng.standard_normal((H, d_nope))
    q_rope = rng.standard_normal((H, d_rope))
    sm = 1 / np.sqrt(d_nope + d_rope)
    # explicit
    ref = np.zeros((H, d_vh))
    for h in range(H):
        k_h = np.concatenate([c @ W_UK[h].T, kr], axis=1)  # [n, d_nope + d_rope]
        v_h = c @ W_UV[h].T
        ref[h] = _sdpa(np.concatenate([q_nope[h], q_rope[h]])[None], k_h, v_h, sm)[0]
    # absorbed, through the oracle's MLA layout (V = first d_lat dims of K)
    K = np.concatenate([c, kr], axis=1)
    q_abs = np.stack([np.concatenate([W_UK[h].T @ q_nope[h], q_rope[h]]) for h in range(H)])
    o_lat, _ = O.dense_attention(q_abs, K, K[:, :d_lat], sm)
    out = np.stack([W_UV[h] @ o_lat[h] for h in range(H)])
    np.testing.assert_allclose(out, ref, atol=1e-12)


# ------------------------------------------------------ calibration scan
def test_calibration_matches_scan():
    rng = np.random.default_rng(15)
    for _ in range(10):
        S, G, d, d_c = 20, 3, 24, 5
        qc = rng.standard_normal((S, G, d))
        kc = rng.standard_normal((30, d))
        ch, s = O.calibrate_channels(qc, kc, d_c)
        ref = np.zeros(d)
        for i in range(d):
            km = max(abs(kc[j, i]) for j in range(30))
            ref[i] = sum(max(abs(qc[t, h, i]) for t in range(S)) * km for h in range(G)) / G
        np.testing.assert_allclose(s, ref, rtol=1e-15)
        assert _is_valid_topk(ref, d_c, list(ch))


def test_errors():
    with pytest.raises(ValueError):
        O.calibrate_channels(np.zeros((1, 1, 4)), np.zeros((1, 4)), 5)
    with pytest.raises(ValueError):
        O.sparse_attention(np.zeros((1, 4)), np.zeros((3, 4)), np.zeros((3, 4)), [], 1.0)
    with pytest.raises(ValueError):
        O.approx_scores(np.zeros((1, 4)), [0], np.zeros((3, 1), np.uint8), np.zeros(3, np.float32), np.zeros(3, np.float32), [], 1.0)
    with pytest.raises(ValueError):
        O.block_ranges(0, 4)
