"""Plain fp64 CPU oracle of AsyncTLS two-level sparse decode attention.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this module.  The product path (``paper_2604_07815_b200``) never imports,
links or executes anything under ``oracle/``, and this module imports nothing
from the product: the two share no code.

Citation key: ``P:n`` = line n of the paper text (``PAPER.md``, LaTeX source of
arXiv 2604.07815); ``S:n`` = line n of ``SPEC.md`` (used for test ideas and the
readings listed in DESIGN.md §3 only).

The oracle follows the paper step by step, one
(batch element, KV-head group) *pair* at a time, with these plain definitions:

* block scores use the paper's *direct* Quest form, not the GEMM form;
* top-k is a full stable sort by (-score, index)  (tie rule: lower index, U2);
* softmax is single pass, max-subtracted, fp64.

Every floating-point step is fp64 except the INT4 quantiser (O5), which is
*defined* in IEEE fp32 (reading U8/U9 in DESIGN.md) so that integer codes are
a well-defined function of the stored keys.

Readings of the paper taken here (all listed in DESIGN.md §3):
  U1  m = ceil(n/B) blocks, last block partial (P:95 writes floor).
  U2  ties in every top-k -> lower index first.
  U3  selections are returned as ascending ids.
  U4  k larger than the candidate count -> select all.
  U5  one channel set C per KV head, passed in.
  U8  INT4 = per-token asymmetric min/max over the d_c channels, fp32 scale/zero.
  U10 alpha-tilde uses the same 1/sqrt(d) (full head dim) as the attention.
  U11 alpha-tilde softmax runs over the candidate tokens only.
  U12 MLA: one shared latent KV head, V = first d_v dims of each K row.
  U13 synchronous operator: candidates are this step's M_t unless a guide
      block set (M_{t-1}) is passed explicitly.

Pins (tests/test_oracle_pins.py): every function here is checked against
something other than itself -- the paper's GEMM identity, brute
force on tiny inputs, dense attention via torch's fp64 SDPA and a hand loop,
closed-form hand cases (tests/golden/hand_cases.json), the quantiser's error
bound, and the absorbed-vs-explicit MLA identity.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "TLSParams",
    "block_ranges",
    "block_summaries",
    "block_scores",
    "block_scores_gemm_form",
    "topk_ids",
    "select_blocks",
    "calibrate_channels",
    "quantize_keys",
    "dequantize",
    "candidate_tokens",
    "approx_scores",
    "select_tokens",
    "sparse_attention",
    "dense_attention",
    "build_index_pair",
    "tls_pair",
    "tls_batch",
]


@dataclass(frozen=True)
class TLSParams:
    """Hyper-parameters of the method (P:397 defaults for the GPU configs)."""

    block_size: int = 64  # B
    top_blocks: int = 128  # k_b
    top_tokens: int = 1024  # k_t (512 / 1024 / 2048)
    sm_scale: float = 1.0 / np.sqrt(128.0)  # 1/sqrt(d) (U10)


# --------------------------------------------------------------------------
# O1-O4: coarse-grained block selection
# --------------------------------------------------------------------------
def block_ranges(n: int, block_size: int) -> list[tuple[int, int]]:
    """O1 (reading U1): token ranges of the m = ceil(n/B) blocks."""
    if n < 1 or block_size < 1:
        raise ValueError("n and block_size must be >= 1")
    m = (n + block_size - 1) // block_size
    return [(i * block_size, min((i + 1) * block_size, n)) for i in range(m)]


def block_summaries(keys: np.ndarray, block_size: int) -> tuple[np.ndarray, np.ndarray]:
    """O2: k_max[i,c] = max_{j in B_i} k[j,c], k_min likewise.

    ``keys`` is [n, d]; returns (k_max, k_min), each [m, d] fp64.
    """
    keys = np.asarray(keys, dtype=np.float64)
    ranges = block_ranges(keys.shape[0], block_size)
    kmax = np.empty((len(ranges), keys.shape[1]))
    kmin = np.empty((len(ranges), keys.shape[1]))
    for i, (s, e) in enumerate(ranges):
        kmax[i] = keys[s:e].max(axis=0)
        kmin[i] = keys[s:e].min(axis=0)
    return kmax, kmin


def block_scores(q: np.ndarray, kmax: np.ndarray, kmin: np.ndarray) -> np.ndarray:
    """O3 (direct Quest form):

        s_i = sum_{h<G} sum_{k<d} max(q[h,k] * kmax[i,k], q[h,k] * kmin[i,k])

    ``q`` is the [G, d] query group sharing one KV head.
    """
    q = np.asarray(q, dtype=np.float64)
    kmax = np.asarray(kmax, dtype=np.float64)
    kmin = np.asarray(kmin, dtype=np.float64)
    s = np.zeros(kmax.shape[0])
    for h in range(q.shape[0]):
        a = q[h][None, :] * kmax  # [m, d]
        b = q[h][None, :] * kmin
        s += np.maximum(a, b).sum(axis=1)
    return s


def block_scores_gemm_form(q: np.ndarray, kmax: np.ndarray, kmin: np.ndarray) -> np.ndarray:
    """The paper's GEMM reformulation, kept only as a pin of O3:

        q^max = max(q, 0), q^min = min(q, 0)
        s = sum_h (Q^max^T K^max + Q^min^T K^min)_h
    """
    q = np.asarray(q, dtype=np.float64)
    qmax = np.maximum(q, 0.0)  # [G, d]
    qmin = np.minimum(q, 0.0)
    per_head = qmax @ np.asarray(kmax, np.float64).T + qmin @ np.asarray(kmin, np.float64).T
    return per_head.sum(axis=0)


def topk_ids(scores: np.ndarray, k: int) -> np.ndarray:
    """O4/O10 (U2-U4): the k largest scores, ties -> lower index.

    Full stable sort by (-score, index); returns the chosen ids ascending.
    k >= len(scores) selects everything.
    """
    scores = np.asarray(scores, dtype=np.float64)
    if k < 0:
        raise ValueError("k must be >= 0")
    idx = np.arange(scores.shape[0])
    order = np.lexsort((idx, -scores))  # primary key: -score, secondary: index
    return np.sort(order[: min(k, scores.shape[0])]).astype(np.int64)


def select_blocks(q, kmax, kmin, top_blocks: int) -> tuple[np.ndarray, np.ndarray]:
    """O3+O4: M_t = top-k_b blocks by s_i. Returns (ids asc, all scores)."""
    s = block_scores(q, kmax, kmin)
    return topk_ids(s, top_blocks), s


# --------------------------------------------------------------------------
# Channel calibration
# --------------------------------------------------------------------------
def calibrate_channels(q_cal: np.ndarray, k_cal: np.ndarray, d_c: int) -> tuple[np.ndarray, np.ndarray]:
    """s_i = (1/G) sum_h (max_D |q_h[i]|) * (max_D |k[i]|); top-d_c -> C.

    ``q_cal`` is [S, G, d] (S calibration queries of the G heads of one KV
    head), ``k_cal`` is [S', d].  Returns (C ascending, channel scores).
    Ties -> lower channel id (reading U5).
    """
    q_cal = np.asarray(q_cal, dtype=np.float64)
    k_cal = np.asarray(k_cal, dtype=np.float64)
    d = k_cal.shape[-1]
    if d_c > d or d_c < 1:
        raise ValueError("d_c must be in [1, d]")
    if q_cal.shape[0] == 0 or k_cal.shape[0] == 0:
        raise ValueError("empty calibration set")
    G = q_cal.shape[1]
    qmax = np.abs(q_cal).max(axis=0)  # [G, d]
    kmax = np.abs(k_cal).max(axis=0)  # [d]
    s = np.zeros(d)
    for h in range(G):
        s += qmax[h] * kmax
    s /= G
    return topk_ids(s, d_c), s


# --------------------------------------------------------------------------
# O5: token index -- channel projection + INT4 quantisation
# --------------------------------------------------------------------------
_F32 = np.float32


def quantize_keys(k_sel: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """O5 ("Quantize", "INT4"; readings U8, U9).

    ``k_sel`` is [n, d_c]: the keys restricted to the channel set C, holding
    the stored key values exactly (bf16 or fp32 inputs are exact in fp32).
    Per token row x (IEEE fp32 arithmetic, round-to-nearest-even, no FMA):

        zero  = min_c x_c
        scale = fp32( fp32(max_c x_c - zero) / 15 )
        code_c = scale > 0 ? clamp(rint_half_even(fp32(fp32(x_c - zero) / scale)), 0, 15) : 0

    Returns (codes uint8 [n, d_c], scale fp32 [n], zero fp32 [n]).
    """
    x = np.asarray(k_sel, dtype=_F32)
    if not np.array_equal(x.astype(np.float64), np.asarray(k_sel, dtype=np.float64)):
        raise ValueError("quantize_keys expects values exactly representable in fp32")
    zero = x.min(axis=1)  # fp32
    mx = x.max(axis=1)
    scale = (mx - zero) / _F32(15.0)  # fp32 subtract, then fp32 divide
    assert scale.dtype == _F32 and zero.dtype == _F32
    codes = np.zeros(x.shape, dtype=np.uint8)
    pos = scale > _F32(0.0)
    t = (x[pos] - zero[pos][:, None]) / scale[pos][:, None]  # fp32 ops, elementwise
    assert t.dtype == _F32
    codes[pos] = np.clip(np.rint(t), 0, 15).astype(np.uint8)  # rint = half-to-even
    return codes, scale, zero


def dequantize(codes: np.ndarray, scale: np.ndarray, zero: np.ndarray) -> np.ndarray:
    """k~ = zero + scale * code, evaluated in fp64 (exact for fp32 scale/zero)."""
    return np.asarray(zero, np.float64)[:, None] + np.asarray(scale, np.float64)[:, None] * np.asarray(
        codes, np.float64
    )


def build_index_pair(keys: np.ndarray, channels: np.ndarray, block_size: int) -> dict:
    """a0 for one KV head: block summaries (O2) and the token index (O5)."""
    kmax, kmin = block_summaries(keys, block_size)
    codes, scale, zero = quantize_keys(np.asarray(keys)[:, np.asarray(channels)])
    return {"kmax": kmax, "kmin": kmin, "codes": codes, "scale": scale, "zero": zero}


# --------------------------------------------------------------------------
# O6-O10: fine-grained token selection
# --------------------------------------------------------------------------
def candidate_tokens(block_ids: np.ndarray, n: int, block_size: int) -> np.ndarray:
    """O6: J = union of the token ranges of the selected blocks, ascending."""
    ranges = block_ranges(n, block_size)
    out = []
    for i in sorted(int(b) for b in block_ids if b >= 0):
        s, e = ranges[i]
        out.extend(range(s, e))
    return np.asarray(out, dtype=np.int64)


def approx_scores(
    q: np.ndarray,
    channels: np.ndarray,
    codes: np.ndarray,
    scale: np.ndarray,
    zero: np.ndarray,
    cand: np.ndarray,
    sm_scale: float,
) -> np.ndarray:
    """O7-O9:

        q~^(h) = q^(h)[C];  k~_j = zero_j + scale_j * code_j
        l[h, j] = q~^(h) . k~_j * sm_scale                     (O7)
        p[h, :] = softmax over the candidates j in J            (O8, U11)
        alpha~_j = (1/G) sum_h p[h, j]                          (O9)
    """
    if len(cand) == 0:
        raise ValueError("empty candidate set")
    q = np.asarray(q, dtype=np.float64)
    qt = q[:, np.asarray(channels)]  # [G, d_c]
    kt = dequantize(codes[cand], scale[cand], zero[cand])  # [|J|, d_c]
    logits = (qt @ kt.T) * sm_scale  # [G, |J|]
    logits = logits - logits.max(axis=1, keepdims=True)
    p = np.exp(logits)
    p /= p.sum(axis=1, keepdims=True)
    return p.mean(axis=0)


def select_tokens(alpha: np.ndarray, cand: np.ndarray, top_tokens: int) -> np.ndarray:
    """O10: S_t = TopK_{k_t}(alpha~ over J); ties -> lower token id."""
    pos = topk_ids(alpha, top_tokens)  # positions in the ascending candidate list
    return np.asarray(cand, dtype=np.int64)[pos]


# --------------------------------------------------------------------------
# O11: sparse attention over the selected tokens
# --------------------------------------------------------------------------
def sparse_attention(q, keys, values, ids, sm_scale: float) -> tuple[np.ndarray, np.ndarray]:
    """O11: o^(h) = softmax(q^(h) K_S^T * sm_scale) V_S, plus lse^(h).

    ``q`` [G, d_k], ``keys`` [n, d_k], ``values`` [n, d_v], ``ids`` the index
    set S.  Returns (out [G, d_v], lse [G]) with lse = log sum_j exp(logit_j).
    """
    ids = np.asarray(ids, dtype=np.int64)
    if ids.size == 0:
        raise ValueError("empty selection")
    q = np.asarray(q, dtype=np.float64)
    ks = np.asarray(keys, dtype=np.float64)[ids]
    vs = np.asarray(values, dtype=np.float64)[ids]
    logits = (q @ ks.T) * sm_scale  # [G, |S|]
    mx = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - mx)
    z = e.sum(axis=1, keepdims=True)
    out = (e / z) @ vs
    lse = (mx + np.log(z))[:, 0]
    return out, lse


def dense_attention(q, keys, values, sm_scale: float) -> tuple[np.ndarray, np.ndarray]:
    """P:66-69 scaled dot-product attention over all n cached tokens."""
    return sparse_attention(q, keys, values, np.arange(np.asarray(keys).shape[0]), sm_scale)


# --------------------------------------------------------------------------
# The whole per-pair pipeline and the batch driver
# --------------------------------------------------------------------------
def tls_pair(
    q: np.ndarray,
    keys: np.ndarray,
    values: np.ndarray,
    channels: np.ndarray,
    params: TLSParams,
    guide_block_ids: np.ndarray | None = None,
    index: dict | None = None,
) -> dict:
    """One decode step of one (batch element, KV head) pair, O0-O11.

    ``q`` [G, d_k] (the G query heads of the group), ``keys`` [n, d_k] and
    ``values`` [n, d_v] hold the n valid tokens.  ``guide_block_ids`` (lag
    mode) replaces this step's M_t as the candidate blocks.
    """
    n = np.asarray(keys).shape[0]
    B = params.block_size
    if index is None:
        index = build_index_pair(keys, channels, B)
    block_ids, s = select_blocks(q, index["kmax"], index["kmin"], params.top_blocks)
    guide = block_ids if guide_block_ids is None else np.sort(np.asarray(guide_block_ids)[np.asarray(guide_block_ids) >= 0])
    cand = candidate_tokens(guide, n, B)
    alpha = approx_scores(q, channels, index["codes"], index["scale"], index["zero"], cand, params.sm_scale)
    token_ids = select_tokens(alpha, cand, params.top_tokens)
    out, lse = sparse_attention(q, keys, values, token_ids, params.sm_scale)
    return {
        "block_scores": s,
        "block_ids": block_ids,
        "candidates": cand,
        "alpha": alpha,
        "token_ids": token_ids,
        "token_alpha": alpha[np.searchsorted(cand, token_ids)],
        "out": out,
        "lse": lse,
    }


def tls_batch(
    q: np.ndarray,
    k_cache: np.ndarray,
    v_cache: np.ndarray | None,
    seq_lens: np.ndarray,
    channels: np.ndarray,
    params: TLSParams,
    layout: str = "gqa",
    d_v: int | None = None,
    pairs: list[tuple[int, int]] | None = None,
) -> dict:
    """Driver over pairs for batch tensors (layouts of DESIGN.md §4).

    GQA: q [Bt, Hq, d], k_cache/v_cache [Bt, Hkv, S, d]; query head h belongs
    to KV group h // G (G = Hq / Hkv).  MLA (U12): k_cache [Bt, S, d_k]
    with one shared latent head, V = K[..., :d_v], q [Bt, H, d_k], G = H.
    ``channels`` is [Hkv, d_c].  ``pairs`` restricts the run to a sample.
    """
    q = np.asarray(q)
    Bt, Hq = q.shape[0], q.shape[1]
    if layout == "mla":
        Hkv = 1
    else:
        Hkv = k_cache.shape[1]
    G = Hq // Hkv
    if pairs is None:
        pairs = [(b, g) for b in range(Bt) for g in range(Hkv)]
    res = {}
    for b, g in pairs:
        n = int(seq_lens[b])
        if layout == "mla":
            keys = k_cache[b, :n]
            values = keys[:, :d_v]
        else:
            keys = k_cache[b, g, :n]
            values = v_cache[b, g, :n]
        res[(b, g)] = tls_pair(q[b, g * G : (g + 1) * G], keys, values, channels[g], params)
    return res
