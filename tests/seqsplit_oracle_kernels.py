"""Test infrastructure: the calls of paper_2604_07815_b200.seqsplit.decode_step (include/tls.h semantics of
tls_block_scores, tls_block_topk, tls_topk_rows, tls_select_range, tls_token_stats, tls_token_keys,
tls_sparse_attend, tls_attn_merge) evaluated in fp64 with the oracle's functions, on CPU tensors.  Lets the
sequence-split orchestration -- ranges, collectives, merges -- be checked on CPU (gloo) against the oracle's
unsplit decode; the CUDA kernels themselves are checked by tests/test_gpu_seqsplit.py."""
from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

import numpy as np
import torch

from oracle import tls_oracle as O

LOG2E = 1.0 / math.log(2.0)


@dataclass
class OracleIndex:
    keys: np.ndarray  # [batch, Hkv, L, d_k] fp64: the rank's local keys
    channels: np.ndarray  # [Hkv, d_c]


def _group(cfg, q, b, g):
    G = cfg.num_q_heads // cfg.num_kv_heads
    return q[b, g * G:(g + 1) * G].double().numpy()


def _pad(vals, ids, k, fill_key=-np.inf):
    ok = np.full(k, fill_key)
    oi = np.full(k, -1, dtype=np.int64)
    ok[: len(vals)] = vals
    oi[: len(ids)] = ids
    return ok, oi


def _logits2(cfg, index, q, b, g, blocks, n):
    """Candidates of the local blocks below n and their logits in log2 units [G, |J|] (O5, O7)."""
    B = cfg.block_size
    ch = index.channels[g]
    keys = index.keys[b, g, :n]
    cand = O.candidate_tokens(np.asarray([x for x in blocks if x >= 0], dtype=np.int64), n, B) if n > 0 else \
        np.zeros(0, np.int64)
    if len(cand) == 0:
        return cand, np.zeros((cfg.num_q_heads // cfg.num_kv_heads, 0))
    codes, scale, zero = O.quantize_keys(keys[:, ch])
    kt = O.dequantize(codes[cand], scale[cand], zero[cand])
    qt = _group(cfg, q, b, g)[:, ch]
    return cand, (qt @ kt.T) * cfg.sm_scale * LOG2E


class OracleKernels:
    @staticmethod
    def block_scores(cfg, q, lens, index):
        M = cfg.num_blocks
        out = torch.full((cfg.batch, cfg.num_kv_heads, M), float("nan"), dtype=torch.float64)
        for b in range(cfg.batch):
            n = int(lens[b])
            if n == 0:
                continue
            for g in range(cfg.num_kv_heads):
                kmax, kmin = O.block_summaries(index.keys[b, g, :n], cfg.block_size)
                s = O.block_scores(_group(cfg, q, b, g), kmax, kmin)
                out[b, g, : len(s)] = torch.from_numpy(s)
        return out

    @staticmethod
    def block_topk(cfg, scores, lens, blk0):
        k = cfg.top_blocks
        ok = torch.empty((cfg.batch, cfg.num_kv_heads, k), dtype=torch.float64)
        oi = torch.empty((cfg.batch, cfg.num_kv_heads, k), dtype=torch.int64)
        for b in range(cfg.batch):
            m = -(-int(lens[b]) // cfg.block_size)
            for g in range(cfg.num_kv_heads):
                s = scores[b, g, :m].numpy()
                sel = O.topk_ids(s, k) if m > 0 else np.zeros(0, np.int64)
                a, c = _pad(s[sel], sel + blk0, k)
                ok[b, g], oi[b, g] = torch.from_numpy(a), torch.from_numpy(c)
        return ok, oi

    @staticmethod
    def topk_rows(keys, ids, k):
        shp = keys.shape[:-1]
        kk = keys.reshape(-1, keys.shape[-1]).numpy()
        ii = ids.reshape(-1, ids.shape[-1]).numpy()
        ok = np.empty((kk.shape[0], k))
        oi = np.empty((kk.shape[0], k), dtype=np.int64)
        cnt = np.empty(kk.shape[0], dtype=np.int64)
        for r in range(kk.shape[0]):
            v = ii[r] >= 0
            vk, vi = kk[r][v], ii[r][v]
            order = np.lexsort((vi, -vk))[:k]  # larger key first, equal keys -> lower id (U2)
            sel = np.sort(order)  # vi is ascending: position order = id order
            ok[r], oi[r] = _pad(vk[sel], vi[sel], k)
            cnt[r] = len(sel)
        return (torch.from_numpy(ok).reshape(*shp, k), torch.from_numpy(oi).reshape(*shp, k),
                torch.from_numpy(cnt).reshape(shp))

    @staticmethod
    def select_range(ids, lo, hi):
        k = ids.shape[-1]
        flat = ids.reshape(-1, k).numpy()
        out = np.full_like(flat, -1)
        cnt = np.zeros(flat.shape[0], dtype=np.int64)
        for r in range(flat.shape[0]):
            sel = flat[r][(flat[r] >= lo) & (flat[r] < hi)] - lo
            out[r, : len(sel)] = sel
            cnt[r] = len(sel)
        return torch.from_numpy(out).reshape(ids.shape), torch.from_numpy(cnt).reshape(ids.shape[:-1])

    @staticmethod
    def token_stats(cfg, q, lens, index, blocks):
        G = cfg.num_q_heads // cfg.num_kv_heads
        st = torch.empty((cfg.batch, cfg.num_kv_heads, G, 2), dtype=torch.float64)
        for b in range(cfg.batch):
            for g in range(cfg.num_kv_heads):
                _, L = _logits2(cfg, index, q, b, g, blocks[b, g].numpy(), int(lens[b]))
                for h in range(G):
                    if L.shape[1] == 0:
                        st[b, g, h] = torch.tensor([-np.inf, 0.0])
                    else:
                        M = L[h].max()
                        st[b, g, h] = torch.tensor([M, np.exp2(L[h] - M).sum()])
        return st

    @staticmethod
    def token_keys(cfg, q, lens, index, blocks, stats_parts, t0):
        G = cfg.num_q_heads // cfg.num_kv_heads
        n_out = cfg.top_blocks * cfg.block_size
        keys = torch.full((cfg.batch, cfg.num_kv_heads, n_out), -np.inf, dtype=torch.float64)
        ids = torch.full((cfg.batch, cfg.num_kv_heads, n_out), -1, dtype=torch.int64)
        sp = stats_parts.numpy()
        for b in range(cfg.batch):
            for g in range(cfg.num_kv_heads):
                lz = np.empty(G)
                for h in range(G):
                    ms, zs = sp[:, b, g, h, 0], sp[:, b, g, h, 1]
                    M = ms.max()
                    lz[h] = M + np.log2(sum(z * np.exp2(m - M) for m, z in zip(ms, zs) if m > -np.inf))
                cand, L = _logits2(cfg, index, q, b, g, blocks[b, g].numpy(), int(lens[b]))
                if len(cand) == 0:
                    continue
                alpha = np.exp2(L - lz[:, None]).mean(axis=0)
                keys[b, g, : len(cand)] = torch.from_numpy(np.log(alpha))
                ids[b, g, : len(cand)] = torch.from_numpy(cand + t0)
        return keys, ids

    @staticmethod
    def sparse_attend(cfg, q, k_cache, v_cache, ids, n, out_f32=True):
        G = cfg.num_q_heads // cfg.num_kv_heads
        out = torch.zeros((cfg.batch, cfg.num_q_heads, cfg.d_v), dtype=torch.float64)
        lse = torch.full((cfg.batch, cfg.num_q_heads), -np.inf, dtype=torch.float64)
        for b in range(cfg.batch):
            for g in range(cfg.num_kv_heads):
                c = int(n[b, g])
                if c == 0:
                    continue
                o, l = O.sparse_attention(_group(cfg, q, b, g), k_cache[b, g].double().numpy(),
                                          v_cache[b, g].double().numpy(), ids[b, g, :c].numpy(), cfg.sm_scale)
                out[b, g * G:(g + 1) * G] = torch.from_numpy(o)
                lse[b, g * G:(g + 1) * G] = torch.from_numpy(l)
        return out, lse

    @staticmethod
    def attn_merge(cfg, parts_out, parts_lse):
        lp = parts_lse.numpy()
        M = lp.max(axis=0)
        w = np.where(np.isfinite(lp), np.exp(lp - M), 0.0)
        tot = M + np.log(w.sum(axis=0))
        wn = np.where(np.isfinite(lp), np.exp(lp - tot), 0.0)
        out = (wn[..., None] * parts_out.numpy()).sum(axis=0)
        return torch.from_numpy(out), torch.from_numpy(tot)


def rank_state(cfg_full, inputs, channels, t0, L):
    """A rank's RankState for the oracle kernels: its slice of the caches (fp64) and a local config."""
    from paper_2604_07815_b200 import seqsplit as SS

    cfg = dataclasses.replace(cfg_full, max_seq_len=L)
    kc = inputs["k_cache"][:, :, t0:t0 + L].double()
    vc = inputs["v_cache"][:, :, t0:t0 + L].double()
    return SS.RankState(cfg=cfg, index=OracleIndex(keys=kc.numpy(), channels=np.asarray(channels)), k_cache=kc,
                        v_cache=vc, t0=t0)
