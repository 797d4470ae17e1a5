"""Torch-tensor front end of libtls.so -- the same names as the C ABI.

PyTorch provides device memory and streams only: every step of the path runs
in the CUDA kernels behind include/tls.h.  Each function checks shapes,
dtypes, devices and contiguity, passes ``data_ptr()`` and the current CUDA
stream, and raises ``TLSError`` on a non-OK status.

Citation key: P:n = line n of PAPER.md (arXiv 2604.07815).
"""
from __future__ import annotations

import ctypes
import os
import math
from dataclasses import dataclass, field

import torch

from . import _lib

__all__ = [
    "TLSConfig",
    "TLSIndex",
    "alloc_index",
    "calibrate_channels",
    "build_index",
    "block_scores",
    "select",
    "sparse_attend",
    "decode",
    "cluster_size",
    "select_mode",
    "kernel_names",
    "KERNELS",
    "timing_enable",
    "TLSTokenCache",
    "alloc_token_cache",
    "host_kv",
    "cache_fetch",
    "offload_decode",
    "timing_read",
    "quest_decode",
    "ds_decode",
]

_DT = {torch.bfloat16: _lib.TLS_BF16, torch.float32: _lib.TLS_FP32}


@dataclass
class TLSConfig:
    """Mirror of ``tls_config`` (include/tls.h).  Defaults follow P:397."""

    batch: int
    num_q_heads: int
    num_kv_heads: int
    d_k: int
    d_v: int
    max_seq_len: int
    block_size: int = 64  # B
    d_c: int = 32  # token-index channels (32 GQA / 128 MLA)
    top_blocks: int = 128  # k_b
    top_tokens: int = 1024  # k_t
    sm_scale: float | None = None  # default 1/sqrt(d_k)
    dtype: torch.dtype = torch.bfloat16
    layout: str = "gqa"  # "gqa" | "mla"
    _c: _lib.TLSConfigC = field(default=None, init=False, repr=False)

    def __post_init__(self):
        if self.sm_scale is None:
            self.sm_scale = 1.0 / math.sqrt(self.d_k)

    @property
    def G(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def num_blocks(self) -> int:
        return (self.max_seq_len + self.block_size - 1) // self.block_size

    @property
    def pairs(self) -> int:
        return self.batch * self.num_kv_heads

    def c(self) -> _lib.TLSConfigC:
        if self.dtype not in _DT:
            raise TypeError(f"dtype must be bf16 or fp32, got {self.dtype}")
        return _lib.TLSConfigC(
            self.batch, self.num_q_heads, self.num_kv_heads, self.d_k, self.d_v, self.max_seq_len, self.block_size,
            self.d_c, self.top_blocks, self.top_tokens, float(self.sm_scale), _DT[self.dtype],
            _lib.TLS_MLA if self.layout == "mla" else _lib.TLS_GQA,
        )


@dataclass
class TLSIndex:
    """The hierarchical index of one KV cache (Fig. 2), device tensors."""

    block_minmax: torch.Tensor  # [batch, Hkv, M, 2, d_k] dtype (k^max, k^min)
    codes: torch.Tensor  # [batch, Hkv, S, d_c/2] uint8 INT4 codes
    scale_zero: torch.Tensor  # [batch, Hkv, S, 2] fp32
    channels: torch.Tensor  # [Hkv, d_c] int32 ascending channel set C

    def c(self) -> _lib.TLSIndexC:
        return _lib.TLSIndexC(self.block_minmax.data_ptr(), self.codes.data_ptr(), self.scale_zero.data_ptr(),
                              self.channels.data_ptr())


_WS: dict = {}


def _workspace(cfg: TLSConfig, dev: torch.device, which: int):
    """Device workspace for tls_select / tls_decode (cached per device and size)."""
    cc = cfg.c()
    nbytes = int(_lib.load().tls_workspace_bytes(ctypes.byref(cc), which))
    if nbytes == ctypes.c_size_t(-1).value or nbytes == 0:  # invalid config: the op call reports why
        return None, 0
    # one zero-filled buffer per (device, stream, configuration): the pair completion words of
    # select_kernel carry state from call to call (tls_workspace_bytes in include/tls.h)
    # (the tuning variables that change the workspace layout -- sub-batch pipeline depth, attention split,
    # the persistent step kernel -- are part of the key: a workspace is only reused with its own layout)
    key = (dev, torch.cuda.current_stream(dev).cuda_stream, bytes(cc), which, nbytes,
           tuple(os.environ.get(v) for v in ("TLS_NSPLIT", "TLS_CLUSTER", "TLS_PSTEP", "TLS_TILE_KB", "TLS_STREAM_SEL")))
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        _lib.check(_lib.load().tls_workspace_init(ctypes.byref(cc), which, buf.data_ptr(), nbytes,
                                                  torch.cuda.current_stream(dev).cuda_stream))
        _WS[key] = buf
    return buf.data_ptr(), nbytes


def _stream(dev: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _need(t: torch.Tensor, name: str, shape: tuple, dtype: torch.dtype, dev: torch.device) -> None:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a tensor")
    if t.device != dev or t.device.type != "cuda":
        raise ValueError(f"{name} must live on {dev} (CUDA); got {t.device}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _kv_shape(cfg: TLSConfig, width: int) -> tuple:
    if cfg.layout == "mla":
        return (cfg.batch, cfg.max_seq_len, width)
    return (cfg.batch, cfg.num_kv_heads, cfg.max_seq_len, width)


def alloc_index(cfg: TLSConfig, channels: torch.Tensor) -> TLSIndex:
    """Allocate the index buffers for ``cfg`` on the device of ``channels``."""
    dev = channels.device
    _need(channels, "channels", (cfg.num_kv_heads, cfg.d_c), torch.int32, dev)
    return TLSIndex(
        block_minmax=torch.empty((cfg.batch, cfg.num_kv_heads, cfg.num_blocks, 2, cfg.d_k), dtype=cfg.dtype, device=dev),
        codes=torch.empty((cfg.batch, cfg.num_kv_heads, cfg.max_seq_len, cfg.d_c // 2), dtype=torch.uint8, device=dev),
        scale_zero=torch.empty((cfg.batch, cfg.num_kv_heads, cfg.max_seq_len, 2), dtype=torch.float32, device=dev),
        channels=channels,
    )


def calibrate_channels(cfg: TLSConfig, q_cal: torch.Tensor, k_cal: torch.Tensor, k_head_stride: int | None = None):
    """Channel set C per KV head on the GPU.

    ``q_cal`` [n_q, Hq, d_k]; ``k_cal`` holds n_k rows of d_k per KV head, head g
    starting ``k_head_stride`` elements after head g-1 (default: a contiguous
    [Hkv, n_k, d_k] tensor).  Returns (channels [Hkv, d_c] int32, scores [Hkv, d_k] fp32).
    """
    lib = _lib.load()
    dev = q_cal.device
    n_q = q_cal.shape[0]
    _need(q_cal, "q_cal", (n_q, cfg.num_q_heads, cfg.d_k), cfg.dtype, dev)
    if k_head_stride is None:
        n_k = k_cal.shape[1]
        _need(k_cal, "k_cal", (cfg.num_kv_heads, n_k, cfg.d_k), cfg.dtype, dev)
        k_head_stride = n_k * cfg.d_k
    else:
        n_k = k_cal.shape[-2]
    ch = torch.empty((cfg.num_kv_heads, cfg.d_c), dtype=torch.int32, device=dev)
    sc = torch.empty((cfg.num_kv_heads, cfg.d_k), dtype=torch.float32, device=dev)
    cc = cfg.c()
    _lib.check(lib.tls_calibrate_channels(ctypes.byref(cc), q_cal.data_ptr(), n_q, k_cal.data_ptr(), n_k,
                                          int(k_head_stride), ch.data_ptr(), sc.data_ptr(), _stream(dev)))
    return ch, sc


def build_index(cfg: TLSConfig, k_cache: torch.Tensor, seq_lens: torch.Tensor, index: TLSIndex,
                start_token: int = 0) -> TLSIndex:
    """Block summaries + INT4 token index, in place."""
    lib = _lib.load()
    dev = k_cache.device
    _need(k_cache, "k_cache", _kv_shape(cfg, cfg.d_k), cfg.dtype, dev)
    _need(seq_lens, "seq_lens", (cfg.batch,), torch.int32, dev)
    _need(index.block_minmax, "block_minmax", (cfg.batch, cfg.num_kv_heads, cfg.num_blocks, 2, cfg.d_k), cfg.dtype, dev)
    _need(index.codes, "codes", (cfg.batch, cfg.num_kv_heads, cfg.max_seq_len, cfg.d_c // 2), torch.uint8, dev)
    _need(index.scale_zero, "scale_zero", (cfg.batch, cfg.num_kv_heads, cfg.max_seq_len, 2), torch.float32, dev)
    _need(index.channels, "channels", (cfg.num_kv_heads, cfg.d_c), torch.int32, dev)
    cc, ic = cfg.c(), index.c()
    _lib.check(lib.tls_build_index(ctypes.byref(cc), k_cache.data_ptr(), seq_lens.data_ptr(), int(start_token),
                                   ctypes.byref(ic), _stream(dev)))
    return index


def block_scores(cfg: TLSConfig, q: torch.Tensor, seq_lens: torch.Tensor, index: TLSIndex, out=None):
    """Block scores s_i of every pair, fp32 [batch, Hkv, M]."""
    lib = _lib.load()
    dev = q.device
    _need(q, "q", (cfg.batch, cfg.num_q_heads, cfg.d_k), cfg.dtype, dev)
    _need(seq_lens, "seq_lens", (cfg.batch,), torch.int32, dev)
    if out is None:
        out = torch.empty((cfg.batch, cfg.num_kv_heads, cfg.num_blocks), dtype=torch.float32, device=dev)
    cc = cfg.c()
    _lib.check(lib.tls_block_scores(ctypes.byref(cc), q.data_ptr(), seq_lens.data_ptr(), index.block_minmax.data_ptr(),
                                    out.data_ptr(), _stream(dev)))
    return out


# ---- sequence-split decode primitives (include/tls.h, seqsplit.cu; orchestration in seqsplit.py)
def topk_rows(keys: torch.Tensor, ids: torch.Tensor, k: int):
    """Exact top-k of each row of (key, id) pairs (ids ascending per row, -1 = empty): larger key first,
    equal keys -> lower id.  Returns (keys [rows, k], ids [rows, k] ascending ids, count [rows])."""
    lib = _lib.load()
    dev = keys.device
    rows, n = keys.reshape(-1, keys.shape[-1]).shape
    _need(keys, "keys", tuple(keys.shape), torch.float32, dev)
    _need(ids, "ids", tuple(keys.shape), torch.int32, dev)
    ok = torch.empty(keys.shape[:-1] + (k,), dtype=torch.float32, device=dev)
    oi = torch.empty(keys.shape[:-1] + (k,), dtype=torch.int32, device=dev)
    cnt = torch.empty(keys.shape[:-1], dtype=torch.int32, device=dev)
    _lib.check(lib.tls_topk_rows(rows, n, keys.data_ptr(), ids.data_ptr(), k, ok.data_ptr(), oi.data_ptr(),
                                 cnt.data_ptr(), _stream(dev)))
    return ok, oi, cnt


def block_topk(cfg: TLSConfig, scores: torch.Tensor, seq_lens: torch.Tensor, block_offset: int):
    """A rank's local top-k_b with global block ids.  Returns (scores, block_ids) [batch, Hkv, k_b]."""
    lib = _lib.load()
    dev = scores.device
    _need(scores, "scores", (cfg.batch, cfg.num_kv_heads, cfg.num_blocks), torch.float32, dev)
    _need(seq_lens, "seq_lens", (cfg.batch,), torch.int32, dev)
    os_ = torch.empty((cfg.batch, cfg.num_kv_heads, cfg.top_blocks), dtype=torch.float32, device=dev)
    ob = torch.empty((cfg.batch, cfg.num_kv_heads, cfg.top_blocks), dtype=torch.int32, device=dev)
    cc = cfg.c()
    _lib.check(lib.tls_block_topk(ctypes.byref(cc), scores.data_ptr(), seq_lens.data_ptr(), int(block_offset),
                                  os_.data_ptr(), ob.data_ptr(), _stream(dev)))
    return os_, ob


def select_range(ids: torch.Tensor, lo: int, hi: int):
    """The ids of each row (ascending, -1 padded) in [lo, hi), shifted by -lo, compacted, -1 padded.
    Returns (ids, count)."""
    lib = _lib.load()
    dev = ids.device
    _need(ids, "ids", tuple(ids.shape), torch.int32, dev)
    k = ids.shape[-1]
    rows = ids.numel() // k
    out = torch.empty_like(ids)
    cnt = torch.empty(ids.shape[:-1], dtype=torch.int32, device=dev)
    _lib.check(lib.tls_select_range(rows, k, ids.data_ptr(), int(lo), int(hi), out.data_ptr(), cnt.data_ptr(),
                                    _stream(dev)))
    return out, cnt


def token_stats(cfg: TLSConfig, q: torch.Tensor, seq_lens: torch.Tensor, index: TLSIndex, block_ids: torch.Tensor):
    """This rank's per-head softmax statistics of a3 over its candidate blocks: [batch, Hkv, G, 2]
    = (max_j L_hj, sum_j 2^(L_hj - max)), L in log2 units."""
    lib = _lib.load()
    dev = q.device
    _need(q, "q", (cfg.batch, cfg.num_q_heads, cfg.d_k), cfg.dtype, dev)
    _need(seq_lens, "seq_lens", (cfg.batch,), torch.int32, dev)
    _need(block_ids, "block_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_blocks), torch.int32, dev)
    st = torch.empty((cfg.batch, cfg.num_kv_heads, cfg.G, 2), dtype=torch.float32, device=dev)
    cc, ic = cfg.c(), index.c()
    _lib.check(lib.tls_token_stats(ctypes.byref(cc), q.data_ptr(), seq_lens.data_ptr(), ctypes.byref(ic),
                                   block_ids.data_ptr(), st.data_ptr(), _stream(dev)))
    return st


def token_keys(cfg: TLSConfig, q: torch.Tensor, seq_lens: torch.Tensor, index: TLSIndex, block_ids: torch.Tensor,
               stats_parts: torch.Tensor, token_offset: int):
    """ln alpha~ of this rank's candidates under the normaliser merged from every rank's token_stats
    (stats_parts [P, batch, Hkv, G, 2]) and their global token ids: ([batch, Hkv, k_b*B] x 2)."""
    lib = _lib.load()
    dev = q.device
    _need(q, "q", (cfg.batch, cfg.num_q_heads, cfg.d_k), cfg.dtype, dev)
    _need(block_ids, "block_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_blocks), torch.int32, dev)
    P = stats_parts.shape[0]
    _need(stats_parts, "stats_parts", (P, cfg.batch, cfg.num_kv_heads, cfg.G, 2), torch.float32, dev)
    n = cfg.top_blocks * cfg.block_size
    keys = torch.empty((cfg.batch, cfg.num_kv_heads, n), dtype=torch.float32, device=dev)
    tids = torch.empty((cfg.batch, cfg.num_kv_heads, n), dtype=torch.int32, device=dev)
    cc, ic = cfg.c(), index.c()
    _lib.check(lib.tls_token_keys(ctypes.byref(cc), q.data_ptr(), seq_lens.data_ptr(), ctypes.byref(ic),
                                  block_ids.data_ptr(), P, stats_parts.data_ptr(), int(token_offset), keys.data_ptr(),
                                  tids.data_ptr(), _stream(dev)))
    return keys, tids


def attn_merge(cfg: TLSConfig, parts_out: torch.Tensor, parts_lse: torch.Tensor):
    """LSE merge of P partial attention results: parts_out [P, batch, Hq, d_v], parts_lse [P, batch, Hq].
    Returns (out, lse)."""
    lib = _lib.load()
    dev = parts_out.device
    P = parts_out.shape[0]
    _need(parts_out, "parts_out", (P, cfg.batch, cfg.num_q_heads, cfg.d_v), torch.float32, dev)
    _need(parts_lse, "parts_lse", (P, cfg.batch, cfg.num_q_heads), torch.float32, dev)
    out = torch.empty((cfg.batch, cfg.num_q_heads, cfg.d_v), dtype=cfg.dtype, device=dev)
    lse = torch.empty((cfg.batch, cfg.num_q_heads), dtype=torch.float32, device=dev)
    cc = cfg.c()
    _lib.check(lib.tls_attn_merge(ctypes.byref(cc), P, parts_out.data_ptr(), parts_lse.data_ptr(), out.data_ptr(),
                                  lse.data_ptr(), _stream(dev)))
    return out, lse


# ---- the paper's comparison operators, from the calls above
def expand_blocks(cfg: TLSConfig, block_ids: torch.Tensor, seq_lens: torch.Tensor, k_out: int):
    """Every token (below the sequence length) of the selected blocks, ascending: (token_ids, num_tokens)."""
    lib = _lib.load()
    dev = block_ids.device
    _need(block_ids, "block_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_blocks), torch.int32, dev)
    tids = torch.empty((cfg.batch, cfg.num_kv_heads, k_out), dtype=torch.int32, device=dev)
    nt = torch.empty((cfg.batch, cfg.num_kv_heads), dtype=torch.int32, device=dev)
    cc = cfg.c()
    _lib.check(lib.tls_expand_blocks(ctypes.byref(cc), block_ids.data_ptr(), seq_lens.data_ptr(), int(k_out),
                                     tids.data_ptr(), nt.data_ptr(), _stream(dev)))
    return tids, nt


def block_iota(cfg: TLSConfig, seq_lens: torch.Tensor):
    """Every block of each sequence as the candidate set ([batch, Hkv, top_blocks], -1 padded)."""
    lib = _lib.load()
    dev = seq_lens.device
    out = torch.empty((cfg.batch, cfg.num_kv_heads, cfg.top_blocks), dtype=torch.int32, device=dev)
    cc = cfg.c()
    _lib.check(lib.tls_block_iota(ctypes.byref(cc), seq_lens.data_ptr(), out.data_ptr(), _stream(dev)))
    return out


def _with(cfg: TLSConfig, **kw) -> TLSConfig:
    import dataclasses

    return dataclasses.replace(cfg, **kw)


def quest_decode(cfg: TLSConfig, q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor | None,
                 seq_lens: torch.Tensor, index: TLSIndex):
    """Quest (the block-level baseline of P:395): the top-k_b blocks by the bound s_i and
    attention over EVERY token of them -- no token-level stage.  Returns (out, lse, block_ids, token_ids,
    num_tokens); k_t of the attention = k_b * B."""
    scores = block_scores(cfg, q, seq_lens, index)
    _, bids = block_topk(cfg, scores, seq_lens, 0)
    kq = cfg.top_blocks * cfg.block_size
    tids, nt = expand_blocks(cfg, bids, seq_lens, kq)
    out, lse = sparse_attend(_with(cfg, top_tokens=kq), q, k_cache, v_cache, tids, nt)
    return out, lse, bids, tids, nt


def ds_decode(cfg: TLSConfig, q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor | None,
              seq_lens: torch.Tensor, index: TLSIndex):
    """DS (the token-level baseline of P:395: alpha~ over the channel-projected INT4 index of EVERY cached token,
    P:127-134, then top-k_t) -- TLS with every block a candidate (k_b = m).  Returns (out, lse,
    token_ids, num_tokens, ln_alpha)."""
    cfg_all = _with(cfg, top_blocks=cfg.num_blocks)
    cand = block_iota(cfg_all, seq_lens)
    stats = token_stats(cfg_all, q, seq_lens, index, cand)
    keys, ids = token_keys(cfg_all, q, seq_lens, index, cand, stats.unsqueeze(0), 0)
    lk, tids, nt = topk_rows(keys, ids, cfg.top_tokens)
    out, lse = sparse_attend(cfg, q, k_cache, v_cache, tids, nt)
    return out, lse, tids, nt, lk


def _sel_outputs(cfg: TLSConfig, dev, out):
    if out is not None:
        return out
    return (
        torch.empty((cfg.batch, cfg.num_kv_heads, cfg.top_blocks), dtype=torch.int32, device=dev),
        torch.empty((cfg.batch, cfg.num_kv_heads, cfg.top_tokens), dtype=torch.int32, device=dev),
        torch.empty((cfg.batch, cfg.num_kv_heads), dtype=torch.int32, device=dev),
        torch.empty((cfg.batch, cfg.num_kv_heads, cfg.top_tokens), dtype=torch.float32, device=dev),
    )


def select(cfg: TLSConfig, q: torch.Tensor, seq_lens: torch.Tensor, index: TLSIndex,
           guide_block_ids: torch.Tensor | None = None, out=None):
    """Two-level selection.  Returns (block_ids, token_ids, num_tokens, token_scores)."""
    lib = _lib.load()
    dev = q.device
    _need(q, "q", (cfg.batch, cfg.num_q_heads, cfg.d_k), cfg.dtype, dev)
    _need(seq_lens, "seq_lens", (cfg.batch,), torch.int32, dev)
    bids, tids, nt, ts = _sel_outputs(cfg, dev, out)
    g = 0
    if guide_block_ids is not None:
        _need(guide_block_ids, "guide_block_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_blocks), torch.int32, dev)
        g = guide_block_ids.data_ptr()
    cc, ic = cfg.c(), index.c()
    ws, wsb = _workspace(cfg, dev, 0)
    _lib.check(lib.tls_select(ctypes.byref(cc), q.data_ptr(), seq_lens.data_ptr(), ctypes.byref(ic), g,
                              bids.data_ptr(), tids.data_ptr(), nt.data_ptr(),
                              ts.data_ptr() if ts is not None else 0, ws, wsb, _stream(dev)))
    return bids, tids, nt, ts


def sparse_attend(cfg: TLSConfig, q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor | None,
                  token_ids: torch.Tensor, num_tokens: torch.Tensor, out=None, lse=None, out_f32: bool = False):
    """Attention over the selected tokens.  Returns (out, lse); out in the cfg dtype, or
    fp32 with out_f32 (tls_sparse_attend_f32: partial results that are merged later)."""
    lib = _lib.load()
    dev = q.device
    _need(q, "q", (cfg.batch, cfg.num_q_heads, cfg.d_k), cfg.dtype, dev)
    _need(k_cache, "k_cache", _kv_shape(cfg, cfg.d_k), cfg.dtype, dev)
    if cfg.layout == "gqa":
        _need(v_cache, "v_cache", _kv_shape(cfg, cfg.d_v), cfg.dtype, dev)
    _need(token_ids, "token_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_tokens), torch.int32, dev)
    _need(num_tokens, "num_tokens", (cfg.batch, cfg.num_kv_heads), torch.int32, dev)
    if out is None:
        out = torch.empty((cfg.batch, cfg.num_q_heads, cfg.d_v), dtype=torch.float32 if out_f32 else cfg.dtype,
                          device=dev)
    if lse is None:
        lse = torch.empty((cfg.batch, cfg.num_q_heads), dtype=torch.float32, device=dev)
    cc = cfg.c()
    ws, wsb = _workspace(cfg, dev, 1)
    fn = lib.tls_sparse_attend_f32 if out_f32 else lib.tls_sparse_attend
    _lib.check(fn(ctypes.byref(cc), q.data_ptr(), k_cache.data_ptr(),
                                     v_cache.data_ptr() if (v_cache is not None and cfg.layout == "gqa") else 0,
                                     token_ids.data_ptr(), num_tokens.data_ptr(), out.data_ptr(), lse.data_ptr(),
                                     ws, wsb, _stream(dev)))
    return out, lse


def decode(cfg: TLSConfig, q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor | None,
           seq_lens: torch.Tensor, index: TLSIndex, guide_block_ids: torch.Tensor | None = None, sel_out=None,
           out=None, lse=None):
    """One decode step of the operator: select + attend in one fused launch.

    Returns (out, lse, block_ids, token_ids, num_tokens, token_scores).
    """
    lib = _lib.load()
    dev = q.device
    _need(q, "q", (cfg.batch, cfg.num_q_heads, cfg.d_k), cfg.dtype, dev)
    _need(k_cache, "k_cache", _kv_shape(cfg, cfg.d_k), cfg.dtype, dev)
    if cfg.layout == "gqa":
        _need(v_cache, "v_cache", _kv_shape(cfg, cfg.d_v), cfg.dtype, dev)
    _need(seq_lens, "seq_lens", (cfg.batch,), torch.int32, dev)
    bids, tids, nt, ts = _sel_outputs(cfg, dev, sel_out)
    if out is None:
        out = torch.empty((cfg.batch, cfg.num_q_heads, cfg.d_v), dtype=cfg.dtype, device=dev)
    if lse is None:
        lse = torch.empty((cfg.batch, cfg.num_q_heads), dtype=torch.float32, device=dev)
    g = 0
    if guide_block_ids is not None:
        _need(guide_block_ids, "guide_block_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_blocks), torch.int32, dev)
        g = guide_block_ids.data_ptr()
    cc, ic = cfg.c(), index.c()
    ws, wsb = _workspace(cfg, dev, 2)
    _lib.check(lib.tls_decode(ctypes.byref(cc), q.data_ptr(), k_cache.data_ptr(),
                              v_cache.data_ptr() if (v_cache is not None and cfg.layout == "gqa") else 0,
                              seq_lens.data_ptr(), ctypes.byref(ic), g, bids.data_ptr(), tids.data_ptr(), nt.data_ptr(),
                              ts.data_ptr() if ts is not None else 0, out.data_ptr(), lse.data_ptr(), ws, wsb,
                              _stream(dev)))
    return out, lse, bids, tids, nt, ts


def cluster_size(cfg: TLSConfig, which: int = 2) -> int:
    """CTAs per (batch, KV-head) pair: token-select kernel (which 0/2) or attention kernel (1)."""
    cc = cfg.c()
    return int(_lib.load().tls_cluster_size(ctypes.byref(cc), which))


# timing slots of the kernel chain (select mode 1) and of the fused step (mode 3, one launch)
KERNELS = ("select_kernel", "token_cluster_kernel", "attend_kernel")
STEP_KERNELS = ("pstep_kernel",)


def select_mode(cfg: TLSConfig) -> int:
    """3: the persistent step kernel (one launch; work items of every stage of every pair claimed from a ticket
    queue, pstep.cu); 1: the kernel chain
    (select_kernel a1-a2, token kernel a3, the attention kernel's prologue a4 + a5)."""
    cc = cfg.c()
    return int(_lib.load().tls_select_mode(ctypes.byref(cc)))


def kernel_names(cfg: TLSConfig) -> tuple:
    """Names of the launches one tls_decode call enqueues (the timing slots of timing_read); the token kernel is
    token_pair_kernel (one, two or four CTAs per pair), token_pair_nt_kernel (G > 8) or token_cluster_kernel (token_reg_kernel /
    token_cluster_kernel: a cluster of chunk CTAs), per ``cluster_size(cfg, 5)``."""
    if select_mode(cfg) == 3:
        return STEP_KERNELS
    form = cluster_size(cfg, 5)
    if form == 6:
        return (KERNELS[0], "token_pair_nt_kernel", KERNELS[2])
    return (KERNELS[0], "token_pair_kernel", KERNELS[2]) if form in (1, 4, 5) else KERNELS


def timing_enable(n_calls: int) -> None:
    """Record CUDA events around each launch of the next select/decode calls
    (tls_timing_enable); 0 disables."""
    _lib.check(_lib.load().tls_timing_enable(int(n_calls)))


def timing_read(cfg: TLSConfig | None = None) -> tuple[dict, int]:
    """(kernel name -> summed ms, number of calls) since the last read (tls_timing_read); the names are those
    of ``kernel_names(cfg)`` (the kernel chain's when cfg is None)."""
    ms = (ctypes.c_double * len(KERNELS))()
    calls = ctypes.c_int64(0)
    _lib.check(_lib.load().tls_timing_read(ms, ctypes.byref(calls)))
    names = kernel_names(cfg) if cfg is not None else KERNELS
    return {k: float(ms[i]) for i, k in enumerate(names)}, int(calls.value)


# ------------------------------------------------------------------ KV offload
@dataclass
class TLSTokenCache:
    """GPU token cache of the offload engine (tls_token_cache, include/tls.h)."""

    capacity: int
    k_slots: torch.Tensor  # [batch, Hkv, capacity, d_k]
    v_slots: torch.Tensor | None  # [batch, Hkv, capacity, d_v] (None for MLA)
    slot_of_token: torch.Tensor  # [batch, Hkv, S] int32, -1 = not resident
    token_of_slot: torch.Tensor  # [batch, Hkv, capacity] int32, -1 = free

    def c(self) -> _lib.TLSTokenCacheC:
        return _lib.TLSTokenCacheC(self.capacity, self.k_slots.data_ptr(),
                                   self.v_slots.data_ptr() if self.v_slots is not None else 0,
                                   self.slot_of_token.data_ptr(), self.token_of_slot.data_ptr())


def alloc_token_cache(cfg: TLSConfig, capacity: int, device) -> TLSTokenCache:
    """An empty token cache of ``capacity`` (>= top_tokens) slots per pair."""
    hk = cfg.num_kv_heads if cfg.layout == "gqa" else 1
    slots = (cfg.batch, hk, capacity) if cfg.layout == "gqa" else (cfg.batch, capacity)  # the k_cache layouts
    return TLSTokenCache(
        capacity=capacity,
        k_slots=torch.empty(slots + (cfg.d_k,), dtype=cfg.dtype, device=device),
        v_slots=torch.empty(slots + (cfg.d_v,), dtype=cfg.dtype, device=device) if cfg.layout == "gqa" else None,
        slot_of_token=torch.full((cfg.batch, hk, cfg.max_seq_len), -1, dtype=torch.int32, device=device),
        token_of_slot=torch.full((cfg.batch, hk, capacity), -1, dtype=torch.int32, device=device),
    )


def host_kv(t: torch.Tensor) -> torch.Tensor:
    """A pinned (page-locked, device-mapped under UVA) host copy of a KV cache tensor."""
    return t.cpu().pin_memory()


def cache_fetch(cfg: TLSConfig, k_host: torch.Tensor, v_host: torch.Tensor | None, token_ids: torch.Tensor,
                num_tokens: torch.Tensor, cache: TLSTokenCache, slot_ids=None, miss_count=None):
    """Make the selection resident in ``cache`` (tls_cache_fetch).  Returns (slot_ids, miss_count)."""
    lib = _lib.load()
    dev = token_ids.device
    if not (k_host.is_pinned() and (v_host is None or v_host.is_pinned())):
        raise ValueError("k_host / v_host must be pinned host tensors (host_kv)")
    _need(token_ids, "token_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_tokens), torch.int32, dev)
    _need(num_tokens, "num_tokens", (cfg.batch, cfg.num_kv_heads), torch.int32, dev)
    if slot_ids is None:
        slot_ids = torch.empty_like(token_ids)
    if miss_count is None:
        miss_count = torch.empty_like(num_tokens)
    cc, kc = cfg.c(), cache.c()
    _lib.check(lib.tls_cache_fetch(ctypes.byref(cc), k_host.data_ptr(),
                                   v_host.data_ptr() if (v_host is not None and cfg.layout == "gqa") else 0,
                                   token_ids.data_ptr(), num_tokens.data_ptr(), ctypes.byref(kc), slot_ids.data_ptr(),
                                   miss_count.data_ptr(), _stream(dev)))
    return slot_ids, miss_count


def offload_decode(cfg: TLSConfig, q: torch.Tensor, k_host: torch.Tensor, v_host: torch.Tensor | None,
                   seq_lens: torch.Tensor, index: TLSIndex, cache: TLSTokenCache, guide_block_ids=None):
    """One decode step with the KV cache in host memory: select on the GPU index (lag mode with
    ``guide_block_ids``), fetch the missed selected tokens into the GPU token cache, attend over the
    cache rows.  Returns (out, lse, block_ids, token_ids, num_tokens, token_scores, slot_ids, miss_count)."""
    bids, tids, nt, ts = select(cfg, q, seq_lens, index, guide_block_ids=guide_block_ids)
    slot_ids, miss = cache_fetch(cfg, k_host, v_host, tids, nt, cache)
    ccfg = TLSConfig(**{**{f: getattr(cfg, f) for f in ("batch", "num_q_heads", "num_kv_heads", "d_k", "d_v",
                                                        "block_size", "d_c", "top_blocks", "top_tokens", "sm_scale",
                                                        "dtype", "layout")}, "max_seq_len": cache.capacity})
    out, lse = sparse_attend(ccfg, q, cache.k_slots, cache.v_slots, slot_ids, nt)
    return out, lse, bids, tids, nt, ts, slot_ids, miss

@dataclass
class TLSBlockCache:
    """GPU block cache of the asynchronous offload engine (tls_block_cache, include/tls.h)."""

    capacity: int  # block slots per pair (>= 2 * top_blocks)
    k_slots: torch.Tensor  # [batch, Hkv, capacity * B, d_k]
    v_slots: torch.Tensor | None  # [batch, Hkv, capacity * B, d_v] (None for MLA)
    slot_of_block: torch.Tensor  # [batch, Hkv, M] int32, -1 = not resident
    block_of_slot: torch.Tensor  # [batch, Hkv, capacity] int32, -1 = free

    def c(self) -> _lib.TLSBlockCacheC:
        return _lib.TLSBlockCacheC(self.capacity, self.k_slots.data_ptr(),
                                   self.v_slots.data_ptr() if self.v_slots is not None else 0,
                                   self.slot_of_block.data_ptr(), self.block_of_slot.data_ptr())


def alloc_block_cache(cfg: TLSConfig, capacity: int, device) -> TLSBlockCache:
    """An empty block cache of ``capacity`` (>= 2 * top_blocks) block slots per pair."""
    hk = cfg.num_kv_heads if cfg.layout == "gqa" else 1
    rows = capacity * cfg.block_size
    lead = (cfg.batch, hk, rows) if cfg.layout == "gqa" else (cfg.batch, rows)  # the k_cache layouts
    return TLSBlockCache(
        capacity=capacity,
        k_slots=torch.empty(lead + (cfg.d_k,), dtype=cfg.dtype, device=device),
        v_slots=torch.empty(lead + (cfg.d_v,), dtype=cfg.dtype, device=device) if cfg.layout == "gqa" else None,
        slot_of_block=torch.full((cfg.batch, hk, cfg.num_blocks), -1, dtype=torch.int32, device=device),
        block_of_slot=torch.full((cfg.batch, hk, capacity), -1, dtype=torch.int32, device=device),
    )


def block_cache_update(cfg: TLSConfig, k_host: torch.Tensor, v_host: torch.Tensor | None, block_ids: torch.Tensor,
                       cache: TLSBlockCache, keep_block_ids=None, miss_count=None, stream=None):
    """Make the blocks ``block_ids`` (M_t) resident, keeping ``keep_block_ids`` (M_{t-1}); enqueued on ``stream``
    (default: the current stream).  Returns miss_count [batch, Hkv] (blocks fetched)."""
    lib = _lib.load()
    dev = block_ids.device
    if not (k_host.is_pinned() and (v_host is None or v_host.is_pinned())):
        raise ValueError("k_host / v_host must be pinned host tensors (host_kv)")
    _need(block_ids, "block_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_blocks), torch.int32, dev)
    if keep_block_ids is not None:
        _need(keep_block_ids, "keep_block_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_blocks), torch.int32, dev)
    if miss_count is None:
        miss_count = torch.empty((cfg.batch, cfg.num_kv_heads), dtype=torch.int32, device=dev)
    cc, bc = cfg.c(), cache.c()
    st = stream.cuda_stream if stream is not None else _stream(dev)
    _lib.check(lib.tls_block_cache_update(ctypes.byref(cc), k_host.data_ptr(),
                                          v_host.data_ptr() if (v_host is not None and cfg.layout == "gqa") else 0,
                                          keep_block_ids.data_ptr() if keep_block_ids is not None else 0,
                                          block_ids.data_ptr(), ctypes.byref(bc), miss_count.data_ptr(), st))
    return miss_count


def block_cache_rows(cfg: TLSConfig, token_ids: torch.Tensor, num_tokens: torch.Tensor, cache: TLSBlockCache,
                     slot_rows=None, absent=None):
    """Cache rows of the selected tokens (tls_block_cache_rows).  Returns (slot_rows, absent)."""
    lib = _lib.load()
    dev = token_ids.device
    _need(token_ids, "token_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_tokens), torch.int32, dev)
    _need(num_tokens, "num_tokens", (cfg.batch, cfg.num_kv_heads), torch.int32, dev)
    if slot_rows is None:
        slot_rows = torch.empty_like(token_ids)
    if absent is None:
        absent = torch.empty_like(num_tokens)
    cc, bc = cfg.c(), cache.c()
    _lib.check(lib.tls_block_cache_rows(ctypes.byref(cc), token_ids.data_ptr(), num_tokens.data_ptr(),
                                        ctypes.byref(bc), slot_rows.data_ptr(), absent.data_ptr(), _stream(dev)))
    return slot_rows, absent


def decode_block_cache(cfg: TLSConfig, q: torch.Tensor, seq_lens: torch.Tensor, index: TLSIndex,
                       cache: TLSBlockCache, guide_block_ids: torch.Tensor | None = None, sel_out=None, out=None,
                       lse=None):
    """tls_decode with the K/V rows read from the block cache (tls_decode_block_cache): every block of the
    candidate set must be resident.  Returns (out, lse, block_ids, token_ids, num_tokens, token_scores)."""
    lib = _lib.load()
    dev = q.device
    _need(q, "q", (cfg.batch, cfg.num_q_heads, cfg.d_k), cfg.dtype, dev)
    _need(seq_lens, "seq_lens", (cfg.batch,), torch.int32, dev)
    bids, tids, nt, ts = _sel_outputs(cfg, dev, sel_out)
    if out is None:
        out = torch.empty((cfg.batch, cfg.num_q_heads, cfg.d_v), dtype=cfg.dtype, device=dev)
    if lse is None:
        lse = torch.empty((cfg.batch, cfg.num_q_heads), dtype=torch.float32, device=dev)
    g = 0
    if guide_block_ids is not None:
        _need(guide_block_ids, "guide_block_ids", (cfg.batch, cfg.num_kv_heads, cfg.top_blocks), torch.int32, dev)
        g = guide_block_ids.data_ptr()
    cc, ic, bc = cfg.c(), index.c(), cache.c()
    ws, wsb = _workspace(cfg, dev, 2)
    _lib.check(lib.tls_decode_block_cache(ctypes.byref(cc), q.data_ptr(), seq_lens.data_ptr(), ctypes.byref(ic), g,
                                          ctypes.byref(bc), bids.data_ptr(), tids.data_ptr(), nt.data_ptr(),
                                          ts.data_ptr() if ts is not None else 0, out.data_ptr(), lse.data_ptr(), ws,
                                          wsb, _stream(dev)))
    return out, lse, bids, tids, nt, ts


class AsyncOffloadDecoder:
    """The asynchronous offload engine: full K/V in pinned host memory, a GPU block cache, one-step
    lag S_t = TokenSelect(q_t, M_{t-1}), and the transfer of M_t's missing blocks on a side stream, overlapped
    with whatever the caller enqueues next.  ``step(q)`` returns (out, lse, block_ids, token_ids, num_tokens,
    token_scores); ``last_miss`` holds the blocks fetched by the latest update."""

    def __init__(self, cfg: TLSConfig, k_host, v_host, seq_lens, index: TLSIndex, capacity: int | None = None):
        self.cfg, self.k_host, self.v_host, self.seq_lens, self.index = cfg, k_host, v_host, seq_lens, index
        dev = seq_lens.device
        self.cache = alloc_block_cache(cfg, capacity or 2 * cfg.top_blocks, dev)
        self.side = torch.cuda.Stream(device=dev)
        self.ready = None  # event: the update that brought M_{t-1} in
        self.prev = None  # M_{t-1}
        self.last_miss = None

    def _update(self, bids, keep):
        main = torch.cuda.current_stream(bids.device)
        sel_done = torch.cuda.Event()
        sel_done.record(main)
        self.side.wait_event(sel_done)
        with torch.cuda.stream(self.side):
            self.last_miss = block_cache_update(self.cfg, self.k_host, self.v_host, bids, self.cache,
                                                keep_block_ids=keep, stream=self.side)
            bids.record_stream(self.side)
            if keep is not None:
                keep.record_stream(self.side)
        ev = torch.cuda.Event()
        ev.record(self.side)
        return ev

    def step(self, q):
        """One decode step: one fused launch chain on the current stream (after the previous step's update),
        then the update of the cache to M_t on the side stream, overlapped with whatever the caller enqueues
        next (the other layers of the model)."""
        cfg = self.cfg
        main = torch.cuda.current_stream(q.device)
        if self.prev is None:  # first step: M_0 from a synchronous selection, fetched before the attention, is
            # the guide (candidates = this step's own M_t, the synchronous form P:137)
            guide = select(cfg, q, self.seq_lens, self.index)[0]
            main.wait_event(self._update(guide, None))
        else:
            guide = self.prev
            main.wait_event(self.ready)  # M_{t-1} resident
        res = decode_block_cache(cfg, q, self.seq_lens, self.index, self.cache, guide_block_ids=guide)
        bids = res[2]
        # M_t's missing blocks go to free slots; M_{t-1} (read by this step) stays
        self.ready = self._update(bids, self.prev)
        self.prev = bids
        return res
