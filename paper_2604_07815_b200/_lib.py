"""ctypes binding of libtls.so (include/tls.h).  Argument marshalling only.

The library must have been built (``__graft_entry__.build()`` or
``python -m paper_2604_07815_b200.build``); loading fails loudly otherwise --
there is no fallback path.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtls.so")

TLS_OK, TLS_ERR_DIM, TLS_ERR_CONFIG, TLS_ERR_INPUT, TLS_ERR_WORKSPACE, TLS_ERR_UNSUPPORTED, TLS_ERR_CUDA = range(7)
TLS_BF16, TLS_FP32 = 0, 1
TLS_GQA, TLS_MLA = 0, 1

# Every symbol include/tls.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "tls_calibrate_channels",
    "tls_build_index",
    "tls_block_scores",
    "tls_select",
    "tls_sparse_attend",
    "tls_decode",
    "tls_topk_rows",
    "tls_block_topk",
    "tls_select_range",
    "tls_token_stats",
    "tls_token_keys",
    "tls_attn_merge",
    "tls_sparse_attend_f32",
    "tls_expand_blocks",
    "tls_block_iota",
    "tls_workspace_bytes",
    "tls_launch_count",
    "tls_cluster_size",
    "tls_select_mode",
    "tls_workspace_init",
    "tls_cache_fetch",
    "tls_block_cache_update",
    "tls_block_cache_rows",
    "tls_decode_block_cache",
    "tls_timing_enable",
    "tls_timing_read",
    "tls_status_string",
    "tls_last_error",
    "tls_version",
)


class TLSConfigC(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32),
        ("num_q_heads", ctypes.c_int32),
        ("num_kv_heads", ctypes.c_int32),
        ("d_k", ctypes.c_int32),
        ("d_v", ctypes.c_int32),
        ("max_seq_len", ctypes.c_int32),
        ("block_size", ctypes.c_int32),
        ("d_c", ctypes.c_int32),
        ("top_blocks", ctypes.c_int32),
        ("top_tokens", ctypes.c_int32),
        ("sm_scale", ctypes.c_float),
        ("dtype", ctypes.c_int32),
        ("layout", ctypes.c_int32),
    ]


class TLSIndexC(ctypes.Structure):
    _fields_ = [
        ("block_minmax", ctypes.c_void_p),
        ("codes", ctypes.c_void_p),
        ("scale_zero", ctypes.c_void_p),
        ("channels", ctypes.c_void_p),
    ]


class TLSTokenCacheC(ctypes.Structure):
    _fields_ = [
        ("capacity", ctypes.c_int32),
        ("k_slots", ctypes.c_void_p),
        ("v_slots", ctypes.c_void_p),
        ("slot_of_token", ctypes.c_void_p),
        ("token_of_slot", ctypes.c_void_p),
    ]


class TLSBlockCacheC(ctypes.Structure):
    _fields_ = [
        ("capacity", ctypes.c_int32),
        ("k_slots", ctypes.c_void_p),
        ("v_slots", ctypes.c_void_p),
        ("slot_of_block", ctypes.c_void_p),
        ("block_of_slot", ctypes.c_void_p),
    ]


class TLSError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        super().__init__(f"{_status_name(status)}: {detail}")


_lib = None
_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_PCFG = ctypes.POINTER(TLSConfigC)
_PIDX = ctypes.POINTER(TLSIndexC)


def _status_name(s: int) -> str:
    names = ["TLS_OK", "TLS_ERR_DIM", "TLS_ERR_CONFIG", "TLS_ERR_INPUT", "TLS_ERR_WORKSPACE", "TLS_ERR_UNSUPPORTED",
             "TLS_ERR_CUDA"]
    return names[s] if 0 <= s < len(names) else f"status {s}"


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libtls.so once; raise if it is missing (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run __graft_entry__.build() (the CUDA path is the only path)")
    lib = ctypes.CDLL(path)
    sig = {
        "tls_calibrate_channels": (_I32, [_PCFG, _P, _I32, _P, _I32, ctypes.c_int64, _P, _P, _P]),
        "tls_build_index": (_I32, [_PCFG, _P, _P, _I32, _PIDX, _P]),
        "tls_block_scores": (_I32, [_PCFG, _P, _P, _P, _P, _P]),
        "tls_topk_rows": (_I32, [_I32, _I32, _P, _P, _I32, _P, _P, _P, _P]),
        "tls_block_topk": (_I32, [_PCFG, _P, _P, _I32, _P, _P, _P]),
        "tls_select_range": (_I32, [_I32, _I32, _P, _I32, _I32, _P, _P, _P]),
        "tls_token_stats": (_I32, [_PCFG, _P, _P, _PIDX, _P, _P, _P]),
        "tls_token_keys": (_I32, [_PCFG, _P, _P, _PIDX, _P, _I32, _P, _I32, _P, _P, _P]),
        "tls_attn_merge": (_I32, [_PCFG, _I32, _P, _P, _P, _P, _P]),
        "tls_sparse_attend_f32": (_I32, [_PCFG, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
        "tls_expand_blocks": (_I32, [_PCFG, _P, _P, _I32, _P, _P, _P]),
        "tls_block_iota": (_I32, [_PCFG, _P, _P, _P]),
        "tls_select": (_I32, [_PCFG, _P, _P, _PIDX, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
        "tls_sparse_attend": (_I32, [_PCFG, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
        "tls_cache_fetch": (_I32, [_PCFG, _P, _P, _P, _P, ctypes.POINTER(TLSTokenCacheC), _P, _P, _P]),
        "tls_block_cache_update": (_I32, [_PCFG, _P, _P, _P, _P, ctypes.POINTER(TLSBlockCacheC), _P, _P]),
        "tls_block_cache_rows": (_I32, [_PCFG, _P, _P, ctypes.POINTER(TLSBlockCacheC), _P, _P, _P]),
        "tls_decode_block_cache": (_I32, [_PCFG, _P, _P, _PIDX, _P, ctypes.POINTER(TLSBlockCacheC), _P, _P, _P, _P,
                                          _P, _P, _P, ctypes.c_size_t, _P]),
        "tls_decode": (_I32, [_PCFG, _P, _P, _P, _P, _PIDX, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
        "tls_workspace_bytes": (ctypes.c_size_t, [_PCFG, _I32]),
        "tls_launch_count": (_I32, [_PCFG, _I32]),
        "tls_cluster_size": (_I32, [_PCFG, _I32]),
        "tls_select_mode": (_I32, [_PCFG]),
        "tls_workspace_init": (_I32, [_PCFG, _I32, _P, ctypes.c_size_t, _P]),
        "tls_timing_enable": (_I32, [_I32]),
        "tls_timing_read": (_I32, [_P, _P]),
        "tls_status_string": (ctypes.c_char_p, [_I32]),
        "tls_last_error": (ctypes.c_char_p, []),
        "tls_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != TLS_OK:
        raise TLSError(status, load().tls_last_error().decode())
