"""B200-native (sm_100a) AsyncTLS two-level sparse decode attention (arXiv 2604.07815).

The compute path is libtls.so (hand-written CUDA, C ABI in include/tls.h);
``ops`` is the torch-tensor front end with the same names.  There is no CPU
fallback: calling an op without the built library raises ImportError.
"""
from .ops import (  # noqa: F401
    TLSConfig,
    TLSIndex,
    alloc_index,
    block_scores,
    build_index,
    calibrate_channels,
    cluster_size,
    decode,
    select,
    select_mode,
    kernel_names,
    sparse_attend,
    KERNELS,
    timing_enable,
    timing_read,
    TLSTokenCache,
    alloc_token_cache,
    host_kv,
    cache_fetch,
    offload_decode,
    TLSBlockCache,
    alloc_block_cache,
    block_cache_update,
    block_cache_rows,
    decode_block_cache,
    AsyncOffloadDecoder,
    quest_decode,
    ds_decode,
)
from ._lib import TLSError, load  # noqa: F401

__version__ = "0.1.0"
