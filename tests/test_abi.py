"""CPU-only checks of the C ABI boundary (no GPU needed, no compute calls):
libtls.so loads, exports every symbol include/tls.h declares, and validates
arguments host-side with the documented status codes before any launch."""
import ctypes
import os
import re

import pytest

from paper_2604_07815_b200 import _lib
from paper_2604_07815_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _lib.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tls.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tls_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), f"libtls.so does not export {s}"
    assert set(syms) == set(_lib.EXPORTS)


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def cfg(**kw):
    base = dict(batch=2, num_q_heads=8, num_kv_heads=2, d_k=128, d_v=128, max_seq_len=4096, block_size=64, d_c=32,
                top_blocks=16, top_tokens=256, sm_scale=0.088, dtype=_lib.TLS_BF16, layout=_lib.TLS_GQA)
    base.update(kw)
    return _lib.TLSConfigC(**base)


def test_status_strings(lib):
    assert lib.tls_status_string(0) == b"TLS_OK"
    assert lib.tls_status_string(5) == b"TLS_ERR_UNSUPPORTED"
    assert lib.tls_version().startswith(b"tls-b200")


@pytest.mark.parametrize("kw,status", [
    (dict(batch=0), _lib.TLS_ERR_INPUT),
    (dict(num_kv_heads=3), _lib.TLS_ERR_DIM),
    (dict(layout=_lib.TLS_MLA), _lib.TLS_ERR_DIM),           # MLA needs one KV head
    (dict(d_c=33), _lib.TLS_ERR_CONFIG),
    (dict(d_c=256), _lib.TLS_ERR_CONFIG),                    # d_c > d_k
    (dict(top_tokens=0), _lib.TLS_ERR_CONFIG),
    (dict(block_size=0), _lib.TLS_ERR_CONFIG),
    (dict(sm_scale=0.0), _lib.TLS_ERR_CONFIG),
    (dict(d_c=48), _lib.TLS_ERR_UNSUPPORTED),
    (dict(block_size=24), _lib.TLS_ERR_UNSUPPORTED),
    (dict(num_q_heads=128, num_kv_heads=2), _lib.TLS_ERR_UNSUPPORTED),
])
def test_config_validation_before_launch(lib, kw, status):
    c = cfg(**kw)
    idx = _lib.TLSIndexC(16, 16, 16, 16)
    st = lib.tls_select(ctypes.byref(c), 16, 16, ctypes.byref(idx), None, 16, 16, 16, None, None, 0, None)
    assert st == status, (st, lib.tls_last_error())
    assert lib.tls_last_error()
    assert lib.tls_workspace_bytes(ctypes.byref(c), 0) == ctypes.c_size_t(-1).value


def test_workspace_required(lib):
    c = cfg()
    idx = _lib.TLSIndexC(16, 16, 16, 16)
    assert lib.tls_select(ctypes.byref(c), 16, 16, ctypes.byref(idx), None, 16, 16, 16, None, None, 0,
                          None) == _lib.TLS_ERR_WORKSPACE
    assert lib.tls_select(ctypes.byref(c), 16, 16, ctypes.byref(idx), None, 16, 16, 16, None, 16, 64,
                          None) == _lib.TLS_ERR_WORKSPACE


def test_null_and_misaligned_pointers(lib):
    c = cfg()
    idx = _lib.TLSIndexC(16, 16, 16, 16)
    assert lib.tls_select(ctypes.byref(c), None, 16, ctypes.byref(idx), None, 16, 16, 16, None, None, 0,
                          None) == _lib.TLS_ERR_INPUT
    assert lib.tls_select(ctypes.byref(c), 18, 16, ctypes.byref(idx), None, 16, 16, 16, None, None, 0,
                          None) == _lib.TLS_ERR_INPUT
    bad = _lib.TLSIndexC(16, 8, 16, 16)
    assert lib.tls_select(ctypes.byref(c), 16, 16, ctypes.byref(bad), None, 16, 16, 16, None, None, 0,
                          None) == _lib.TLS_ERR_INPUT
    assert lib.tls_build_index(ctypes.byref(c), 16, 16, -1, ctypes.byref(idx), None) == _lib.TLS_ERR_INPUT
    assert lib.tls_calibrate_channels(ctypes.byref(c), 16, 0, 16, 4, 0, 16, None, None) == _lib.TLS_ERR_INPUT


def test_workspace_and_plan(lib, monkeypatch):
    # bf16 GQA, d 128, G <= 8, d_c 32, B 64: the persistent step kernel (one launch) when opted in
    c = cfg()
    monkeypatch.setenv("TLS_PSTEP", "0")
    assert lib.tls_select_mode(ctypes.byref(c)) == 3
    assert lib.tls_launch_count(ctypes.byref(c), 2) == 1
    assert lib.tls_launch_count(ctypes.byref(c), 0) == 1
    assert lib.tls_workspace_bytes(ctypes.byref(c), 2) >= lib.tls_workspace_bytes(ctypes.byref(c), 0) > 0
    assert lib.tls_cluster_size(ctypes.byref(c), 2) == 1  # 256 selected tokens: one attention slice
    monkeypatch.delenv("TLS_PSTEP")
    assert lib.tls_select_mode(ctypes.byref(c)) == 1
    # every other configuration runs the kernel chain
    c = cfg(dtype=_lib.TLS_FP32)
    assert lib.tls_workspace_bytes(ctypes.byref(c), 2) >= 2 * 2 * 64 * 4
    assert lib.tls_workspace_bytes(ctypes.byref(c), 1) > 0
    assert lib.tls_workspace_bytes(ctypes.byref(c), 2) == lib.tls_workspace_bytes(ctypes.byref(c), 0) + lib.tls_workspace_bytes(ctypes.byref(c), 1)
    assert lib.tls_select_mode(ctypes.byref(c)) == 1  # select_kernel a1-a2, token kernel a3, attend a4(+a5)
    assert lib.tls_launch_count(ctypes.byref(c), 2) == 4
    assert lib.tls_launch_count(ctypes.byref(c), 0) == 4
    cs = lib.tls_cluster_size(ctypes.byref(c), 2)
    assert cs in (1, 2, 4, 8, 16)
    # headline shapes plan without error
    c3 = cfg(batch=32, num_q_heads=64, num_kv_heads=8, max_seq_len=98304, top_blocks=128, top_tokens=1024)
    assert lib.tls_cluster_size(ctypes.byref(c3), 2) == 1 and lib.tls_select_mode(ctypes.byref(c3)) == 1
    c2 = cfg(batch=16, num_q_heads=32, num_kv_heads=8, max_seq_len=49152, top_blocks=128, top_tokens=1024)
    assert lib.tls_select_mode(ctypes.byref(c2)) == 1
    c4 = cfg(batch=32, num_q_heads=32, num_kv_heads=1, d_k=576, d_v=512, max_seq_len=65536, d_c=128,
             top_blocks=128, top_tokens=1024, layout=_lib.TLS_MLA)
    assert lib.tls_cluster_size(ctypes.byref(c4), 2) > 0
    assert lib.tls_launch_count(ctypes.byref(c4), 2) == 4
    # token-kernel form: one CTA per pair where G <= 8 and the pair's candidate index fits shared memory
    assert lib.tls_cluster_size(ctypes.byref(c3), 5) == 4 and lib.tls_cluster_size(ctypes.byref(c2), 5) == 4
    monkeypatch.setenv("TLS_K2_FORM", "1")
    assert lib.tls_cluster_size(ctypes.byref(c3), 5) == 1
    monkeypatch.delenv("TLS_K2_FORM")
    assert lib.tls_cluster_size(ctypes.byref(c4), 5) == 6  # MLA, G = 32: token_pair_nt_kernel
    c3kb = cfg(batch=32, num_q_heads=64, num_kv_heads=8, max_seq_len=98304, top_blocks=256, top_tokens=1024)
    assert lib.tls_cluster_size(ctypes.byref(c3kb), 5) in (2, 3)  # 384 KB of candidates: too large for one CTA
    monkeypatch.setenv("TLS_K2_FORM", "cluster")
    assert lib.tls_cluster_size(ctypes.byref(c3), 5) == 2
    assert lib.tls_cluster_size(ctypes.byref(c4), 5) in (2, 3)
    monkeypatch.delenv("TLS_K2_FORM")


def test_cluster_override(lib, monkeypatch):
    c = cfg()
    for cs in (1, 2, 4, 8, 16):
        monkeypatch.setenv("TLS_CLUSTER", str(cs))
        assert lib.tls_cluster_size(ctypes.byref(c), 2) == cs
        assert lib.tls_cluster_size(ctypes.byref(c), 1) == cs


def test_workspace_init_validates(lib):
    c = cfg()
    need = lib.tls_workspace_bytes(ctypes.byref(c), 2)
    # too small -> TLS_ERR_WORKSPACE before anything is enqueued (no GPU needed)
    assert lib.tls_workspace_init(ctypes.byref(c), 2, 16, need - 1, None) == _lib.TLS_ERR_WORKSPACE
    assert lib.tls_workspace_init(ctypes.byref(c), 7, 16, need, None) == _lib.TLS_ERR_INPUT
