"""GPU tests of the KV-offload engine (tls_cache_fetch; SURVEY §8(f)
f1): the K/V caches in pinned host memory, a GPU token cache, zero-copy
fetch of the missed selected tokens.

Parity: the offloaded step attends over exactly the selected tokens, so its
selections equal the resident tls_decode's bit for bit and its output matches
within the attention tolerance (the rows are gathered from cache slots in the
same selection order).  Cache invariants: after a fetch every selected token is
resident, the two slot maps are mutually consistent, and with capacity = k_t
the number of rows fetched equals |S_t \\ S_{t-1}| (the step-to-step locality
the paper exploits).

The asynchronous block-granular engine (tls_block_cache_update / _rows,
AsyncOffloadDecoder): with the one-step lag its selections equal the
resident lag-mode tls_decode (guide_block_ids = M_{t-1}) bit for bit, its output
matches within the attention tolerance, every selected token's block is
resident when the attention runs, the cache holds M_{t-1} u M_t, and each
update fetches at most |M_t minus M_{t-1}| blocks.
"""
from __future__ import annotations

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

tls = pytest.importorskip("paper_2604_07815_b200")
from paper_2604_07815_b200 import workloads as W  # noqa: E402
from tests.test_gpu_parity import setup_case  # noqa: E402

CASES = {
    "gqa": W.Workload("o-gqa", 2, 16, 2, 128, 128, 6000, top_blocks=16, top_tokens=256),
    "mla": W.Workload("o-mla", 2, 16, 1, 576, 512, 4133, d_c=128, top_blocks=16, top_tokens=256, layout="mla",
                      sm_scale=1.0 / math.sqrt(192.0)),
}


def check_cache(cfg, cache, tids, nt, slots):
    rows = cfg.batch * (cfg.num_kv_heads if cfg.layout == "gqa" else 1)
    sot = cache.slot_of_token.reshape(rows, -1)
    tos = cache.token_of_slot.reshape(rows, -1)
    t2, s2, n2 = tids.reshape(rows, -1), slots.reshape(rows, -1), nt.reshape(-1)
    for r in range(rows):
        k = int(n2[r])
        sel = t2[r, :k].long()
        sl = s2[r, :k].long()
        assert torch.equal(sot[r][sel].long(), sl)  # every selected token resident, in its slot
        assert torch.equal(tos[r][sl].long(), sel)  # and the slot points back to it
        assert int((tos[r] >= 0).sum()) == k  # the cache holds exactly the current selection


@pytest.mark.parametrize("name", list(CASES))
def test_offload_matches_resident_decode(name):
    w = CASES[name]
    cfg, inputs, idx = setup_case(w, seed=7)
    k_host = tls.host_kv(inputs["k_cache"])
    v_host = tls.host_kv(inputs["v_cache"]) if inputs["v_cache"] is not None else None
    cache = tls.alloc_token_cache(cfg, cfg.top_tokens, inputs["k_cache"].device)
    ref = tls.decode(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    res = tls.offload_decode(cfg, inputs["q"], k_host, v_host, inputs["seq_lens"], idx, cache)
    torch.cuda.synchronize()
    for a, b in zip(ref[2:6], res[2:6]):
        assert torch.equal(a, b)
    torch.testing.assert_close(res[0].float(), ref[0].float(), rtol=0, atol=2e-2)
    torch.testing.assert_close(res[1], ref[1], rtol=0, atol=1e-3)
    check_cache(cfg, cache, res[3], res[4], res[6])
    assert torch.equal(res[7], res[4])  # first step: every selected token was a miss


def test_offload_steps_fetch_only_the_new_tokens():
    w = CASES["gqa"]
    cfg, inputs, idx = setup_case(w, seed=8)
    k_host = tls.host_kv(inputs["k_cache"])
    v_host = tls.host_kv(inputs["v_cache"])
    cache = tls.alloc_token_cache(cfg, cfg.top_tokens, inputs["k_cache"].device)
    q = inputs["q"].clone()
    g = torch.Generator(device=q.device).manual_seed(3)
    prev = None
    for step in range(4):
        res = tls.offload_decode(cfg, q, k_host, v_host, inputs["seq_lens"], idx, cache)
        ref = tls.decode(cfg, q, inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
        torch.cuda.synchronize()
        assert torch.equal(res[3], ref[3])
        torch.testing.assert_close(res[0].float(), ref[0].float(), rtol=0, atol=2e-2)
        check_cache(cfg, cache, res[3], res[4], res[6])
        tids, nt = res[3], res[4]
        if prev is not None:
            for b in range(cfg.batch):
                for h in range(cfg.num_kv_heads):
                    cur = set(tids[b, h, : int(nt[b, h])].tolist())
                    old = set(prev[0][b, h, : int(prev[1][b, h])].tolist())
                    assert int(res[7][b, h]) == len(cur - old)
        prev = (tids.clone(), nt.clone())
        # a drifting query: the selection changes a little from step to step
        q = (q.float() + 0.05 * torch.randn(q.shape, generator=g, device=q.device)).to(q.dtype)


def check_block_cache(cfg, cache, keep_sets):
    """slot_of_block / block_of_slot are mutually consistent and hold every block of the kept sets."""
    rows = cfg.batch * cfg.num_kv_heads
    sob = cache.slot_of_block.reshape(rows, -1)
    bos = cache.block_of_slot.reshape(rows, -1)
    for r in range(rows):
        res = (sob[r] >= 0).nonzero().flatten()
        assert torch.equal(bos[r][sob[r][res].long()].long(), res)  # slot -> block -> slot round trip
        assert int((bos[r] >= 0).sum()) == len(res)
        for ks in keep_sets:
            for blk in ks[r]:
                assert int(sob[r][blk]) >= 0


@pytest.mark.parametrize("name", list(CASES))
def test_async_offload_matches_lag_mode_decode(name):
    w = CASES[name]
    cfg, inputs, idx = setup_case(w, seed=9)
    k_host = tls.host_kv(inputs["k_cache"])
    v_host = tls.host_kv(inputs["v_cache"]) if inputs["v_cache"] is not None else None
    eng = tls.AsyncOffloadDecoder(cfg, k_host, v_host, inputs["seq_lens"], idx)
    q = inputs["q"].clone()
    g = torch.Generator(device=q.device).manual_seed(5)
    prev = None
    rows = cfg.batch * cfg.num_kv_heads
    for step in range(4):
        res = eng.step(q)
        ref = tls.decode(cfg, q, inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx, guide_block_ids=prev)
        torch.cuda.synchronize()
        for a, b in zip(ref[2:6], res[2:6]):
            assert torch.equal(a, b)
        torch.testing.assert_close(res[0].float(), ref[0].float(), rtol=0, atol=2e-2)
        torch.testing.assert_close(res[1], ref[1], rtol=0, atol=1e-3)
        # the rows the attention read are the selected tokens' rows of resident blocks
        _, absent = tls.block_cache_rows(cfg, res[3], res[4], eng.cache)
        torch.cuda.synchronize()
        assert int(absent.sum()) == 0
        bids = res[2].reshape(rows, -1)
        cur = [[int(x) for x in bids[r] if int(x) >= 0] for r in range(rows)]
        keep = [cur] if prev is None else [cur, [[int(x) for x in prev.reshape(rows, -1)[r] if int(x) >= 0]
                                                  for r in range(rows)]]
        check_block_cache(cfg, eng.cache, keep)
        if prev is not None:  # blocks fetched = M_t minus what was resident before the update
            miss = eng.last_miss.reshape(-1)
            for r in range(rows):
                assert int(miss[r]) <= len(set(cur[r]) - set(keep[1][r]))
        prev = res[2].clone()
        q = (q.float() + 0.05 * torch.randn(q.shape, generator=g, device=q.device)).to(q.dtype)


def test_block_cache_rejects_small_capacity():
    w = CASES["gqa"]
    cfg, inputs, idx = setup_case(w, seed=1)
    k_host = tls.host_kv(inputs["k_cache"])
    v_host = tls.host_kv(inputs["v_cache"])
    cache = tls.alloc_block_cache(cfg, cfg.top_blocks, inputs["k_cache"].device)  # < 2 * top_blocks
    bids = torch.zeros((cfg.batch, cfg.num_kv_heads, cfg.top_blocks), dtype=torch.int32, device=k_host.device
                       if k_host.is_cuda else inputs["k_cache"].device)
    with pytest.raises(tls.TLSError):
        tls.block_cache_update(cfg, k_host, v_host, bids, cache)
