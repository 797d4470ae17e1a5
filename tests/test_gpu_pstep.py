"""GPU parity of the persistent step kernel (pstep.cu: one launch, ready-queue scheduled work items of every
stage of every pair) against the fp64 oracle, with the same per-pair checks as the kernel chain
(tests/test_gpu_parity.py check_pair): block/token sets, ln alpha~, attention output and lse.

Covers the supported specialisation (bf16 GQA, d = 128, G <= 8, d_c = 32, B = 64): ragged lengths, several
attention slices per pair, tls_select alone (no ATT items), repeated calls on one workspace (the
scheduler and per-pair counters reset themselves), and the full C2/C3 sizes.
"""
from __future__ import annotations

import pytest
import torch

from oracle import tls_oracle as O
from tests import parity as P
from tests import test_gpu_parity as T

pytestmark = pytest.mark.gpu

tls = pytest.importorskip("paper_2604_07815_b200")
from paper_2604_07815_b200 import workloads as W  # noqa: E402

CASES = {
    "g4": W.Workload("p-g4", 3, 16, 4, 128, 128, 5000, top_blocks=16, top_tokens=256),
    "g8": W.Workload("p-g8", 2, 16, 2, 128, 128, 8192, top_blocks=32, top_tokens=512),
    "g2_long": W.Workload("p-g2", 2, 8, 4, 128, 128, 20000, top_blocks=128, top_tokens=1024),
}


@pytest.fixture(autouse=True)
def _pstep(monkeypatch):
    monkeypatch.setenv("TLS_PSTEP", "1")


def check_all(w, cfg, inputs, idx, res):
    stats = {"block_near_ties": 0, "token_near_ties": 0}
    for b in range(w.batch):
        for g in range(w.num_kv_heads):
            T.check_pair(w, cfg, inputs, idx, res, b, g, stats)
    return stats


@pytest.mark.parametrize("name", list(CASES))
def test_pstep_decode_parity(name):
    w = CASES[name]
    cfg, inputs, idx = T.setup_case(w)
    assert tls.select_mode(cfg) == 3
    res = T.run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    print(f"{name}: near-ties {check_all(w, cfg, inputs, idx, res)}")


@pytest.mark.parametrize("ns", [1, 3, 8])
def test_pstep_attention_slices(ns, monkeypatch):
    monkeypatch.setenv("TLS_CLUSTER", str(ns))
    w = CASES["g4"]
    cfg, inputs, idx = T.setup_case(w, seed=1, pattern="peaked")
    assert tls.cluster_size(cfg, 2) == ns
    res = T.run_decode(cfg, inputs, idx)
    torch.cuda.synchronize()
    check_all(w, cfg, inputs, idx, res)


def test_pstep_repeated_calls_and_select_only():
    """Ten calls with changing queries on one workspace (decode and select-only interleaved) equal fresh
    results of the kernel chain's selections: the scheduler words and per-pair counters reset themselves."""
    w = CASES["g8"]
    cfg, inputs, idx = T.setup_case(w, seed=4)
    first = None
    for it in range(10):
        q = inputs["q"] if it % 2 == 0 else torch.flip(inputs["q"], dims=[1]).contiguous()
        if it % 3 == 2:
            bids, tids, ntok, tsc = tls.select(cfg, q, inputs["seq_lens"], idx)
            res = None
        else:
            res = tls.decode(cfg, q, inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
            bids, tids, ntok = res[2], res[3], res[4]
        torch.cuda.synchronize()
        if it == 0:
            first = (bids.clone(), tids.clone(), ntok.clone(), res[0].clone())
        if it % 2 == 0:
            assert torch.equal(bids, first[0]) and torch.equal(tids, first[1]) and torch.equal(ntok, first[2])
            if res is not None:
                assert torch.equal(res[0], first[3])
    check_all(w, cfg, inputs, idx, T.run_decode(cfg, inputs, idx))


def test_pstep_has_no_lag_mode():
    """Lag mode (guide_block_ids) is not implemented by the persistent kernel: reported, not run."""
    w = CASES["g4"]
    cfg, inputs, idx = T.setup_case(w, seed=5)
    guide = T.run_decode(cfg, inputs, idx)[2].clone()
    torch.cuda.synchronize()
    with pytest.raises(tls.TLSError, match="UNSUPPORTED"):
        tls.decode(cfg, inputs["q"], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx,
                   guide_block_ids=guide)


@pytest.mark.slow
@pytest.mark.parametrize("pattern", ["outlier", "uniform"])
@pytest.mark.parametrize("name", ["c2", "c3"])
def test_pstep_full_size(name, pattern):
    stats = T.run_full(W.CONFIGS[name], pattern)
    print(stats)
