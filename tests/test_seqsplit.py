"""Sequence-split decode (paper_2604_07815_b200/seqsplit.py) on CPU: the orchestration
-- block-aligned ranges, local top-k_b -> all_gather -> global top-k_b, per-rank softmax statistics ->
all_gather -> globally normalised alpha~, local top-k_t -> all_gather -> global top-k_t,
per-rank partial attention -> all_gather -> LSE merge -- reproduces the oracle's UNSPLIT decode of
every pair exactly (same M_t and S_t; output to fp64 rounding).  The per-call semantics are evaluated by the
fp64 oracle (tests/seqsplit_oracle_kernels.py); the CUDA kernels are checked on the GPU by
tests/test_gpu_seqsplit.py.  P = 2 over gloo (two processes), P = 3 and 4 in one process."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tls_oracle as O
from paper_2604_07815_b200 import ops
from paper_2604_07815_b200 import seqsplit as SS
from paper_2604_07815_b200 import workloads as W
from tests import seqsplit_oracle_kernels as K

WL = W.Workload("ss-cpu", 2, 8, 2, 64, 64, 3000, block_size=64, d_c=16, top_blocks=8, top_tokens=96,
                dtype=torch.float32)


def _setup():
    inputs = W.make_inputs(WL, seed=7, device="cpu", pattern="peaked", seq_lens=[3000, 2333])
    channels = [np.arange(g, WL.d_k, WL.d_k // WL.d_c)[: WL.d_c] for g in range(WL.num_kv_heads)]
    cfg = ops.TLSConfig(**WL.config_kwargs())
    return cfg, inputs, channels


def _states(cfg, inputs, channels, P):
    return [K.rank_state(cfg, inputs, channels, t0, L) for t0, L in SS.split_ranges(cfg.max_seq_len, cfg.block_size, P)]


def _check_against_unsplit(cfg, inputs, channels, res):
    out, lse, m_glob, s_glob, n_glob = res
    G = WL.num_q_heads // WL.num_kv_heads
    prm = O.TLSParams(block_size=WL.block_size, top_blocks=WL.top_blocks, top_tokens=WL.top_tokens, sm_scale=WL.scale)
    for b in range(WL.batch):
        n = int(inputs["seq_lens"][b])
        for g in range(WL.num_kv_heads):
            q = inputs["q"][b, g * G:(g + 1) * G].double().numpy()
            keys = inputs["k_cache"][b, g, :n].double().numpy()
            vals = inputs["v_cache"][b, g, :n].double().numpy()
            ref = O.tls_pair(q, keys, vals, channels[g], prm)
            mb = m_glob[b, g].numpy()
            assert np.array_equal(mb[mb >= 0], ref["block_ids"]), (b, g)
            nt = int(n_glob[b, g])
            assert nt == len(ref["token_ids"])
            assert np.array_equal(s_glob[b, g, :nt].numpy(), ref["token_ids"]), (b, g)
            assert (s_glob[b, g, nt:] == -1).all()
            np.testing.assert_allclose(out[b, g * G:(g + 1) * G].numpy(), ref["out"], rtol=0, atol=1e-10)
            np.testing.assert_allclose(lse[b, g * G:(g + 1) * G].numpy(), ref["lse"], rtol=0, atol=1e-10)


def test_split_ranges_cover_the_sequence():
    for S, B, P in [(3000, 64, 2), (3000, 64, 3), (4096, 64, 4), (65, 64, 2), (98304, 64, 8)]:
        r = SS.split_ranges(S, B, P)
        assert r[0][0] == 0 and all(t0 % B == 0 for t0, _ in r)
        assert sum(L for _, L in r) == S
        assert all(r[i][0] + r[i][1] == r[i + 1][0] for i in range(P - 1) if r[i + 1][1] > 0)


@pytest.mark.parametrize("P", [1, 3, 4])
def test_in_process_ranks_match_unsplit_oracle(P):
    cfg, inputs, channels = _setup()
    res = SS.run_ranks(_states(cfg, inputs, channels, P), inputs["q"], inputs["seq_lens"], kern=K.OracleKernels)
    for r in res:  # every rank ends with the same result
        for a, b in zip(r, res[0]):
            assert torch.equal(a, b)
    _check_against_unsplit(cfg, inputs, channels, res[0])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, inputs, channels = _setup()
        t0, L = SS.split_ranges(cfg.max_seq_len, cfg.block_size, world)[rank]
        st = K.rank_state(cfg, inputs, channels, t0, L)
        res = SS.decode_step(st, inputs["q"], inputs["seq_lens"], SS.TorchDistComm(), kern=K.OracleKernels)
        if rank == 0:
            _check_against_unsplit(cfg, inputs, channels, res)
        q.put((rank, "ok"))
    except BaseException as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_match_unsplit_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert got == {0: "ok", 1: "ok"}, got
