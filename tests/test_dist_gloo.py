"""Multi-process (gloo, world size 2, CPU) tests of the multi-GPU host logic:
the (batch, KV-head) pair partition covers every pair exactly once, each rank
computing its shard independently (here with the fp64 oracle standing in for
the per-GPU kernels) and gathering reproduces the single-process result, and
the max-over-ranks timing reduction bench.py uses."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tls_oracle as O
from paper_2604_07815_b200 import dist as D
from paper_2604_07815_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pair_outputs(w, inputs, channels, bsl, hsl):
    """Oracle decode of the pairs in the shard: out [b, Hq_shard, d_v]."""
    G = w.num_q_heads // w.num_kv_heads
    prm = O.TLSParams(block_size=w.block_size, top_blocks=w.top_blocks, top_tokens=w.top_tokens, sm_scale=w.scale)
    outs = []
    for b in range(bsl.start, bsl.stop):
        n = int(inputs["seq_lens"][b])
        heads = []
        for g in range(hsl.start, hsl.stop):
            q = inputs["q"][b, g * G:(g + 1) * G].double().numpy()
            if w.layout == "mla":
                keys = inputs["k_cache"][b, :n].double().numpy()
                vals = keys[:, : w.d_v]
            else:
                keys = inputs["k_cache"][b, g, :n].double().numpy()
                vals = inputs["v_cache"][b, g, :n].double().numpy()
            heads.append(O.tls_pair(q, keys, vals, channels[g], prm)["out"])
        outs.append(np.concatenate(heads, 0))
    return torch.tensor(np.stack(outs))


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = WORKLOADS[name]
        inputs = W.make_inputs(w, seed=4, device="cpu")
        channels = [np.arange(0, w.d_k, w.d_k // w.d_c)[: w.d_c] for _ in range(w.num_kv_heads)]
        plan = D.shard_plan(w.batch, w.num_kv_heads, w.layout, world)
        bsl, hsl = D.shard_ranges(w.batch, w.num_kv_heads, w.layout, rank, world)
        local = _pair_outputs(w, inputs, channels, bsl, hsl)
        full = D.gather_outputs(local, plan["axis"])
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py's max-over-ranks step time
        if rank == 0:
            ref = _pair_outputs(w, inputs, channels, slice(0, w.batch), slice(0, w.num_kv_heads))
            q.put((plan["axis"], float((full - ref).abs().max()), tuple(full.shape), float(t)))
    finally:
        dist.destroy_process_group()


WORKLOADS = {
    "gqa": W.Workload("d-gqa", 2, 8, 4, 64, 64, 700, top_blocks=4, top_tokens=64, dtype=torch.float32),
    "mla": W.Workload("d-mla", 4, 8, 1, 64, 32, 500, top_blocks=4, top_tokens=64, dtype=torch.float32,
                      layout="mla"),
}


@pytest.mark.parametrize("name,axis", [("gqa", "kv_head"), ("mla", "batch")])
def test_sharded_equals_single_process(name, axis):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, name, q), nprocs=2, join=True, start_method="spawn")
    got_axis, err, shape, tmax = q.get(timeout=60)
    w = WORKLOADS[name]
    assert got_axis == axis
    assert shape == (w.batch, w.num_q_heads, w.d_v)
    assert err == 0.0
    assert tmax == 2.0


def test_partition_covers_every_pair_once():
    for batch, hkv, layout, world in [(32, 8, "gqa", 8), (32, 8, "gqa", 2), (16, 8, "gqa", 4), (32, 1, "mla", 8),
                                      (6, 4, "gqa", 3)]:
        seen = []
        for r in range(world):
            bsl, hsl = D.shard_ranges(batch, hkv, layout, r, world)
            seen += [(b, g) for b in range(bsl.start, bsl.stop) for g in range(hsl.start, hsl.stop)]
        assert sorted(seen) == [(b, g) for b in range(batch) for g in range(hkv)]
    with pytest.raises(ValueError):
        D.shard_plan(5, 3, "gqa", 2)


def test_shard_workload_strong_scaling():
    w = W.CONFIGS["c3"]
    parts = [D.shard_workload(w, r, 8) for r in range(8)]
    assert all(p.num_kv_heads == 1 and p.num_q_heads == 8 for p in parts)
    w4 = W.CONFIGS["c4"]
    parts = [D.shard_workload(w4, r, 4) for r in range(4)]
    assert sum(p.batch for p in parts) == w4.batch


def test_bench_self_launches_n_ranks():
    """`bench.py --gpus 2` without a launcher re-execs itself under torch.distributed.run (two ranks, gloo on
    a CPU box): rank 0 prints n_gpus 2 and the strong-scaling KV-head shard plan of BASELINE.json configs[2]."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["plan"] == {"axis": "kv_head", "per_rank": 4}
    assert sorted(tuple(x) for x in line["ranks"]) == [(0, 0, 32, 0, 4), (1, 0, 32, 4, 8)]
