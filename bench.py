#!/usr/bin/env python
"""Benchmark of the AsyncTLS decode operator on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl tls|reference]

One *step* = one tls_decode call (4 launches) = the whole hot path (block scores,
top-k_b, token scores, top-k_t, sparse attention) for every (batch, KV-head)
pair of one synthetic decode batch, with the KV cache and index resident in
HBM.  Default workload: configs[2] of BASELINE.json (Qwen3-32B shape, 96k
context, batch 32) -- the north star's headline "96k context on 1 GPU".
Prints ONE JSON line (rank 0).  See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TLS decode op µs/step & HBM GB/s vs roofline at 48k/96k; decode tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--pattern", default="outlier", choices=["uniform", "outlier", "peaked"])
    ap.add_argument("--impl", default="tls", choices=["tls", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default, BASELINE.json configs[2]): the fixed problem sharded by KV head (GQA) "
                         "or batch (MLA) over the ranks; weak: every rank a full copy")
    ap.add_argument("--dry-run", action="store_true",
                    help="start the ranks, plan the shards, all_gather the plan, print one JSON line; no timing "
                         "(runs on CPU with gloo: checks the launcher)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    return ap.parse_args()


# ----------------------------------------------------------------- accounting
def algorithmic_bytes_per_pair(w) -> float:
    """SURVEY §8(d) / DESIGN.md §5: m*2*d_k*s + K_b*B*(d_c/2 + 8) + K_t*row + G*(d_k + d_v)*s."""
    s = 2 if w.dtype == torch.bfloat16 else 4
    G = w.num_q_heads // w.num_kv_heads
    m = math.ceil(w.context / w.block_size)
    kb = min(w.top_blocks, m)
    cand = min(kb * w.block_size, w.context)
    kt = min(w.top_tokens, cand)
    row = w.d_k * s if w.layout == "mla" else (w.d_k + w.d_v) * s
    return m * 2 * w.d_k * s + cand * (w.d_c // 2 + 8) + kt * row + G * (w.d_k + w.d_v) * s


def kernel_bytes_per_pair(w, mode: int = 2, token_kernel: str = "token_cluster_kernel") -> dict:
    """Algorithmic bytes per (batch, kv-head) pair of each launch of the step
    (the terms of algorithmic_bytes_per_pair split by the kernel that moves
    them; q is read by every kernel that uses it; intermediates -- scores,
    ids, token keys -- are excluded as in SURVEY §8(d))."""
    s = 2 if w.dtype == torch.bfloat16 else 4
    G = w.num_q_heads // w.num_kv_heads
    m = math.ceil(w.context / w.block_size)
    kb = min(w.top_blocks, m)
    cand = min(kb * w.block_size, w.context)
    kt = min(w.top_tokens, cand)
    row = w.d_k * s if w.layout == "mla" else (w.d_k + w.d_v) * s
    q = G * w.d_k * s
    a1 = m * 2 * w.d_k * s + q  # block summaries
    a3 = cand * (w.d_c // 2 + 8)  # INT4 codes + scale/zero of the candidate tokens
    a5 = kt * row + q + G * w.d_v * s  # selected K/V rows, o
    if mode == 3:  # the persistent step kernel: a1-a5 in one launch
        return {"pstep_kernel": a1 + a3 + a5}
    return {"select_kernel": a1, token_kernel: a3 + q, "attend_kernel": a5}


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload, {}).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms in the background."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [s for (t, s) in self.samples if t0 - 0.06 <= t <= t1 + 0.06] or [s for (_, s) in self.samples[-3:]]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            parts = [p.strip() for p in r.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except Exception:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ------------------------------------------------------------------ workload
def build_state(w, seed, device, pattern):
    import paper_2604_07815_b200 as tls
    from paper_2604_07815_b200 import workloads as W

    inputs = W.make_inputs(w, seed=seed, pattern=pattern, device=device)
    cfg = tls.TLSConfig(**w.config_kwargs())
    q_cal, k_cal = W.calibration_sample(w, inputs, seed=seed, pattern=pattern)
    channels, _ = tls.calibrate_channels(cfg, q_cal, k_cal)
    idx = tls.alloc_index(cfg, channels)
    tls.build_index(cfg, inputs["k_cache"], inputs["seq_lens"], idx)
    queries = W.make_queries(w, 8, seed=seed, pattern=pattern, device=device)
    torch.cuda.synchronize()
    return cfg, inputs, idx, queries


def time_steps(fn, steps, warmup, flush, stream, on_timed_start=None):
    """Device time of `steps` calls of fn(i), L2 flushed before each (not timed)."""
    for i in range(warmup):
        flush()
        fn(i)
    torch.cuda.synchronize()
    if on_timed_start:
        on_timed_start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush()
        starts[i].record(stream)
        fn(i)
        ends[i].record(stream)
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


_POOL_PAIRS: dict = {}


def _pool_pair(key):
    """One sampled pair in a forked worker (1 BLAS thread): the oracle's decode step O3-O11, timed."""
    from oracle import tls_oracle as O

    try:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(1)
    except Exception:  # pragma: no cover
        ctx = None
    qg, keys, values, ch, index, prm = _POOL_PAIRS[key]
    t0 = time.perf_counter()
    O.tls_pair(qg, keys, values, ch, prm, index=index)
    return time.perf_counter() - t0


def cpu_baseline(w, inputs, idx_channels, budget_s, label):
    """The fp64 oracle as it stands (never tuned), timed on this host on a bounded sample of pairs:
    (i) one process, 1 BLAS thread; (ii) a multiprocessing.Pool over every core this process may use,
    each worker 1 BLAS thread, the sampled pairs spread over the workers (value = workers / mean per-pair
    time under that concurrent load).  The prefill index build (O2, O5) is not part of a decode step and is
    not timed."""
    import multiprocessing as mp

    import numpy as np

    from oracle import tls_oracle as O

    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    G = w.num_q_heads // w.num_kv_heads
    prm = O.TLSParams(block_size=w.block_size, top_blocks=w.top_blocks, top_tokens=w.top_tokens, sm_scale=w.scale)
    pairs = [(b, g) for b in range(w.batch) for g in range(w.num_kv_heads)]
    rng = np.random.default_rng(0)
    rng.shuffle(pairs)
    cores = len(os.sched_getaffinity(0))

    def pair_data(b, g):
        n = int(inputs["seq_lens"][b])
        qg = inputs["q"][b, g * G:(g + 1) * G].double().cpu().numpy()
        if w.layout == "mla":
            keys = inputs["k_cache"][b, :n].double().cpu().numpy()
            values = keys[:, : w.d_v]
        else:
            keys = inputs["k_cache"][b, g, :n].double().cpu().numpy()
            values = inputs["v_cache"][b, g, :n].double().cpu().numpy()
        ch = idx_channels[g].cpu().numpy()
        return qg, keys, values, ch, O.build_index_pair(keys, ch, w.block_size), prm

    done, spent = 0, 0.0
    ctx = threadpool_limits(1) if threadpool_limits else None
    if ctx:
        ctx.__enter__()
    try:
        for b, g in pairs:
            qg, keys, values, ch, index, _ = pair_data(b, g)
            t0 = time.perf_counter()
            O.tls_pair(qg, keys, values, ch, prm, index=index)
            spent += time.perf_counter() - t0
            done += 1
            if spent >= budget_s or done >= 64:
                break
    finally:
        if ctx:
            ctx.__exit__(None, None, None)
    per_pair = spent / done
    tokens_per_s = (1.0 / w.num_kv_heads) / per_pair  # a pair is 1/Hkv of one sequence's decode token
    runs = [{"value": tokens_per_s, "cores": 1, "sample": f"{done} pairs, one process",
             "ms_per_pair": per_pair * 1e3}]
    value, used = tokens_per_s, 1
    if cores > 1:  # (ii) every core: fork workers that inherit the sampled pairs (no pickling of the caches)
        n_pool = min(len(pairs), 2 * cores, 64)
        _POOL_PAIRS.clear()
        for b, g in pairs[:n_pool]:
            _POOL_PAIRS[(b, g)] = pair_data(b, g)
        try:
            with mp.get_context("fork").Pool(cores) as pool:
                ts = pool.map(_pool_pair, list(_POOL_PAIRS.keys()), chunksize=1)
            mean = sum(ts) / len(ts)
            v = cores * (1.0 / w.num_kv_heads) / mean
            runs.append({"value": v, "cores": cores, "sample": f"{len(ts)} pairs over a {cores}-process pool",
                         "ms_per_pair": mean * 1e3})
            value, used = v, cores
        except Exception as e:  # pragma: no cover - reported, not fatal
            runs.append({"error": repr(e)})
        finally:
            _POOL_PAIRS.clear()
    return {"value": value, "unit": "tokens/s", "cores": used, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"(batch, kv-head) pairs of {label}: the oracle's decode step O3-O11 per pair (fp64 numpy, "
                      f"1 BLAS thread per process; prefill index build untimed), extrapolated to tokens/s",
            "runs": runs}


# ---------------------------------------------------------------------- arms
def run_reference(args, w, rank, world):
    """--impl reference: the oracle as it stands on host cores (rank 0 only)."""
    if rank != 0:
        return
    import numpy as np

    from oracle import tls_oracle as O
    from paper_2604_07815_b200 import workloads as W

    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    # the same seeded workload as the tls arm; the oracle reads a fresh pair per step
    inputs = W.make_inputs(w, seed=0, pattern=args.pattern, device=dev)
    q_cal, k_cal = W.calibration_sample(w, inputs, seed=0, pattern=args.pattern)
    G = w.num_q_heads // w.num_kv_heads
    chans = [O.calibrate_channels(q_cal[:, g * G:(g + 1) * G].double().cpu().numpy(),
                                  k_cal[g].double().cpu().numpy(), w.d_c)[0] for g in range(w.num_kv_heads)]
    prm = O.TLSParams(block_size=w.block_size, top_blocks=w.top_blocks, top_tokens=w.top_tokens, sm_scale=w.scale)
    pairs = [(b, g) for b in range(w.batch) for g in range(w.num_kv_heads)]
    cache = {}

    def prep(i):
        b, g = pairs[i % len(pairs)]
        if (b, g) not in cache:
            n = int(inputs["seq_lens"][b])
            qg = inputs["q"][b, g * G:(g + 1) * G].double().cpu().numpy()
            if w.layout == "mla":
                keys = inputs["k_cache"][b, :n].double().cpu().numpy()
                values = keys[:, : w.d_v]
            else:
                keys = inputs["k_cache"][b, g, :n].double().cpu().numpy()
                values = inputs["v_cache"][b, g, :n].double().cpu().numpy()
            cache.clear()
            cache[(b, g)] = (qg, keys, values, chans[g], O.build_index_pair(keys, chans[g], w.block_size))
        return cache[(b, g)]

    ctx = threadpool_limits(1) if threadpool_limits else None
    if ctx:
        ctx.__enter__()
    for i in range(args.warmup):
        qg, keys, values, ch, index = prep(i)
        O.tls_pair(qg, keys, values, ch, prm, index=index)
    times = []
    for i in range(args.steps):
        qg, keys, values, ch, index = prep(args.warmup + i)
        t0 = time.perf_counter()
        O.tls_pair(qg, keys, values, ch, prm, index=index)
        times.append(time.perf_counter() - t0)
    if ctx:
        ctx.__exit__(None, None, None)
    per_pair = sum(times) / len(times)
    value = (1.0 / w.num_kv_heads) / per_pair
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_pair * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "step": "one (batch, kv-head) pair per step (bounded sample)",
                   "batch": w.batch, "context": w.context},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{args.steps} pairs of {w.name}, O3-O11 per pair, fp64 numpy, 1 BLAS thread"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_tls(args, w, rank, world, local_rank):
    import paper_2604_07815_b200 as tls

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    w_full = w
    plan = None
    if args.scaling == "strong" and world > 1:
        # shard the fixed problem: KV heads (GQA) or batch (MLA) across ranks (dist.py; no collective in the step)
        from paper_2604_07815_b200.dist import shard_plan, shard_workload
        plan = shard_plan(w.batch, w.num_kv_heads, w.layout, world)
        w = shard_workload(w, rank, world)
    seed = rank if args.scaling == "weak" else 0
    cfg, inputs, idx, queries = build_state(w, seed, dev, args.pattern)
    stream = torch.cuda.current_stream(dev)
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # 2x the 126 MB L2

    def flush():
        flush_buf.fill_(1)

    out = torch.empty((w.batch, w.num_q_heads, w.d_v), dtype=w.dtype, device=dev)
    lse = torch.empty((w.batch, w.num_q_heads), dtype=torch.float32, device=dev)
    sel = (torch.empty((w.batch, w.num_kv_heads, w.top_blocks), dtype=torch.int32, device=dev),
           torch.empty((w.batch, w.num_kv_heads, w.top_tokens), dtype=torch.int32, device=dev),
           torch.empty((w.batch, w.num_kv_heads), dtype=torch.int32, device=dev),
           torch.empty((w.batch, w.num_kv_heads, w.top_tokens), dtype=torch.float32, device=dev))

    def step(i):
        tls.decode(cfg, queries[i % queries.shape[0]], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"],
                   idx, sel_out=sel, out=out, lse=lse)

    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    # the step as deployed: the token / attention kernels start under PDL while the previous one drains
    times = time_steps(step, args.steps, args.warmup, flush, stream)
    t_wall1 = time.time()
    if world > 1:
        torch.distributed.barrier()
    clocks.stop()
    # live per-kernel durations: a second timed pass with library events around each launch, on the
    # launch stream (events between launches also serialise them, so this pass runs without PDL overlap)
    n_k = max(10, min(args.steps, 200))
    tls.timing_enable(n_k + 3)
    kern_step_times = time_steps(step, n_k, 3, flush, stream, on_timed_start=lambda: tls.timing_read(cfg))
    kern_ms, kern_calls = tls.timing_read(cfg)
    tls.timing_enable(0)
    # e2e through the public API with HOST buffers: H2D q (pinned), decode, D2H out+lse
    q_host = queries.cpu().pin_memory()
    out_host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    lse_host = torch.empty(lse.shape, dtype=lse.dtype).pin_memory()
    q_dev = torch.empty_like(queries[0])

    def e2e_step(i):
        q_dev.copy_(q_host[i % q_host.shape[0]], non_blocking=True)
        tls.decode(cfg, q_dev, inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx, sel_out=sel,
                   out=out, lse=lse)
        out_host.copy_(out, non_blocking=True)
        lse_host.copy_(lse, non_blocking=True)

    e2e_times = time_steps(e2e_step, max(10, args.steps // 4), 3, flush, stream)
    assembly_us = None
    if world > 1 and plan is not None:  # NCCL all_gather of the sharded outputs: verification only, timed apart
        from paper_2604_07815_b200.dist import gather_outputs

        torch.distributed.barrier()
        ga = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(3):
            gather_outputs(out, plan["axis"])
        torch.cuda.synchronize()
        ga[0].record(stream)
        for _ in range(20):
            gather_outputs(out, plan["axis"])
        ga[1].record(stream)
        torch.cuda.synchronize()
        assembly_us = ga[0].elapsed_time(ga[1]) * 1e3 / 20

    ms = sum(times) / len(times)
    ms_e2e = sum(e2e_times) / len(e2e_times)
    names = tls.kernel_names(cfg)
    kavg = [kern_ms[k] / max(1, kern_calls) for k in names]
    if world > 1:
        t = torch.tensor([ms, ms_e2e, assembly_us or 0.0] + kavg, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, ms_e2e, assembly_us = float(t[0]), float(t[1]), (float(t[2]) if assembly_us is not None else None)
        kavg = [float(x) for x in t[3:]]
    if rank != 0:
        return
    # one decode token per sequence: weak -> every rank its own batch; strong -> the one (sharded) batch
    tokens_per_step = w.batch * world if args.scaling == "weak" else w_full.batch
    bytes_step = algorithmic_bytes_per_pair(w) * w.batch * w.num_kv_heads * world  # all ranks' pairs
    peak, peak_src = hbm_peak()
    achieved = bytes_step / (ms * 1e-3) / 1e9
    clk = clocks.summary(t_wall0, t_wall1)
    pairs = w.batch * w.num_kv_heads
    mode = tls.select_mode(cfg)
    kbytes = kernel_bytes_per_pair(w, mode, names[1] if len(names) > 1 else "token_cluster_kernel")
    ms_ser = sum(kern_step_times) / len(kern_step_times)
    kernels = {k: {"avg_us": kavg[i] * 1e3, "share": kavg[i] / ms_ser,
                   "algorithmic_bytes_per_launch": kbytes[k] * pairs,
                   "gbs": kbytes[k] * pairs / (kavg[i] * 1e-3) / 1e9 if kavg[i] > 0 else None}
               for i, k in enumerate(names)}
    dom = max(names, key=lambda k: kernels[k]["avg_us"])
    dom_ach = kernels[dom]["gbs"]
    line = {
        "metric": METRIC,
        "value": tokens_per_step / (ms * 1e-3),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "bf16" if w.dtype == torch.bfloat16 else "f32",
        "data": "synthetic",
        "config": {
            "workload": w_full.name, "batch_per_gpu": w.batch, "kv_heads_per_gpu": w.num_kv_heads,
            "global_batch": w.batch * world if args.scaling == "weak" else w_full.batch,
            "context": w.context, "num_q_heads": w.num_q_heads, "num_kv_heads": w.num_kv_heads, "d_k": w.d_k,
            "d_v": w.d_v, "layout": w.layout, "block_size": w.block_size, "d_c": w.d_c, "K_b": w.top_blocks,
            "K_t": w.top_tokens, "pattern": args.pattern, "cluster_size": tls.cluster_size(cfg, 2),
            "token_kernel": tls.kernel_names(cfg)[1] if mode != 3 else None,
            "select_mode": mode,
            "l2": "flushed before every timed step (256 MiB write, untimed)",
            "parallelism": (f"{world} rank(s), " + (f"{plan['axis']} shard of the fixed problem" if plan else
                            "each rank a full copy" if world > 1 else "one GPU") +
                            "; (batch, kv-head) pairs independent, no collective in the step"),
            "layer": "one attention layer (tokens/s = batch / layer-step time)",
        },
        "us_per_step": ms * 1e3,
        "per_gpu_us_per_step": ms * 1e3,
        "assembly_allgather_us": assembly_us,
        "hbm_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": dom_ach, "peak": peak, "unit": "GB/s", "frac": dom_ach / peak,
                     "traffic": ncu_traffic(w.name, dom), "peak_source": peak_src, "kernel": dom,
                     "algorithmic_bytes_per_launch": kernels[dom]["algorithmic_bytes_per_launch"],
                     "avg_launch_us": kernels[dom]["avg_us"],
                     "timing": f"CUDA events around each launch on its stream, {kern_calls} timed steps of a "
                               f"separate pass without PDL overlap (step {sum(kern_step_times) / len(kern_step_times) * 1e3:.1f} us "
                               f"there vs {ms * 1e3:.1f} us overlapped)"},
        "step_roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                          "algorithmic_bytes_per_step": bytes_step},
        "kernels": kernels,
        "e2e": {"value": tokens_per_step / (ms_e2e * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(queries[0].numel() * queries.element_size()),
                "d2h_bytes_per_step": int(out.numel() * out.element_size() + lse.numel() * 4),
                "ms_per_step": ms_e2e, "api": "paper_2604_07815_b200.decode (tls_decode) with pinned host q/out"},
        "gpu_launches": args.steps * tls.load().tls_launch_count(__import__("ctypes").byref(cfg.c()), 2),
        "clocks": clk,
        "p10_p90_ms": [sorted(times)[len(times) // 10], sorted(times)[(9 * len(times)) // 10]],
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(w, inputs, idx.channels, args.cpu_budget_s, w.name)
    elif not args.no_cpu_baseline:
        line["cpu_baseline"] = None
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args) -> int:
    """`--gpus N` without a launcher: re-exec this command under torch.distributed.run, one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
    return subprocess.call(cmd + sys.argv[1:])


def dry_run(args, w, rank, world):
    """Launcher check: every rank plans its shard, the plans are all_gathered, rank 0 prints one line."""
    import torch.distributed as dist

    from paper_2604_07815_b200.dist import shard_plan, shard_ranges

    mine = [rank, 0, 0, 0, 0]
    if world > 1 and args.scaling == "strong":
        bsl, hsl = shard_ranges(w.batch, w.num_kv_heads, w.layout, rank, world)
        mine = [rank, bsl.start, bsl.stop, hsl.start, hsl.stop]
    t = torch.tensor(mine)
    parts = [torch.empty_like(t) for _ in range(world)]
    if world > 1:
        dist.all_gather(parts, t)
    else:
        parts = [t]
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "scaling": args.scaling,
                          "config": {"workload": w.name},
                          "plan": shard_plan(w.batch, w.num_kv_heads, w.layout, world) if world > 1 else None,
                          "ranks": [p.tolist() for p in parts]}), flush=True)


def main():
    args = parse()
    from paper_2604_07815_b200 import workloads as W

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    w = W.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return
    if world > 1:
        if torch.cuda.is_available():
            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group("gloo")
    try:
        if args.dry_run:
            dry_run(args, w, rank, world)
        else:
            run_tls(args, w, rank, world, local_rank)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
