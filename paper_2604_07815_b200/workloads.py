"""Seeded synthetic decode workloads (DESIGN.md §4 "input recipe").

This module only draws random inputs; it holds none of the method's
arithmetic, so it may serve both the CUDA path and the oracle (tests,
bench.py).  Shapes follow BASELINE.json's configs; value distributions are a
proxy for the paper's RULER / LongBench workloads, which need real
models:

* ``uniform``  q, K, V ~ N(0, 1)
* ``outlier``  as uniform, with 8 fixed channels of q and K scaled x4 (the
               key statistics that motivate channel selection)
* ``peaked``   outlier + 32 planted tokens per pair whose keys are pushed
               towards the group's mean query (a needle-in-a-haystack analogue,
               SPEC S:614): K_j += beta * sqrt(d) * qbar / |qbar|, beta = 4

Every random role (q, K, V, positions, calibration queries) has its own
``torch.Generator`` seeded from (seed, role), so inputs are reproducible on
either device.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import torch

ROLES = {"q": 1, "k": 2, "v": 3, "plant": 4, "qcal": 5, "outlier": 6, "lens": 7}


@dataclass(frozen=True)
class Workload:
    name: str
    batch: int
    num_q_heads: int
    num_kv_heads: int
    d_k: int
    d_v: int
    context: int  # n, tokens already in the cache
    block_size: int = 64  # B
    d_c: int = 32  # 32 GQA / 128 MLA
    top_blocks: int = 128  # k_b
    top_tokens: int = 1024  # k_t (1024 = the LongBench budget P:406)
    dtype: torch.dtype = torch.bfloat16
    layout: str = "gqa"
    sm_scale: float | None = None
    max_seq_len: int | None = None

    @property
    def S(self) -> int:
        return self.max_seq_len or self.context

    @property
    def scale(self) -> float:
        return self.sm_scale if self.sm_scale is not None else 1.0 / math.sqrt(self.d_k)

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)

    def config_kwargs(self) -> dict:
        return dict(batch=self.batch, num_q_heads=self.num_q_heads, num_kv_heads=self.num_kv_heads, d_k=self.d_k,
                    d_v=self.d_v, max_seq_len=self.S, block_size=self.block_size, d_c=self.d_c,
                    top_blocks=self.top_blocks, top_tokens=self.top_tokens, sm_scale=self.scale, dtype=self.dtype,
                    layout=self.layout)


# BASELINE.json configs[0..4]
CONFIGS = {
    # single-sequence GQA, fp32, oracle runs in seconds
    "c1": Workload("c1-gqa-fp32-4k", 1, 4, 1, 128, 128, 4096, top_blocks=8, top_tokens=128, dtype=torch.float32),
    # Qwen3-8B shape: 32 q / 8 KV heads, d=128, 48k context, batch 16
    "c2": Workload("c2-qwen3-8b-48k-b16", 16, 32, 8, 128, 128, 48 * 1024),
    # Qwen3-32B shape: 64 q / 8 KV heads, d=128, 96k context, batch 32 (headline, 1 GPU)
    "c3": Workload("c3-qwen3-32b-96k-b32", 32, 64, 8, 128, 128, 96 * 1024),
    # GLM-4.7-Flash-shaped MLA: 32 heads, one latent head d_k = 512 + 64 rope, d_v = 512 (reading U12)
    "c4": Workload("c4-glm47flash-mla-64k-b32", 32, 32, 1, 576, 512, 64 * 1024, d_c=128, layout="mla",
                   sm_scale=1.0 / math.sqrt(192.0)),
    # offload: Qwen3-8B shape at 96k, batch 64 (GPU-side operator shape)
    "c5": Workload("c5-offload-qwen3-8b-96k-b64", 64, 32, 8, 128, 128, 96 * 1024),
}


def _gen(seed: int, role: str, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + ROLES[role] * 7919) & 0x7FFF_FFFF_FFFF)
    return g


def _outlier_channels(w: Workload, seed: int) -> torch.Tensor:
    g = _gen(seed, "outlier", "cpu")
    return torch.randperm(w.d_k, generator=g)[:8]


def make_inputs(w: Workload, seed: int = 0, pattern: str = "outlier", device="cuda", seq_lens=None,
                ragged: bool = False) -> dict:
    """q [B, Hq, d_k], k_cache / v_cache (GQA [B, Hkv, S, d]; MLA k only [B, S, d_k]), seq_lens int32 [B]."""
    dev = torch.device(device)
    dt = w.dtype
    mla = w.layout == "mla"
    if seq_lens is None:
        if ragged:
            g = _gen(seed, "lens", "cpu")
            lo = max(1, w.context // 2)
            seq_lens = torch.randint(lo, w.context + 1, (w.batch,), generator=g, dtype=torch.int32)
        else:
            seq_lens = torch.full((w.batch,), w.context, dtype=torch.int32)
    seq_lens = torch.as_tensor(seq_lens, dtype=torch.int32).to(dev)
    gq = _gen(seed, "q", dev)
    q = torch.randn((w.batch, w.num_q_heads, w.d_k), generator=gq, device=dev, dtype=torch.float32)
    kshape = (w.batch, w.S, w.d_k) if mla else (w.batch, w.num_kv_heads, w.S, w.d_k)
    k = torch.empty(kshape, dtype=dt, device=dev)
    gk = _gen(seed, "k", dev)
    for b in range(w.batch):  # per batch row: bounded temporaries at 96k x batch 32
        k[b] = torch.randn(kshape[1:], generator=gk, device=dev, dtype=torch.float32).to(dt)
    v = None
    if not mla:
        v = torch.empty((w.batch, w.num_kv_heads, w.S, w.d_v), dtype=dt, device=dev)
        gv = _gen(seed, "v", dev)
        for b in range(w.batch):
            v[b] = torch.randn(v.shape[1:], generator=gv, device=dev, dtype=torch.float32).to(dt)
    if pattern in ("outlier", "peaked"):
        oc = _outlier_channels(w, seed).to(dev)
        q[..., oc] *= 4.0
        k[..., oc] = (k[..., oc].float() * 4.0).to(dt)
    if pattern == "peaked":
        gp = _gen(seed, "plant", dev)
        G = w.num_q_heads // w.num_kv_heads
        beta = 4.0
        for b in range(w.batch):
            n = int(seq_lens[b].item())
            for gi in range(w.num_kv_heads):
                qbar = q[b, gi * G:(gi + 1) * G].mean(0)
                push = beta * math.sqrt(w.d_k) * qbar / qbar.norm()
                pos = torch.randint(0, n, (32,), generator=gp, device=dev)
                if mla:
                    k[b, pos] = (k[b, pos].float() + push).to(dt)
                else:
                    k[b, gi, pos] = (k[b, gi, pos].float() + push).to(dt)
    q = q.to(dt)
    return {"q": q, "k_cache": k, "v_cache": v, "seq_lens": seq_lens}


def make_queries(w: Workload, count: int, seed: int = 0, pattern: str = "outlier", device="cuda") -> torch.Tensor:
    """``count`` further decode queries of the same distribution: [count, B, Hq, d_k]."""
    dev = torch.device(device)
    g = _gen(seed + 17, "q", dev)
    q = torch.randn((count, w.batch, w.num_q_heads, w.d_k), generator=g, device=dev, dtype=torch.float32)
    if pattern in ("outlier", "peaked"):
        q[..., _outlier_channels(w, seed).to(dev)] *= 4.0
    return q.to(w.dtype)


def calibration_sample(w: Workload, inputs: dict, seed: int = 0, n_q: int = 64, n_k: int = 1024,
                       pattern: str = "outlier"):
    """Held-out calibration set D_cal (reading U6): fresh queries of the same
    distribution [n_q, Hq, d_k] and the first n_k cached keys of sequence 0 per KV
    head [Hkv, n_k, d_k]."""
    dev = inputs["q"].device
    g = _gen(seed, "qcal", dev)
    qc = torch.randn((n_q, w.num_q_heads, w.d_k), generator=g, device=dev, dtype=torch.float32)
    if pattern in ("outlier", "peaked"):
        qc[..., _outlier_channels(w, seed).to(dev)] *= 4.0
    qc = qc.to(w.dtype)
    n_k = min(n_k, int(inputs["seq_lens"][0].item()))
    k = inputs["k_cache"]
    if w.layout == "mla":
        kc = k[0, :n_k].unsqueeze(0).contiguous()
    else:
        kc = k[0, :, :n_k].contiguous()
    return qc, kc
