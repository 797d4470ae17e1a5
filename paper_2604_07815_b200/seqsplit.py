"""Sequence-split decode: one very long context split along the sequence over P ranks,
merged exactly.

Pairs (batch element, KV head) shard with no collective (dist.py).  A single sequence too long for one GPU is
split instead along the sequence: rank r holds the block-aligned token range [t0_r, t0_r + L) of every sequence
-- its slice of the KV cache and an index built over that slice.  One decode step then needs four small
exchanges, because three decisions of the method are global over the whole sequence:

1. top-k_b: each rank scores its blocks (a1) and keeps its local top-k_b (score, global block id);
   the global top-k_b is contained in the union of the local ones, so all_gather + one more exact top-k over
   the P*k_b candidates gives every rank the same M_t.
2. alpha~ is a softmax over ALL candidate tokens J of M_t, which are spread over the ranks: each rank
   computes per-head (max, sum) over its candidates, all_gather, and every rank merges them (LSE identity)
   inside the key kernel -> globally normalised ln alpha~ for its own candidates.
3. top-k_t: local top-k_t, all_gather, global top-k_t -> the same S_t everywhere.
4. attention: each rank attends over the tokens of S_t it holds -> partial (out, lse); all_gather;
   LSE merge -> the output.

Every arithmetic step runs in libtls.so kernels (include/tls.h: tls_block_scores, tls_block_topk,
tls_topk_rows, tls_select_range, tls_token_stats, tls_token_keys, tls_sparse_attend_f32, tls_attn_merge); this
module only sequences the calls and the collectives.  ``comm`` performs the all_gathers (NCCL over NVLink in
production, any torch.distributed backend, or a loopback that simulates P ranks in one process); ``kern``
defaults to the CUDA binding (ops.py) -- tests substitute other implementations of the same calls to check
the orchestration on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops


def split_ranges(max_seq_len: int, block_size: int, world: int) -> list[tuple[int, int]]:
    """Block-aligned token ranges [t0, t0 + L) of the P ranks (the last may be shorter)."""
    nblocks = -(-max_seq_len // block_size)
    per = -(-nblocks // world)
    out = []
    for r in range(world):
        t0 = min(r * per * block_size, max_seq_len)
        out.append((t0, min(per * block_size, max_seq_len - t0)))
    return out


def local_seq_lens(seq_lens: torch.Tensor, t0: int, length: int) -> torch.Tensor:
    """Tokens of each sequence that fall in [t0, t0 + length)."""
    return (seq_lens.to(torch.int64) - t0).clamp(0, length).to(torch.int32)


class TorchDistComm:
    """all_gather over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """[P, *t.shape] in rank order."""
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.stack(parts)


@dataclass
class RankState:
    """What rank r holds for one layer: its config over the local range, index, KV slice and the range."""

    cfg: ops.TLSConfig  # max_seq_len = L (the local cache length); top_blocks / top_tokens as the operator's
    index: ops.TLSIndex
    k_cache: torch.Tensor
    v_cache: torch.Tensor | None
    t0: int  # first global token of the range (a multiple of block_size)


def decode_step(st: RankState, q: torch.Tensor, seq_lens: torch.Tensor, comm, kern=ops):
    """One exact decode step of the sequence-split operator on this rank.

    seq_lens: GLOBAL sequence lengths [batch] (int32, on the rank's device).  Returns
    (out [batch, Hq, d_v], lse [batch, Hq], block_ids [batch, Hkv, k_b] global M_t,
    token_ids [batch, Hkv, k_t] global S_t, num_tokens [batch, Hkv]) -- identical on every rank.
    """
    cfg = st.cfg
    B = cfg.block_size
    blk0 = st.t0 // B
    L = cfg.max_seq_len
    lens = local_seq_lens(seq_lens, st.t0, L)
    # 1. a1 on the local blocks, local top-k_b, global top-k_b
    scores = kern.block_scores(cfg, q, lens, st.index)
    lk, lb = kern.block_topk(cfg, scores, lens, blk0)
    gk = comm.all_gather(lk)  # [P, batch, Hkv, k_b]
    gb = comm.all_gather(lb)
    _, m_glob, _ = kern.topk_rows(_cat_parts(gk), _cat_parts(gb), cfg.top_blocks)  # M_t, ascending global ids
    # 2. this rank's blocks of M_t; its softmax statistics of a3
    m_loc, _ = kern.select_range(m_glob, blk0, blk0 + (L + B - 1) // B)
    stats = kern.token_stats(cfg, q, lens, st.index, m_loc)
    stats_parts = comm.all_gather(stats)  # [P, batch, Hkv, G, 2]
    # 3. globally normalised ln alpha~ of the local candidates; local then global top-k_t
    keys, tids = kern.token_keys(cfg, q, lens, st.index, m_loc, stats_parts, st.t0)
    tk, tt, _ = kern.topk_rows(keys, tids, cfg.top_tokens)
    gtk = comm.all_gather(tk)
    gtt = comm.all_gather(tt)
    _, s_glob, n_glob = kern.topk_rows(_cat_parts(gtk), _cat_parts(gtt), cfg.top_tokens)  # S_t
    # 4. attention over the local tokens of S_t, LSE merge of the P partials
    s_loc, n_loc = kern.select_range(s_glob, st.t0, st.t0 + L)
    o_part, lse_part = kern.sparse_attend(cfg, q, st.k_cache, st.v_cache, s_loc, n_loc, out_f32=True)
    out, lse = kern.attn_merge(cfg, comm.all_gather(o_part), comm.all_gather(lse_part))
    return out, lse, m_glob, s_glob, n_glob


def _cat_parts(x: torch.Tensor) -> torch.Tensor:
    """[P, batch, Hkv, k] -> [batch, Hkv, P * k] (rank order: ids stay ascending, ranks hold ascending ranges)."""
    P = x.shape[0]
    return x.permute(1, 2, 0, 3).reshape(x.shape[1], x.shape[2], P * x.shape[3]).contiguous()


def run_ranks(states: list[RankState], q: torch.Tensor, seq_lens: torch.Tensor, kern=ops):
    """Run decode_step for P simulated ranks in one process, the all_gathers served in lockstep
    (a generator per rank yields at each collective)."""
    import threading

    P = len(states)
    barrier = threading.Barrier(P)
    slots: list = [None] * P
    results: list = [None] * P
    errors: list = []
    stream_dev = q.device

    class _Comm:
        world = P

        def __init__(self, rank):
            self.rank = rank

        def all_gather(self, t):
            slots[self.rank] = t
            barrier.wait()
            out = torch.stack([s.to(t.device) for s in slots])
            barrier.wait()
            return out

    def worker(r):
        try:
            if stream_dev.type == "cuda":
                torch.cuda.set_device(stream_dev)
            results[r] = decode_step(states[r], q, seq_lens, _Comm(r), kern)
        except BaseException as e:  # surface the first failure, release the others
            errors.append(e)
            barrier.abort()

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return results
