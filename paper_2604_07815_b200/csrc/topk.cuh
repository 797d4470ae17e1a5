// topk.cuh -- emission of an exact top-k selection (readings U2-U4) over
// order-preserving uint32 keys held in shared memory.  A selection is
// described by TopK: {key > thr} plus, when several keys equal thr, the first
// take_eq of them in index order (ascending ids) -- the paper-silent tie rule
// U2.  Key 0 means "not a candidate" and is never taken.  The threshold
// itself comes from fast_topk (fasttopk.cuh).
#pragma once

#include "common.cuh"

namespace tls {

constexpr int kMaxCluster = 16;

struct TopKCtl {
  int scan[kWarps + 2];
};

struct TopK {
  uint32_t thr;
  int take_eq;
  int offset;
  int total;
  bool eq_mode;
};

// Emit this CTA's selected elements in local-index order: f(local_index,
// out_pos).  Warp w owns a contiguous segment of the keys and walks it 32
// consecutive keys at a time (coalesced, conflict-free shared loads); ranks
// come from ballot / popc prefixes and one block-level scan over the warps.
template <class F>
__device__ void topk_emit(const uint32_t* keys, int nloc, const TopK& t, TopKCtl& ctl, F f) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int seg = (((nloc + kWarps - 1) / kWarps) + 31) & ~31;
  const int s0 = min(warp * seg, nloc), s1 = min(s0 + seg, nloc);
  int cgt = 0, ceq = 0;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + lane;
    const uint32_t k = i < s1 ? keys[i] : 0u;
    cgt += __popc(__ballot_sync(0xffffffffu, k > t.thr));
    ceq += __popc(__ballot_sync(0xffffffffu, t.eq_mode && k != 0u && k == t.thr));
  }
  __shared__ int wgt[kWarps], weq[kWarps], wsel[kWarps], weqb[kWarps];
  if (lane == 0) {
    wgt[warp] = cgt;
    weq[warp] = ceq;
  }
  __syncthreads();
  if (tid == 0) {
    int eb = 0, sb = 0;
    for (int w = 0; w < kWarps; ++w) {
      weqb[w] = eb;
      wsel[w] = sb;
      const int take = t.eq_mode ? min(max(t.take_eq - eb, 0), weq[w]) : 0;
      eb += weq[w];
      sb += wgt[w] + take;
    }
  }
  __syncthreads();
  int eq_seen = weqb[warp], pos = t.offset + wsel[warp];
  for (int base = s0; base < s1; base += 32) {
    const int i = base + lane;
    const uint32_t k = i < s1 ? keys[i] : 0u;
    const bool gt = k > t.thr;
    const bool eq = t.eq_mode && k != 0u && k == t.thr;
    const unsigned beq = __ballot_sync(0xffffffffu, eq);
    const bool sel = gt || (eq && eq_seen + __popc(beq & lt) < t.take_eq);
    const unsigned bsel = __ballot_sync(0xffffffffu, sel);
    if (sel) f(i, pos + __popc(bsel & lt));
    pos += __popc(bsel);
    eq_seen += __popc(beq);
  }
  __syncthreads();
}


// One-pass emit when the caller already knows, for the segmentation used by
// topk_emit (warp w owns [w*seg, (w+1)*seg), seg = ceil(n/8) rounded up to
// 128), each warp's count of keys > thr (wgt_in) and == thr (weq_in).  Four
// 32-key groups per iteration (independent ballots first, then the writes).
template <class F>
__device__ void topk_emit_counted(const uint32_t* keys, int nloc, const TopK& t, const int* wgt_in, const int* weq_in,
                                  F f) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int seg = (((nloc + kWarps - 1) / kWarps) + 127) & ~127;
  const int s0 = min(warp * seg, nloc), s1 = min(s0 + seg, nloc);
  int eq_seen = 0, pos = t.offset;
  for (int w = 0; w < warp; ++w) {
    const int take = t.eq_mode ? min(max(t.take_eq - eq_seen, 0), weq_in[w]) : 0;
    pos += wgt_in[w] + take;
    eq_seen += weq_in[w];
  }
  for (int base = s0; base < s1; base += 128) {
    uint32_t k[4];
    unsigned beq[4], bgt[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = base + 32 * u + lane;
      k[u] = i < s1 ? keys[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bgt[u] = __ballot_sync(0xffffffffu, k[u] > t.thr);
      beq[u] = __ballot_sync(0xffffffffu, t.eq_mode && k[u] != 0u && k[u] == t.thr);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      // ties taken in index order: this group's eq lanes below `lane` plus all earlier ones
      const int room = t.take_eq - eq_seen;  // ties still allowed before this group
      unsigned tie_ok = 0u;
      if (beq[u]) {
        if (room >= __popc(beq[u])) {
          tie_ok = beq[u];
        } else if (room > 0) {
          unsigned m = beq[u];
          for (int r = 0; r < room; ++r) {
            const unsigned low = m & (~m + 1u);
            tie_ok |= low;
            m &= m - 1u;
          }
        }
      }
      const unsigned bsel = bgt[u] | tie_ok;
      if ((bsel >> lane) & 1u) f(base + 32 * u + lane, pos + __popc(bsel & lt));
      pos += __popc(bsel);
      eq_seen += __popc(beq[u]);
    }
  }
  __syncthreads();
}

}  // namespace tls
