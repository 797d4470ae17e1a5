// fasttopk.cuh -- exact CTA-local top-k with the lower-index tie rule (U2)
// over order-preserving uint32 keys in shared memory (0 = not a candidate).
//
// Sample-bracket select (no atomics on the large array): 256 evenly spaced
// keys are ranked by comparison, a bracket [lo, hi] of sample values around
// the k-th position is counted over all keys with ballot / popc, and only the
// keys inside the bracket (typically a few hundred) are gathered and resolved
// by a range-histogram select.  A bracket that misses (rare) falls back to
// the range-histogram select over all keys.  Shared-memory atomics cost ~2
// cycles per lane on this part, so the histogram runs only on small sets.
#pragma once

#include "common.cuh"
#include "params.h"
#include "topk.cuh"

namespace tls {

constexpr int kFastBins = 2048;
constexpr int kBracketCap = kBracketWords;

struct FastTopKCtl {
  uint32_t hist[kFastBins];
  uint32_t samp[256];
  uint32_t red_min[kWarps], red_max[kWarps];
  int red_a[kWarps], red_b[kWarps];
  uint32_t lo, hi;
  int krem, bsel, above, bcount, cnt_a, cnt_b;
  uint32_t bkeys[32];
  uint32_t thr;
  int take_eq;
  int nvalid;
};

// Block-wide sums of two ints (every thread gets both totals).
__device__ __forceinline__ void block_sum2(int& a, int& b, FastTopKCtl& c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
    c.red_a[warp] = a;
    c.red_b[warp] = b;
  }
  __syncthreads();
  a = 0;
  b = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    a += c.red_a[w];
    b += c.red_b[w];
  }
  __syncthreads();
}

// Range-histogram select of the krem-th largest key value among the nonzero
// keys of `keys` within [lo, hi] (callers guarantee >= krem such keys).
// Returns the value in c.thr (ties are not resolved here).
__device__ inline void range_select(const uint32_t* keys, int n, uint32_t lo, uint32_t hi, int krem, FastTopKCtl& c,
                             TopKCtl& tk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    c.lo = lo;
    c.hi = hi;
    c.krem = krem;
  }
  __syncthreads();
  for (int iter = 0; iter < 8; ++iter) {
    const uint32_t l = c.lo, h = c.hi;
    const int kr0 = c.krem;
    const uint32_t span = h - l;
    const int shift = span == 0 ? 0 : max(0, 32 - __clz(span) - 11);
    const int nb = (int)(span >> shift) + 1;  // <= 2048
    for (int i = tid; i < nb; i += kThreads) c.hist[i] = 0;
    if (tid == 0) c.bcount = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kThreads) {
      const uint32_t k = keys[i];
      if (k >= l && k <= h && k) atomicAdd(&c.hist[(k - l) >> shift], 1u);
    }
    __syncthreads();
    int cnt[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int bi = nb - 1 - 8 * tid - j;
      cnt[j] = bi >= 0 ? (int)c.hist[bi] : 0;
      sum += cnt[j];
    }
    int total;
    const int excl = block_exclusive_scan(sum, tk.scan, &total);
    if (excl < kr0 && kr0 <= excl + sum) {
      int above = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (above + cnt[j] >= kr0) {
          c.bsel = nb - 1 - 8 * tid - j;
          c.above = above;
          break;
        }
        above += cnt[j];
      }
    }
    __syncthreads();
    const int b = c.bsel;
    const int kr = kr0 - c.above;
    const uint32_t blo = l + ((uint32_t)b << shift);
    const uint32_t bhi = shift == 0 ? blo : min(h, blo + ((1u << shift) - 1u));
    const int bc = (int)c.hist[b];
    if (shift == 0 || blo == bhi) {
      if (tid == 0) c.thr = blo;
      __syncthreads();
      return;
    }
    if (bc <= 32) {
      for (int i = tid; i < n; i += kThreads) {
        const uint32_t k = keys[i];
        if (k >= blo && k <= bhi && k) c.bkeys[atomicAdd(&c.bcount, 1)] = k;
      }
      __syncthreads();
      if (warp == 0) {
        const uint32_t mine = lane < bc ? c.bkeys[lane] : 0u;
        int rank = 0, eqn = 0;
        for (int j = 0; j < bc; ++j) {
          rank += c.bkeys[j] > mine;
          eqn += c.bkeys[j] == mine;
        }
        const bool is_thr = lane < bc && rank < kr && rank + eqn >= kr;
        const unsigned bal = __ballot_sync(0xffffffffu, is_thr);
        if (lane == __ffs(bal) - 1) c.thr = mine;
      }
      __syncthreads();
      return;
    }
    if (tid == 0) {
      c.lo = blo;
      c.hi = bhi;
      c.krem = kr;
    }
    __syncthreads();
  }
}

// Count keys > a and keys >= b over the array (ballot / popc, no atomics).
__device__ __forceinline__ void count_two(const uint32_t* keys, int n, uint32_t a, uint32_t b, int& ca, int& cb,
                                          FastTopKCtl& c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = 0, y = 0;
  for (int base = warp * 32; base < n; base += kThreads) {
    const int i = base + lane;
    const uint32_t k = i < n ? keys[i] : 0u;
    x += __popc(__ballot_sync(0xffffffffu, k > a && k));
    y += __popc(__ballot_sync(0xffffffffu, k >= b && k));
  }
  if (lane != 0) x = y = 0;
  block_sum2(x, y, c);
  ca = x;
  cb = y;
}

// Top-k over n keys.  Returns a TopK for topk_emit (offset 0, total = K).
// take_all (K >= number of nonzero keys) selects every nonzero key.
__device__ inline TopK fast_topk(const uint32_t* keys, int n, int K, bool take_all, FastTopKCtl& c, TopKCtl& tk,
                          uint32_t* scratch /* >= kBracketCap words of smem, or NULL */) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TopK r;
  r.offset = 0;
  r.total = K;
  if (take_all || K <= 0) {
    r.thr = 0;
    r.eq_mode = false;
    r.take_eq = 0;
    return r;
  }
  uint32_t thr = 0;
  bool done = false;
  if (n >= 1024 && scratch != nullptr) {
    // ---- 1. rank 256 evenly spaced samples (descending) ----
    const uint32_t sv = keys[(int)(((long long)tid * n) >> 8)];
    c.samp[tid] = sv;
    __syncthreads();
    int rank = 0;
    for (int j = 0; j < 256; ++j) {
      const uint32_t o = c.samp[j];
      rank += (o > sv) || (o == sv && j < tid);
    }
    __syncthreads();
    c.samp[rank] = sv;
    __syncthreads();
    // ---- 2. bracket around position K: count over all keys ----
    const int pidx = (int)(((long long)K << 8) / n);
    const int hi_i = max(0, pidx - 12), lo_i = min(255, pidx + 12);
    const uint32_t hiT = c.samp[hi_i], loT = c.samp[lo_i];
    int cgt, cge;
    count_two(keys, n, hiT, loT, cgt, cge, c);
    const bool hi_ok = cgt < K;
    const bool lo_ok = loT != 0u && cge >= K;
    if (hi_ok && lo_ok && cge - cgt <= kBracketCap) {
      // ---- 3. gather the bracket [loT, hiT] (ballot compaction) ----
      if (tid == 0) c.bcount = 0;
      __syncthreads();
      for (int base = warp * 32; base < n; base += kThreads) {
        const int i = base + lane;
        const uint32_t k = i < n ? keys[i] : 0u;
        const bool in = k && k >= loT && k <= hiT;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        int off = 0;
        if (lane == 0 && bal) off = atomicAdd(&c.bcount, __popc(bal));
        off = __shfl_sync(0xffffffffu, off, 0);
        if (in) scratch[off + __popc(bal & ((1u << lane) - 1u))] = k;
      }
      __syncthreads();
      const int nb = c.bcount;
      const int kr = K - cgt;
      if (nb <= 1024) {  // exact threshold by rank: the kr-th largest bracketed key
        if (tid == 0) c.thr = 0u;
        __syncthreads();
        for (int i = tid; i < nb; i += kThreads) {
          const uint32_t v = scratch[i];
          int gtc = 0, eqc = 0;
          for (int j = 0; j < nb; ++j) {
            const uint32_t o = scratch[j];
            gtc += o > v;
            eqc += o == v;
          }
          if (gtc < kr && gtc + eqc >= kr) c.thr = v;  // all writers write the same value
        }
        __syncthreads();
      } else {
        range_select(scratch, nb, loT, hiT, kr, c, tk);
      }
      thr = c.thr;
      done = true;
    }
  }
  if (!done) {
    // min / max of the nonzero keys, then range-histogram select over all keys
    uint32_t mn = 0xffffffffu, mx = 0u;
    for (int i = tid; i < n; i += kThreads) {
      const uint32_t k = keys[i];
      if (k) {
        mn = min(mn, k);
        mx = max(mx, k);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
      c.red_min[warp] = mn;
      c.red_max[warp] = mx;
    }
    __syncthreads();
    uint32_t a = 0xffffffffu, b = 0u;
    for (int w = 0; w < kWarps; ++w) {
      a = min(a, c.red_min[w]);
      b = max(b, c.red_max[w]);
    }
    __syncthreads();
    range_select(keys, n, a, b, K, c, tk);
    thr = c.thr;
  }
  // ---- ties at thr: take K - #(keys > thr) of them, lowest index first ----
  int cgt, cge;
  count_two(keys, n, thr, thr, cgt, cge, c);
  r.thr = thr;
  r.eq_mode = true;
  r.take_eq = K - cgt;
  return r;
}

// Number of nonzero keys (block-wide).
__device__ __forceinline__ int count_nonzero(const uint32_t* keys, int n, FastTopKCtl& c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = 0, y = 0;
  for (int base = warp * 32; base < n; base += kThreads) {
    const int i = base + lane;
    x += __popc(__ballot_sync(0xffffffffu, i < n && keys[i] != 0u));
  }
  if (lane != 0) x = 0;
  block_sum2(x, y, c);
  return x;
}

}  // namespace tls
