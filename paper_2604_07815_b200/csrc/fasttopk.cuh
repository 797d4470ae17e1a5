// fasttopk.cuh -- exact CTA-local top-k with the lower-index tie rule (U2)
// over order-preserving uint32 keys in shared memory (0 = not a candidate).
//
// Range-histogram select: the keys' actual range [lo, hi] is cut into <= 2048
// power-of-two-wide bins; one histogram pass finds the bin holding the k-th
// largest key, whose range becomes the new [lo, hi].  The search stops when
// that boundary bin is a single key value (then ties are taken in index
// order, as in topk_emit) or holds <= 32 keys, which one warp resolves
// exactly.  Typically one histogram pass instead of radix select's four.
#pragma once

#include "common.cuh"
#include "topk.cuh"

namespace tls {

constexpr int kFastBins = 2048;

struct FastTopKCtl {
  uint32_t hist[kFastBins];
  int scan[kWarps + 2];
  uint32_t red_min[kWarps], red_max[kWarps];
  uint32_t lo, hi;
  int krem, found, bsel, above;
  uint32_t bkeys[32];
  int bcount;
  uint32_t thr;
  int take_eq;
};

// Returns a TopK usable with topk_emit (offset 0).  K <= number of nonzero
// keys unless take_all.
__device__ TopK fast_topk(const uint32_t* keys, int n, int K, bool take_all, FastTopKCtl& c, TopKCtl& tk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TopK r;
  r.offset = 0;
  if (take_all || K <= 0) {
    r.thr = 0;
    r.eq_mode = false;
    r.take_eq = 0;
    r.total = 0;  // caller knows the count
    return r;
  }
  // ---- min / max of the candidate keys ----
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
  if (tid == 0) {
    uint32_t a = 0xffffffffu, b = 0u;
    for (int w = 0; w < kWarps; ++w) {
      a = min(a, c.red_min[w]);
      b = max(b, c.red_max[w]);
    }
    c.lo = a;
    c.hi = b;
    c.krem = K;
    c.found = 0;
  }
  __syncthreads();
  for (int iter = 0; iter < 8; ++iter) {
    const uint32_t lo = c.lo, hi = c.hi;
    const int krem = c.krem;
    const uint32_t span = hi - lo;
    const int shift = span == 0 ? 0 : max(0, 32 - __clz(span) - 11);
    const int nb = (int)(span >> shift) + 1;  // <= 2048
    for (int i = tid; i < nb; i += kThreads) c.hist[i] = 0;
    if (tid == 0) c.bcount = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kThreads) {
      const uint32_t k = keys[i];
      if (k >= lo && k <= hi && k) atomicAdd(&c.hist[(k - lo) >> shift], 1u);
    }
    __syncthreads();
    // suffix search: thread t owns the 8 bins [nb-1-8t .. nb-8-8t] (descending)
    int cnt[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int bi = nb - 1 - 8 * tid - j;
      cnt[j] = bi >= 0 ? (int)c.hist[bi] : 0;
      sum += cnt[j];
    }
    int total;
    const int excl = block_exclusive_scan(sum, tk.scan, &total);
    if (excl < krem && krem <= excl + sum) {
      int above = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (above + cnt[j] >= krem) {
          c.bsel = nb - 1 - 8 * tid - j;
          c.above = above;
          break;
        }
        above += cnt[j];
      }
    }
    __syncthreads();
    const int b = c.bsel;
    const int kr = krem - c.above;  // keys still needed from bin b
    const uint32_t blo = lo + ((uint32_t)b << shift);
    const uint32_t bhi = shift == 0 ? blo : min(hi, blo + ((1u << shift) - 1u));
    const int bc = (int)c.hist[b];
    if (shift == 0 || blo == bhi) {  // a single key value: ties by index in topk_emit
      if (tid == 0) {
        c.thr = blo;
        c.take_eq = kr;
      }
      __syncthreads();
      break;
    }
    if (bc <= 32) {  // resolve the boundary bin exactly in one warp
      for (int i = tid; i < n; i += kThreads) {
        const uint32_t k = keys[i];
        if (k >= blo && k <= bhi) c.bkeys[atomicAdd(&c.bcount, 1)] = k;
      }
      __syncthreads();
      if (warp == 0) {
        const uint32_t mine = lane < bc ? c.bkeys[lane] : 0u;
        int rank = 0;  // number of boundary keys strictly greater than mine
        for (int j = 0; j < bc; ++j) rank += c.bkeys[j] > mine;
        // the kr-th largest value: rank < kr and rank + (#equal) >= kr
        int eqn = 0;
        for (int j = 0; j < bc; ++j) eqn += c.bkeys[j] == mine;
        const bool is_thr = lane < bc && rank < kr && rank + eqn >= kr;
        const unsigned bal = __ballot_sync(0xffffffffu, is_thr);
        if (lane == __ffs(bal) - 1) {
          c.thr = mine;
          c.take_eq = kr - rank;
        }
      }
      __syncthreads();
      break;
    }
    if (tid == 0) {
      c.lo = blo;
      c.hi = bhi;
      c.krem = kr;
    }
    __syncthreads();
  }
  r.thr = c.thr;
  r.eq_mode = true;
  r.take_eq = c.take_eq;
  r.total = K;
  __syncthreads();
  return r;
}

}  // namespace tls
