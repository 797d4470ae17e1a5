// tokensel.cuh -- a4: S_t = the top-k_t candidate tokens from
// order-preserving ranking keys held in shared memory plus their fixed-bin
// histogram (kKeyBins bins of 1/16 log2 unit; bins ascend as keys descend),
// ties -> lower slot (U2).  Used by the attention kernel's selection prologue
// (attend.cu).
//
// Cost model: the selection runs once per pair in one CTA, so it is written
// to keep the per-key work to a few instructions: the boundary bin is turned
// into a key interval once (a 32-ary warp search over key space), keys are
// classified by two integer compares, and the selected slots are first
// compacted into a list so the per-token output work runs only for the K
// selected tokens, with every lane busy.
#pragma once

#include "common.cuh"
#include "fasttopk.cuh"
#include "params.h"
#include "topk.cuh"

namespace tls {

struct HistSel {  // shared-memory state of one selection (plan -> emit)
  int wgt[kWarps], weq[kWarps];
  int bsel, above, jtot;
  uint32_t klo, khi;  // key interval [klo, khi] of the boundary bin
};
struct HistPlan {
  TopK t;
  int K;
  bool need_full;
};

// Smallest key k >= 1 with key_bin(key2f(k)) <= b (key_bin(key2f(.)) is
// non-increasing in the key): a 32-ary search by one warp, <= 7 rounds.
__device__ __forceinline__ uint32_t first_key_with_bin_le(int b) {
  const int lane = threadIdx.x & 31;
  // invariant: predicate false at lo (or lo = 0, no key), true at hi
  uint64_t lo = 0, hi = 0xffffffffull;
  while (hi - lo > 1) {
    const uint64_t step = (hi - lo + 31) / 32;
    const uint64_t probe = lo + step * (uint64_t)(lane + 1);
    const bool ok = probe >= hi || key_bin(key2f((uint32_t)probe)) <= b;
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    const int f = __ffs(bal) - 1;  // lane 31's probe is >= hi, so bal != 0
    const uint64_t nhi = lo + step * (uint64_t)(f + 1);
    lo = lo + step * (uint64_t)f;
    hi = nhi < hi ? nhi : hi;
  }
  return (uint32_t)hi;
}

// skeys[nslots] (0 = not a candidate), shist[kKeyBins] (exact counts of the
// nonzero keys per bin, bins by key_bin(key2f(key))), scratch >= 2048 words.
// Plans the selection of the K = min(Kt, #valid) largest keys;
// hist_topk_emit then emits it.  Contains __syncthreads(); every thread of
// the CTA must call it.
__device__ inline HistPlan hist_topk_plan(const uint32_t* skeys, int nslots, const uint32_t* shist, int Kt,
                                          uint32_t* scratch, FastTopKCtl& fk, TopKCtl& tk, HistSel& hs,
                                          unsigned long long* dbg = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* wgt = hs.wgt;
  int* weq = hs.weq;
  // boundary bin of the histogram (bins ascend as keys descend): 4 bins per thread
  int c4[4], sum = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    c4[j] = (int)shist[4 * tid + j];
    sum += c4[j];
  }
  int jtot;
  const int excl = block_exclusive_scan(sum, tk.scan, &jtot);  // jtot = number of valid candidates
  const int K = min(Kt, jtot);
  if (tid == 0) {
    hs.bsel = -1;
    hs.jtot = jtot;
  }
  __syncthreads();
  if (K < jtot && excl < K && K <= excl + sum) {
    int above = excl;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (above + c4[j] >= K) {
        hs.bsel = 4 * tid + j;
        hs.above = above;
        break;
      }
      above += c4[j];
    }
  }
  __syncthreads();
  TopK t;
  t.offset = 0;
  t.total = K;
  const int bsel = hs.bsel;
  bool need_full = false;
  // per-warp segment counts for the one-pass emit (segments as in hist_topk_emit)
  const int seg = (((nslots + kWarps - 1) / kWarps) + 127) & ~127;
  const int s0 = min(warp * seg, nslots), s1 = min(s0 + seg, nslots);
  if (K >= jtot) {
    t.thr = 0;  // take every valid candidate
    t.eq_mode = false;
    t.take_eq = 0;
    int c = 0;
    for (int base = s0; base < s1; base += 32) {
      const int i = base + lane;
      c += __popc(__ballot_sync(0xffffffffu, i < s1 && skeys[i] != 0u));
    }
    if (lane == 0) {
      wgt[warp] = c;
      weq[warp] = 0;
    }
    __syncthreads();
  } else {
    // the boundary bin as a key interval [klo, khi]: keys > khi lie in bins above it
    if (warp < 2) {
      const uint32_t k = first_key_with_bin_le(warp == 0 ? bsel : bsel - 1);
      if (lane == 0) {
        if (warp == 0) hs.klo = k;
        else hs.khi = bsel > 0 ? k - 1u : 0xffffffffu;
      }
    }
    if (tid == 0) fk.bcount = 0;
    __syncthreads();
    const uint32_t klo = hs.klo, khi = hs.khi;
    const int kr = K - hs.above;
    // One pass over the keys: count keys above the boundary bin per warp
    // segment, and gather the boundary bin's keys (with their segment).
    int above_w = 0;
    for (int base = s0; base < s1; base += 128) {  // four independent 32-key groups per step
      uint32_t k[4];
      unsigned bal[4];
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + 32 * u + lane;
        k[u] = i < s1 ? skeys[i] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        above_w += __popc(__ballot_sync(0xffffffffu, k[u] > khi));
        bal[u] = __ballot_sync(0xffffffffu, k[u] != 0u && k[u] >= klo && k[u] <= khi);
        cnt += __popc(bal[u]);
      }
      if (cnt) {
        int off = 0;
        if (lane == 0) off = atomicAdd(&fk.bcount, cnt);
        off = __shfl_sync(0xffffffffu, off, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int dst = off + __popc(bal[u] & ((1u << lane) - 1u));
          if (((bal[u] >> lane) & 1u) && dst < 1024) {
            scratch[dst] = k[u];
            scratch[1024 + dst] = (uint32_t)warp;
          }
          off += __popc(bal[u]);
        }
      }
    }
    __syncthreads();
    const int nbk = fk.bcount;
    if (dbg && threadIdx.x == 0) {  // diagnostics: gather-pass end, boundary-bin size
      dbg[6] = gtimer();
      dbg[7] = (unsigned long long)nbk;
    }
    if (nbk <= 1024) {
      // exact threshold: the kr-th largest boundary key (rank by comparison)
      if (tid == 0) fk.thr = 0u;
      __syncthreads();
      for (int i = tid; i < nbk; i += kThreads) {
        const uint32_t v = scratch[i];
        int gtc = 0, eqc = 0;
        for (int j = 0; j < nbk; ++j) {
          const uint32_t o = scratch[j];
          gtc += o > v;
          eqc += o == v;
        }
        if (gtc < kr && gtc + eqc >= kr) fk.thr = v;  // every writer writes the same value
      }
      __syncthreads();
      const uint32_t thr = fk.thr;
      // per-warp counts: keys above the boundary bin + boundary keys > thr / == thr
      int gb = 0, eb = 0;
      for (int i = lane; i < nbk; i += 32) {
        if ((int)scratch[1024 + i] == warp) {
          gb += scratch[i] > thr;
          eb += scratch[i] == thr;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gb += __shfl_xor_sync(0xffffffffu, gb, o);
        eb += __shfl_xor_sync(0xffffffffu, eb, o);
      }
      if (lane == 0) {
        wgt[warp] = above_w + gb;
        weq[warp] = eb;
      }
      __syncthreads();
      int gtot = 0;
      for (int w = 0; w < kWarps; ++w) gtot += wgt[w];
      t.thr = thr;
      t.eq_mode = true;
      t.take_eq = K - gtot;
    } else {
      need_full = true;
    }
  }
  if (need_full) {  // rare: an oversized boundary bin -> generic select
    t = fast_topk(skeys, nslots, K, false, fk, tk, scratch);
  }
  HistPlan pl;
  pl.t = t;
  pl.K = K;
  pl.need_full = need_full;
  return pl;
}

// Emit a planned selection: put(slot, pos) for every selected slot, pos
// ascending with slot (ties at the threshold -> lower slot first, U2).  The
// selected slots are first compacted into slist[0 .. K) (>= K ints of shared
// memory, not aliasing skeys), then put runs once per selected slot with
// every lane busy.
template <class F>
__device__ void hist_topk_emit(const uint32_t* skeys, int nslots, const HistPlan& pl, HistSel& hs, TopKCtl& tk,
                               int* slist, F put) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const TopK& t = pl.t;
  if (pl.need_full) {
    topk_emit(skeys, nslots, t, tk, [&](int i, int pos) { slist[pos] = i; });
  } else {
    const int seg = (((nslots + kWarps - 1) / kWarps) + 127) & ~127;
    const int s0 = min(warp * seg, nslots), s1 = min(s0 + seg, nslots);
    int eq_seen = 0, pos = 0;
    for (int w = 0; w < warp; ++w) {
      const int take = t.eq_mode ? min(max(t.take_eq - eq_seen, 0), hs.weq[w]) : 0;
      pos += hs.wgt[w] + take;
      eq_seen += hs.weq[w];
    }
    for (int base = s0; base < s1; base += 128) {  // four independent 32-key groups per step (ILP)
      uint32_t k[4];
      unsigned bgt[4], beq[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + 32 * u + lane;
        k[u] = i < s1 ? skeys[i] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        bgt[u] = __ballot_sync(0xffffffffu, k[u] > t.thr);
        beq[u] = __ballot_sync(0xffffffffu, t.eq_mode && k[u] != 0u && k[u] == t.thr);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        unsigned tie_ok = 0u;
        if (beq[u]) {  // ties taken in slot order
          const int room = t.take_eq - eq_seen;
          if (room >= __popc(beq[u])) {
            tie_ok = beq[u];
          } else if (room > 0) {
            unsigned m = beq[u];
            for (int r = 0; r < room; ++r) {
              tie_ok |= m & (~m + 1u);
              m &= m - 1u;
            }
          }
        }
        const unsigned bsel = bgt[u] | tie_ok;
        if ((bsel >> lane) & 1u) slist[pos + __popc(bsel & lt)] = base + 32 * u + lane;
        pos += __popc(bsel);
        eq_seen += __popc(beq[u]);
      }
    }
    __syncthreads();
  }
  for (int p = tid; p < pl.K; p += kThreads) put(slist[p], p);
  __syncthreads();
}

// Smallest key k >= 1 with key_bin(key2f(k)) <= b, 0 <= b < 1023, by one warp
// in one round when possible: key_bin(f) <= b iff (6 - f) * 16 < b + 1, whose
// exact boundary f* = 6 - (b + 1) / 16 is an fp32 value, so the answer lies
// within a few ulps of f2key(f*); the 32 keys around it are tested at once and
// the 32-ary search runs only if the window misses.
__device__ __forceinline__ uint32_t bin_lower_key(int b) {
  const int lane = threadIdx.x & 31;
  const uint32_t kc = f2key(6.0f - (float)(b + 1) * 0.0625f);
  const uint32_t probe = kc - 15u + (uint32_t)lane;
  const bool ok = probe >= 1u && probe <= 0xfffffff0u && key_bin(key2f(probe)) <= b;
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  if (bal != 0u && !(bal & 1u) && (bal >> 31)) {  // false .. true inside the window: monotone boundary found
    return kc - 15u + (uint32_t)(__ffs(bal) - 1);
  }
  return first_key_with_bin_le(b);
}

// One-pass form of plan + emit for nslots <= kSelRunMax * kThreads: thread t
// owns the contiguous slots [t*R, t*R + R), R = 4 * ceil(nslots / (4 *
// kThreads)), read as 16-byte chunks in a rotated order (conflict-free banks),
// and keeps two bitmasks over them: keys above the boundary bin and keys in it.
// The boundary bin's few keys are gathered and ranked exactly; one packed block
// scan of (#greater, #equal-to-threshold) per thread then gives every thread
// its output position, and it emits its selected slots in slot order.  Same
// result as hist_topk_plan + hist_topk_emit (ties at the threshold -> lower
// slot, U2).  on_k(K) runs once per thread as soon as K is known, then
// put(slot, pos) once per selected slot.  Returns K.
constexpr int kSelRunMax = 64;  // keys per thread (two 32-bit masks)

template <class FK, class F>
__device__ int hist_topk_select(const uint32_t* skeys, int nslots, const uint32_t* shist, int Kt, uint32_t* scratch,
                                FastTopKCtl& fk, TopKCtl& tk, HistSel& hs, int* slist, FK on_k, F put,
                                unsigned long long* dbg = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long cyc0 = clock64();
#define TLS_CYC(i) \
  if (dbg && tid == 0) dbg[65536 * 4 + (i)] = (unsigned long long)(clock64() - cyc0);
  // this thread's run of keys (issued first; consumed after the interval is known)
  const int nch = (nslots + 4 * kThreads - 1) / (4 * kThreads);  // 16-byte chunks per thread (<= 16)
  const int r0 = tid * 4 * nch;
  const int c0 = nch > 0 ? tid % nch : 0;
  const uint4* k4 = reinterpret_cast<const uint4*>(skeys) + (r0 >> 2);
  uint4 kv[kSelRunMax / 4];
#pragma unroll
  for (int j = 0; j < kSelRunMax / 4; ++j) {
    if (j < nch) {
      int c = c0 + j;  // rotated: the 8 threads of a phase hit distinct banks
      if (c >= nch) c -= nch;
      kv[j] = k4[c];
    }
  }
  // boundary bin of the histogram (bins ascend as keys descend): 4 bins per thread
  int c4[4], sum = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    c4[j] = (int)shist[4 * tid + j];
    sum += c4[j];
  }
  int jtot;
  const int excl = block_exclusive_scan(sum, tk.scan, &jtot);  // jtot = number of valid candidates
  const int K = min(Kt, jtot);
  on_k(K);
  if (tid == 0) {
    hs.bsel = -1;
    fk.bcount = 0;
  }
  __syncthreads();
  if (K < jtot && excl < K && K <= excl + sum) {
    int above = excl;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (above + c4[j] >= K) {
        hs.bsel = 4 * tid + j;
        hs.above = above;
        break;
      }
      above += c4[j];
    }
  }
  __syncthreads();
  TLS_CYC(0)
  const int bsel = hs.bsel;
  const bool take_all = K >= jtot;
  if (!take_all && warp < 2) {  // the boundary bin as a key interval [klo, khi]
    if (warp == 0) {
      const uint32_t k = bsel >= 1023 ? 1u : bin_lower_key(bsel);
      if (lane == 0) hs.klo = k;
    } else {
      const uint32_t k = bsel > 0 ? bin_lower_key(bsel - 1) - 1u : 0xffffffffu;
      if (lane == 0) hs.khi = k;
    }
  }
  __syncthreads();
  TLS_CYC(1)
  // keys above the boundary bin (every valid key when all are taken) and keys in it
  const uint32_t khi = take_all ? 0u : hs.khi;
  const uint32_t klo = take_all ? 0xffffffffu : hs.klo;
  const uint32_t span = khi - klo;  // in-bin test: key - klo <= span (unsigned)
  uint64_t gt = 0, bd = 0;
#pragma unroll
  for (int j = 0; j < kSelRunMax / 4; ++j) {
    if (j < nch) {
      int c = c0 + j;
      if (c >= nch) c -= nch;
      const uint32_t e[4] = {kv[j].x, kv[j].y, kv[j].z, kv[j].w};
      uint32_t na = 0, nb = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        na |= (uint32_t)(e[u] > khi) << u;
        nb |= (uint32_t)(e[u] - klo <= span) << u;
      }
      gt |= (uint64_t)na << (4 * c);
      bd |= (uint64_t)nb << (4 * c);
    }
  }
  {  // slots past nslots are not candidates
    const int lim = nslots - r0;
    const uint64_t live = lim >= 64 ? ~0ull : (lim <= 0 ? 0ull : (1ull << lim) - 1ull);
    gt &= live;
    bd = take_all ? 0ull : (bd & live);
  }
  const int nb_own = __popcll(bd);
  if (nb_own) {  // gather the boundary bin's keys (few)
    int dst = atomicAdd(&fk.bcount, nb_own);
    for (uint64_t m = bd; m; m &= m - 1, ++dst) {
      const int bit = __ffsll((long long)m) - 1;
      if (dst < 1024) scratch[dst] = skeys[r0 + bit];
    }
  }
  __syncthreads();
  TLS_CYC(2)
  int nbk = take_all ? 0 : fk.bcount;
  int kr = take_all ? 0 : K - hs.above;  // rank of the threshold among the boundary keys
  if (dbg && tid == 0) {  // diagnostics: classification-pass end, boundary-bin size
    dbg[6] = gtimer();
    dbg[7] = (unsigned long long)nbk;
  }
  if (nbk > 32) {
    // a large boundary bin (flat alpha~, e.g. uniform inputs: hundreds of keys, whose O(n^2) rank cost ~11 us):
    // refine it with 256 sub-bins linear in the key over [klo, khi] (monotone); keys of higher sub-bins join
    // gt, the sub-bin holding the kr-th largest boundary key becomes the new boundary
    __shared__ uint32_t s_sub[kThreads];
    s_sub[tid] = 0u;
    __syncthreads();
    const uint64_t span = (uint64_t)khi - (uint64_t)klo + 1ull;
    auto sub_of = [&](uint32_t k) -> int { return (int)(((uint64_t)(k - klo) << 8) / span); };
    for (uint64_t m = bd; m; m &= m - 1) atomicAdd(&s_sub[sub_of(skeys[r0 + __ffsll((long long)m) - 1])], 1u);
    __syncthreads();
    const int c = (int)s_sub[kThreads - 1 - tid];
    if (tid == 0) hs.bsel = -1;  // (ordered before the writer below by the scan's barriers)
    int tot_;
    const int ab = block_exclusive_scan(c, tk.scan, &tot_);
    if (ab < kr && kr <= ab + c) {
      hs.bsel = kThreads - 1 - tid;
      hs.above = ab;
    }
    if (tid == 0) fk.bcount = 0;
    __syncthreads();
    const int sb = hs.bsel;
    if (sb < 0) {  // the sub-bin counts do not bracket rank kr (cannot happen for an exact histogram): take
                   // the generic select below instead of emitting a wrong set
      nbk = 1 << 30;
      goto generic_select;
    }
    kr -= hs.above;
    uint64_t nbd = 0;
    for (uint64_t m = bd; m; m &= m - 1) {
      const int bit = __ffsll((long long)m) - 1;
      const int sbin = sub_of(skeys[r0 + bit]);
      if (sbin > sb) gt |= 1ull << bit;
      else if (sbin == sb) nbd |= 1ull << bit;
    }
    bd = nbd;
    const int nb2 = __popcll(bd);
    if (nb2) {
      int dst = atomicAdd(&fk.bcount, nb2);
      for (uint64_t m = bd; m; m &= m - 1, ++dst) {
        const int bit = __ffsll((long long)m) - 1;
        if (dst < 1024) scratch[dst] = skeys[r0 + bit];
      }
    }
    __syncthreads();
    nbk = fk.bcount;
  }
generic_select:
  if (nbk > 1024) {  // rare (e.g. thousands of equal keys): generic select into slist
    const TopK t = fast_topk(skeys, nslots, K, false, fk, tk, scratch);
    topk_emit(skeys, nslots, t, tk, [&](int i, int pos) { slist[pos] = i; });
    for (int p = tid; p < K; p += kThreads) put(slist[p], p);
    __syncthreads();
    return K;
  }
  uint32_t thr = 0u;
  if (!take_all) {
    // exact threshold: the kr-th largest boundary key (rank by comparison)
    if (nbk <= 32) {  // one warp, keys in lanes, the others' keys by shuffle
      if (warp == 0) {
        const uint32_t v = lane < nbk ? scratch[lane] : 0u;
        int gtc = 0, eqc = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t o = __shfl_sync(0xffffffffu, v, j);
          gtc += o > v;
          eqc += o == v;
        }
        if (lane < nbk && gtc < kr && gtc + eqc >= kr) fk.thr = v;  // every writer writes the same value
      }
    } else {
      for (int i = tid; i < nbk; i += kThreads) {
        const uint32_t v = scratch[i];
        int gtc = 0, eqc = 0;
        for (int j = 0; j < nbk; ++j) {
          const uint32_t o = scratch[j];
          gtc += o > v;
          eqc += o == v;
        }
        if (gtc < kr && gtc + eqc >= kr) fk.thr = v;  // every writer writes the same value
      }
    }
    __syncthreads();
    thr = fk.thr;
  }
  TLS_CYC(3)
  // boundary keys of this run: > thr joins gt, == thr is a tie
  uint64_t eq = 0;
  for (uint64_t m = bd; m; m &= m - 1) {
    const int bit = __ffsll((long long)m) - 1;
    const uint32_t k = skeys[r0 + bit];
    if (k > thr) gt |= 1ull << bit;
    else if (k == thr) eq |= 1ull << bit;
  }
  const int ngt = __popcll(gt), neq = __popcll(eq);
  int tot;
  const int pre = block_exclusive_scan(ngt | (neq << 16), tk.scan, &tot);
  TLS_CYC(4)
  const int gt_before = pre & 0xffff, eq_before = pre >> 16;
  const int take_eq = K - (tot & 0xffff);  // ties taken in slot order
  int ntake = min(max(take_eq - eq_before, 0), neq);
  uint64_t selm = gt;
  for (uint64_t m = eq; ntake > 0; --ntake, m &= m - 1) selm |= m & (~m + 1ull);
  int pos = gt_before + min(eq_before, max(take_eq, 0));
  // selected slots -> slist in slot order, then put over the list with every lane busy
  for (uint64_t m = selm; m; m &= m - 1) slist[pos++] = r0 + __ffsll((long long)m) - 1;
  __syncthreads();
  for (int p = tid; p < K; p += kThreads) put(slist[p], p);
  __syncthreads();
  TLS_CYC(5)
#undef TLS_CYC
  return K;
}

// Exact top-K of n order-preserving keys (no key 0 among the first n) for the
// block selection a2, ties -> lower index (U2), emitted ascending: put(i, pos).
// One pass in registers: thread t owns keys [t*R, t*R + R) (R = 4*ceil(n/1024)
// <= 4*MAXC, 16-byte chunks loaded in rotated order); a 256-bin histogram that is
// linear in the key's fp32 value between the min and max key (monotone in the
// key, so bins never reorder keys) gives the boundary bin; its keys are ranked
// exactly; one packed block scan places every thread's selected keys.  Returns
// false (nothing emitted) when the boundary bin holds > 1024 keys: the caller
// then runs the generic select.
template <int MAXC, class F>
__device__ bool range_topk_select(const uint32_t* keys, int n, int K, uint32_t* scratch, FastTopKCtl& fk, TopKCtl& tk,
                                  HistSel& hs, F put) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint32_t s_hist[kThreads];
  __shared__ uint32_t s_mn[kWarps], s_mx[kWarps];
  const int nch = (n + 4 * kThreads - 1) / (4 * kThreads);  // <= MAXC (caller: n <= 4 * MAXC * kThreads)
  const int r0 = tid * 4 * nch;
  const int c0 = nch > 0 ? tid % nch : 0;
  const uint4* k4 = reinterpret_cast<const uint4*>(keys) + (r0 >> 2);
  const int lim = n - r0;  // valid keys of this run
  uint4 kv[MAXC];
  uint32_t mnk = 0xffffffffu, mxk = 0u;
#pragma unroll
  for (int j = 0; j < MAXC; ++j) {
    if (j < nch) {
      int c = c0 + j;
      if (c >= nch) c -= nch;
      kv[j] = 4 * c < lim ? k4[c] : make_uint4(0u, 0u, 0u, 0u);
      const uint32_t e[4] = {kv[j].x, kv[j].y, kv[j].z, kv[j].w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (4 * c + u < lim) {
          mnk = min(mnk, e[u]);
          mxk = max(mxk, e[u]);
        }
    }
  }
  s_hist[tid] = 0u;
  mnk = __reduce_min_sync(0xffffffffu, mnk);
  mxk = __reduce_max_sync(0xffffffffu, mxk);
  if (lane == 0) {
    s_mn[warp] = mnk;
    s_mx[warp] = mxk;
  }
  __syncthreads();
  mnk = s_mn[0];
  mxk = s_mx[0];
#pragma unroll
  for (int w = 1; w < kWarps; ++w) {
    mnk = min(mnk, s_mn[w]);
    mxk = max(mxk, s_mx[w]);
  }
  if (mnk == mxk) {  // every key equal: the first K
    for (int i = tid; i < K; i += kThreads) put(i, i);
    __syncthreads();
    return true;
  }
  const float mn = key2f(mnk);
  const float inv = 256.0f / (key2f(mxk) - mn);  // bins by value (inf / 0 range -> everything in one bin)
  auto bin_of = [&](uint32_t k) -> int {
    const float x = (key2f(k) - mn) * inv;
    return x >= 255.f ? 255 : (x > 0.f ? (int)x : 0);
  };
#pragma unroll
  for (int j = 0; j < MAXC; ++j) {
    if (j < nch) {
      int c = c0 + j;
      if (c >= nch) c -= nch;
      const uint32_t e[4] = {kv[j].x, kv[j].y, kv[j].z, kv[j].w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (4 * c + u < lim) atomicAdd(&s_hist[bin_of(e[u])], 1u);
    }
  }
  __syncthreads();
  // boundary bin: thread t holds bin 255 - t, so the exclusive prefix counts the keys in higher bins
  const int cnt = (int)s_hist[kThreads - 1 - tid];
  int tot;
  const int above = block_exclusive_scan(cnt, tk.scan, &tot);
  if (tid == 0) fk.bcount = 0;
  if (above < K && K <= above + cnt) {
    hs.bsel = kThreads - 1 - tid;
    hs.above = above;
  }
  __syncthreads();
  const int bsel = hs.bsel, kr = K - hs.above;
  uint64_t gt = 0, bd = 0;
#pragma unroll
  for (int j = 0; j < MAXC; ++j) {
    if (j < nch) {
      int c = c0 + j;
      if (c >= nch) c -= nch;
      const uint32_t e[4] = {kv[j].x, kv[j].y, kv[j].z, kv[j].w};
      uint32_t na = 0, nb = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool ok = 4 * c + u < lim;
        const int bn = bin_of(e[u]);
        na |= (uint32_t)(ok && bn > bsel) << u;
        nb |= (uint32_t)(ok && bn == bsel) << u;
      }
      gt |= (uint64_t)na << (4 * c);
      bd |= (uint64_t)nb << (4 * c);
    }
  }
  const int nb_own = __popcll(bd);
  if (nb_own) {
    int dst = atomicAdd(&fk.bcount, nb_own);
    for (uint64_t m = bd; m; m &= m - 1, ++dst) {
      const int bit = __ffsll((long long)m) - 1;
      if (dst < 1024) scratch[dst] = keys[r0 + bit];
    }
  }
  __syncthreads();
  const int nbk = fk.bcount;
  if (nbk > 1024) return false;  // uniform: every thread read the same count
  if (nbk <= 32) {
    if (warp == 0) {
      const uint32_t v = lane < nbk ? scratch[lane] : 0u;
      int gtc = 0, eqc = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t o = __shfl_sync(0xffffffffu, v, j);
        gtc += o > v;
        eqc += o == v;
      }
      if (lane < nbk && gtc < kr && gtc + eqc >= kr) fk.thr = v;
    }
  } else {
    for (int i = tid; i < nbk; i += kThreads) {
      const uint32_t v = scratch[i];
      int gtc = 0, eqc = 0;
      for (int j = 0; j < nbk; ++j) {
        const uint32_t o = scratch[j];
        gtc += o > v;
        eqc += o == v;
      }
      if (gtc < kr && gtc + eqc >= kr) fk.thr = v;
    }
  }
  __syncthreads();
  const uint32_t thr = fk.thr;
  uint64_t eq = 0;
  for (uint64_t m = bd; m; m &= m - 1) {
    const int bit = __ffsll((long long)m) - 1;
    const uint32_t k = keys[r0 + bit];
    if (k > thr) gt |= 1ull << bit;
    else if (k == thr) eq |= 1ull << bit;
  }
  const int ngt = __popcll(gt), neq = __popcll(eq);
  int tot2;
  const int pre = block_exclusive_scan(ngt | (neq << 16), tk.scan, &tot2);
  const int gt_before = pre & 0xffff, eq_before = pre >> 16;
  const int take_eq = K - (tot2 & 0xffff);
  int ntake = min(max(take_eq - eq_before, 0), neq);
  uint64_t selm = gt;
  for (uint64_t m = eq; ntake > 0; --ntake, m &= m - 1) selm |= m & (~m + 1ull);
  int pos = gt_before + min(eq_before, max(take_eq, 0));
  for (uint64_t m = selm; m; m &= m - 1) put(r0 + __ffsll((long long)m) - 1, pos++);
  __syncthreads();
  return true;
}

}  // namespace tls
