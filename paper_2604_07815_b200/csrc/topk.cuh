// topk.cuh -- exact top-k with the lower-index tie rule (readings U2-U4) over
// order-preserving uint32 keys held in shared memory, for one CTA or for a
// thread-block cluster (keys distributed over the CTAs in rank order).
//
// Radix select with 8-bit digits, most significant first: each pass builds a
// warp-aggregated histogram of the keys that match the digits fixed so far,
// (cluster: sums the cs CTAs' histograms through DSMEM, the remote loads
// issued back to back), and one warp picks the digit holding the k-th
// largest key.  A pass that takes its whole bin ends the search early.  The
// selected set is {key > thr} plus, when several keys equal thr, the first
// ones in (CTA rank, local index) order -- ascending ids -- which is the
// paper-silent tie rule U2.  Key 0 means "not a candidate" and is never taken.
#pragma once

#include "common.cuh"

namespace tls {

constexpr int kMaxCluster = 16;

struct TopKCtl {
  uint32_t hist[2][256];  // double-buffered (read remotely)
  uint32_t tot[256];
  int scan[kWarps + 2];
  int xc[2];  // (count > thr, count == thr) of this CTA (read remotely)
  int dig, krem, bincnt;
  int r_take, r_off, r_total;
};

struct TopK {
  uint32_t thr;
  int take_eq;
  int offset;
  int total;
  bool eq_mode;
};

// CLUSTER = false: a single CTA (cs must be 1, rank 0).
template <bool CLUSTER>
__device__ TopK radix_topk(const uint32_t* keys, int nloc, int K, bool take_all, int cs, unsigned rank,
                           TopKCtl& ctl) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t prefix = 0, mask = 0, thr = 0;
  int krem = K;
  bool eq_mode = false;
  if (!take_all) {
    bool done = false;
    for (int pass = 0; pass < 4 && !done; ++pass) {
      const int shift = 24 - 8 * pass, buf = pass & 1;
      for (int i = tid; i < 256; i += kThreads) ctl.hist[buf][i] = 0;
      __syncthreads();
      for (int base = 0; base < nloc; base += kThreads) {
        const int i = base + tid;
        const uint32_t k = i < nloc ? keys[i] : 0u;
        const bool cand = k != 0u && (k & mask) == prefix;
        const uint32_t digit = cand ? ((k >> shift) & 255u) : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        if (cand && lane == __ffs(peers) - 1) atomicAdd(&ctl.hist[buf][digit], (uint32_t)__popc(peers));
      }
      if constexpr (CLUSTER) {
        cluster_sync_all();
        uint32_t v[kMaxCluster];
#pragma unroll
        for (int rr = 0; rr < kMaxCluster; ++rr) v[rr] = rr < cs ? *dsmem(&ctl.hist[buf][tid], rr) : 0u;
        uint32_t s = 0;
#pragma unroll
        for (int rr = 0; rr < kMaxCluster; ++rr) s += v[rr];
        ctl.tot[tid] = s;
      } else {
        __syncthreads();
        ctl.tot[tid] = ctl.hist[buf][tid];
      }
      __syncthreads();
      if (warp == 0) {
        int c[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          c[j] = (int)ctl.tot[255 - 8 * lane - j];
          sum += c[j];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const int excl = incl - sum;
        if (excl < krem && krem <= incl) {
          int above = excl;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (above + c[j] >= krem) {
              ctl.dig = 255 - 8 * lane - j;
              ctl.krem = krem - above;
              ctl.bincnt = c[j];
              break;
            }
            above += c[j];
          }
        }
      }
      __syncthreads();
      prefix |= (uint32_t)ctl.dig << shift;
      mask |= 0xffu << shift;
      krem = ctl.krem;
      if (krem == ctl.bincnt) {  // the whole bin is taken: select k >= prefix
        done = true;
        thr = prefix ? prefix - 1u : 0u;
      }
    }
    if (!done) {
      thr = prefix;
      eq_mode = true;
    }
  }
  int gt = 0, eq = 0;
  for (int i = tid; i < nloc; i += kThreads) {
    const uint32_t k = keys[i];
    gt += k > thr;
    eq += (eq_mode && k == thr);
  }
  int gtot, etot;
  block_exclusive_scan(gt, ctl.scan, &gtot);
  block_exclusive_scan(eq, ctl.scan, &etot);
  if constexpr (CLUSTER) {
    if (tid == 0) {
      ctl.xc[0] = gtot;
      ctl.xc[1] = etot;
    }
    cluster_sync_all();
    if (tid == 0) {
      int g[kMaxCluster], e[kMaxCluster];
#pragma unroll
      for (int rr = 0; rr < kMaxCluster; ++rr) {
        g[rr] = rr < cs ? *dsmem(&ctl.xc[0], rr) : 0;
        e[rr] = rr < cs ? *dsmem(&ctl.xc[1], rr) : 0;
      }
      int eq_before = 0, off = 0, total = 0, my_take = 0;
      for (int rr = 0; rr < cs; ++rr) {
        int take = eq_mode ? min(max(krem - eq_before, 0), e[rr]) : 0;
        eq_before += e[rr];
        const int s = g[rr] + take;
        if (rr < (int)rank) off += s;
        if (rr == (int)rank) my_take = take;
        total += s;
      }
      ctl.r_take = my_take;
      ctl.r_off = off;
      ctl.r_total = total;
    }
  } else {
    if (tid == 0) {
      ctl.r_take = eq_mode ? min(krem, etot) : 0;
      ctl.r_off = 0;
      ctl.r_total = gtot + ctl.r_take;
    }
  }
  __syncthreads();
  TopK r;
  r.thr = thr;
  r.eq_mode = eq_mode;
  r.take_eq = ctl.r_take;
  r.offset = ctl.r_off;
  r.total = ctl.r_total;
  __syncthreads();
  return r;
}

// Emit this CTA's selected elements in local-index order: f(local_index, out_pos).
template <class F>
__device__ void topk_emit(const uint32_t* keys, int nloc, const TopK& t, TopKCtl& ctl, F f) {
  const int tid = threadIdx.x;
  const int per = (nloc + kThreads - 1) / kThreads;
  const int b = min(tid * per, nloc), e = min(b + per, nloc);
  int eqc = 0;
  if (t.eq_mode)
    for (int i = b; i < e; ++i) eqc += keys[i] == t.thr;
  int tot;
  const int eqbase = block_exclusive_scan(eqc, ctl.scan, &tot);
  int selc = 0, eqs = eqbase;
  for (int i = b; i < e; ++i) {
    const uint32_t k = keys[i];
    bool s = k > t.thr;
    if (t.eq_mode && k == t.thr) s = (eqs++ < t.take_eq);
    selc += s;
  }
  int pos = t.offset + block_exclusive_scan(selc, ctl.scan, &tot);
  eqs = eqbase;
  for (int i = b; i < e; ++i) {
    const uint32_t k = keys[i];
    bool s = k > t.thr;
    if (t.eq_mode && k == t.thr) s = (eqs++ < t.take_eq);
    if (s) f(i, pos++);
  }
}

}  // namespace tls
