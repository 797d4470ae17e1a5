// step.cu -- the whole decode step of AsyncTLS (arXiv 2604.07815) for one
// (batch, KV-head) pair in ONE thread-block cluster, for sm_100a:
//
//   step_kernel, grid (nc, pairs), cluster (nc, 1, 1); CTA rank r of pair p:
//     a1  s_i = Q+ . k^max_i + Q- . k^min_i (P:99 via the P:110 identity and
//         linearity of sum_h) for the blocks [r*mb, (r+1)*mb) of the pair:
//         block-summary rows streamed by TMA bulk copies through a ring of
//         8-row slots, one GEMV dot product per row
//     a2  M_t = top-k_b blocks, exact, ties -> lower block id (U2):
//         a cluster-wide radix select over the CTAs' score keys (cluster_topk)
//     a3  alpha~_j over the candidate tokens: CTA r stages the
//         INT4 token index of candidate blocks [r*cb, (r+1)*cb) of M_t by TMA,
//         logits on tensor cores (mma.sync, codes x q~), per-head softmax
//         statistics merged over DSMEM, ranking keys log2 sum_h 2^(L_hj - lz_h)
//     a4  S_t = top-k_t tokens, exact, ties -> lower token id:
//         cluster_topk over the CTAs' ranking keys
//     a5  o = softmax(q K_S^T sm_scale) V_S: CTA r attends over
//         positions [K r / nc, K (r+1) / nc) of S_t (K/V rows gathered by
//         cp.async, tensor cores), the nc partials merged over DSMEM with the
//         LSE identity (T10)
//
// There is no global workspace and no inter-kernel hand-off: every
// intermediate (scores, candidate lists, softmax statistics, ranking keys,
// selected lists, attention partials) lives in the cluster's shared memory,
// and the phases are ordered by cluster barriers.  Pairs are independent, so
// the clusters of different pairs overlap freely: while one pair waits on a
// barrier or a top-k round, the other CTAs on the SM stream their rows.
//
// Specialisation (the BASELINE.json GQA configs): bf16, GQA with d_k = d_v =
// 128, G <= 8 query heads per KV head, d_c = 32 channels, block size 64.
// Every other configuration runs the kernel chain of fused.cu / select.cu /
// attend.cu.
//
// Citation key: P:n = line n of PAPER.md.  Readings U1..U20: DESIGN.md §3.
#include <math_constants.h>

#include "common.cuh"
#include "launch.h"
#include "params.h"
#include "token.cuh"

namespace tls {

namespace {

constexpr int kD = 128;           // head dim (d_k = d_v)
constexpr int kRowBytes = 2 * kD * 2;  // one block's [k^max | k^min] row, bf16: 512 B
constexpr int kGroupBytes = 8 * kRowBytes;  // one 8-row TMA group: 4 KB
constexpr int kRing = 16;         // a1 ring slots (8 rows each): 64 KB
constexpr int kTC = 64;           // a5 tokens per staged chunk
constexpr int kStages = 2;        // a5 cp.async stages (2 x (64 K + 64 V rows) = 64 KB)
constexpr int kKS = 2;            // a3 k-steps: d_c / 16
constexpr int kTPW = 8;           // a3 16-token tiles per warp (register-resident logits)
constexpr int kMaxNC = 16;
constexpr float kKeyOff = 64.f;   // a3 ranking-key scale (reading U20)
constexpr size_t kUBytes = (size_t)kStages * 2 * kTC * kD * 2;  // union region: 64 KB

constexpr size_t kKeys3Off = 32 * 1024;  // a3 ranking keys inside U (after the <= 24 KB index stage)
constexpr size_t kPartOff = 17408;       // a5 CTA partial inside U (after the 4 x 8 x 132 + 64 float scratch)
static_assert(kUBytes >= (size_t)kRing * kGroupBytes, "a1 ring fits the union region");
static_assert(kPartOff >= (4 * 8 * (kD + 4) + 64) * 4 && kPartOff + (8 * kD + 16) * 4 <= kUBytes, "a5 partial");
static_assert(kKeys3Off + 4 * 1024 * 4 <= kUBytes, "a3 keys");

struct StepCtl {
  int scan[kWarps + 2];
  int bin, above, cnt;          // cluster_topk: boundary bin of the current round
  int gt_before, eq_before;     // cluster_topk: counts of the lower-ranked CTAs
  int kb, kt;                   // |M_t|, |S_t|
  float wm[kWarps][8], ws[kWarps][8];  // a3 per-warp head statistics
  float hlz[8];                 // a3 lz_h = M_h + log2 Z_h
  float mw[kMaxNC][8], minv[8]; // a5 merge weights
};

}  // namespace

namespace {

// ---------------------------------------------------------------------------
// Exact cluster-wide top-K (readings U2-U4) over order-preserving keys: CTA q
// of the cluster holds `nloc` keys in shared memory (key 0 = not a
// candidate), thread t owns the slots [4t, 4t + 4).  The global order of the
// slots is (CTA rank, slot), which is ascending id order for both selections,
// so "ties -> lower id" is "ties -> earlier slot".  Radix select, 8 bits per
// round from the top: each CTA histograms the keys that match the prefix
// found so far, one cluster barrier, every CTA sums the nc histograms over
// DSMEM in the same order and finds the same boundary bin; a round whose
// boundary bin is taken whole ends the search.  The selection is
// {key > prefix class} + the first `need` members of the class in slot order.
// Returns K = min(Kreq, #candidates); sel = this thread's selected slots
// (bit u = slot 4t + u) and pos = the global output position of the first.
// Every thread of the cluster must call it.
// ---------------------------------------------------------------------------
struct TopkRes {
  int K;
  uint32_t sel;
  int pos;
};

__device__ __forceinline__ TopkRes cluster_topk(const uint32_t* keys, int nloc, int Kreq, uint32_t* hist2,
                                                int* xcnt, StepCtl& ctl, unsigned nc, unsigned rank) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t kv[4];
  {
    const int s0 = 4 * tid;
    if (s0 + 4 <= nloc) {
      const uint4 v = *reinterpret_cast<const uint4*>(keys + s0);
      kv[0] = v.x, kv[1] = v.y, kv[2] = v.z, kv[3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) kv[u] = s0 + u < nloc ? keys[s0 + u] : 0u;
    }
  }
  uint32_t prefix = 0u, mask = 0u;
  int need = 0, K = 0;
#pragma unroll 1
  for (int round = 0; round < 4; ++round) {
    const int shift = 24 - 8 * round;
    uint32_t* h = hist2 + (round & 1) * 256;
    h[tid] = 0u;  // read by the other CTAs two rounds ago at the latest (ordered by the last cluster barrier)
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (kv[u] != 0u && (kv[u] & mask) == prefix) atomicAdd(&h[(kv[u] >> shift) & 255u], 1u);
    cluster_sync_all();
    const int bin = 255 - tid;  // thread order = descending bins
    uint32_t part[kMaxNC];
#pragma unroll
    for (int q = 0; q < kMaxNC; ++q) part[q] = (unsigned)q < nc ? *dsmem(h + bin, (unsigned)q) : 0u;
    int tot = 0;
#pragma unroll
    for (int q = 0; q < kMaxNC; ++q) tot += (int)part[q];
    int total;
    const int above = block_exclusive_scan(tot, ctl.scan, &total);
    if (round == 0) {
      K = min(Kreq, total);
      need = K;
      if (K >= total) break;  // every candidate is taken: class = all nonzero keys (prefix = mask = 0)
    }
    if (above < need && need <= above + tot) {
      ctl.bin = bin;
      ctl.above = above;
      ctl.cnt = tot;
    }
    __syncthreads();
    prefix |= (uint32_t)ctl.bin << shift;
    mask |= 255u << shift;
    need -= ctl.above;
    if (ctl.cnt == need) break;  // the whole boundary bin is taken
  }
  // this thread's keys above the class, and class members
  uint32_t gtm = 0u, eqm = 0u;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (kv[u] == 0u) continue;
    const uint32_t km = kv[u] & mask;
    if (km > prefix) gtm |= 1u << u;
    else if (km == prefix) eqm |= 1u << u;
  }
  const int ngt = __popc(gtm), neq = __popc(eqm);
  int tot2;
  const int pre = block_exclusive_scan(ngt | (neq << 16), ctl.scan, &tot2);
  if (tid == 0) {
    xcnt[0] = tot2 & 0xffff;
    xcnt[1] = tot2 >> 16;
  }
  cluster_sync_all();
  if (warp == 0) {  // counts of the lower-ranked CTAs
    const bool lower = (unsigned)lane < rank;
    int g = lower ? *dsmem(xcnt, (unsigned)lane) : 0;
    int e = lower ? *dsmem(xcnt + 1, (unsigned)lane) : 0;
    g = (int)warp_sum_u32((uint32_t)g);
    e = (int)warp_sum_u32((uint32_t)e);
    if (lane == 0) {
      ctl.gt_before = g;
      ctl.eq_before = e;
    }
  }
  __syncthreads();
  const int E = need;  // class members to take, in slot order over the cluster
  const int eq_r = tot2 >> 16;
  const int take_r = min(max(E - ctl.eq_before, 0), eq_r);
  const int cta_base = ctl.gt_before + min(E, ctl.eq_before);
  const int gt_b = pre & 0xffff, eq_b = pre >> 16;
  int take_t = min(max(take_r - eq_b, 0), neq);
  uint32_t sel = gtm;
  for (uint32_t m = eqm; take_t > 0; --take_t, m &= m - 1u) sel |= m & (~m + 1u);
  TopkRes res;
  res.K = K;
  res.sel = sel;
  res.pos = cta_base + gt_b + min(eq_b, take_r);
  return res;
}

// Rank of the CTA whose a5 slice [K q / nc, K (q+1) / nc) holds position pos.
__device__ __forceinline__ int slice_owner(int pos, int K, int nc) {
  int o = (int)(((long long)pos * nc) / K);
  while (o + 1 < nc && (int)(((long long)K * (o + 1)) / nc) <= pos) ++o;
  while (o > 0 && (int)(((long long)K * o) / nc) > pos) --o;
  return o;
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 3) step_kernel(const __grid_constant__ StepKParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t ring_bar[kRing];
  __shared__ __align__(8) uint64_t idx_bar;
  __shared__ StepCtl ctl;
  __shared__ int xcnt[2];
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rank = blockIdx.x, nc = (unsigned)p.nc;
  const int pair = blockIdx.y;
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int G = d.G;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;  // reading U1
  // shared memory (plan_step): U is the a1 ring, then the a3 index stage (+ the a3 ranking keys at kKeys3Off),
  // then the a5 K/V staging (+ the warp-partial scratch and this CTA's partial at kPartOff); QQ (a1 only)
  // aliases the radix histograms (a2 on); the a5 P buffers alias [a1 keys .. cand] (dead by then)
  uint8_t* U = smem + p.off_u;
  uint32_t* keys1 = reinterpret_cast<uint32_t*>(smem + p.off_keys);  // a1 score keys
  uint32_t* keys = reinterpret_cast<uint32_t*>(U + kKeys3Off);        // a3 ranking keys
  uint32_t* hist2 = reinterpret_cast<uint32_t*>(smem + p.off_hist);
  int* cand = reinterpret_cast<int*>(smem + p.off_cand);
  int* sel = reinterpret_cast<int*>(smem + p.off_sel);
  float* QQ = reinterpret_cast<float*>(smem + p.off_hist);
  uint32_t* qb = reinterpret_cast<uint32_t*>(smem + p.off_qb);
  float* qsum = reinterpret_cast<float*>(smem + p.off_qb + kKS * 256);
  float* xm = reinterpret_cast<float*>(smem + p.off_xs);  // [kMaxNC][8] per-CTA head max, then [kMaxNC][8] sums
  float* xz = xm + kMaxNC * 8;
  const __nv_bfloat16* qg = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b * d.Hq + (size_t)g * G) * kD;

  // ===================== a1: block scores of rows [i0, i0 + nrows) =====================
  const int i0 = (int)rank * p.mb;
  const int nrows = max(0, min(p.mb, m - i0));
  const int ngrp = (nrows + 7) >> 3;
  const uint8_t* bsrc = reinterpret_cast<const uint8_t*>(p.block_minmax) + ((size_t)pair * d.M + i0) * kRowBytes;
  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(&ring_bar[s], 1);
    mbar_init(&idx_bar, 1);
    mbar_fence_init();
    for (int s = 0; s < min(kRing, ngrp); ++s) {
      const int rows = min(8, nrows - 8 * s);
      mbar_arrive_expect_tx(&ring_bar[s], (uint32_t)(rows * kRowBytes));
      tma_bulk_g2s(U + (size_t)s * kGroupBytes, bsrc + (size_t)s * kGroupBytes, (uint32_t)(rows * kRowBytes),
                   &ring_bar[s]);
    }
  }
  // QQ = [Q+ | Q-] of the pair (fp32), the head-collapsed query of the P:110 GEMV
  if (tid < kD) {
    float qp = 0.f, qn = 0.f;
    for (int h = 0; h < G; ++h) {
      const float v = __bfloat162float(qg[(size_t)h * kD + tid]);
      qp += fmaxf(v, 0.f);
      qn += fminf(v, 0.f);
    }
    QQ[tid] = qp;
    QQ[kD + tid] = qn;
  }
  // q~_h[c] = q_h[C_c] as the B fragments of the a3 mma (channel order of token_tile_mma)
  {
    const int* ch = p.channels + (size_t)g * d.d_c;
    // 64 fragment words x 2 bf16 pairs: lane ln, k-step s; head ln >> 2; channels cb, cb+1, cb+4, cb+5
    if (tid < kKS * 32) {
      const int ln = tid & 31, s = tid >> 5;
      const int h = ln >> 2;
      const int cb = 8 * (ln & 3) + 2 * s;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (h < G) {
        const int cc[4] = {cb, cb + 4, cb + 1, cb + 5};
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = __bfloat162float(qg[(size_t)h * kD + __ldg(ch + cc[e])]);
      }
      qb[2 * tid] = pack_bf16x2(v[0], v[1]);
      qb[2 * tid + 1] = pack_bf16x2(v[2], v[3]);
    }
    if (tid >= 64 && tid < 64 + 8) {  // sum_c q~_h[c]
      const int h = tid - 64;
      float s = 0.f;
      if (h < G)
        for (int c = 0; c < d.d_c; ++c) s += __bfloat162float(qg[(size_t)h * kD + __ldg(ch + c)]);
      qsum[h] = s;
    }
  }
  __syncthreads();  // QQ, q~ ready; ring barriers initialised
  {
    float qreg[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) qreg[e] = QQ[lane * 8 + e];
    for (int gq = warp; gq < ngrp; gq += kWarps) {
      const int slot = gq % kRing;
      mbar_wait(&ring_bar[slot], (uint32_t)((gq / kRing) & 1));
      const uint8_t* tile = U + (size_t)slot * kGroupBytes;
      const int r8 = gq * 8;
      float acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc[u] = 0.f;
        if (r8 + u < nrows) {
          float f[8];
          unpack16<__nv_bfloat16>(reinterpret_cast<const uint4*>(tile + (size_t)u * kRowBytes)[lane], f);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[u] = fmaf(qreg[e], f[e], acc[u]);
        }
      }
      __syncwarp();
      if (lane == 0 && gq + kRing < ngrp) {  // refill this slot with group gq + kRing (same warp)
        const int g2 = gq + kRing;
        const int rows = min(8, nrows - 8 * g2);
        mbar_arrive_expect_tx(&ring_bar[slot], (uint32_t)(rows * kRowBytes));
        tma_bulk_g2s(U + (size_t)slot * kGroupBytes, bsrc + (size_t)g2 * kGroupBytes, (uint32_t)(rows * kRowBytes),
                     &ring_bar[slot]);
      }
      // transposed butterfly: lanes 4u..4u+3 end with the dot product of row u
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool up = lane & 16;
        const float send = up ? acc[j] : acc[j + 4];
        const float keep = up ? acc[j + 4] : acc[j];
        acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const bool up = lane & 8;
        const float send = up ? acc[j] : acc[j + 2];
        const float keep = up ? acc[j + 2] : acc[j];
        acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
      {
        const bool up = lane & 4;
        const float send = up ? acc[0] : acc[1];
        const float keep = up ? acc[1] : acc[0];
        acc[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 2);
      acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
      const int u = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      if ((lane & 3) == 0 && r8 + u < nrows) keys1[r8 + u] = f2key(acc[0]);
    }
  }
  __syncthreads();  // every score key of this CTA stored

  // ===================== a2: M_t = top-k_b blocks over the cluster =====================
  const TopkRes tb = cluster_topk(keys1, nrows, d.Kb, hist2, xcnt, ctl, nc, rank);
  const int Kb = tb.K;  // = min(k_b, m)
  {
    int pos = tb.pos;
    int* bout = p.block_ids + (size_t)pair * d.Kb;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (!((tb.sel >> u) & 1u)) continue;
      const int blk = i0 + 4 * tid + u;
      bout[pos] = blk;
      if (p.guide == nullptr) *dsmem(cand + pos % p.cb, (unsigned)(pos / p.cb)) = blk;  // a3 owner CTA
      ++pos;
    }
    if (rank == 0)
      for (int q = Kb + tid; q < d.Kb; q += kThreads) bout[q] = -1;
  }
  int nbl;  // this CTA's candidate blocks
  if (p.guide == nullptr) {
    cluster_sync_all();  // candidate lists complete
    nbl = max(0, min(p.cb, Kb - (int)rank * p.cb));
  } else {
    // lag mode: the candidates are the guide's valid ids (< m), in order; this CTA takes its slice
    const int* gd = p.guide + (size_t)pair * d.Kb;
    const int per = (d.Kb + kThreads - 1) / kThreads;
    const int lo = min(tid * per, d.Kb), hi = min(lo + per, d.Kb);
    int cnt = 0;
    for (int i = lo; i < hi; ++i) cnt += (gd[i] >= 0 && gd[i] < m);
    int total;
    int pos = block_exclusive_scan(cnt, ctl.scan, &total);
    const int kc = min(total, min(d.Kb, d.M));
    const int c0 = (int)rank * p.cb;
    for (int i = lo; i < hi; ++i)
      if (gd[i] >= 0 && gd[i] < m) {
        if (pos >= c0 && pos < min(c0 + p.cb, kc)) cand[pos - c0] = gd[i];
        ++pos;
      }
    nbl = max(0, min(p.cb, kc - c0));
    __syncthreads();
  }

  // ===================== a3: ranking keys of this CTA's candidate tokens =====================
  const int rowb = d.d_c / 2;  // 16 B of codes per token
  uint8_t* stc = U;
  float2* stz = reinterpret_cast<float2*>(U + (size_t)p.cb * d.B * rowb);
  if (warp == 0) {
    const uint8_t* cbase = p.codes + (size_t)pair * d.S * rowb;
    const float2* zbase = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * d.S;
    uint32_t bytes = 0;
    for (int k = lane; k < nbl; k += 32) bytes += (uint32_t)(min(d.B, d.S - cand[k] * d.B) * (rowb + 8));
    bytes = warp_sum_u32(bytes);
    if (lane == 0 && nbl > 0) mbar_arrive_expect_tx(&idx_bar, bytes);
    __syncwarp();
    for (int k = lane; k < nbl; k += 32) {
      const int blk = cand[k];
      const int rows = min(d.B, d.S - blk * d.B);
      tma_bulk_g2s(stc + (size_t)k * d.B * rowb, cbase + (size_t)blk * d.B * rowb, rows * rowb, &idx_bar);
      tma_bulk_g2s(stz + k * d.B, zbase + (size_t)blk * d.B, rows * 8, &idx_bar);
    }
  }
  if (nbl > 0) mbar_wait(&idx_bar, 0);
  const int q4 = lane & 3, r0 = lane >> 2;
  const float sm2 = d.sm_scale * kLog2e;
  float sq[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) sq[e] = sm2 * qsum[2 * q4 + e];
  const uint2* qb2 = reinterpret_cast<const uint2*>(qb);
  const int ntiles = nbl << (d.log2B - 4);
  const int tshift = d.log2B - 4;
  // pass 1: logits L of every tile (tile = warp + t * kWarps), per-warp head max
  float ev[kTPW][4];
  float hm[2] = {-CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
  for (int t = 0; t < kTPW; ++t) {
    const int tile = warp + t * kWarps;
    if (tile < ntiles) {
      float acc[1][4];
      token_tile_mma<kKS, 1, 1>(stc + (size_t)tile * 16 * rowb, qb2, acc);
      const int blk = cand[tile >> tshift];
      const int tok0 = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
      const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
      const float2 z0 = stz[tile * 16 + r0], z1 = stz[tile * 16 + r0 + 8];
      const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        ev[t][e] = v0 ? fmaf(s0, acc[0][e], z0.y * sq[e]) : -CUDART_INF_F;
        ev[t][2 + e] = v1 ? fmaf(s1, acc[0][2 + e], z1.y * sq[e]) : -CUDART_INF_F;
        hm[e] = fmaxf(hm[e], fmaxf(ev[t][e], ev[t][2 + e]));
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) ev[t][e] = -CUDART_INF_F;
    }
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) hm[e] = fmaxf(hm[e], __shfl_xor_sync(0xffffffffu, hm[e], o));
    const float mref = hm[e] == -CUDART_INF_F ? 0.f : hm[e];
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < kTPW; ++t) {
      ev[t][e] = fexp2(ev[t][e] - mref);
      ev[t][2 + e] = fexp2(ev[t][2 + e] - mref);
      s += ev[t][e] + ev[t][2 + e];
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (r0 == 0) {
      ctl.wm[warp][2 * q4 + e] = hm[e];
      ctl.ws[warp][2 * q4 + e] = s;
    }
  }
  __syncthreads();
  {  // CTA merge of the 8 warps' (max, sum) per head (8 lanes per head), pushed to every CTA of the pair
    const int w = tid & 7, h = tid >> 3;  // h < 32: warp-uniform shuffles
    const bool okh = h < G;
    const float mv = okh ? ctl.wm[w][h] : -CUDART_INF_F, sv = okh ? ctl.ws[w][h] : 0.f;
    float M = mv;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float S = (mv == -CUDART_INF_F) ? 0.f : sv * fexp2(mv - M);
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
    if (okh)
      for (unsigned rr = (unsigned)w; rr < nc; rr += 8) {
        *dsmem(&xm[rank * 8 + h], rr) = M;
        *dsmem(&xz[rank * 8 + h], rr) = S;
      }
  }
  cluster_sync_all();  // every CTA's statistics landed in every CTA
  {  // lz_h = M_h + log2 Z_h over the nc CTAs (16 lanes per head, rank order: deterministic)
    const int rr = tid & 15, h = tid >> 4;
    if (h < 16) {
      const bool ok = (unsigned)rr < nc && h < G;
      const float mv = ok ? xm[rr * 8 + h] : -CUDART_INF_F, sv = ok ? xz[rr * 8 + h] : 0.f;
      float M = mv;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      float S = (mv == -CUDART_INF_F) ? 0.f : sv * fexp2(mv - M);
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
      if (rr == 0 && h < 8) ctl.hlz[h] = h < G ? M + flog2(S) : CUDART_INF_F;
    }
  }
  __syncthreads();
  // pass 2: key_j = log2 sum_h 2^(L_hj - lz_h) (= log2 (G alpha~_j), reading U15) of every candidate slot
  {
    float cf[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int h = 2 * q4 + e;
      cf[e] = (h < G && hm[e] != -CUDART_INF_F) ? fexp2(hm[e] - ctl.hlz[h] + kKeyOff) : 0.f;
    }
    const bool bit0 = q4 & 1, bit1 = q4 & 2;
#pragma unroll
    for (int t = 0; t < kTPW; t += 2) {
      if (warp + t * kWarps >= ntiles) break;  // warp-uniform
      const float pa = ev[t][0] * cf[0] + ev[t][1] * cf[1];
      const float pb = ev[t][2] * cf[0] + ev[t][3] * cf[1];
      const float pc = ev[t + 1][0] * cf[0] + ev[t + 1][1] * cf[1];
      const float pd = ev[t + 1][2] * cf[0] + ev[t + 1][3] * cf[1];
      float k1 = bit0 ? pb : pa, k2 = bit0 ? pd : pc;
      k1 += __shfl_xor_sync(0xffffffffu, bit0 ? pa : pb, 1);
      k2 += __shfl_xor_sync(0xffffffffu, bit0 ? pc : pd, 1);
      float mine = bit1 ? k2 : k1;
      mine += __shfl_xor_sync(0xffffffffu, bit1 ? k1 : k2, 2);
      const int tile = warp + (t + (bit1 ? 1 : 0)) * kWarps;
      const int row = r0 + (bit0 ? 8 : 0);
      if (tile < ntiles) {
        const int blk = cand[tile >> tshift];
        const int tok = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + row;
        keys[tile * 16 + row] = tok < n ? f2key(flog2(mine) - kKeyOff) : 0u;
      }
    }
  }
  __syncthreads();

  // ===================== a4: S_t = top-k_t tokens over the cluster =====================
  const int nslots = nbl << d.log2B;
  const TopkRes tt = cluster_topk(keys, nslots, d.Kt, hist2, xcnt, ctl, nc, rank);
  const int Kt = tt.K;
  {
    int pos = tt.pos;
    int* tout = p.token_ids + (size_t)pair * d.Kt;
    float* sout = p.token_scores ? p.token_scores + (size_t)pair * d.Kt : nullptr;
    const float lnG = logf((float)G);
    const int* sob = p.slot_of_block ? p.slot_of_block + (size_t)pair * d.M : nullptr;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (!((tt.sel >> u) & 1u)) continue;
      const int s = 4 * tid + u;
      const int tok = (cand[s >> d.log2B] << d.log2B) + (s & (d.B - 1));
      tout[pos] = tok;
      if (sout) sout[pos] = key2f(keys[s]) * kLn2 - lnG;
      if (p.attend) {
        const int o = slice_owner(pos, Kt, (int)nc);
        const int t0o = (int)(((long long)Kt * o) / (int)nc);
        int row = tok;
        if (sob) {  // block cache: the token's row in the slot arrays (its block must be resident)
          const int sl = sob[tok >> d.log2B];
          row = sl >= 0 ? (sl << d.log2B) + (tok & (d.B - 1)) : 0;
        }
        *dsmem(sel + (pos - t0o), (unsigned)o) = row;
      }
      ++pos;
    }
    if (rank == 0) {
      for (int q = Kt + tid; q < d.Kt; q += kThreads) {
        tout[q] = -1;
        if (sout) sout[q] = -CUDART_INF_F;
      }
      if (tid == 0) p.num_tokens[pair] = Kt;
    }
  }
  cluster_sync_all();  // every CTA's selected-token slice complete (and every remote read of xcnt done)
  if (!p.attend) return;  // selection only (tls_select)

  // ===================== a5: attention over this CTA's slice of S_t =====================
  const int t0 = (int)(((long long)Kt * rank) / nc);
  const int tloc = (int)(((long long)Kt * (rank + 1)) / nc) - t0;
  float* part = reinterpret_cast<float*>(U + kPartOff);  // [8 heads][kD] o, then [8][2] (m, l)
  {
    constexpr int CPR = kD / 8;
    const int r = lane >> 2, q = lane & 3;
    const int tg = warp >> 1, dh = warp & 1;
    __nv_bfloat16* sbuf = reinterpret_cast<__nv_bfloat16*>(U);  // [kStages][K kTC*kD | V kTC*kD]
    __nv_bfloat16* pbuf = reinterpret_cast<__nv_bfloat16*>(keys1) + warp * 256;  // [2 pieces][8 heads][16 tokens]
    const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_cache) + (size_t)pair * p.kv_rows * kD;
    const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(p.v_cache) + (size_t)pair * p.kv_rows * kD;
    const int nchunks = (tloc + kTC - 1) / kTC;
    auto load_chunk = [&](int c, int stage) {
      __nv_bfloat16* sK = sbuf + (size_t)stage * 2 * kTC * kD;
      __nv_bfloat16* sV = sK + kTC * kD;
      const int ntk = min(kTC, tloc - c * kTC);
#pragma unroll
      for (int it = 0; it < (kTC * CPR) / kThreads; ++it) {
        const int i = tid + it * kThreads;
        const int row = i / CPR, chk = i - row * CPR;
        const bool ok = row < ntk;
        const int tok = ok ? sel[c * kTC + row] : 0;
        const int dst = row * kD + ((chk ^ (row & 7)) << 3);
        cp_async16(sK + dst, kb + (size_t)tok * kD + chk * 8, ok);
        cp_async16(sV + dst, vb + (size_t)tok * kD + chk * 8, ok);
      }
      cp_async_commit();
    };
#pragma unroll
    for (int c = 0; c < kStages - 1; ++c) {
      if (c < nchunks) load_chunk(c, c);
      else cp_async_commit();
    }
    // Q^T as the B operand: b0 = Q[head r][16k + 2q, +1], b1 = Q[head r][16k + 2q + 8, +9] (heads >= G: 0)
    uint32_t qf[kD / 16][2];
#pragma unroll
    for (int k = 0; k < kD / 16; ++k) {
      qf[k][0] = r < G ? *reinterpret_cast<const uint32_t*>(qg + r * kD + 16 * k + 2 * q) : 0u;
      qf[k][1] = r < G ? *reinterpret_cast<const uint32_t*>(qg + r * kD + 16 * k + 2 * q + 8) : 0u;
    }
    float mrun[2] = {-CUDART_INF_F, -CUDART_INF_F}, lrun[2] = {0.f, 0.f};  // heads 2q, 2q + 1
    float o[4][4];  // O^T: m-tile mt = dims 64 dh + 16 mt + (r, r + 8), heads (2q, 2q + 1)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    for (int c = 0; c < nchunks; ++c) {
      if (c + kStages - 1 < nchunks) load_chunk(c + kStages - 1, (c + kStages - 1) % kStages);
      else cp_async_commit();
      cp_async_wait<kStages - 1>();
      __syncthreads();  // chunk c landed for every thread's copies
      const __nv_bfloat16* sK = sbuf + (size_t)(c % kStages) * 2 * kTC * kD;
      const __nv_bfloat16* sV = sK + kTC * kD;
      const int ntk = min(kTC, tloc - c * kTC);
      const int tb0 = tg * 16;
      if (tb0 < ntk) {
        // S^T (16 tokens x 8 heads) = K Q^T
        float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const int row = tb0 + (lane & 7) + ((lane >> 3) & 1) * 8;
          const int chk = 2 * k + (lane >> 4);
          uint32_t a[4];
          ldsm_x4(a, sK + row * kD + ((chk ^ (row & 7)) << 3));
          mma_bf16_16816(s, a, qf[k][0], qf[k][1]);
        }
        const bool v0 = tb0 + r < ntk, v1 = tb0 + r + 8 < ntk;
        s[0] = v0 ? s[0] * sm2 : -CUDART_INF_F;
        s[1] = v0 ? s[1] * sm2 : -CUDART_INF_F;
        s[2] = v1 ? s[2] * sm2 : -CUDART_INF_F;
        s[3] = v1 ? s[3] * sm2 : -CUDART_INF_F;
        float x0 = fmaxf(s[0], s[2]), x1 = fmaxf(s[1], s[3]);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, off));
          x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, off));
        }
        // lazy rescaling: the reference max moves only when a score exceeds it by > 8 (log2 units)
        const bool g0 = x0 > mrun[0] + 8.f, g1 = x1 > mrun[1] + 8.f;
        const float n0 = g0 ? x0 : mrun[0], n1 = g1 ? x1 : mrun[1];
        const float a0 = g0 ? fexp2(mrun[0] - n0) : 1.f, a1 = g1 ? fexp2(mrun[1] - n1) : 1.f;
        const float p0 = fexp2(s[0] - n0), p1 = fexp2(s[1] - n1), p2 = fexp2(s[2] - n0), p3 = fexp2(s[3] - n1);
        float r0s = p0 + p2, r1s = p1 + p3;
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          r0s += __shfl_xor_sync(0xffffffffu, r0s, off);
          r1s += __shfl_xor_sync(0xffffffffu, r1s, off);
        }
        lrun[0] = lrun[0] * a0 + r0s;
        lrun[1] = lrun[1] * a1 + r1s;
        mrun[0] = n0;
        mrun[1] = n1;
        if (__any_sync(0xffffffffu, g0 || g1)) {
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            o[mt][0] *= a0;
            o[mt][1] *= a1;
            o[mt][2] *= a0;
            o[mt][3] *= a1;
          }
        }
        // P^T as two bf16 pieces (hi + lo: the PV product keeps ~16 bits of P) into the B layout
        const float pv[4] = {p0, p1, p2, p3};
        const int pi[4] = {(2 * q) * 16 + r, (2 * q + 1) * 16 + r, (2 * q) * 16 + r + 8, (2 * q + 1) * 16 + r + 8};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const __nv_bfloat16 hi = __float2bfloat16_rn(pv[e]);
          pbuf[pi[e]] = hi;
          pbuf[128 + pi[e]] = __float2bfloat16_rn(pv[e] - __bfloat162float(hi));
        }
        __syncwarp();
        const uint32_t ph0 = *reinterpret_cast<const uint32_t*>(pbuf + r * 16 + 2 * q);
        const uint32_t ph1 = *reinterpret_cast<const uint32_t*>(pbuf + r * 16 + 2 * q + 8);
        const uint32_t pl0 = *reinterpret_cast<const uint32_t*>(pbuf + 128 + r * 16 + 2 * q);
        const uint32_t pl1 = *reinterpret_cast<const uint32_t*>(pbuf + 128 + r * 16 + 2 * q + 8);
        __syncwarp();
        // O^T (64 dims x 8 heads) += V^T (dims x 16 tokens) P^T
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const int token = tb0 + (lane & 7) + ((lane >> 4) & 1) * 8;
          const int chk = (dh * 64 + 16 * mt) / 8 + ((lane >> 3) & 1);
          uint32_t a[4];
          ldsm_x4_trans(a, sV + token * kD + ((chk ^ (token & 7)) << 3));
          mma_bf16_16816(o[mt], a, ph0, ph1);
          mma_bf16_16816(o[mt], a, pl0, pl1);
        }
      }
      __syncthreads();  // stage c % kStages consumed before it is refilled
    }
    cp_async_wait<0>();
    // merge the 4 token groups of this CTA (the staging buffers become scratch) -> part
    constexpr int WS = kD + 4;
    float* wo = reinterpret_cast<float*>(U);  // [tg][8 heads][WS]
    float* wml = wo + 4 * 8 * WS;             // [tg][8 heads][2]
    if (dh == 0 && r == 0) {
      wml[(tg * 8 + 2 * q) * 2] = mrun[0];
      wml[(tg * 8 + 2 * q) * 2 + 1] = lrun[0];
      wml[(tg * 8 + 2 * q + 1) * 2] = mrun[1];
      wml[(tg * 8 + 2 * q + 1) * 2 + 1] = lrun[1];
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int d0 = dh * 64 + 16 * mt + r;
      wo[(tg * 8 + 2 * q) * WS + d0] = o[mt][0];
      wo[(tg * 8 + 2 * q + 1) * WS + d0] = o[mt][1];
      wo[(tg * 8 + 2 * q) * WS + d0 + 8] = o[mt][2];
      wo[(tg * 8 + 2 * q + 1) * WS + d0 + 8] = o[mt][3];
    }
    __syncthreads();
    const int ngroups = min(4, (min(tloc, kTC) + 15) / 16);  // token groups that saw at least one token
    for (int idx = tid; idx < G * kD; idx += kThreads) {
      const int h = idx / kD, dcol = idx - h * kD;
      float M = -CUDART_INF_F;
      for (int t = 0; t < ngroups; ++t) M = fmaxf(M, wml[(t * 8 + h) * 2]);
      float L = 0.f, acc = 0.f;
      if (M != -CUDART_INF_F) {
        for (int t = 0; t < ngroups; ++t) {
          const float mw = wml[(t * 8 + h) * 2];
          const float sc = mw == -CUDART_INF_F ? 0.f : fexp2(mw - M);
          L = fmaf(wml[(t * 8 + h) * 2 + 1], sc, L);
          acc = fmaf(wo[(t * 8 + h) * WS + dcol], sc, acc);
        }
      }
      part[idx] = acc;
      if (dcol == 0) {
        part[8 * kD + 2 * h] = M;
        part[8 * kD + 2 * h + 1] = L;
      }
    }
  }
  cluster_sync_all();  // every CTA's partial (o, m, l) visible
  // ---- merge the nc partials (flash-decoding LSE identity, T10); CTA rank writes a 1/nc slice ----
  {
    if (tid < G) {
      float M = -CUDART_INF_F;
      float mq[kMaxNC], lq[kMaxNC];
#pragma unroll
      for (int qq = 0; qq < kMaxNC; ++qq) {
        mq[qq] = (unsigned)qq < nc ? *dsmem(part + 8 * kD + 2 * tid, (unsigned)qq) : -CUDART_INF_F;
        lq[qq] = (unsigned)qq < nc ? *dsmem(part + 8 * kD + 2 * tid + 1, (unsigned)qq) : 0.f;
        M = fmaxf(M, mq[qq]);
      }
      float L = 0.f;
#pragma unroll
      for (int qq = 0; qq < kMaxNC; ++qq) {
        const float w = (M == -CUDART_INF_F || mq[qq] == -CUDART_INF_F) ? 0.f : fexp2(mq[qq] - M);
        L = fmaf(lq[qq], w, L);
        if (qq < kMaxNC) ctl.mw[qq][tid] = w;
      }
      ctl.minv[tid] = L > 0.f ? 1.f / L : 0.f;
      if (rank == 0 && p.lse != nullptr)
        p.lse[(size_t)b * d.Hq + (size_t)g * G + tid] = L > 0.f ? (M + flog2(L)) * kLn2 : -CUDART_INF_F;
    }
    __syncthreads();
    const int tot = G * kD;
    const int lo = (int)(((long long)tot * rank) / nc), hi = (int)(((long long)tot * (rank + 1)) / nc);
    __nv_bfloat16* outg = reinterpret_cast<__nv_bfloat16*>(p.out) + ((size_t)b * d.Hq + (size_t)g * G) * kD;
    for (int idx = lo + tid; idx < hi; idx += kThreads) {
      const int h = idx / kD;
      float v[kMaxNC];
#pragma unroll
      for (int qq = 0; qq < kMaxNC; ++qq) v[qq] = (unsigned)qq < nc ? *dsmem(part + idx, (unsigned)qq) : 0.f;
      float acc = 0.f;
#pragma unroll
      for (int qq = 0; qq < kMaxNC; ++qq)
        if ((unsigned)qq < nc) acc = fmaf(v[qq], ctl.mw[qq][h], acc);
      outg[idx] = __float2bfloat16_rn(acc * ctl.minv[h]);
    }
  }
  cluster_sync_all();  // keep this CTA's partial alive until every remote reader is done
}

// ============================================================== host side
// Whether the fused step kernel handles this configuration (else the kernel
// chain runs), and its plan.
bool step_supported(const Dims& d) {
  return d.bf16 && !d.mla && d.d_k == kD && d.d_v == kD && d.G <= 8 && d.d_c == 32 && d.B == 64 && (d.S % 2) == 0;
}

bool plan_step(StepKParams& p, int nc) {
  const Dims& d = p.d;
  p.nc = nc;
  const int kb_eff = kb_effective(d);
  p.mb = (((d.M + nc - 1) / nc) + 7) & ~7;
  p.cb = (kb_eff + nc - 1) / nc;
  const int kt_eff = kt_effective(d);
  p.tok_max = (kt_eff + nc - 1) / nc;
  if (p.mb > 4 * kThreads) return false;            // a1 keys per CTA (4 per thread)
  if (p.cb * d.B > 4 * kThreads) return false;      // a3 candidate slots per CTA (4 per thread, 8 tiles per warp)
  if ((size_t)p.cb * d.B * (d.d_c / 2 + 8) > kKeys3Off) return false;  // a3 index stage below the a3 keys
  size_t o = 0;
  p.off_u = (unsigned)o;
  o += kUBytes;
  p.off_keys = (unsigned)o;  // a1 score keys (the a5 P buffers, 8 warps x 512 B, alias keys .. cand)
  o = align16(o + (size_t)(p.mb > 128 ? p.mb : 128) * 4);
  p.off_hist = (unsigned)o;  // 2 x 256 bins (double-buffered radix rounds); QQ during a1
  o = align16(o + 2 * 256 * 4);
  p.off_xs = (unsigned)o;
  o = align16(o + 2 * kMaxNC * 8 * 4);
  p.off_qb = (unsigned)o;
  o = align16(o + kKS * 256 + 8 * 4);
  p.off_cand = (unsigned)o;
  o = align16(o + (size_t)p.cb * 4);
  if (o < p.off_keys + (size_t)kWarps * 512) o = p.off_keys + (size_t)kWarps * 512;
  p.off_sel = (unsigned)o;
  o = align16(o + (size_t)(p.tok_max + 1) * 4);
  p.off_qq = p.off_hist;
  p.off_part = (unsigned)(p.off_u + kPartOff);
  p.smem_bytes = (unsigned)o;
  return true;
}

cudaError_t launch_step(const StepKParams& p, cudaStream_t st) {
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(step_kernel), p.smem_bytes, p.nc > 8);
  if (e != cudaSuccess) return e;
  return launch_ex(step_kernel, dim3((unsigned)p.nc, (unsigned)(p.d.batch * p.d.Hkv), 1), kThreads, p.smem_bytes, st,
                   LaunchOpts{}, (unsigned)p.nc, p);
}

}  // namespace tls
