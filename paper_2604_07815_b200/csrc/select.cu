// select.cu -- token scoring (a3) of AsyncTLS (arXiv 2604.07815) for sm_100a.
//
// The decode step's kernels: qq_kernel + select_kernel (fused.cu: a1 block
// scores as an HBM-streaming GEMV, a2 top-k_b in each pair's last tile CTA),
// then K2 here, then attend_kernel (attend.cu: a4 top-k_t prologue + a5).
//   K2 token_pair_kernel    a3  (default, G <= 8) one cluster of 1 / 2 / 4 CTAs
//                               per pair holding the pair's whole candidate
//                               index in shared memory (cp.async staging in
//                               mbarrier groups), logits on the tensor cores
//                               (mma.sync) kept in TMEM between the two passes
//   K2 token_pair_nt_kernel a3  (G > 8, MLA) the same with NT n-tiles of 8
//                               heads: a cluster of 8 / 16 CTAs, statistics by
//                               a second pass over TMEM
//   K2 token_reg_kernel     a3  alpha~_j over the candidate tokens:
//                               a cluster of nch chunk CTAs per pair, logits on
//                               the tensor cores (mma.sync, INT4 codes -> bf16)
//                               kept in registers, softmax statistics merged
//                               over DSMEM, ranking keys and their histogram ->
//                               workspace
//   K2 token_cluster_kernel a3  the same contract when a chunk exceeds the
//                               registers (two tensor-core passes over smem)
// Citation key: P:n = line n of PAPER.md.  Readings U1..U20: DESIGN.md §3.
#include <math_constants.h>

#include "common.cuh"
#include "params.h"
#include "topk.cuh"
#include "fasttopk.cuh"
#include "launch.h"
#include "token.cuh"

namespace tls {

// ============================================================== K2: a3
// token_cluster_kernel: grid (nch, pairs), one cluster of nch CTAs per pair;
// CTA c owns candidate blocks [c*cb, (c+1)*cb) of M_t (or of the lag-mode
// guide), staged once into shared memory with one TMA bulk copy per block and
// run (single-use mbarrier).  Pass 1: online per-head (max, sum) of the
// chunk's logits; the nch chunks' statistics are merged through DSMEM in chunk
// order (deterministic) into lz_h = M_h + log2 Z_h.  Pass 2 (same staged
// index): the ranking key log2 sum_h exp2(L_hj - lz_h) of every candidate slot
// -> workspace keys (0 past the sequence end), plus a fixed-bin histogram of
// the keys (red.add into the pair's histogram, zeroed by K1).
// The logits L_hj = sm_scale*log2e*(zero_j*sum_c q~_h[c] + scale_j*(q~_h.code_j))
// are formed on tensor cores (token_tile_mma).
struct SelCtl {
  TopKCtl tk;
  int kc;
  float hlz[32];
  float wm[kWarps][32], ws[kWarps][32];
  int chan[128];
};

template <typename T, int KS, int NT, int NSPLIT>
__global__ void __launch_bounds__(kThreads, (NT == 1 && KS * NSPLIT <= 2) ? 5 : 3) token_cluster_kernel(const __grid_constant__ SelectParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ SelCtl ctl;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t lhist[kKeyBins];
  __shared__ float s_hm[32], s_hz[32];
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q4 = lane & 3, r0 = lane >> 2;
  const int chunk = blockIdx.x, pair = blockIdx.y;
  unsigned long long* dbg = p.dbg ? p.dbg + ((size_t)pair * 8 + chunk) * 8 : nullptr;
#define TLS_STAMP(i) \
  if (dbg && tid == 0) dbg[i] = gtimer();
  TLS_STAMP(0)
  launch_dependents();
  if (tid == 0) wait_ready(p.ready_in + pair, p.epoch);  // select_kernel's a2 outputs for this pair
  __syncthreads();
  for (int i = tid; i < kKeyBins; i += kThreads) lhist[i] = 0u;
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;
  int* cblk = reinterpret_cast<int*>(smem + p.off_cblk);
  uint32_t* qb = reinterpret_cast<uint32_t*>(smem + p.off_qb);
  float* qsum = reinterpret_cast<float*>(smem + p.off_qsum);
  float* qc = reinterpret_cast<float*>(smem + p.off_qc);
  uint8_t* stc = smem + p.off_stage;
  float2* stz = reinterpret_cast<float2*>(smem + p.off_stage + (size_t)p.cb * d.B * (d.d_c / 2));
  __shared__ __align__(8) uint64_t qbar;
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * d.Hq + (size_t)g * d.G) * d.d_k;
  T* qrows = reinterpret_cast<T*>(smem + p.off_qrows);
  int* chan_s = reinterpret_cast<int*>(smem + p.off_qrows + (size_t)d.G * d.d_k * sizeof(T));
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&qbar, 1);
    mbar_fence_init();
    if (p.qfrag != nullptr) {  // the pair's q~ fragment blob built by qq_kernel: one TMA bulk copy
      const uint32_t qfb = (uint32_t)(NSPLIT * NT * KS * 256 + NT * 32);
      mbar_arrive_expect_tx(&qbar, qfb);
      tma_bulk_g2s(smem + p.off_qb, p.qfrag + (size_t)pair * qfb, qfb, &qbar);
    } else if (p.qtma) {  // the pair's q rows and channel ids: two TMA bulk copies
      const uint32_t qb_ = (uint32_t)(d.G * d.d_k * sizeof(T)), cb_ = (uint32_t)(d.d_c * 4);
      mbar_arrive_expect_tx(&qbar, qb_ + cb_);
      tma_bulk_g2s(qrows, qg, qb_, &qbar);
      tma_bulk_g2s(chan_s, p.channels + (size_t)g * d.d_c, cb_, &qbar);
    }
  }
  if (p.qfrag == nullptr && !p.qtma && tid < KS * 16) ctl.chan[tid] = p.channels[(size_t)g * d.d_c + tid];
  const int* cand = p.guide ? p.guide + (size_t)pair * d.Kb : p.block_ids + (size_t)pair * d.Kb;
  // ---- candidate blocks (ascending): M_t from K1 (block_ids) or the lag-mode guide ----
  {
    const int per = (d.Kb + kThreads - 1) / kThreads;
    const int lo = min(tid * per, d.Kb), hi = min(lo + per, d.Kb);
    int cnt = 0;
    for (int i = lo; i < hi; ++i) cnt += (cand[i] >= 0 && cand[i] < m);
    int total;
    int pos = block_exclusive_scan(cnt, ctl.tk.scan, &total);
    for (int i = lo; i < hi; ++i)
      if (cand[i] >= 0 && cand[i] < m && pos < p.kb_eff) cblk[pos++] = cand[i];
    if (tid == 0) ctl.kc = min(total, p.kb_eff);
  }
  __syncthreads();
  const int kc = ctl.kc;
  const int cb0 = chunk * p.cb, cb1 = min(cb0 + p.cb, kc);
  const int nbl = cb1 - cb0;
  const int rowbytes = d.d_c / 2;
  const uint8_t* cbase = p.codes + (size_t)pair * d.S * rowbytes;
  const float2* zbase = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * d.S;
  const bool zal = (d.S & 1) == 0;  // every block's scale/zero rows 16-byte aligned and sized -> TMA
  if (nbl > 0 && tid == 0) {  // stage this chunk's candidate index (TMA bulk, one barrier)
    uint32_t bytes = 0;
    for (int k = 0; k < nbl; ++k) {
      const int rows = min(d.B, d.S - cblk[cb0 + k] * d.B);
      bytes += rows * rowbytes + (zal ? rows * 8 : 0);
    }
    mbar_arrive_expect_tx(&bar, bytes);
    for (int k = 0; k < nbl; ++k) {
      const int blk = cblk[cb0 + k];
      const int rows = min(d.B, d.S - blk * d.B);
      tma_bulk_g2s(stc + (size_t)k * d.B * rowbytes, cbase + (size_t)blk * d.B * rowbytes, rows * rowbytes, &bar);
      if (zal) tma_bulk_g2s(stz + k * d.B, zbase + (size_t)blk * d.B, rows * 8, &bar);
    }
  }
  // ---- channel-projected query q~, its B fragments and sum ----
  constexpr int DC = KS * 16;
  if (p.qfrag != nullptr) {
    mbar_wait(&qbar, 0);
  } else {
  if (p.qtma) {
    mbar_wait(&qbar, 0);
    for (int i = tid; i < NT * 8 * DC; i += kThreads) {
      const int h = i / DC, c = i - h * DC;
      qc[i] = h < d.G ? to_f32<T>(qrows[(size_t)h * d.d_k + chan_s[c]]) : 0.f;
    }
  } else {
    for (int i = tid; i < NT * 8 * DC; i += kThreads) {
      const int h = i / DC, c = i - h * DC;
      qc[i] = h < d.G ? to_f32<T>(qg[(size_t)h * d.d_k + ctl.chan[c]]) : 0.f;
    }
  }
  __syncthreads();
  constexpr int WPT = KS / 2;
  for (int idx = tid; idx < NSPLIT * NT * KS * 32; idx += kThreads) {
    const int ln = idx & 31, rest = idx >> 5;
    const int s = rest % KS, nt = (rest / KS) % NT, sp = rest / (KS * NT);
    const float* qh = qc + (nt * 8 + (ln >> 2)) * DC;
    const int cb = 8 * ((ln & 3) * WPT + (s >> 1)) + 2 * (s & 1);
    qb[2 * idx] = pack_bf16x2(split_piece(qh[cb], sp), split_piece(qh[cb + 4], sp));
    qb[2 * idx + 1] = pack_bf16x2(split_piece(qh[cb + 1], sp), split_piece(qh[cb + 5], sp));
  }
  if (tid < NT * 8) {
    float s = 0.f;
    for (int c = 0; c < DC; ++c) s += qc[tid * DC + c];
    qsum[tid] = s;
  }
  __syncthreads();
  }
  TLS_STAMP(1)
  if (nbl > 0) mbar_wait(&bar, 0);
  TLS_STAMP(2)
  const float sm2 = d.sm_scale * kLog2e;
  float sq[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) sq[nt][e] = sm2 * qsum[nt * 8 + 2 * q4 + e];
  const uint2* qb2 = reinterpret_cast<const uint2*>(qb);
  const int tshift = d.log2B - 4;
  const int ntiles = nbl << tshift;
  const float2* zglob = zbase;
  {  // pass 1: per-head online (max, sum) of this chunk's logits
    float rm[NT][2], rs[NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i) rm[i][0] = rm[i][1] = -CUDART_INF_F, rs[i][0] = rs[i][1] = 0.f;
    for (int tp = warp * 2; tp < ntiles; tp += kWarps * 2) {  // two independent tiles per step
      float acc[2][NT][4];
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (tp + u < ntiles) token_tile_mma<KS, NT, NSPLIT>(stc + (size_t)(tp + u) * 16 * rowbytes, qb2, acc[u]);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int tile = tp + u;
        if (tile >= ntiles) break;
        const int blk = cblk[cb0 + (tile >> tshift)];
        const int tok0 = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
        const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
        const float2 z0 = zal ? stz[tile * 16 + r0] : (v0 ? __ldg(zglob + tok0) : make_float2(0.f, 0.f));
        const float2 z1 = zal ? stz[tile * 16 + r0 + 8] : (v1 ? __ldg(zglob + tok0 + 8) : make_float2(0.f, 0.f));
        const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float l0 = v0 ? fmaf(s0, acc[u][nt][e], z0.y * sq[nt][e]) : -CUDART_INF_F;
            const float l1 = v1 ? fmaf(s1, acc[u][nt][2 + e], z1.y * sq[nt][e]) : -CUDART_INF_F;
            const float mt = fmaxf(l0, l1);
            if (mt > rm[nt][e]) {  // rescale only when the running max grows
              rs[nt][e] *= fexp2(rm[nt][e] - mt);
              rm[nt][e] = mt;
            }
            if (mt != -CUDART_INF_F) rs[nt][e] += fexp2(l0 - rm[nt][e]) + fexp2(l1 - rm[nt][e]);
          }
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          const float om = __shfl_xor_sync(0xffffffffu, rm[nt][e], o);
          const float os = __shfl_xor_sync(0xffffffffu, rs[nt][e], o);
          stat_merge(rm[nt][e], rs[nt][e], om, os);
        }
    if (r0 == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          ctl.wm[warp][nt * 8 + 2 * q4 + e] = rm[nt][e];
          ctl.ws[warp][nt * 8 + 2 * q4 + e] = rs[nt][e];
        }
    }
    __syncthreads();
    if (tid < d.G) {  // warps merged in a fixed order (deterministic)
      float mm = -CUDART_INF_F, ss = 0.f;
      for (int w = 0; w < kWarps; ++w) stat_merge(mm, ss, ctl.wm[w][tid], ctl.ws[w][tid]);
      s_hm[tid] = mm;
      s_hz[tid] = ss;
    }
  }
  // ---- merge the nch chunks' statistics of the pair through DSMEM, in chunk order ----
  TLS_STAMP(3)
  cluster_sync_all();
  TLS_STAMP(4)
  if (chunk == 0 && tid == 0) p.ready_in[pair] = 0u;  // every CTA of the pair passed its wait
  if (tid < d.G) {
    float M = -CUDART_INF_F, Z = 0.f;
    for (int rr = 0; rr < (int)gridDim.x; ++rr) stat_merge(M, Z, *dsmem(&s_hm[tid], rr), *dsmem(&s_hz[tid], rr));
    ctl.hlz[tid] = M + flog2(Z);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");  // remote reads done
  __syncthreads();
  {  // pass 2: ranking keys
    float lz[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int h = nt * 8 + 2 * q4 + e;
        lz[nt][e] = h < d.G ? ctl.hlz[h] : CUDART_INF_F;  // padded heads: exp2(-inf) = 0
      }
    uint32_t* kout = p.keys + (size_t)pair * p.kb_eff * d.B + ((size_t)cb0 << d.log2B);
    for (int tp = warp * 2; tp < ntiles; tp += kWarps * 2) {  // two independent tiles per step
      float acc[2][NT][4];
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (tp + u < ntiles) token_tile_mma<KS, NT, NSPLIT>(stc + (size_t)(tp + u) * 16 * rowbytes, qb2, acc[u]);
      float mx[2][2], es[2][2];
      bool vv[2][2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int tile = min(tp + u, ntiles - 1);
        const int blk = cblk[cb0 + (tile >> tshift)];
        const int tok0 = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
        vv[u][0] = tp + u < ntiles && tok0 < n;
        vv[u][1] = tp + u < ntiles && tok0 + 8 < n;
        const float2 z0 = zal ? stz[tile * 16 + r0] : (vv[u][0] ? __ldg(zglob + tok0) : make_float2(0.f, 0.f));
        const float2 z1 = zal ? stz[tile * 16 + r0 + 8] : (vv[u][1] ? __ldg(zglob + tok0 + 8) : make_float2(0.f, 0.f));
        const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
        float t0[NT][2], t1[NT][2];
        float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            t0[nt][e] = fmaf(s0, acc[u][nt][e], fmaf(z0.y, sq[nt][e], -lz[nt][e]));
            t1[nt][e] = fmaf(s1, acc[u][nt][2 + e], fmaf(z1.y, sq[nt][e], -lz[nt][e]));
            m0 = fmaxf(m0, t0[nt][e]);
            m1 = fmaxf(m1, t1[nt][e]);
          }
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
        float e0 = 0.f, e1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            e0 += fexp2(t0[nt][e] - m0);
            e1 += fexp2(t1[nt][e] - m1);
          }
        e0 += __shfl_xor_sync(0xffffffffu, e0, 1);
        e0 += __shfl_xor_sync(0xffffffffu, e0, 2);
        e1 += __shfl_xor_sync(0xffffffffu, e1, 1);
        e1 += __shfl_xor_sync(0xffffffffu, e1, 2);
        mx[u][0] = m0;
        mx[u][1] = m1;
        es[u][0] = e0;
        es[u][1] = e1;
      }
      // lane q4 = 0 finishes row r0, lane q4 = 1 row r0 + 8 (of both tiles)
      if (q4 < 2) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (tp + u >= ntiles) break;
          const int j = (tp + u) * 16 + r0 + 8 * q4;
          const bool v = q4 == 0 ? vv[u][0] : vv[u][1];
          const float kf = (q4 == 0 ? mx[u][0] : mx[u][1]) + flog2(q4 == 0 ? es[u][0] : es[u][1]);
          kout[j] = v ? f2key(kf) : 0u;
          if (v) atomicAdd(&lhist[key_bin(kf)], 1u);
        }
      }
    }
    __syncthreads();
    uint32_t* gh = p.khist + (size_t)pair * kKeyBins;
    for (int i = tid; i < kKeyBins; i += kThreads)
      if (lhist[i]) atomicAdd(&gh[i], lhist[i]);
  }
  TLS_STAMP(5)
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");  // keep smem alive for remote readers
  __syncthreads();
  if (tid == 0)  // hand-off: one count per chunk CTA (the attention kernel waits for nch); a release add,
                  // cumulative over the CTA barrier
    red_release_add_gpu(p.ready_out + pair, 1u);
  TLS_STAMP(6)
#undef TLS_STAMP
}

// ----------------------------------------------------------------------------
// K2, register-resident form (used whenever a CTA's tiles fit: <= TPW 16-token
// tiles per warp, TPW = 8 / NT).  Same arithmetic contract as
// token_cluster_kernel, one tensor-core pass instead of two:
//   pass 1: L_hj for every staged tile (token_tile_mma, once); per-warp head
//           max m_h^w; E_hj = exp2(L_hj - m_h^w) kept in registers; per-warp
//           sums -> CTA -> cluster (DSMEM, chunk order) -> lz_h = M_h + log2 Z_h.
//   pass 2: sum_h exp2(L_hj - lz_h) = 2^r_w sum_h E_hj * c_h^w with the
//           per-(warp, head) factor c_h^w = exp2(m_h^w - lz_h - r_w), r_w its
//           max over heads, reduced over the four lanes that hold a token's
//           heads with a transposed butterfly (3 shuffles per 4 tokens); every
//           lane emits one key.  A warp whose logits of some head span more
//           than kUnder (attention-sink-like keys) keeps L instead of E and
//           forms its keys in the log domain (reading U20: exact for any logit
//           span; test_sink_tokens_wide_logit_span).
constexpr float kUnder = 100.f;

// 4 CTAs / SM (64 registers) where the variant fits without spilling, else 3.
template <int KS, int NT, int NSPLIT>
constexpr int k2_min_blocks() { return (NT == 1 && KS * NSPLIT <= 6) ? 4 : 3; }

template <typename T, int KS, int NT, int NSPLIT, int TPW>
__global__ void __launch_bounds__(kThreads, k2_min_blocks<KS, NT, NSPLIT>()) token_reg_kernel(const __grid_constant__ SelectParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ SelCtl ctl;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t qbar;
  __shared__ uint32_t lhist[kKeyBins];
  __shared__ float s_cm[16][32], s_cz[16][32];  // [chunk rank][head]: every chunk's stats, pushed by that chunk
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q4 = lane & 3, r0 = lane >> 2;
  const int chunk = blockIdx.x, pair = blockIdx.y;
  unsigned long long* dbg = p.dbg && chunk < 8 ? p.dbg + ((size_t)pair * 8 + chunk) * 8 : nullptr;
#define TLS_STAMP(i) \
  if (dbg && tid == 0) dbg[i] = gtimer();
  TLS_STAMP(0)
  launch_dependents();
  for (int i = tid; i < kKeyBins; i += kThreads) lhist[i] = 0u;  // (overlaps the wait below)
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;
  int* cblk = reinterpret_cast<int*>(smem + p.off_cblk);
  float* qsum = reinterpret_cast<float*>(smem + p.off_qsum);
  uint8_t* stc = smem + p.off_stage;
  float2* stz = reinterpret_cast<float2*>(smem + p.off_stage + (size_t)p.cb * d.B * (d.d_c / 2));
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&qbar, 1);
    mbar_fence_init();
    wait_ready(p.ready_in + pair, p.epoch);  // select_kernel's a2 outputs for this pair
    // the pair's q-fragment blob from K1b: one TMA bulk copy into [off_qb, off_qsum + NT*32)
    const uint32_t qfb = (uint32_t)(NSPLIT * NT * KS * 256 + NT * 32);
    mbar_arrive_expect_tx(&qbar, qfb);
    tma_bulk_g2s(smem + p.off_qb, p.qfrag + (size_t)pair * qfb, qfb, &qbar);
  }
  __syncthreads();  // mbarriers initialised; the hand-off observed by thread 0 (cumulative through the barrier)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");  // started (matched before the DSMEM push)
  const int rowbytes = d.d_c / 2;
  const uint8_t* cbase = p.codes + (size_t)pair * d.S * rowbytes;
  const float2* zbase = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * d.S;
  const bool zal = (d.S & 1) == 0;  // every block's scale/zero rows 16-byte aligned and sized -> TMA
  const int cb0 = chunk * p.cb;
  int nbl;
  if (p.guide == nullptr) {
    // K1b's M_t is already compact: min(kb_eff, m) ascending valid ids, -1 padded.
    // Warp 0 reads this chunk's ids and issues the TMA copies straight away.
    // (-1 padding marks the end, so no dependence on seq_lens.)
    nbl = 0;
    if (warp == 0) {
      const int* cand = p.block_ids + (size_t)pair * d.Kb + cb0;
      const int lim = min(p.cb, p.kb_eff - cb0);
      uint32_t bytes = 0;
      int cntv = 0;
      for (int k0 = 0; k0 < lim; k0 += 32) {
        const int k = k0 + lane;
        const int blk = k < lim ? cand[k] : -1;
        const bool ok = blk >= 0;
        cntv += __popc(__ballot_sync(0xffffffffu, ok));
        if (ok) {
          cblk[cb0 + k] = blk;
          const int rows = min(d.B, d.S - blk * d.B);
          bytes += rows * rowbytes + (zal ? rows * 8 : 0);
        }
      }
      bytes = warp_sum_u32(bytes);
      if (lane == 0) {
        ctl.kc = cntv;
        if (cntv > 0) mbar_arrive_expect_tx(&bar, bytes);
      }
      __syncwarp();
      for (int k = lane; k < cntv; k += 32) {
        const int blk = cblk[cb0 + k];
        const int rows = min(d.B, d.S - blk * d.B);
        tma_bulk_g2s(stc + (size_t)k * d.B * rowbytes, cbase + (size_t)blk * d.B * rowbytes, rows * rowbytes, &bar);
        if (zal) tma_bulk_g2s(stz + k * d.B, zbase + (size_t)blk * d.B, rows * 8, &bar);
      }
    }
  } else {  // lag mode: the guide may hold ids past this step's m or -1: compact it first
    const int* cand = p.guide + (size_t)pair * d.Kb;
    const int per = (d.Kb + kThreads - 1) / kThreads;
    const int lo = min(tid * per, d.Kb), hi = min(lo + per, d.Kb);
    int cnt = 0;
    for (int i = lo; i < hi; ++i) cnt += (cand[i] >= 0 && cand[i] < m);
    int total;
    int pos = block_exclusive_scan(cnt, ctl.tk.scan, &total);
    for (int i = lo; i < hi; ++i)
      if (cand[i] >= 0 && cand[i] < m && pos < p.kb_eff) cblk[pos++] = cand[i];
    __syncthreads();
    const int kc = min(total, p.kb_eff);
    nbl = max(0, min(p.cb, kc - cb0));
    if (warp == 0 && nbl > 0) {
      uint32_t bytes = 0;
      for (int k = lane; k < nbl; k += 32) {
        const int rows = min(d.B, d.S - cblk[cb0 + k] * d.B);
        bytes += rows * rowbytes + (zal ? rows * 8 : 0);
      }
      bytes = warp_sum_u32(bytes);
      if (lane == 0) mbar_arrive_expect_tx(&bar, bytes);
      __syncwarp();
      for (int k = lane; k < nbl; k += 32) {
        const int blk = cblk[cb0 + k];
        const int rows = min(d.B, d.S - blk * d.B);
        tma_bulk_g2s(stc + (size_t)k * d.B * rowbytes, cbase + (size_t)blk * d.B * rowbytes, rows * rowbytes, &bar);
        if (zal) tma_bulk_g2s(stz + k * d.B, zbase + (size_t)blk * d.B, rows * 8, &bar);
      }
    }
  }
  __syncthreads();  // cblk / ctl.kc published
  if (p.guide == nullptr) nbl = ctl.kc;
  TLS_STAMP(1)
  mbar_wait(&qbar, 0);
  if (nbl > 0) mbar_wait(&bar, 0);
  TLS_STAMP(2)
  const float sm2 = d.sm_scale * kLog2e;
  float sq[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) sq[nt][e] = sm2 * qsum[nt * 8 + 2 * q4 + e];
  const uint2* qb2 = reinterpret_cast<const uint2*>(smem + p.off_qb);
  const int tshift = d.log2B - 4;
  const int ntiles = nbl << tshift;
  // ---- pass 1: logits of every tile (tile = warp + t * kWarps), L = sm_scale log2(e) (zero sum q~ + scale q~.code)
  // from the tensor-core product of token_tile_mma, -inf past the sequence; per-warp head max and min ----
  float ev[TPW][NT][4];
  float hm[NT][2], hl[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) hm[nt][0] = hm[nt][1] = -CUDART_INF_F, hl[nt][0] = hl[nt][1] = CUDART_INF_F;
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int tile = warp + t * kWarps;
    if (tile < ntiles) {
      float acc[NT][4];
      token_tile_mma<KS, NT, NSPLIT>(stc + (size_t)tile * 16 * rowbytes, qb2, acc);
      const int blk = cblk[cb0 + (tile >> tshift)];
      const int tok0 = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
      const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
      const float2 z0 = zal ? stz[tile * 16 + r0] : (v0 ? __ldg(zbase + tok0) : make_float2(0.f, 0.f));
      const float2 z1 = zal ? stz[tile * 16 + r0 + 8] : (v1 ? __ldg(zbase + tok0 + 8) : make_float2(0.f, 0.f));
      const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float l0 = fmaf(s0, acc[nt][e], z0.y * sq[nt][e]), l1 = fmaf(s1, acc[nt][2 + e], z1.y * sq[nt][e]);
          // the min also sees the rows past the sequence (stale staging; at worst a needless log-domain warp)
          hl[nt][e] = fminf(hl[nt][e], fminf(l0, l1));
          ev[t][nt][e] = v0 ? l0 : -CUDART_INF_F;
          ev[t][nt][2 + e] = v1 ? l1 : -CUDART_INF_F;
          hm[nt][e] = fmaxf(hm[nt][e], fmaxf(ev[t][nt][e], ev[t][nt][2 + e]));
        }
    } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) ev[t][nt][e] = -CUDART_INF_F;
    }
  }
  // A warp whose logits of some head span more than kUnder (attention-sink-like keys) keeps L in registers and
  // forms its keys in the log domain (pass 2); every other warp keeps E_hj = 2^(L_hj - m_h^w) >= 2^-kUnder.
  bool wide = false;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        hm[nt][e] = fmaxf(hm[nt][e], __shfl_xor_sync(0xffffffffu, hm[nt][e], o));
        hl[nt][e] = fminf(hl[nt][e], __shfl_xor_sync(0xffffffffu, hl[nt][e], o));
      }
      wide |= hm[nt][e] - hl[nt][e] > kUnder;  // NaN (stale rows) compares false; -inf min -> true
    }
  wide = __any_sync(0xffffffffu, wide);
  float hs[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float mref = hm[nt][e] == -CUDART_INF_F ? 0.f : hm[nt][e];
      float s = 0.f;
      if (wide) {
#pragma unroll
        for (int t = 0; t < TPW; ++t) s += fexp2(ev[t][nt][e] - mref) + fexp2(ev[t][nt][2 + e] - mref);
      } else {
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          ev[t][nt][e] = fexp2(ev[t][nt][e] - mref);
          ev[t][nt][2 + e] = fexp2(ev[t][nt][2 + e] - mref);
          s += ev[t][nt][e] + ev[t][nt][2 + e];
        }
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      hs[nt][e] = s;
    }
  if (r0 == 0) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        ctl.wm[warp][nt * 8 + 2 * q4 + e] = hm[nt][e];
        ctl.ws[warp][nt * 8 + 2 * q4 + e] = hs[nt][e];
      }
  }
  __syncthreads();
  {  // CTA merge of the 8 warps' (max, sum) per head: 8 lanes per head; push the result to every chunk CTA
    const int w = tid & 7, nch = (int)gridDim.x;
    const unsigned my = blockIdx.x;
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");  // every chunk CTA has started (DSMEM rule)
    {
      const int h = tid >> 3;  // G <= 32 = kThreads / 8: one pass, warp-uniform shuffles
      const bool okh = h < d.G;
      const float mv = okh ? ctl.wm[w][h] : -CUDART_INF_F, sv = okh ? ctl.ws[w][h] : 0.f;
      float M = mv;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      float S = (mv == -CUDART_INF_F) ? 0.f : sv * fexp2(mv - M);
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
      if (okh)
        for (int rr = w; rr < nch; rr += 8) {
          *dsmem(&s_cm[my][h], rr) = M;
          *dsmem(&s_cz[my][h], rr) = S;
        }
    }
  }
  TLS_STAMP(3)
  cluster_sync_all();  // every chunk's statistics have landed in every CTA
  if (chunk == 0 && tid == 0) p.ready_in[pair] = 0u;  // every CTA of the pair passed its wait
  TLS_STAMP(4)
  {  // cluster merge, local: 16 lanes per head over the nch chunk ranks
    const int r = tid & 15, nch = (int)gridDim.x;
    for (int h = tid >> 4; h < ((d.G + 15) & ~15); h += kThreads / 16) {
      const bool ok = r < nch && h < d.G;
      const float mv = ok ? s_cm[r][h] : -CUDART_INF_F, sv = ok ? s_cz[r][h] : 0.f;
      float M = mv;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      float S = (mv == -CUDART_INF_F) ? 0.f : sv * fexp2(mv - M);
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
      if (r == 0 && h < d.G) ctl.hlz[h] = M + flog2(S);
    }
  }
  __syncthreads();
  // ---- pass 2: ranking keys log2 sum_h exp2(L_hj - lz_h) (the head sum reduced over the four lanes that hold a
  // token's heads with a transposed butterfly, 3 shuffles per 4 tokens; every lane emits one key) ----
  // Narrow warp: key = r_w + log2 sum_h E_hj c_h^w with c_h^w = 2^(m_h^w - lz_h - r_w), r_w = max_h (m_h^w - lz_h),
  // so the largest factor is 1.  Every token's largest term x = L_hj - lz_h then has x - r_w >= min_h (min_j L_hj -
  // m_h^w) >= -kUnder, and a head whose factor or E underflows contributes below 2^-26 of it: the keys are exact
  // to fp32 rounding.
  // Wide warp: key = mx + log2 sum_h 2^(L_hj - lz_h - mx) with mx = max_h (L_hj - lz_h), whose largest term is 1
  // -- exact for any span (reading U20).
  float cf[NT][2], hz[NT][2];
  float rw = -CUDART_INF_F;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int h = nt * 8 + 2 * q4 + e;
      hz[nt][e] = h < d.G ? ctl.hlz[h] : CUDART_INF_F;  // x = L - (+inf) = -inf: no term
      if (h < d.G && hm[nt][e] != -CUDART_INF_F) rw = fmaxf(rw, hm[nt][e] - hz[nt][e]);
    }
  rw = fmaxf(rw, __shfl_xor_sync(0xffffffffu, rw, 1));
  rw = fmaxf(rw, __shfl_xor_sync(0xffffffffu, rw, 2));
  if (rw == -CUDART_INF_F) rw = 0.f;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      cf[nt][e] = (nt * 8 + 2 * q4 + e < d.G && hm[nt][e] != -CUDART_INF_F) ? fexp2(hm[nt][e] - hz[nt][e] - rw) : 0.f;
  uint32_t* kout = p.keys + (size_t)pair * p.kb_eff * d.B + ((size_t)cb0 << d.log2B);
  const bool bit0 = q4 & 1, bit1 = q4 & 2;
#pragma unroll
  for (int t = 0; t < TPW; t += 2) {
    if (warp + t * kWarps >= ntiles) break;  // warp-uniform
    float pa = 0.f, pb = 0.f, pc = 0.f, pd = 0.f;  // (tile t, r0), (t, r0+8), (t+1, r0), (t+1, r0+8)
    float ra = rw, rb = rw, rc = rw, rd = rw;  // log2 of the factor the sums carry
    if (!wide) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          pa = fmaf(ev[t][nt][e], cf[nt][e], pa);
          pb = fmaf(ev[t][nt][2 + e], cf[nt][e], pb);
          pc = fmaf(ev[t + 1][nt][e], cf[nt][e], pc);
          pd = fmaf(ev[t + 1][nt][2 + e], cf[nt][e], pd);
        }
    } else {
      float ma = -CUDART_INF_F, mb = -CUDART_INF_F, mc = -CUDART_INF_F, md = -CUDART_INF_F;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          ma = fmaxf(ma, ev[t][nt][e] - hz[nt][e]);
          mb = fmaxf(mb, ev[t][nt][2 + e] - hz[nt][e]);
          mc = fmaxf(mc, ev[t + 1][nt][e] - hz[nt][e]);
          md = fmaxf(md, ev[t + 1][nt][2 + e] - hz[nt][e]);
        }
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, o));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o));
        mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
        md = fmaxf(md, __shfl_xor_sync(0xffffffffu, md, o));
      }
      ra = ma == -CUDART_INF_F ? 0.f : ma, rb = mb == -CUDART_INF_F ? 0.f : mb;
      rc = mc == -CUDART_INF_F ? 0.f : mc, rd = md == -CUDART_INF_F ? 0.f : md;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          pa += fexp2(ev[t][nt][e] - hz[nt][e] - ra);
          pb += fexp2(ev[t][nt][2 + e] - hz[nt][e] - rb);
          pc += fexp2(ev[t + 1][nt][e] - hz[nt][e] - rc);
          pd += fexp2(ev[t + 1][nt][2 + e] - hz[nt][e] - rd);
        }
    }
    // transposed butterfly: lane q4 ends with the head-sum of token q4 of (pa, pb, pc, pd)
    float k1 = bit0 ? pb : pa, k2 = bit0 ? pd : pc;
    k1 += __shfl_xor_sync(0xffffffffu, bit0 ? pa : pb, 1);
    k2 += __shfl_xor_sync(0xffffffffu, bit0 ? pc : pd, 1);
    float mine = bit1 ? k2 : k1;
    mine += __shfl_xor_sync(0xffffffffu, bit1 ? k1 : k2, 2);
    const float mx = bit1 ? (bit0 ? rd : rc) : (bit0 ? rb : ra);
    const int tile = warp + (t + (bit1 ? 1 : 0)) * kWarps;
    const int row = r0 + (bit0 ? 8 : 0);
    if (tile < ntiles) {
      const int blk = cblk[cb0 + (tile >> tshift)];
      const int tok = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + row;
      const bool v = tok < n;
      const float kf = mx + flog2(mine);
      kout[tile * 16 + row] = v ? f2key(kf) : 0u;
      if (v) atomicAdd(&lhist[key_bin(kf)], 1u);
    }
  }
  __syncthreads();
  uint32_t* gh = p.khist + (size_t)pair * kKeyBins;
  for (int i = tid; i < kKeyBins; i += kThreads)
    if (lhist[i]) atomicAdd(&gh[i], lhist[i]);
  TLS_STAMP(5)
  __syncthreads();
  if (tid == 0)  // hand-off: one count per chunk CTA (no cluster barrier; the attention kernel waits for nch);
                  // a release add: this CTA's keys and histogram counts (cumulative over the CTA barrier)
    red_release_add_gpu(p.ready_out + pair, 1u);
  TLS_STAMP(6)
#undef TLS_STAMP
}

// ----------------------------------------------------------------------------
// K2, one or two CTAs per pair (token_pair_kernel; G <= 8 and the pair's
// candidate index in shared memory -- C2/C3: 128 blocks x 64 tokens x 24 B =
// 192 KB): NCH = 1 is one 1024-thread CTA holding all of it; NCH = 2 is a
// cluster of two 512-thread CTAs holding half each (two CTAs per SM, so one
// CTA's start-up latency hides under the other's work).  Either way the
// per-CTA fixed costs (hand-off wait, block-id read, merges, histogram) are
// paid once or twice per pair instead of once per 1024 candidates, and the
// softmax statistics merge inside the CTA (plus one DSMEM exchange for NCH 2).
// Staging: every thread copies 16-byte chunks with cp.async (a block = B rows
// of codes + B scale/zero pairs; rows past the cache end zero-filled) and
// arrives on its staging group's mbarrier, so pass 1 runs on the first groups
// while the rest land.  Two tensor-core passes over the staged codes (the same
// L_hj = sm_scale log2(e) (zero sum q~ + scale q~.code) as the other forms,
// P:129-133):
//   pass 1: per-lane sum of 2^(L_hj - r) against a per-lane reference r =
//           (largest logit seen) + kPairSlack, raised (warp-uniform branch)
//           only when a logit exceeds it -> lanes -> warps -> CTA (-> cluster),
//           fixed order -> lz_h = M_h + log2 Z_h;
//   pass 2: L_hj recomputed (two mma + dequantisation per 16-token tile is
//           cheaper than holding 8192 x G logits), x = L_hj - lz_h, key =
//           log2 sum_h 2^x (the head sum over the four lanes that hold a
//           token's heads by a transposed butterfly, 3 shuffles per 2 tiles).
//           A token whose sum falls below 2^-100 (terms near the bottom of
//           fp32's range: attention-sink-like logit spans, reading U20) is
//           re-keyed in the log domain, mx + log2 sum_h 2^(x - mx): exact to
//           fp32 rounding for any span.
// The key histogram is built in shared memory; one release add per CTA hands
// the pair to the attention kernel (ready count = NCH).
constexpr int kPairThreads = 1024;
constexpr float kPairSlack = 48.f;  // log2 units above the largest logit seen: terms <= 2^-48, no overflow

// TMEM as the pair kernel's logit store: lane i of a warp writes / reads TMEM lane 32 (warp % 4) + i,
// 4 (x4) or 8 (x8) consecutive 32-bit columns
__device__ __forceinline__ void tm_st4(uint32_t taddr, float a, float b, float c, float d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr), "r"(__float_as_uint(a)),
               "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d))
               : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void cp_async16_u(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0));
}

// acc = codes(16-token tile) x q~ (B fragments preloaded in registers, or read from shared memory per tile)
template <int KS, int NSPLIT, bool PRE>
__device__ __forceinline__ void pair_tile(const uint8_t* codes, const uint2 (&qbr)[PRE ? NSPLIT : 1][PRE ? KS : 1],
                                          const uint2* qb2, float (&acc)[4]) {
  CodeWords<KS> cw;
  load_code_words<KS>(codes, true, true, cw);
  constexpr int WPT = KS / 2;
  uint32_t a[KS][4];
#pragma unroll
  for (int u = 0; u < WPT; ++u) {
    uint32_t x0[4], x1[4];
    unpack_nibbles8(cw.w0[u], x0);
    unpack_nibbles8(cw.w1[u], x1);
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      a[2 * u + v][0] = x0[2 * v];
      a[2 * u + v][1] = x1[2 * v];
      a[2 * u + v][2] = x0[2 * v + 1];
      a[2 * u + v][3] = x1[2 * v + 1];
    }
  }
  acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 0; s < KS; ++s)
#pragma unroll
    for (int sp = 0; sp < NSPLIT; ++sp) {
      uint2 bb;
      if constexpr (PRE) bb = qbr[sp][s];
      else bb = qb2[(sp * KS + s) * 32 + lane];
      mma_bf16_16816(acc, a[s], bb.x, bb.y);
    }
}

template <typename T, int KS, int NSPLIT, int NCH>
__global__ void __launch_bounds__(kPairThreads / NCH, NCH) token_pair_kernel(const __grid_constant__ SelectParams p) {
  constexpr int NTH = kPairThreads / NCH, NW = NTH / 32;
  constexpr int rowbytes = KS * 8, lcpr = KS == 2 ? 0 : (KS == 4 ? 1 : 2);  // 16-byte chunks per code row: 2^lcpr
  constexpr bool PRE = NSPLIT * KS <= 4;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t gbar[kPairGroups];
  __shared__ __align__(8) uint64_t qbar;
  __shared__ uint32_t lhist[kKeyBins];
  __shared__ float s_wm[NW][8], s_ws[NW][8], s_lz[8];
  __shared__ float s_cm[NCH][8], s_cz[NCH][8];  // [chunk][head]: every chunk's statistics, pushed by that chunk
  __shared__ int s_kc, s_pslot;
  __shared__ uint32_t s_tmem;
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q4 = lane & 3, r0 = lane >> 2;
  const int chunk = NCH > 1 ? (int)blockIdx.x : 0, pair = blockIdx.y;
  unsigned long long* dbg = p.dbg ? p.dbg + ((size_t)pair * 8 + chunk) * 8 : nullptr;
#define TLS_STAMP(i) \
  if (dbg && tid == 0) dbg[i] = gtimer();
  TLS_STAMP(0)
  launch_dependents();
#pragma unroll
  for (int i = 0; i < kKeyBins / NTH; ++i) lhist[tid + i * NTH] = 0u;
  if constexpr (NCH > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");  // started
  const int b = pair / d.Hkv;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;
  int* cblk = reinterpret_cast<int*>(smem + p.off_cblk);
  const float* qsum = reinterpret_cast<const float*>(smem + p.off_qsum);
  const uint8_t* stc = smem + p.off_stage;
  const float2* stz = reinterpret_cast<const float2*>(smem + p.off_stage + ((size_t)p.cb << d.log2B) * rowbytes);
  if (warp == 0) {
    // TMEM columns for the pass-1 logits (L_hj of every staged token, 4 columns per 16-token tile per warp)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&s_tmem)),
                 "r"((uint32_t)p.tmcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    if (lane == 0) {
      for (int i = 0; i < kPairGroups; ++i) mbar_init(&gbar[i], NTH);  // one cp.async arrival per thread
      mbar_init(&qbar, 1);
      mbar_fence_init();
      s_pslot = -1;
      wait_ready(p.ready_in + pair, p.epoch);  // select_kernel's a2 outputs for this pair
      if (NCH == 1) p.ready_in[pair] = 0u;     // the hand-off's only consumer
      const uint32_t qfb = (uint32_t)(NSPLIT * KS * 256 + 32);  // the pair's q-fragment blob (qq_kernel)
      mbar_arrive_expect_tx(&qbar, qfb);
      tma_bulk_g2s(smem + p.off_qb, p.qfrag + (size_t)pair * qfb, qfb, &qbar);
    }
    __syncwarp();  // lane 0's acquire orders the warp's reads of the candidate list below
    // candidate blocks: a2's M_t (ascending, -1 padded) or the lag-mode guide, compacted in list order to
    // the valid ids (< m), at most kb_eff -- the same slots the attention prologue maps back to tokens
    const int* cand = (p.guide ? p.guide : p.block_ids) + (size_t)pair * d.Kb;
    constexpr int kMaxIt = 16;  // Kb <= 512 (plan)
    int cv[kMaxIt];
#pragma unroll
    for (int i = 0; i < kMaxIt; ++i) cv[i] = i * 32 + lane < d.Kb ? cand[i * 32 + lane] : -1;  // loads in flight
    int base = 0;
#pragma unroll
    for (int i = 0; i < kMaxIt; ++i) {
      if (i * 32 >= d.Kb) break;
      const int blk = cv[i];
      const bool ok = blk >= 0 && blk < m;
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      const int pos = base + __popc(bal & ((1u << lane) - 1u));
      if (ok && pos < p.kb_eff) {
        cblk[pos] = blk;
        if (blk == m - 1) s_pslot = pos;  // the sequence's last (possibly partial) block
      }
      base += __popc(bal);
    }
    if (lane == 0) s_kc = min(base, p.kb_eff);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();  // cblk, s_kc, s_pslot, lhist zeroed, barriers initialised, TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  TLS_STAMP(7)
  // this warp's TMEM region: lanes of its quarter, columns (warp / 4) * 4 * tiles-per-warp ..
  const uint32_t tmw = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 4 * p.tmtpw);
  const int c0 = chunk * p.cb;                           // this CTA's first candidate slot
  const int nbl = max(0, min(p.cb, s_kc - c0));          // and its number of candidate blocks
  const int gsh = p.gsh;                                 // staging group = 2^gsh candidate blocks
  {  // staging (cp.async, 16-byte chunks): warp w copies candidate blocks w, w + NW, ... (B rows of codes, then
     // B scale/zero pairs), group by group; every thread arrives on a group's barrier once its copies landed
    const uint32_t stc_u = smem_u32(stc), stz_u = smem_u32(stz);
    const int ccb = d.B << lcpr, zcb = d.B >> 1;  // 16-byte chunks per block: codes, scale/zero
    const uint8_t* cdb = p.codes + (size_t)pair * d.S * rowbytes + (size_t)lane * 16;
    const float2* szb = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * d.S + 2 * lane;
    int k = warp;
    for (int g = 0; g < kPairGroups; ++g) {
      const int kend = min((g + 1) << gsh, nbl);
      for (; k < kend; k += NW) {
        const int blk = cblk[c0 + k], rows = d.S - (blk << d.log2B);
        const uint8_t* cs = cdb + (size_t)blk * (d.B * rowbytes);
        const uint32_t cd = stc_u + (uint32_t)(k * ccb + lane) * 16u;
        for (int c = 0; c < ccb; c += 32)
          cp_async16_u(cd + (uint32_t)c * 16u, cs + (size_t)c * 16, ((c + lane) >> lcpr) < rows);
        const float2* zs = szb + ((size_t)blk << d.log2B);
        const uint32_t zd = stz_u + (uint32_t)(k * zcb + lane) * 16u;
        for (int c = 0; c < zcb; c += 32) cp_async16_u(zd + (uint32_t)c * 16u, zs + 2 * c, 2 * (c + lane) < rows);
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&gbar[g])) : "memory");
    }
  }
  const int nvl = n - (m - 1) * d.B;  // valid tokens of block m - 1
  const int tshift = d.log2B - 4;
  const int ntl = nbl << tshift;      // this CTA's 16-token tiles
  // tiles holding rows past the sequence end: [tp0, tp1), inside block m - 1 (if this CTA holds it)
  const int lp = s_pslot - c0;
  const bool hasp = s_pslot >= 0 && lp >= 0 && lp < nbl && nvl < d.B;
  const int tp0 = hasp ? (lp << tshift) + (nvl >> 4) : 0, tpn = hasp ? ((lp + 1) << tshift) - tp0 : 0;
  TLS_STAMP(1)
  const float sm2 = d.sm_scale * kLog2e;
  mbar_wait(&qbar, 0);
  float sq[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) sq[e] = sm2 * qsum[2 * q4 + e];  // padded heads: q~ = 0, sum 0
  const uint2* qb2 = reinterpret_cast<const uint2*>(smem + p.off_qb);
  uint2 qbr[PRE ? NSPLIT : 1][PRE ? KS : 1];
  if constexpr (PRE) {
#pragma unroll
    for (int sp = 0; sp < NSPLIT; ++sp)
#pragma unroll
      for (int s2 = 0; s2 < KS; ++s2) qbr[sp][s2] = qb2[(sp * KS + s2) * 32 + lane];
  }
  // ---- pass 1: per-lane sums of heads 2q4, 2q4 + 1 against the lane's reference rf (packed fp32x2 math:
  // .x = head 2q4, .y = head 2q4 + 1) ----
  const float2 sq2 = make_float2(sq[0], sq[1]);
  // the reference starts at the lane's first finite logit + kPairSlack (fx / fy: none seen yet); the logits go
  // to TMEM (pass 2 reads them back instead of recomputing them)
  float2 rf2 = make_float2(0.f, 0.f), hs2 = make_float2(0.f, 0.f);
  bool fx = true, fy = true;
  int gdone = -1;
  for (int i = 0, t = warp; t < ntl; ++i, t += NW) {
    const int grp = t >> (tshift + gsh);
    while (gdone < grp) mbar_wait(&gbar[++gdone], 0);
    float acc[4];
    pair_tile<KS, NSPLIT, PRE>(stc + (size_t)t * 16 * rowbytes, qbr, qb2, acc);
    const float2 z0 = stz[t * 16 + r0], z1 = stz[t * 16 + r0 + 8];
    const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
    // L for rows r0 (la) and r0 + 8 (lb), heads (2q4, 2q4 + 1)
    float2 la = __ffma2_rn(make_float2(s0, s0), make_float2(acc[0], acc[1]), __fmul2_rn(make_float2(z0.y, z0.y), sq2));
    float2 lb = __ffma2_rn(make_float2(s1, s1), make_float2(acc[2], acc[3]), __fmul2_rn(make_float2(z1.y, z1.y), sq2));
    if ((unsigned)(t - tp0) < (unsigned)tpn) {  // warp-uniform: the sequence's partial last block
      const int o = (t & ((1 << tshift) - 1)) << 4;
      if (o + r0 >= nvl) la = make_float2(-CUDART_INF_F, -CUDART_INF_F);
      if (o + r0 + 8 >= nvl) lb = make_float2(-CUDART_INF_F, -CUDART_INF_F);
    }
    tm_st4(tmw + 4 * i, la.x, la.y, lb.x, lb.y);
    const float2 mt = make_float2(fmaxf(la.x, lb.x), fmaxf(la.y, lb.y));
    if (__any_sync(0xffffffffu, fx || fy || mt.x > rf2.x || mt.y > rf2.y)) {  // first tile, then rare
      if (mt.x > rf2.x || (fx && mt.x != -CUDART_INF_F)) {
        const float nr = mt.x + kPairSlack;
        hs2.x *= fexp2(rf2.x - nr);
        rf2.x = nr, fx = false;
      }
      if (mt.y > rf2.y || (fy && mt.y != -CUDART_INF_F)) {
        const float nr = mt.y + kPairSlack;
        hs2.y *= fexp2(rf2.y - nr);
        rf2.y = nr, fy = false;
      }
    }
    const float2 nrf = make_float2(-rf2.x, -rf2.y);
    la = __fadd2_rn(la, nrf);
    lb = __fadd2_rn(lb, nrf);
    hs2 = __fadd2_rn(hs2, __fadd2_rn(make_float2(fexp2(la.x), fexp2(la.y)), make_float2(fexp2(lb.x), fexp2(lb.y))));
  }
  float rf[2] = {fx ? -1e30f : rf2.x, fy ? -1e30f : rf2.y}, hs[2] = {hs2.x, hs2.y};
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, rf[e], o), os = __shfl_xor_sync(0xffffffffu, hs[e], o);
      const float nm = fmaxf(rf[e], om);
      hs[e] = hs[e] * fexp2(rf[e] - nm) + os * fexp2(om - nm);
      rf[e] = nm;
    }
  if (r0 == 0) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      s_wm[warp][2 * q4 + e] = rf[e];
      s_ws[warp][2 * q4 + e] = hs[e];
    }
  }
  TLS_STAMP(2)
  __syncthreads();
  TLS_STAMP(3)
  if (warp < 8) {  // head h = warp: the warps' (reference, sum) merged in a fixed order
    const float mv = lane < NW ? s_wm[lane][warp] : -1e30f, sv = lane < NW ? s_ws[lane][warp] : 0.f;
    const float M = warp_max(mv);
    const float S = warp_sum(sv * fexp2(mv - M));
    if constexpr (NCH == 1) {
      if (lane == 0) s_lz[warp] = (warp < d.G && S > 0.f) ? M + flog2(S) : CUDART_INF_F;
    } else {
      asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");  // every chunk CTA has started (DSMEM rule)
      if (lane < NCH) {
        *dsmem(&s_cm[chunk][warp], (unsigned)lane) = M;
        *dsmem(&s_cz[chunk][warp], (unsigned)lane) = S;
      }
    }
  }
  if constexpr (NCH > 1) {
    if (warp >= 8) asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    cluster_sync_all();  // every chunk's statistics have landed in every CTA
    if (chunk == 0 && tid == 0) p.ready_in[pair] = 0u;  // every CTA of the pair passed its wait
    if (tid < 8) {
      float M = -1e30f, S = 0.f;
#pragma unroll
      for (int c = 0; c < NCH; ++c) M = fmaxf(M, s_cm[c][tid]);
#pragma unroll
      for (int c = 0; c < NCH; ++c) S += s_cz[c][tid] * fexp2(s_cm[c][tid] - M);
      s_lz[tid] = (tid < d.G && S > 0.f) ? M + flog2(S) : CUDART_INF_F;
    }
  }
  __syncthreads();
  TLS_STAMP(4)
  // ---- pass 2: ranking keys, two tiles per step (every lane emits one key per step) ----
  float nlz[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) nlz[e] = -s_lz[2 * q4 + e];  // padded heads: -inf -> no term
  const float2 nlz2 = make_float2(nlz[0], nlz[1]);
  uint32_t* kout = p.keys + (size_t)pair * p.kb_eff * d.B + ((size_t)c0 << d.log2B);
  const bool bit0 = q4 & 1, bit1 = q4 & 2;
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");  // this warp's logits are in TMEM
  for (int i = 0, ta = warp; ta < ntl; i += 2, ta += 2 * NW) {
    float x[2][2][2];  // [tile a / b][head e][row r0, r0 + 8]: L_hj - lz_h (tile b past the end: unused)
    {
      float v[8];
      tm_ld8(tmw + 4 * i, v);
      const float2 xa0 = __fadd2_rn(make_float2(v[0], v[1]), nlz2), xb0 = __fadd2_rn(make_float2(v[2], v[3]), nlz2);
      const float2 xa1 = __fadd2_rn(make_float2(v[4], v[5]), nlz2), xb1 = __fadd2_rn(make_float2(v[6], v[7]), nlz2);
      x[0][0][0] = xa0.x, x[0][1][0] = xa0.y, x[0][0][1] = xb0.x, x[0][1][1] = xb0.y;
      x[1][0][0] = xa1.x, x[1][1][0] = xa1.y, x[1][0][1] = xb1.x, x[1][1][1] = xb1.y;
    }
    float pa = fexp2(x[0][0][0]) + fexp2(x[0][1][0]), pb = fexp2(x[0][0][1]) + fexp2(x[0][1][1]);
    float pc = fexp2(x[1][0][0]) + fexp2(x[1][1][0]), pd = fexp2(x[1][0][1]) + fexp2(x[1][1][1]);
    // transposed butterfly: lane q4 ends with the head sum of (tile bit1, row r0 + 8 bit0)
    float k1 = bit0 ? pb : pa, k2 = bit0 ? pd : pc;
    k1 += __shfl_xor_sync(0xffffffffu, bit0 ? pa : pb, 1);
    k2 += __shfl_xor_sync(0xffffffffu, bit0 ? pc : pd, 1);
    float mine = bit1 ? k2 : k1;
    mine += __shfl_xor_sync(0xffffffffu, bit1 ? k1 : k2, 2);
    const int t = ta + (bit1 ? NW : 0);
    const int row = r0 + (bit0 ? 8 : 0);
    const bool v = t < ntl && !((unsigned)(t - tp0) < (unsigned)tpn && ((t & ((1 << tshift) - 1)) << 4) + row >= nvl);
    float kf = flog2(mine);
    if (__any_sync(0xffffffffu, v && !(mine >= 0x1p-100f))) {  // log domain for this step (reading U20)
      float ma = fmaxf(x[0][0][0], x[0][1][0]), mb = fmaxf(x[0][0][1], x[0][1][1]);
      float mc = fmaxf(x[1][0][0], x[1][1][0]), md = fmaxf(x[1][0][1], x[1][1][1]);
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, o));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o));
        mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
        md = fmaxf(md, __shfl_xor_sync(0xffffffffu, md, o));
      }
      ma = ma == -CUDART_INF_F ? 0.f : ma, mb = mb == -CUDART_INF_F ? 0.f : mb;
      mc = mc == -CUDART_INF_F ? 0.f : mc, md = md == -CUDART_INF_F ? 0.f : md;
      pa = fexp2(x[0][0][0] - ma) + fexp2(x[0][1][0] - ma), pb = fexp2(x[0][0][1] - mb) + fexp2(x[0][1][1] - mb);
      pc = fexp2(x[1][0][0] - mc) + fexp2(x[1][1][0] - mc), pd = fexp2(x[1][0][1] - md) + fexp2(x[1][1][1] - md);
      k1 = bit0 ? pb : pa, k2 = bit0 ? pd : pc;
      k1 += __shfl_xor_sync(0xffffffffu, bit0 ? pa : pb, 1);
      k2 += __shfl_xor_sync(0xffffffffu, bit0 ? pc : pd, 1);
      mine = bit1 ? k2 : k1;
      mine += __shfl_xor_sync(0xffffffffu, bit1 ? k1 : k2, 2);
      kf = (bit1 ? (bit0 ? md : mc) : (bit0 ? mb : ma)) + flog2(mine);
    }
    if (t < ntl) {
      kout[t * 16 + row] = v ? f2key(kf) : 0u;
      if (v) atomicAdd(&lhist[key_bin(kf)], 1u);
    }
  }
  __syncthreads();
  uint32_t* gh = p.khist + (size_t)pair * kKeyBins;
#pragma unroll
  for (int i = 0; i < kKeyBins / NTH; ++i) {
    const int j = tid + i * NTH;
    if constexpr (NCH == 1) gh[j] = lhist[j];  // the pair's whole histogram
    else if (lhist[j]) atomicAdd(&gh[j], lhist[j]);  // zeroed by qq_kernel
  }
  TLS_STAMP(5)
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(s_tmem), "r"((uint32_t)p.tmcols));
  if (tid == 0)  // hand-off: a release add (this CTA's keys and histogram, cumulative over the CTA barrier)
    red_release_add_gpu(p.ready_out + pair, 1u);
  TLS_STAMP(6)
#undef TLS_STAMP
}

template <typename T, int KS, int NSPLIT>
static cudaError_t launch_k2_pair(const SelectParams& p, cudaStream_t st, const LaunchOpts& o) {
  const unsigned pairs = (unsigned)(p.d.batch * p.d.Hkv);
  if (p.pairk == 4) {
    auto kern = token_pair_kernel<T, KS, NSPLIT, 4>;
    cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, false);
    if (e != cudaSuccess) return e;
    return launch_ex(kern, dim3(4u, pairs, 1), kPairThreads / 4, p.smem_bytes, st, o, 4u, p);
  }
  if (p.pairk == 2) {
    auto kern = token_pair_kernel<T, KS, NSPLIT, 2>;
    cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, false);
    if (e != cudaSuccess) return e;
    return launch_ex(kern, dim3(2u, pairs, 1), kPairThreads / 2, p.smem_bytes, st, o, 2u, p);
  }
  auto kern = token_pair_kernel<T, KS, NSPLIT, 1>;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, false);
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3(1u, pairs, 1), kPairThreads, p.smem_bytes, st, o, 0u, p);
}

// ----------------------------------------------------------------------------
// K2 for G > 8 (MLA: G = 32, d_c = 128): token_pair_nt_kernel -- the token_pair_kernel design for NT = ceil(G/8)
// n-tiles of 8 heads: a cluster of NCH 256-thread CTAs per pair, each holding cb candidate blocks in shared memory
// (C4: 8 blocks x 64 tokens x 72 B), the logits of every tile in TMEM (NT x 4 columns per tile per warp).  With
// 2 NT heads per lane a per-lane running (reference, sum) for each head would not fit the 64-register budget of
// four CTAs per SM, so the softmax statistics take one more pass over TMEM:
//   pass 1:  dequantised codes x q~ (NT x KS mma per tile), L -> TMEM, per-lane maxima;
//   CTA max M_h (lanes -> warps, fixed order);
//   pass 1b: TMEM -> per-lane sums of 2^(L - M_h) -> CTA sums (fixed order);
//   cluster: every chunk's (M, S) pushed over DSMEM, merged in chunk order -> lz_h (identical in every CTA);
//   pass 2:  TMEM -> key = log2 sum_h 2^(L - lz_h) (a lane's 2 NT heads, then the transposed butterfly over the
//            four lanes holding a token's heads), the log-domain recomputation below 2^-100 (reading U20),
//            keys + histogram, one release add per CTA.
constexpr int kNtThreads = 256, kNtWarps = kNtThreads / 32;
__device__ __forceinline__ int i_count(int ntl, int warp, int nw) { return warp < ntl ? (ntl - warp + nw - 1) / nw : 0; }

template <typename T, int KS, int NSPLIT, int NCH, int NT>
__global__ void __launch_bounds__(kNtThreads, 4) token_pair_nt_kernel(const __grid_constant__ SelectParams p) {
  constexpr int NW = kNtWarps, NH = NT * 8;
  constexpr int rowbytes = KS * 8, lcpr = KS == 2 ? 0 : (KS == 4 ? 1 : 2);
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t gbar[kPairGroups];
  __shared__ __align__(8) uint64_t qbar;
  __shared__ uint32_t lhist[kKeyBins];
  __shared__ float s_w[NW][NH], s_mx[NH], s_lz[NH];
  __shared__ float s_cm[NCH][NH], s_cz[NCH][NH];  // [chunk][head]: every chunk's statistics, pushed by that chunk
  __shared__ int s_kc, s_pslot;
  __shared__ uint32_t s_tmem;
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q4 = lane & 3, r0 = lane >> 2;
  const int chunk = (int)blockIdx.x, pair = blockIdx.y;
  unsigned long long* dbg = p.dbg && chunk < 8 ? p.dbg + ((size_t)pair * 8 + chunk) * 8 : nullptr;
#define TLS_STAMP(i) \
  if (dbg && tid == 0) dbg[i] = gtimer();
  TLS_STAMP(0)
  launch_dependents();
#pragma unroll
  for (int i = 0; i < kKeyBins / kNtThreads; ++i) lhist[tid + i * kNtThreads] = 0u;
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");  // started (matched before the DSMEM push)
  const int b = pair / d.Hkv;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;
  int* cblk = reinterpret_cast<int*>(smem + p.off_cblk);
  const float* qsum = reinterpret_cast<const float*>(smem + p.off_qsum);
  const uint8_t* stc = smem + p.off_stage;
  const float2* stz = reinterpret_cast<const float2*>(smem + p.off_stage + ((size_t)p.cb << d.log2B) * rowbytes);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&s_tmem)),
                 "r"((uint32_t)p.tmcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    if (lane == 0) {
      for (int i = 0; i < kPairGroups; ++i) mbar_init(&gbar[i], kNtThreads);
      mbar_init(&qbar, 1);
      mbar_fence_init();
      s_pslot = -1;
      wait_ready(p.ready_in + pair, p.epoch);  // select_kernel's a2 outputs for this pair
      const uint32_t qfb = (uint32_t)(NSPLIT * NT * KS * 256 + NT * 32);  // the pair's q-fragment blob (qq_kernel)
      mbar_arrive_expect_tx(&qbar, qfb);
      tma_bulk_g2s(smem + p.off_qb, p.qfrag + (size_t)pair * qfb, qfb, &qbar);
    }
    __syncwarp();
    const int* cand = (p.guide ? p.guide : p.block_ids) + (size_t)pair * d.Kb;
    constexpr int kMaxIt = 16;  // Kb <= 512 (plan)
    int cv[kMaxIt];
#pragma unroll
    for (int i = 0; i < kMaxIt; ++i) cv[i] = i * 32 + lane < d.Kb ? cand[i * 32 + lane] : -1;
    int base = 0;
#pragma unroll
    for (int i = 0; i < kMaxIt; ++i) {
      if (i * 32 >= d.Kb) break;
      const int blk = cv[i];
      const bool ok = blk >= 0 && blk < m;
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      const int pos = base + __popc(bal & ((1u << lane) - 1u));
      if (ok && pos < p.kb_eff) {
        cblk[pos] = blk;
        if (blk == m - 1) s_pslot = pos;
      }
      base += __popc(bal);
    }
    if (lane == 0) s_kc = min(base, p.kb_eff);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  TLS_STAMP(7)
  const int c0 = chunk * p.cb;
  const int nbl = max(0, min(p.cb, s_kc - c0));
  const int gsh = p.gsh;
  // TMEM: warp w -> lanes of quarter w % 4, columns (w / 4) * 4 NT * tiles-per-warp ..
  const uint32_t tmw = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 4 * NT * p.tmtpw);
  {  // staging: warp w copies candidate blocks w, w + NW, ... (cp.async), group by group
    const uint32_t stc_u = smem_u32(stc), stz_u = smem_u32(stz);
    const int ccb = d.B << lcpr, zcb = d.B >> 1;
    const uint8_t* cdb = p.codes + (size_t)pair * d.S * rowbytes + (size_t)lane * 16;
    const float2* szb = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * d.S + 2 * lane;
    int k = warp;
    for (int g = 0; g < kPairGroups; ++g) {
      const int kend = min((g + 1) << gsh, nbl);
      for (; k < kend; k += NW) {
        const int blk = cblk[c0 + k], rows = d.S - (blk << d.log2B);
        const uint8_t* cs = cdb + (size_t)blk * (d.B * rowbytes);
        const uint32_t cd = stc_u + (uint32_t)(k * ccb + lane) * 16u;
        for (int c = 0; c < ccb; c += 32)
          cp_async16_u(cd + (uint32_t)c * 16u, cs + (size_t)c * 16, ((c + lane) >> lcpr) < rows);
        const float2* zs = szb + ((size_t)blk << d.log2B);
        const uint32_t zd = stz_u + (uint32_t)(k * zcb + lane) * 16u;
        for (int c = 0; c < zcb; c += 32) cp_async16_u(zd + (uint32_t)c * 16u, zs + 2 * c, 2 * (c + lane) < rows);
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&gbar[g])) : "memory");
    }
  }
  const int nvl = n - (m - 1) * d.B;
  const int tshift = d.log2B - 4;
  const int ntl = nbl << tshift;
  const int lp = s_pslot - c0;
  const bool hasp = s_pslot >= 0 && lp >= 0 && lp < nbl && nvl < d.B;
  const int tp0 = hasp ? (lp << tshift) + (nvl >> 4) : 0, tpn = hasp ? ((lp + 1) << tshift) - tp0 : 0;
  TLS_STAMP(1)
  const float sm2 = d.sm_scale * kLog2e;
  mbar_wait(&qbar, 0);
  const uint2* qb2 = reinterpret_cast<const uint2*>(smem + p.off_qb);
  const float2* qs2 = reinterpret_cast<const float2*>(qsum);  // [nt * 4 + q4]: heads nt*8 + 2q4, +1
  // ---- pass 1: L -> TMEM, per-lane maxima of heads nt*8 + 2q4 + e ----
  float2 mx[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) mx[nt] = make_float2(-CUDART_INF_F, -CUDART_INF_F);
  int gdone = -1;
  for (int i = 0, t = warp; t < ntl; ++i, t += NW) {
    const int grp = t >> (tshift + gsh);
    while (gdone < grp) mbar_wait(&gbar[++gdone], 0);
    CodeWords<KS> cw;
    load_code_words<KS>(stc + (size_t)t * 16 * rowbytes, true, true, cw);
    uint32_t a[KS][4];
#pragma unroll
    for (int u = 0; u < KS / 2; ++u) {
      uint32_t x0[4], x1[4];
      unpack_nibbles8(cw.w0[u], x0);
      unpack_nibbles8(cw.w1[u], x1);
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        a[2 * u + v][0] = x0[2 * v];
        a[2 * u + v][1] = x1[2 * v];
        a[2 * u + v][2] = x0[2 * v + 1];
        a[2 * u + v][3] = x1[2 * v + 1];
      }
    }
    const float2 z0 = stz[t * 16 + r0], z1 = stz[t * 16 + r0 + 8];
    const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
    const bool part = (unsigned)(t - tp0) < (unsigned)tpn;  // warp-uniform: the sequence's partial last block
    const int o = (t & ((1 << tshift) - 1)) << 4;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int s2 = 0; s2 < KS; ++s2)
#pragma unroll
        for (int sp = 0; sp < NSPLIT; ++sp) {
          const uint2 bb = qb2[((sp * NT + nt) * KS + s2) * 32 + lane];
          mma_bf16_16816(acc, a[s2], bb.x, bb.y);
        }
      const float2 sq2 = __fmul2_rn(make_float2(sm2, sm2), qs2[nt * 4 + q4]);
      float2 la = __ffma2_rn(make_float2(s0, s0), make_float2(acc[0], acc[1]), __fmul2_rn(make_float2(z0.y, z0.y), sq2));
      float2 lb = __ffma2_rn(make_float2(s1, s1), make_float2(acc[2], acc[3]), __fmul2_rn(make_float2(z1.y, z1.y), sq2));
      if (part) {
        if (o + r0 >= nvl) la = make_float2(-CUDART_INF_F, -CUDART_INF_F);
        if (o + r0 + 8 >= nvl) lb = make_float2(-CUDART_INF_F, -CUDART_INF_F);
      }
      tm_st4(tmw + (uint32_t)((i * NT + nt) * 4), la.x, la.y, lb.x, lb.y);
      mx[nt] = make_float2(fmaxf(mx[nt].x, fmaxf(la.x, lb.x)), fmaxf(mx[nt].y, fmaxf(la.y, lb.y)));
    }
  }
  const int ntw = i_count(ntl, warp, NW);
  // CTA maxima per head (lanes -> warps -> CTA)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int o2 = 4; o2 < 32; o2 <<= 1) {
      mx[nt].x = fmaxf(mx[nt].x, __shfl_xor_sync(0xffffffffu, mx[nt].x, o2));
      mx[nt].y = fmaxf(mx[nt].y, __shfl_xor_sync(0xffffffffu, mx[nt].y, o2));
    }
  if (r0 == 0) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      s_w[warp][nt * 8 + 2 * q4] = mx[nt].x;
      s_w[warp][nt * 8 + 2 * q4 + 1] = mx[nt].y;
    }
  }
  TLS_STAMP(2)
  __syncthreads();
  if (tid < NH) {
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, s_w[w][tid]);
    s_mx[tid] = M;
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");  // this warp's logits are in TMEM
  __syncthreads();
  // ---- pass 1b: per-lane sums of 2^(L - M_h) from TMEM ----
  float2 hs[NT], nm[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    hs[nt] = make_float2(0.f, 0.f);
    const float a0 = s_mx[nt * 8 + 2 * q4], a1 = s_mx[nt * 8 + 2 * q4 + 1];
    nm[nt] = make_float2(a0 == -CUDART_INF_F ? 0.f : -a0, a1 == -CUDART_INF_F ? 0.f : -a1);
  }
  for (int i = 0; i < ntw; ++i) {
#pragma unroll
    for (int h2 = 0; h2 < NT; h2 += 2) {  // 8 columns = two n-tiles per load
      float v[8];
      tm_ld8(tmw + (uint32_t)((i * NT + h2) * 4), v);
#pragma unroll
      for (int u = 0; u < 2 && h2 + u < NT; ++u) {
        const float2 xa = __fadd2_rn(make_float2(v[4 * u], v[4 * u + 1]), nm[h2 + u]);
        const float2 xb = __fadd2_rn(make_float2(v[4 * u + 2], v[4 * u + 3]), nm[h2 + u]);
        hs[h2 + u] = __fadd2_rn(hs[h2 + u], __fadd2_rn(make_float2(fexp2(xa.x), fexp2(xa.y)),
                                                       make_float2(fexp2(xb.x), fexp2(xb.y))));
      }
    }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int o2 = 4; o2 < 32; o2 <<= 1) {
      hs[nt].x += __shfl_xor_sync(0xffffffffu, hs[nt].x, o2);
      hs[nt].y += __shfl_xor_sync(0xffffffffu, hs[nt].y, o2);
    }
  if (r0 == 0) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      s_w[warp][nt * 8 + 2 * q4] = hs[nt].x;
      s_w[warp][nt * 8 + 2 * q4 + 1] = hs[nt].y;
    }
  }
  __syncthreads();
  TLS_STAMP(3)
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");  // every chunk CTA has started (DSMEM rule)
  if (tid < NH) {  // this CTA's (M_h, S_h) to every chunk CTA
    float S = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) S += s_w[w][tid];
    const float M = s_mx[tid];
    for (int rr = 0; rr < NCH; ++rr) {
      *dsmem(&s_cm[chunk][tid], (unsigned)rr) = M;
      *dsmem(&s_cz[chunk][tid], (unsigned)rr) = S;
    }
  }
  cluster_sync_all();  // every chunk's statistics have landed in every CTA
  if (chunk == 0 && tid == 0) p.ready_in[pair] = 0u;  // every CTA of the pair passed its wait
  if (tid < NH) {
    float M = -CUDART_INF_F;
    for (int c = 0; c < NCH; ++c) M = fmaxf(M, s_cm[c][tid]);
    float S = 0.f;
    if (M != -CUDART_INF_F)
      for (int c = 0; c < NCH; ++c)
        if (s_cm[c][tid] != -CUDART_INF_F) S += s_cz[c][tid] * fexp2(s_cm[c][tid] - M);
    s_lz[tid] = (tid < d.G && S > 0.f) ? M + flog2(S) : CUDART_INF_F;
  }
  __syncthreads();
  TLS_STAMP(4)
  // ---- pass 2: ranking keys, two tiles per step ----
  float2 nlz[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) nlz[nt] = make_float2(-s_lz[nt * 8 + 2 * q4], -s_lz[nt * 8 + 2 * q4 + 1]);
  uint32_t* kout = p.keys + (size_t)pair * p.kb_eff * d.B + ((size_t)c0 << d.log2B);
  const bool bit0 = q4 & 1, bit1 = q4 & 2;
  for (int i = 0, ta = warp; ta < ntl; i += 2, ta += 2 * NW) {
    // p[u][r]: the lane's 2 NT heads of (tile u, row r); mxx[u][r]: their maximum (log domain)
    float pr[2][2], mxx[2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      pr[u][0] = pr[u][1] = 0.f;
      mxx[u][0] = mxx[u][1] = -CUDART_INF_F;
      if (u == 1 && ta + NW >= ntl) continue;  // warp-uniform
#pragma unroll
      for (int h2 = 0; h2 < NT; h2 += 2) {
        float v[8];
        tm_ld8(tmw + (uint32_t)(((i + u) * NT + h2) * 4), v);
#pragma unroll
        for (int w2 = 0; w2 < 2 && h2 + w2 < NT; ++w2) {
          const float2 xa = __fadd2_rn(make_float2(v[4 * w2], v[4 * w2 + 1]), nlz[h2 + w2]);
          const float2 xb = __fadd2_rn(make_float2(v[4 * w2 + 2], v[4 * w2 + 3]), nlz[h2 + w2]);
          pr[u][0] += fexp2(xa.x) + fexp2(xa.y);
          pr[u][1] += fexp2(xb.x) + fexp2(xb.y);
          mxx[u][0] = fmaxf(mxx[u][0], fmaxf(xa.x, xa.y));
          mxx[u][1] = fmaxf(mxx[u][1], fmaxf(xb.x, xb.y));
        }
      }
    }
    float pa = pr[0][0], pb = pr[0][1], pc = pr[1][0], pd = pr[1][1];
    float k1 = bit0 ? pb : pa, k2 = bit0 ? pd : pc;
    k1 += __shfl_xor_sync(0xffffffffu, bit0 ? pa : pb, 1);
    k2 += __shfl_xor_sync(0xffffffffu, bit0 ? pc : pd, 1);
    float mine = bit1 ? k2 : k1;
    mine += __shfl_xor_sync(0xffffffffu, bit1 ? k1 : k2, 2);
    const int t = ta + (bit1 ? NW : 0);
    const int row = r0 + (bit0 ? 8 : 0);
    const bool v = t < ntl && !((unsigned)(t - tp0) < (unsigned)tpn && ((t & ((1 << tshift) - 1)) << 4) + row >= nvl);
    float kf = flog2(mine);
    if (__any_sync(0xffffffffu, v && !(mine >= 0x1p-100f))) {  // log domain for this step (reading U20)
      float ma = mxx[0][0], mb = mxx[0][1], mc = mxx[1][0], md = mxx[1][1];
#pragma unroll
      for (int o2 = 1; o2 < 4; o2 <<= 1) {
        ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, o2));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o2));
        mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o2));
        md = fmaxf(md, __shfl_xor_sync(0xffffffffu, md, o2));
      }
      ma = ma == -CUDART_INF_F ? 0.f : ma, mb = mb == -CUDART_INF_F ? 0.f : mb;
      mc = mc == -CUDART_INF_F ? 0.f : mc, md = md == -CUDART_INF_F ? 0.f : md;
      const float mm[2][2] = {{ma, mb}, {mc, md}};
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        pr[u][0] = pr[u][1] = 0.f;
        if (u == 1 && ta + NW >= ntl) continue;
#pragma unroll
        for (int h2 = 0; h2 < NT; h2 += 2) {
          float vv[8];
          tm_ld8(tmw + (uint32_t)(((i + u) * NT + h2) * 4), vv);
#pragma unroll
          for (int w2 = 0; w2 < 2 && h2 + w2 < NT; ++w2) {
            const float2 xa = __fadd2_rn(make_float2(vv[4 * w2], vv[4 * w2 + 1]), nlz[h2 + w2]);
            const float2 xb = __fadd2_rn(make_float2(vv[4 * w2 + 2], vv[4 * w2 + 3]), nlz[h2 + w2]);
            pr[u][0] += fexp2(xa.x - mm[u][0]) + fexp2(xa.y - mm[u][0]);
            pr[u][1] += fexp2(xb.x - mm[u][1]) + fexp2(xb.y - mm[u][1]);
          }
        }
      }
      pa = pr[0][0], pb = pr[0][1], pc = pr[1][0], pd = pr[1][1];
      k1 = bit0 ? pb : pa, k2 = bit0 ? pd : pc;
      k1 += __shfl_xor_sync(0xffffffffu, bit0 ? pa : pb, 1);
      k2 += __shfl_xor_sync(0xffffffffu, bit0 ? pc : pd, 1);
      mine = bit1 ? k2 : k1;
      mine += __shfl_xor_sync(0xffffffffu, bit1 ? k1 : k2, 2);
      kf = (bit1 ? (bit0 ? md : mc) : (bit0 ? mb : ma)) + flog2(mine);
    }
    if (t < ntl) {
      kout[t * 16 + row] = v ? f2key(kf) : 0u;
      if (v) atomicAdd(&lhist[key_bin(kf)], 1u);
    }
  }
  __syncthreads();
  uint32_t* gh = p.khist + (size_t)pair * kKeyBins;
#pragma unroll
  for (int i = 0; i < kKeyBins / kNtThreads; ++i) {
    const int j = tid + i * kNtThreads;
    if (lhist[j]) atomicAdd(&gh[j], lhist[j]);  // zeroed by qq_kernel
  }
  TLS_STAMP(5)
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(s_tmem), "r"((uint32_t)p.tmcols));
  if (tid == 0) red_release_add_gpu(p.ready_out + pair, 1u);
  TLS_STAMP(6)
#undef TLS_STAMP
}

template <typename T, int KS, int NSPLIT, int NT>
static cudaError_t launch_k2_nt(const SelectParams& p, cudaStream_t st, const LaunchOpts& o) {
  const unsigned pairs = (unsigned)(p.d.batch * p.d.Hkv);
  if (p.pairk == 16) {
    auto kern = token_pair_nt_kernel<T, KS, NSPLIT, 16, NT>;
    cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, true);
    if (e != cudaSuccess) return e;
    return launch_ex(kern, dim3(16u, pairs, 1), kNtThreads, p.smem_bytes, st, o, 16u, p);
  }
  auto kern = token_pair_nt_kernel<T, KS, NSPLIT, 8, NT>;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, false);
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3(8u, pairs, 1), kNtThreads, p.smem_bytes, st, o, 8u, p);
}

// ============================================================== launchers
template <typename T, int KS, int NT, int NSPLIT>
static cudaError_t launch_k2(const SelectParams& p, cudaStream_t st, const LaunchOpts& o) {
  auto kern = p.tpw > 0 ? token_reg_kernel<T, KS, NT, NSPLIT, 8 / NT> : token_cluster_kernel<T, KS, NT, NSPLIT>;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, p.nch > 8);
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3((unsigned)p.nch, (unsigned)(p.d.batch * p.d.Hkv), 1), kThreads, p.smem_bytes, st, o,
                   (unsigned)p.nch, p);
}

// Supported (d_c, G) combinations: KS = d_c/16 in {2, 4, 8}, NT = ceil(G/8) in {1, 2, 4}.
bool select_supported(int d_c, int G) {
  const int ks = d_c / 16, nt = (G + 7) / 8;
  return (ks == 2 || ks == 4 || ks == 8) && (nt >= 1 && nt <= 4) && d_c % 32 == 0;
}

template <typename T, int NS>
static cudaError_t dispatch_k2(const SelectParams& p, cudaStream_t st, const LaunchOpts& o) {
  const int ks = p.d.d_c / 16, nt = (p.d.G + 7) / 8;
  if (p.pairk >= 8) {  // token_pair_nt_kernel (G > 8; the q-fragment blob's n-tiles: 2 or 4)
    if constexpr (NS == 1) {
      const int ntb = nt <= 2 ? 2 : 4;
      if (ks == 8 && ntb == 4) return launch_k2_nt<T, 8, NS, 4>(p, st, o);
      if (ks == 8 && ntb == 2) return launch_k2_nt<T, 8, NS, 2>(p, st, o);
      if (ks == 2 && ntb == 2) return launch_k2_nt<T, 2, NS, 2>(p, st, o);
      if (ks == 2 && ntb == 4) return launch_k2_nt<T, 2, NS, 4>(p, st, o);
    }
    return cudaErrorInvalidValue;
  }
  if (p.pairk) {
    if (ks == 2) return launch_k2_pair<T, 2, NS>(p, st, o);
    if (ks == 4) return launch_k2_pair<T, 4, NS>(p, st, o);
    if (ks == 8) return launch_k2_pair<T, 8, NS>(p, st, o);
    return cudaErrorInvalidValue;
  }
#define TLS_K2(KS_, NT_) \
  if (ks == KS_ && nt <= NT_) return launch_k2<T, KS_, NT_, NS>(p, st, o);
  TLS_K2(2, 1) TLS_K2(2, 2) TLS_K2(2, 4)
  TLS_K2(4, 1) TLS_K2(4, 2) TLS_K2(4, 4)
  TLS_K2(8, 1) TLS_K2(8, 2) TLS_K2(8, 4)
#undef TLS_K2
  return cudaErrorInvalidValue;
}

cudaError_t launch_token_cluster(const SelectParams& p, cudaStream_t st, const LaunchOpts& o) {
  return p.d.bf16 ? dispatch_k2<__nv_bfloat16, 1>(p, st, o) : dispatch_k2<float, 3>(p, st, o);
}

}  // namespace tls
