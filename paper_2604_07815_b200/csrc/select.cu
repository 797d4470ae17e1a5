// select.cu -- two-level selection of AsyncTLS (arXiv 2604.07815) for sm_100a.
//
//   K1 block_score_kernel   a1  s_i = Q+ . k^max_i + Q- . k^min_i  (P:99 via the
//                               P:110 identity and linearity of sum_h): an
//                               HBM-streaming GEMV over every block of every
//                               pair, fp32 scores -> workspace.
//   K2 token_select_kernel  a2  M_t = top-k_b blocks
//                           a3  alpha~_j over the candidate tokens
//                           a4  S_t = top-k_t tokens
//                               one thread-block CLUSTER of cs CTAs per pair.
//
// Citation key: P:n = line n of PAPER.md.  Readings U1..U19: DESIGN.md §3.
#include <math_constants.h>

#include "common.cuh"
#include "params.h"
#include "topk.cuh"
#include "fasttopk.cuh"

namespace tls {

// ============================================================== K1: a1
// grid (ceil(m_max / tb), pairs).  A CTA scores blocks [i0, i0 + tb) of one
// pair: one thread streams the tile of block summaries (tb rows of
// [k^max | k^min], contiguous, <= 32 KB) into shared memory with TMA bulk
// copies in kSub sub-chunks, each completing on its own single-use mbarrier;
// the warps score a sub-chunk as soon as it lands.  QQ = [Q+ | Q-] (2*d_k
// fp32), so s_i = QQ . row_i: 1 flop per byte, HBM-bound.  Each warp scores 8
// blocks at a time and reduces the 8 dot products with a transposed butterfly
// (9 shuffles instead of 40).
constexpr int kSub = 4;

template <typename T, int CPL>
__global__ void __launch_bounds__(kThreads) block_score_kernel(const __grid_constant__ ScoreParams p) {
  constexpr int EPC = 16 / sizeof(T);
  extern __shared__ __align__(128) uint8_t tile[];
  __shared__ float QQ[32 * CPL * EPC];
  __shared__ __align__(8) uint64_t bars[kSub];
  const Dims& d = p.d;
  const int pair = blockIdx.y;
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) / d.B;  // reading U1
  const int i0 = blockIdx.x * p.tb;
  if (i0 >= m) return;
  const int nb = min(p.tb, m - i0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rowbytes = 2 * d.d_k * (int)sizeof(T);
  const uint8_t* src = reinterpret_cast<const uint8_t*>(p.block_minmax) + ((size_t)pair * d.M + i0) * rowbytes;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kSub; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
#pragma unroll
    for (int s = 0; s < kSub; ++s) {
      const int s0 = nb * s / kSub, s1 = nb * (s + 1) / kSub;
      if (s1 > s0) {
        mbar_arrive_expect_tx(&bars[s], (uint32_t)((s1 - s0) * rowbytes));
        tma_bulk_g2s(tile + (size_t)s0 * rowbytes, src + (size_t)s0 * rowbytes, (uint32_t)((s1 - s0) * rowbytes),
                     &bars[s]);
      }
    }
  }
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * d.Hq + (size_t)g * d.G) * d.d_k;
  for (int c = tid; c < d.d_k; c += kThreads) {
    float qv[32];
#pragma unroll
    for (int h = 0; h < 32; ++h)
      if (h < d.G) qv[h] = to_f32<T>(qg[(size_t)h * d.d_k + c]);
    float qp = 0.f, qn = 0.f;
#pragma unroll
    for (int h = 0; h < 32; ++h)
      if (h < d.G) {
        qp += fmaxf(qv[h], 0.f);
        qn += fminf(qv[h], 0.f);
      }
    QQ[c] = qp;
    QQ[d.d_k + c] = qn;
  }
  __syncthreads();  // QQ ready, barriers initialised
  const int nchunk = rowbytes / 16;
  float qreg[CPL][EPC];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int ch = lane + 32 * c;
#pragma unroll
    for (int e = 0; e < EPC; ++e) qreg[c][e] = ch < nchunk ? QQ[ch * EPC + e] : 0.f;
  }
  float* out = p.scores + (size_t)pair * d.M + i0;
#pragma unroll 1
  for (int s = 0; s < kSub; ++s) {
    const int s0 = nb * s / kSub, s1 = nb * (s + 1) / kSub;
    if (s1 <= s0) continue;
    mbar_wait(&bars[s], 0);
    for (int r8 = s0 + warp * 8; r8 < s1; r8 += kWarps * 8) {
      float acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc[u] = 0.f;
        if (r8 + u < s1) {
          const uint4* row = reinterpret_cast<const uint4*>(tile + (size_t)(r8 + u) * rowbytes);
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nchunk) {
              float f[EPC];
              unpack16<T>(row[ch], f);
#pragma unroll
              for (int e = 0; e < EPC; ++e) acc[u] = fmaf(qreg[c][e], f[e], acc[u]);
            }
          }
        }
      }
      // transposed butterfly: afterwards lanes 4u..4u+3 hold the sum of block u
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
      if ((lane & 3) == 0 && r8 + u < s1) out[r8 + u] = acc[0];
    }
  }
}

// ============================================================== K2: a2-a4
struct SelCtl {
  TopKCtl tk;
  FastTopKCtl fk;
  int kc, nvalid, jtot;
  float hm[32], hz[32];  // per-head local (max, sum) (read remotely)
  float hlz[32];         // per-head log2 normaliser M_h + log2 Z_h
  float wm[kWarps][32], ws[kWarps][32];
  int chan[128];
};

// bf16 piece `sp` of x: x ~= hi + mid + lo (sp = 0, 1, 2), each exact in bf16.
__device__ __forceinline__ float split_piece(float x, int sp) {
  float hi = __bfloat162float(__float2bfloat16_rn(x));
  if (sp == 0) return hi;
  float r1 = x - hi;
  float mid = __bfloat162float(__float2bfloat16_rn(r1));
  if (sp == 1) return mid;
  return __bfloat162float(__float2bfloat16_rn(r1 - mid));
}

// merge two online-softmax states (m, s) in log2 units
__device__ __forceinline__ void stat_merge(float& m, float& s, float om, float os) {
  const float nm = fmaxf(m, om);
  if (nm == -CUDART_INF_F) return;
  s = (m == -CUDART_INF_F ? 0.f : s * fexp2(m - nm)) + (om == -CUDART_INF_F ? 0.f : os * fexp2(om - nm));
  m = nm;
}

// acc[nt][*] = codes(16-token tile at `codes`) x q-fragments, for the NT n-tiles
// of 8 heads.  A = codes (16 tokens x 16 channels per k-step), nibbles -> exact
// bf16; the channel order inside the MMA's K dimension is a permutation
// (thread q4 owns the contiguous code word(s) q4*WPT..), applied identically to
// the B fragments built in token_select_kernel.
template <int KS, int NT, int NSPLIT>
__device__ __forceinline__ void token_tile_mma(const uint8_t* codes, const uint2* qb2, float (&acc)[NT][4]) {
  constexpr int WPT = KS / 2;
  constexpr int ROWB = KS * 8;  // d_c / 2
  const int lane = threadIdx.x & 31, q4 = lane & 3, r0 = lane >> 2;
  const uint8_t* p0 = codes + r0 * ROWB + q4 * WPT * 4;
  const uint8_t* p1 = p0 + 8 * ROWB;
  uint32_t w0[WPT], w1[WPT];
  if constexpr (WPT == 4) {
    const uint4 x = *reinterpret_cast<const uint4*>(p0), y = *reinterpret_cast<const uint4*>(p1);
    w0[0] = x.x; w0[1] = x.y; w0[2] = x.z; w0[3] = x.w;
    w1[0] = y.x; w1[1] = y.y; w1[2] = y.z; w1[3] = y.w;
  } else if constexpr (WPT == 2) {
    const uint2 x = *reinterpret_cast<const uint2*>(p0), y = *reinterpret_cast<const uint2*>(p1);
    w0[0] = x.x; w0[1] = x.y;
    w1[0] = y.x; w1[1] = y.y;
  } else {
    w0[0] = *reinterpret_cast<const uint32_t*>(p0);
    w1[0] = *reinterpret_cast<const uint32_t*>(p1);
  }
  uint32_t a[KS][4];
#pragma unroll
  for (int u = 0; u < WPT; ++u) {
    uint32_t x0[4], x1[4];
    unpack_nibbles8(w0[u], x0);
    unpack_nibbles8(w1[u], x1);
#pragma unroll
    for (int v = 0; v < 2; ++v) {  // k-step 2u+v uses nibble pairs (2v, 2v+4) and (2v+1, 2v+5)
      a[2 * u + v][0] = x0[2 * v];
      a[2 * u + v][1] = x1[2 * v];
      a[2 * u + v][2] = x0[2 * v + 1];
      a[2 * u + v][3] = x1[2 * v + 1];
    }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
    for (int s = 0; s < KS; ++s)
#pragma unroll
      for (int sp = 0; sp < NSPLIT; ++sp) {
        const uint2 bb = qb2[((sp * NT + nt) * KS + s) * 32 + lane];
        mma_bf16_16816(acc[nt], a[s], bb.x, bb.y);
      }
  }
}

constexpr int kRing = 3;  // stages of the candidate-index ring (~16 KB each)

// The token index of this CTA's candidate blocks streams through a kRing-stage
// ring TWICE (pass 1: softmax statistics, pass 2: ranking keys), as one
// sequence of 2*ngroups groups of p.rb blocks: group gq lives in slot
// gq % kRing and is loaded by one TMA bulk copy per block and run (codes, and
// (scale, zero) when 16-byte aligned), completing on the slot's mbarrier.  A
// slot is refilled by the last warp to release it (no CTA-wide barrier), so
// warps run ahead independently and pass-2 loads overlap the end of pass 1.
struct IndexRing {
  const SelectParams* p;
  const uint8_t* cbase;
  const float2* zbase;
  const int* cblk;
  int cb0, nbl, ngroups;
  bool zal;
  uint8_t* ring;
  uint64_t* full;
  int* slot_cnt;
  __device__ int group_blocks(int gi) const { return min(p->rb, nbl - gi * p->rb); }
  __device__ uint8_t* slot_codes(int slot) const { return ring + (size_t)slot * p->ring_stage_bytes; }
  __device__ float2* slot_sz(int slot) const {
    return reinterpret_cast<float2*>(ring + (size_t)slot * p->ring_stage_bytes + (size_t)p->rb * p->d.B * (p->d.d_c / 2));
  }
  // issue sequence element gq (one thread)
  __device__ void issue(int gq) const {
    const Dims& d = p->d;
    const int gi = gq % ngroups, slot = gq % kRing;
    const int rowbytes = d.d_c / 2;
    const int nb = group_blocks(gi);
    uint32_t bytes = 0;
    for (int k = 0; k < nb; ++k) {
      const int blk = cblk[cb0 + gi * p->rb + k];
      const int rows = min(d.B, d.S - blk * d.B);
      bytes += rows * rowbytes + (zal ? rows * 8 : 0);
    }
    mbar_arrive_expect_tx(&full[slot], bytes);
    for (int k = 0; k < nb; ++k) {
      const int blk = cblk[cb0 + gi * p->rb + k];
      const int rows = min(d.B, d.S - blk * d.B);
      tma_bulk_g2s(slot_codes(slot) + (size_t)k * d.B * rowbytes, cbase + (size_t)blk * d.B * rowbytes,
                   rows * rowbytes, &full[slot]);
      if (zal) tma_bulk_g2s(slot_sz(slot) + k * d.B, zbase + (size_t)blk * d.B, rows * 8, &full[slot]);
    }
  }
  __device__ void wait(int gq) const { mbar_wait(&full[gq % kRing], (gq / kRing) & 1); }
  // every warp calls this after consuming gq; the last one refills the slot
  __device__ void release(int gq) const {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      __threadfence_block();
      const int slot = gq % kRing;
      if (atomicAdd(&slot_cnt[slot], 1) == kWarps - 1) {
        slot_cnt[slot] = 0;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (gq + kRing < 2 * ngroups) issue(gq + kRing);
      }
    }
  }
};

template <typename T, int KS, int NT, int NSPLIT>
__global__ void __launch_bounds__(kThreads, 2) token_select_kernel(const __grid_constant__ SelectParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ SelCtl ctl;
  __shared__ __align__(8) uint64_t full[kRing];
  __shared__ int slot_cnt[kRing];
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q4 = lane & 3, r0 = lane >> 2;
  const unsigned rank = blockIdx.x;  // cluster = the cs CTAs of blockIdx.y
  const int cs = p.cs;
  const int pair = blockIdx.y;
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;
  uint32_t* bkeys = reinterpret_cast<uint32_t*>(smem + p.off_bkeys);
  int* cblk = reinterpret_cast<int*>(smem + p.off_cblk);
  uint32_t* qb = reinterpret_cast<uint32_t*>(smem + p.off_qb);
  float* qsum = reinterpret_cast<float*>(smem + p.off_qsum);
  float* qc = reinterpret_cast<float*>(smem + p.off_qc);
  uint8_t* ring = smem + p.off_ring;
  uint32_t* tkeys = reinterpret_cast<uint32_t*>(smem + p.off_tkeys);
  unsigned long long* dbg = p.dbg ? p.dbg + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 : nullptr;
#define TLS_STAMP(i) \
  if (dbg && tid == 0) dbg[i] = gtimer();
  TLS_STAMP(0)
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&full[s], 1);
      slot_cnt[s] = 0;
    }
    mbar_fence_init();
  }
  // ---- channel-projected query q~_h[c] = q_h[C_c], gathered once ----
  constexpr int DC = KS * 16;
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * d.Hq + (size_t)g * d.G) * d.d_k;
  if (tid < DC) ctl.chan[tid] = p.channels[(size_t)g * d.d_c + tid];
  // ---- a2 input: keys of the m block scores (K1's output, L2-resident) ----
  const float* sc = p.scores + (size_t)pair * d.M;
  for (int i = tid; i < m; i += kThreads) bkeys[i] = f2key(sc[i]);
  __syncthreads();
  for (int i = tid; i < NT * 8 * DC; i += kThreads) {
    const int h = i / DC, c = i - h * DC;
    qc[i] = h < d.G ? to_f32<T>(qg[(size_t)h * d.d_k + ctl.chan[c]]) : 0.f;
  }
  // ---- a2: M_t = top-k_b blocks.  Every CTA of the cluster selects
  // redundantly from identical data, so the candidate list needs no exchange.
  const bool sync_mode = p.guide == nullptr;
  {
    const int K = min(d.Kb, m);
    const TopK t = fast_topk(bkeys, m, K, d.Kb >= m, ctl.fk, ctl.tk);
    int* bout = p.block_ids + (size_t)pair * d.Kb;
    topk_emit(bkeys, m, t, ctl.tk, [&](int i, int pos) {
      if (sync_mode) cblk[pos] = i;
      if (rank == 0) bout[pos] = i;
    });
    if (rank == 0)
      for (int pos = K + tid; pos < d.Kb; pos += kThreads) bout[pos] = -1;
    if (sync_mode) {
      if (tid == 0) ctl.kc = K;
    } else {
      // one-step-lag mode: candidates = the guide blocks (ascending, -1 padded)
      const int* gd = p.guide + (size_t)pair * d.Kb;
      const int per = (d.Kb + kThreads - 1) / kThreads;
      const int lo = min(tid * per, d.Kb), hi = min(lo + per, d.Kb);
      int cnt = 0;
      for (int i = lo; i < hi; ++i) cnt += (gd[i] >= 0 && gd[i] < m);
      int total;
      int pos = block_exclusive_scan(cnt, ctl.tk.scan, &total);
      for (int i = lo; i < hi; ++i)
        if (gd[i] >= 0 && gd[i] < m && pos < p.kb_eff) cblk[pos++] = gd[i];
      if (tid == 0) ctl.kc = min(total, p.kb_eff);
    }
    __syncthreads();
  }
  TLS_STAMP(1)
  // ---- a3 setup: this CTA's share of the candidate blocks, streamed ----
  const int kc = ctl.kc;
  const int cb0 = (int)((long long)kc * rank / cs), cb1 = (int)((long long)kc * (rank + 1) / cs);
  IndexRing rg;
  rg.p = &p;
  rg.cbase = p.codes + (size_t)pair * d.S * (d.d_c / 2);
  rg.zbase = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * d.S;
  rg.cblk = cblk;
  rg.cb0 = cb0;
  rg.nbl = cb1 - cb0;
  rg.ngroups = (rg.nbl + p.rb - 1) / p.rb;
  rg.zal = (((size_t)pair * d.S) & 1) == 0;
  rg.ring = ring;
  rg.full = full;
  rg.slot_cnt = slot_cnt;
  if (tid == 0)
    for (int gq = 0; gq < min(kRing, 2 * rg.ngroups); ++gq) rg.issue(gq);
  // warm L2 with the rest of this CTA's candidate index (the ring then refills from L2)
  if (warp == 1) {
    const int rowbytes_ = d.d_c / 2;
    for (int k = kRing * p.rb + lane; k < rg.nbl; k += 32) {
      const int blk = cblk[cb0 + k];
      const int rows = min(d.B, d.S - blk * d.B);
      tma_prefetch_l2(rg.cbase + (size_t)blk * d.B * rowbytes_, rows * rowbytes_);
      if (rg.zal) tma_prefetch_l2(rg.zbase + (size_t)blk * d.B, rows * 8);
    }
  }
  // B fragments of the token contraction and sum_c q~_h[c] (overlaps the first loads)
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
  if (tid == 0) {
    int nv = 0;
    for (int k = cb0; k < cb1; ++k) nv += min(d.B, n - (cblk[k] << d.log2B));
    ctl.nvalid = nv;
  }
  __syncthreads();
  const float sm2 = d.sm_scale * kLog2e;
  float sq[NT][2];  // sm2 * sum_c q~_h[c] for this thread's heads
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) sq[nt][e] = sm2 * qsum[nt * 8 + 2 * q4 + e];
  const uint2* qb2 = reinterpret_cast<const uint2*>(qb);
  const int tshift = d.log2B - 4;  // 16-token tiles per block = 2^tshift
  const int rowbytes = d.d_c / 2;
  const float2* zglob = rg.zbase;

  // ---- pass 1: online per-head (max, sum) of
  //      L_hj = sm2 * (zero_j * sum_c q~_h[c] + scale_j * (q~_h . code_j)) ----
  {
    float rm[NT][2], rs[NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i) rm[i][0] = rm[i][1] = -CUDART_INF_F, rs[i][0] = rs[i][1] = 0.f;
    for (int gi = 0; gi < rg.ngroups; ++gi) {
      const int gq = gi, slot = gq % kRing;
      rg.wait(gq);
      const uint8_t* gcodes = rg.slot_codes(slot);
      const float2* gsz = rg.slot_sz(slot);
      const int ntiles = rg.group_blocks(gi) << tshift;
      for (int tile = warp; tile < ntiles; tile += kWarps) {
        float acc[NT][4];
        token_tile_mma<KS, NT, NSPLIT>(gcodes + (size_t)tile * 16 * rowbytes, qb2, acc);
        const int kb = tile >> tshift;
        const int blk = cblk[cb0 + gi * p.rb + kb];
        const int tok0 = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
        const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
        const float2 z0 = rg.zal ? gsz[tile * 16 + r0] : (v0 ? __ldg(zglob + tok0) : make_float2(0.f, 0.f));
        const float2 z1 = rg.zal ? gsz[tile * 16 + r0 + 8] : (v1 ? __ldg(zglob + tok0 + 8) : make_float2(0.f, 0.f));
        const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
        if (tok0 - r0 + 16 <= n) {  // warp-uniform: every token of the tile is valid
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float l0 = fmaf(s0, acc[nt][e], z0.y * sq[nt][e]);
              const float l1 = fmaf(s1, acc[nt][2 + e], z1.y * sq[nt][e]);
              const float mt = fmaxf(l0, l1);
              if (mt > rm[nt][e]) {  // rescale only when the running max grows
                rs[nt][e] *= fexp2(rm[nt][e] - mt);
                rm[nt][e] = mt;
              }
              rs[nt][e] += fexp2(l0 - rm[nt][e]) + fexp2(l1 - rm[nt][e]);
            }
        } else {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float l0 = v0 ? fmaf(s0, acc[nt][e], z0.y * sq[nt][e]) : -CUDART_INF_F;
              const float l1 = v1 ? fmaf(s1, acc[nt][2 + e], z1.y * sq[nt][e]) : -CUDART_INF_F;
              const float mt = fmaxf(l0, l1);
              if (mt > rm[nt][e]) {
                rs[nt][e] *= fexp2(rm[nt][e] - mt);
                rm[nt][e] = mt;
              }
              if (mt != -CUDART_INF_F) rs[nt][e] += fexp2(l0 - rm[nt][e]) + fexp2(l1 - rm[nt][e]);
            }
        }
      }
      rg.release(gq);
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
      ctl.hm[tid] = mm;
      ctl.hz[tid] = ss;
    }
  }
  TLS_STAMP(2)
  if (cs > 1) {
    cluster_sync_all();
    if (tid < d.G) {  // the cs CTAs' (max, sum) merged in rank order
      float hm[kMaxCluster], hz[kMaxCluster];
#pragma unroll
      for (int rr = 0; rr < kMaxCluster; ++rr) {
        hm[rr] = rr < cs ? *dsmem(&ctl.hm[tid], rr) : -CUDART_INF_F;
        hz[rr] = rr < cs ? *dsmem(&ctl.hz[tid], rr) : 0.f;
      }
      float M = -CUDART_INF_F, Z = 0.f;
#pragma unroll
      for (int rr = 0; rr < kMaxCluster; ++rr) stat_merge(M, Z, hm[rr], hz[rr]);
      ctl.hlz[tid] = M + flog2(Z);
    }
    if (tid == 32) {
      int nv[kMaxCluster];
#pragma unroll
      for (int rr = 0; rr < kMaxCluster; ++rr) nv[rr] = rr < cs ? *dsmem(&ctl.nvalid, rr) : 0;
      int jt = 0;
#pragma unroll
      for (int rr = 0; rr < kMaxCluster; ++rr) jt += nv[rr];
      ctl.jtot = jt;
    }
  } else {
    if (tid < d.G) ctl.hlz[tid] = ctl.hm[tid] + flog2(ctl.hz[tid]);
    if (tid == 32) ctl.jtot = ctl.nvalid;
  }
  __syncthreads();
  TLS_STAMP(3)
  // ---- pass 2: ranking key log2 alpha~_j + log2 G = log2 sum_h exp2(L_hj - lz_h)
  // (reading U15), written into rank 0's key array (DSMEM when cs > 1) ----
  {
    float lz[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int h = nt * 8 + 2 * q4 + e;
        lz[nt][e] = h < d.G ? ctl.hlz[h] : CUDART_INF_F;  // padded heads: exp2(-inf) = 0
      }
    uint32_t* keys0 = cs > 1 ? dsmem(tkeys, 0) : tkeys;
    for (int gi = 0; gi < rg.ngroups; ++gi) {
      const int gq = rg.ngroups + gi, slot = gq % kRing;
      rg.wait(gq);
      const uint8_t* gcodes = rg.slot_codes(slot);
      const float2* gsz = rg.slot_sz(slot);
      const int ntiles = rg.group_blocks(gi) << tshift;
      for (int tile = warp; tile < ntiles; tile += kWarps) {
        float acc[NT][4];
        token_tile_mma<KS, NT, NSPLIT>(gcodes + (size_t)tile * 16 * rowbytes, qb2, acc);
        const int kb = tile >> tshift;
        const int blk = cblk[cb0 + gi * p.rb + kb];
        const int tok0 = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
        const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
        const float2 z0 = rg.zal ? gsz[tile * 16 + r0] : (v0 ? __ldg(zglob + tok0) : make_float2(0.f, 0.f));
        const float2 z1 = rg.zal ? gsz[tile * 16 + r0 + 8] : (v1 ? __ldg(zglob + tok0 + 8) : make_float2(0.f, 0.f));
        const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
        float t0[NT][2], t1[NT][2];
        float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            t0[nt][e] = fmaf(s0, acc[nt][e], fmaf(z0.y, sq[nt][e], -lz[nt][e]));
            t1[nt][e] = fmaf(s1, acc[nt][2 + e], fmaf(z1.y, sq[nt][e], -lz[nt][e]));
            mx0 = fmaxf(mx0, t0[nt][e]);
            mx1 = fmaxf(mx1, t1[nt][e]);
          }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        float e0 = 0.f, e1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            e0 += fexp2(t0[nt][e] - mx0);
            e1 += fexp2(t1[nt][e] - mx1);
          }
        e0 += __shfl_xor_sync(0xffffffffu, e0, 1);
        e0 += __shfl_xor_sync(0xffffffffu, e0, 2);
        e1 += __shfl_xor_sync(0xffffffffu, e1, 1);
        e1 += __shfl_xor_sync(0xffffffffu, e1, 2);
        if (q4 == 0) {
          const int j0 = ((cb0 + gi * p.rb + kb) << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
          keys0[j0] = v0 ? f2key(mx0 + flog2(e0)) : 0u;
          keys0[j0 + 8] = v1 ? f2key(mx1 + flog2(e1)) : 0u;
        }
      }
      rg.release(gq);
    }
  }
  TLS_STAMP(4)
  if (cs > 1) {
    cluster_sync_all();  // every CTA's keys are in rank 0's smem
    if (rank != 0) return;
  }
  TLS_STAMP(5)
  // ---- a4: S_t = top-k_t tokens, rank 0 over all kc*B candidate slots ----
  {
    const int jtot = ctl.jtot;
    const int K = min(d.Kt, jtot);
    const int nslots = kc << d.log2B;
    const TopK t = fast_topk(tkeys, nslots, K, d.Kt >= jtot, ctl.fk, ctl.tk);
    int* tout = p.token_ids + (size_t)pair * d.Kt;
    float* sout = p.token_scores ? p.token_scores + (size_t)pair * d.Kt : nullptr;
    const float lnG = logf((float)d.G);
    topk_emit(tkeys, nslots, t, ctl.tk, [&](int i, int pos) {
      tout[pos] = (cblk[i >> d.log2B] << d.log2B) + (i & (d.B - 1));
      if (sout) sout[pos] = key2f(tkeys[i]) * kLn2 - lnG;
    });
    for (int pos = K + tid; pos < d.Kt; pos += kThreads) {
      tout[pos] = -1;
      if (sout) sout[pos] = -CUDART_INF_F;
    }
    if (tid == 0) p.num_tokens[pair] = K;
  }
  TLS_STAMP(6)
  TLS_STAMP(7)
#undef TLS_STAMP
}

// ============================================================== launchers
int score_cpl(int d_k, size_t elem_bytes) {
  const int nchunk = (int)(2 * d_k * elem_bytes / 16);
  if (nchunk <= 32) return 1;
  if (nchunk <= 64) return 2;
  if (nchunk <= 160) return 5;
  return -1;
}

template <typename T, int CPL>
static cudaError_t launch_k1(const ScoreParams& p, cudaStream_t st) {
  auto kern = block_score_kernel<T, CPL>;
  const int smem = p.tb * 2 * p.d.d_k * (int)sizeof(T);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((p.d.M + p.tb - 1) / p.tb), (unsigned)(p.d.batch * p.d.Hkv), 1);
  kern<<<grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_block_scores(const ScoreParams& p, cudaStream_t st) {
  const int cpl = score_cpl(p.d.d_k, p.d.bf16 ? 2 : 4);
  if (p.d.bf16) {
    if (cpl == 1) return launch_k1<__nv_bfloat16, 1>(p, st);
    if (cpl == 2) return launch_k1<__nv_bfloat16, 2>(p, st);
    return launch_k1<__nv_bfloat16, 5>(p, st);
  }
  if (cpl == 1) return launch_k1<float, 1>(p, st);
  if (cpl == 2) return launch_k1<float, 2>(p, st);
  return launch_k1<float, 5>(p, st);
}

template <typename T, int KS, int NT, int NSPLIT>
static cudaError_t launch_k2(const SelectParams& p, cudaStream_t st) {
  auto kern = token_select_kernel<T, KS, NT, NSPLIT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  if (p.cs > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)p.cs, (unsigned)(p.d.batch * p.d.Hkv), 1);
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.dynamicSmemBytes = p.smem_bytes;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, kern, p);
}

// Supported (d_c, G) combinations: KS = d_c/16 in {2, 4, 8}, NT = ceil(G/8) in {1, 2, 4}.
bool select_supported(int d_c, int G) {
  const int ks = d_c / 16, nt = (G + 7) / 8;
  return (ks == 2 || ks == 4 || ks == 8) && (nt == 1 || nt == 2 || nt == 3 || nt == 4) && d_c % 32 == 0;
}

template <typename T, int NS>
static cudaError_t dispatch_k2(const SelectParams& p, cudaStream_t st) {
  const int ks = p.d.d_c / 16, nt = (p.d.G + 7) / 8;
#define TLS_K2(KS_, NT_) \
  if (ks == KS_ && nt <= NT_) return launch_k2<T, KS_, NT_, NS>(p, st);
  TLS_K2(2, 1) TLS_K2(2, 2) TLS_K2(2, 4)
  TLS_K2(4, 1) TLS_K2(4, 2) TLS_K2(4, 4)
  TLS_K2(8, 1) TLS_K2(8, 2) TLS_K2(8, 4)
#undef TLS_K2
  return cudaErrorInvalidValue;
}

cudaError_t launch_token_select(const SelectParams& p, cudaStream_t st) {
  return p.d.bf16 ? dispatch_k2<__nv_bfloat16, 1>(p, st) : dispatch_k2<float, 3>(p, st);
}

}  // namespace tls
