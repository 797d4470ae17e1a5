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

namespace tls {

// ============================================================== K1: a1
// grid (ceil(m_max / tb), pairs).  A CTA scores blocks [i0, i0 + tb) of one
// pair: one thread streams the tile of block summaries (tb rows of
// [k^max | k^min], contiguous, <= 32 KB) into shared memory with TMA bulk
// copies in kSub sub-chunks, each completing on its own mbarrier; the warps
// score a sub-chunk as soon as it lands.  QQ = [Q+ | Q-] (2*d_k fp32), so
// s_i = QQ . row_i: 1 flop per byte, HBM-bound.
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
    float qp = 0.f, qn = 0.f;
    for (int h = 0; h < d.G; ++h) {
      const float v = to_f32<T>(qg[(size_t)h * d.d_k + c]);
      qp += fmaxf(v, 0.f);
      qn += fminf(v, 0.f);
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
    for (int i = s0 + warp; i < s1; i += kWarps) {
      const uint4* row = reinterpret_cast<const uint4*>(tile + (size_t)i * rowbytes);
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
        if (ch < nchunk) {
          float f[EPC];
          unpack16<T>(row[ch], f);
#pragma unroll
          for (int e = 0; e < EPC; ++e) acc = fmaf(qreg[c][e], f[e], acc);
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) out[i] = acc;
    }
  }
}

// ============================================================== K2: a2-a4
struct SelCtl {
  TopKCtl tk;
  int kc, nvalid, jtot;
  float hm[32], hz[32];  // per-head local (max, sum) (read remotely)
  float hlz[32];         // per-head log2 normaliser M_h + log2 Z_h
  float wm[kWarps][32], ws[kWarps][32];
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

// Stage codes + (scale, zero) of candidate blocks cblk[c0 .. c0+nbl) in smem:
// one TMA bulk copy per block for the codes (B*d_c/2 contiguous bytes) and one
// for (scale, zero) (B*8 bytes) on one mbarrier; 8-byte cp.async for a
// (scale, zero) run that is not 16-byte aligned (odd max_seq_len).
__device__ void stage_token_index(const SelectParams& p, int pair, const int* cblk, int c0, int nbl, uint8_t* stc,
                                  float2* stz, uint64_t* bar) {
  const Dims& d = p.d;
  const int rowbytes = d.d_c / 2;
  const uint8_t* cbase = p.codes + (size_t)pair * d.S * rowbytes;
  const float2* zbase = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * d.S;
  const bool zal = (((size_t)pair * d.S) & 1) == 0;
  const int tid = threadIdx.x;
  if (tid < 32) {
    uint32_t total = 0;
    for (int kb = 0; kb < nbl; ++kb) {
      const int rows = min(d.B, d.S - cblk[c0 + kb] * d.B);
      total += rows * rowbytes + ((zal && !(rows & 1)) ? rows * 8 : 0);
    }
    if (tid == 0) mbar_arrive_expect_tx(bar, total);
    __syncwarp();
    for (int kb = tid; kb < nbl; kb += 32) {
      const int blk = cblk[c0 + kb];
      const int rows = min(d.B, d.S - blk * d.B);
      tma_bulk_g2s(stc + (size_t)kb * d.B * rowbytes, cbase + (size_t)blk * d.B * rowbytes, rows * rowbytes, bar);
      if (zal && !(rows & 1)) tma_bulk_g2s(stz + kb * d.B, zbase + (size_t)blk * d.B, rows * 8, bar);
    }
  }
  for (int kb = 0; kb < nbl; ++kb) {  // rare fallback: unaligned (scale, zero) runs
    const int blk = cblk[c0 + kb];
    const int rows = min(d.B, d.S - blk * d.B);
    if (zal && !(rows & 1)) continue;
    for (int r = tid; r < rows; r += kThreads)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(stz + kb * d.B + r)),
                   "l"(zbase + (size_t)blk * d.B + r));
  }
  cp_async_commit();
  cp_async_wait<0>();
  mbar_wait(bar, 0);
  __syncthreads();
}

// acc[nt][*] = codes(tile) x q-fragments, for the NT n-tiles of 8 heads.
// A = codes (16 tokens x 16 channels per k-step), nibbles -> exact bf16; the
// channel order inside the MMA's K dimension is a permutation (thread q4 owns
// the contiguous code word(s) q4*WPT..), applied identically to the B
// fragments built in token_select_kernel.
template <int KS, int NT, int NSPLIT>
__device__ __forceinline__ void token_tile_mma(const uint8_t* stc, const uint2* qb2, int tile, float (&acc)[NT][4]) {
  constexpr int WPT = KS / 2;
  constexpr int ROWB = KS * 8;  // d_c / 2
  const int lane = threadIdx.x & 31, q4 = lane & 3, r0 = lane >> 2;
  const uint8_t* p0 = stc + (size_t)(tile * 16 + r0) * ROWB + q4 * WPT * 4;
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
  for (int s = 0; s < KS; ++s) {
    const int u = s >> 1, sel = 2 * (s & 1);
    a[s][0] = nib2bf16(w0[u], sel);
    a[s][1] = nib2bf16(w1[u], sel);
    a[s][2] = nib2bf16(w0[u], sel + 1);
    a[s][3] = nib2bf16(w1[u], sel + 1);
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

template <typename T, int KS, int NT, int NSPLIT>
__global__ void __launch_bounds__(kThreads, 2) token_select_kernel(const __grid_constant__ SelectParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ SelCtl ctl;
  __shared__ __align__(8) uint64_t stage_bar;
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
  uint8_t* stc = smem + p.off_stc;
  float2* stz = reinterpret_cast<float2*>(smem + p.off_stz);
  uint32_t* tkeys = reinterpret_cast<uint32_t*>(smem + p.off_tkeys);
  unsigned long long* dbg = p.dbg ? p.dbg + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 : nullptr;
#define TLS_STAMP(i) \
  if (dbg && tid == 0) dbg[i] = gtimer();
  TLS_STAMP(0)
  if (tid == 0) {
    mbar_init(&stage_bar, 1);
    mbar_fence_init();
  }
  // ---- channel-projected query q~_h[c] = q_h[C_c], gathered once ----
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * d.Hq + (size_t)g * d.G) * d.d_k;
  const int* chan = p.channels + (size_t)g * d.d_c;
  constexpr int DC = KS * 16;
  for (int i = tid; i < NT * 8 * DC; i += kThreads) {
    const int h = i / DC, c = i - h * DC;
    qc[i] = h < d.G ? to_f32<T>(qg[(size_t)h * d.d_k + chan[c]]) : 0.f;
  }
  // ---- a2 input: keys of the m block scores (K1's output, L2-resident) ----
  const float* sc = p.scores + (size_t)pair * d.M;
  for (int i = tid; i < m; i += kThreads) bkeys[i] = f2key(sc[i]);
  __syncthreads();
  // B fragments of the token contraction (MMA K order = channel permutation,
  // thread q4 owns code words q4*WPT..; see token_tile_mma), and sum_c q~_h[c]
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
  TLS_STAMP(1)
  // ---- a2: M_t = top-k_b blocks.  Every CTA of the cluster selects
  // redundantly from identical data, so the candidate list needs no exchange.
  const bool sync_mode = p.guide == nullptr;
  {
    const TopK t = radix_topk<false>(bkeys, m, min(d.Kb, m), d.Kb >= m, 1, 0, ctl.tk);
    int* bout = p.block_ids + (size_t)pair * d.Kb;
    topk_emit(bkeys, m, t, ctl.tk, [&](int i, int pos) {
      if (sync_mode) cblk[pos] = i;
      if (rank == 0) bout[pos] = i;
    });
    if (rank == 0)
      for (int pos = t.total + tid; pos < d.Kb; pos += kThreads) bout[pos] = -1;
    if (sync_mode) {
      if (tid == 0) ctl.kc = t.total;
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

  // ---- a3: token scores of this CTA's share of the candidate blocks ----
  const int kc = ctl.kc;
  const int cb0 = (int)((long long)kc * rank / cs), cb1 = (int)((long long)kc * (rank + 1) / cs);
  const int nbl = cb1 - cb0;
  const int lc = nbl << d.log2B;
  const int tshift = d.log2B - 4;  // 16-token tiles per block = 2^tshift
  const int ntiles = lc >> 4;
  TLS_STAMP(2)
  stage_token_index(p, pair, cblk, cb0, nbl, stc, stz, &stage_bar);
  TLS_STAMP(3)
  if (tid == 0) {
    int nv = 0;
    for (int k = cb0; k < cb1; ++k) nv += min(d.B, n - (cblk[k] << d.log2B));
    ctl.nvalid = nv;
  }
  const float sm2 = d.sm_scale * kLog2e;
  // per-thread head constants: L = zero * (sm2*qsum_h) + scale * (sm2 * acc)
  float sq[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) sq[nt][e] = sm2 * qsum[nt * 8 + 2 * q4 + e];
  const uint2* qb2 = reinterpret_cast<const uint2*>(qb);
  {  // pass 1: online per-head (max, sum)
    float rm[NT][2], rs[NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i) rm[i][0] = rm[i][1] = -CUDART_INF_F, rs[i][0] = rs[i][1] = 0.f;
    for (int tile = warp; tile < ntiles; tile += kWarps) {
      float acc[NT][4];
      token_tile_mma<KS, NT, NSPLIT>(stc, qb2, tile, acc);
      const int j0 = tile * 16 + r0;
      const int tok0 = (cblk[cb0 + (tile >> tshift)] << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
      const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
      const float2 z0 = stz[j0], z1 = stz[j0 + 8];
      const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float l0 = v0 ? fmaf(s0, acc[nt][e], z0.y * sq[nt][e]) : -CUDART_INF_F;
          const float l1 = v1 ? fmaf(s1, acc[nt][2 + e], z1.y * sq[nt][e]) : -CUDART_INF_F;
          const float mt = fmaxf(l0, l1);
          if (mt != -CUDART_INF_F) {
            const float nm = fmaxf(rm[nt][e], mt);
            rs[nt][e] = rs[nt][e] * fexp2(rm[nt][e] - nm) + fexp2(l0 - nm) + fexp2(l1 - nm);
            rm[nt][e] = nm;
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
      ctl.hm[tid] = mm;
      ctl.hz[tid] = ss;
    }
  }
  TLS_STAMP(4)
  cluster_sync_all();
  if (tid < d.G) {  // the cs CTAs' (max, sum) merged in rank order: lz_h = M_h + log2 Z_h
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
  __syncthreads();
  // pass 2: ranking key log2 alpha~_j + log2 G = log2 sum_h exp2(L_hj - lz_h)  (reading U15)
  {
    float lz[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int h = nt * 8 + 2 * q4 + e;
        lz[nt][e] = h < d.G ? ctl.hlz[h] : CUDART_INF_F;  // padded heads contribute exp2(-inf) = 0
      }
    for (int tile = warp; tile < ntiles; tile += kWarps) {
      float acc[NT][4];
      token_tile_mma<KS, NT, NSPLIT>(stc, qb2, tile, acc);
      const int j0 = tile * 16 + r0;
      const int tok0 = (cblk[cb0 + (tile >> tshift)] << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
      const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
      const float2 z0 = stz[j0], z1 = stz[j0 + 8];
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
        tkeys[j0] = v0 ? f2key(mx0 + flog2(e0)) : 0u;
        tkeys[j0 + 8] = v1 ? f2key(mx1 + flog2(e1)) : 0u;
      }
    }
  }
  __syncthreads();

  TLS_STAMP(5)
  // ---- a4: S_t = top-k_t tokens over the cluster ----
  {
    const int jtot = ctl.jtot;
    const int K = min(d.Kt, jtot);
    const TopK t = radix_topk<true>(tkeys, lc, K, d.Kt >= jtot, cs, rank, ctl.tk);
    int* tout = p.token_ids + (size_t)pair * d.Kt;
    float* sout = p.token_scores ? p.token_scores + (size_t)pair * d.Kt : nullptr;
    const float lnG = logf((float)d.G);
    topk_emit(tkeys, lc, t, ctl.tk, [&](int i, int pos) {
      tout[pos] = (cblk[cb0 + (i >> d.log2B)] << d.log2B) + (i & (d.B - 1));
      if (sout) sout[pos] = key2f(tkeys[i]) * kLn2 - lnG;
    });
    if (rank == 0) {
      for (int pos = K + tid; pos < d.Kt; pos += kThreads) {
        tout[pos] = -1;
        if (sout) sout[pos] = -CUDART_INF_F;
      }
      if (tid == 0) p.num_tokens[pair] = K;
    }
  }
  TLS_STAMP(6)
  cluster_sync_all();  // no CTA leaves while its smem may still be read remotely
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
