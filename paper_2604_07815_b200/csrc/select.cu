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
// grid (ceil(M / kScoreChunk), pairs); a CTA scores blocks [i0, i0 + 128) of
// one pair.  QQ = [Q+ | Q-] (2*d_k fp32); a block's summary row is
// [k^max | k^min], so s_i = QQ . row_i.  Each warp keeps U blocks (U*CPL
// 16-byte loads per lane) in flight.
template <typename T, int CPL>
__global__ void __launch_bounds__(kThreads) block_score_kernel(const __grid_constant__ ScoreParams p) {
  constexpr int EPC = 16 / sizeof(T);
  constexpr int U = CPL == 1 ? 8 : (CPL == 2 ? 4 : 2);
  __shared__ float QQ[2 * 32 * CPL * EPC];
  const Dims& d = p.d;
  const int pair = blockIdx.y;
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) / d.B;  // reading U1
  const int i0 = blockIdx.x * kScoreChunk;
  if (i0 >= m) return;
  const int i1 = min(i0 + kScoreChunk, m);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
  __syncthreads();
  const int nchunk = 2 * d.d_k / EPC;
  float qreg[CPL][EPC];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int ch = lane + 32 * c;
#pragma unroll
    for (int e = 0; e < EPC; ++e) qreg[c][e] = ch < nchunk ? QQ[ch * EPC + e] : 0.f;
  }
  const T* bm = reinterpret_cast<const T*>(p.block_minmax) + (size_t)pair * d.M * 2 * d.d_k;
  float* out = p.scores + (size_t)pair * d.M;
  for (int i = i0 + warp * U; i < i1; i += kWarps * U) {
    uint4 v[U][CPL];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
        v[u][c] = (i + u < i1 && ch < nchunk) ? ldg_stream16(bm + (size_t)(i + u) * 2 * d.d_k + (size_t)ch * EPC)
                                               : make_uint4(0u, 0u, 0u, 0u);
      }
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[u] = 0.f;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        float f[EPC];
        unpack16<T>(v[u][c], f);
#pragma unroll
        for (int e = 0; e < EPC; ++e) acc[u] = fmaf(qreg[c][e], f[e], acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = warp_sum(acc[u]);
    if (lane < U && i + lane < i1) {
      float mine = acc[0];
#pragma unroll
      for (int u = 1; u < U; ++u)
        if (lane == u) mine = acc[u];
      out[i + lane] = mine;
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
  s = (m == -CUDART_INF_F ? 0.f : s * exp2f(m - nm)) + (om == -CUDART_INF_F ? 0.f : os * exp2f(om - nm));
  m = nm;
}

// Stage codes + (scale, zero) of candidate blocks cblk[c0 .. c0+nbl) in smem.
__device__ void stage_token_index(const SelectParams& p, int pair, const int* cblk, int c0, int nbl, uint8_t* stc,
                                  float2* stz) {
  const Dims& d = p.d;
  const int rowbytes = d.d_c / 2;
  const int cpb = d.B * rowbytes / 16;  // 16-byte pieces of codes per block
  const int per = cpb + d.B;            // + one 8-byte (scale, zero) per token
  const uint8_t* cbase = p.codes + (size_t)pair * d.S * rowbytes;
  const float2* zbase = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * d.S;
  const size_t cend = (size_t)d.S * rowbytes;
  for (int i = threadIdx.x; i < nbl * per; i += kThreads) {
    const int kb = i / per;
    const int r = i - kb * per;
    const int blk = cblk[c0 + kb];
    if (r < cpb) {
      const size_t off = (size_t)blk * d.B * rowbytes + (size_t)r * 16;
      const bool ok = off + 16 <= cend;
      cp_async16(stc + (size_t)kb * d.B * rowbytes + (size_t)r * 16, cbase + (ok ? off : 0), ok);
    } else {
      const int t = blk * d.B + (r - cpb);
      const bool ok = t < d.S;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(stz + kb * d.B + (r - cpb))),
                   "l"(zbase + (ok ? t : 0)), "r"(ok ? 8 : 0));
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
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
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ SelCtl ctl;
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q4 = lane & 3, r0 = lane >> 2;
  const unsigned rank = blockIdx.x;  // cluster = the cs CTAs of blockIdx.y
  const int cs = p.cs;
  const int pair = blockIdx.y;
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) / d.B;
  uint32_t* bkeys = reinterpret_cast<uint32_t*>(smem + p.off_bkeys);
  int* cblk = reinterpret_cast<int*>(smem + p.off_cblk);
  uint32_t* qb = reinterpret_cast<uint32_t*>(smem + p.off_qb);
  float* qsum = reinterpret_cast<float*>(smem + p.off_qsum);
  uint8_t* stc = smem + p.off_stc;
  float2* stz = reinterpret_cast<float2*>(smem + p.off_stz);
  uint32_t* tkeys = reinterpret_cast<uint32_t*>(smem + p.off_tkeys);
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * d.Hq + (size_t)g * d.G) * d.d_k;
  const int* chan = p.channels + (size_t)g * d.d_c;

  // ---- query fragments for the token contraction, and sum_c q_h[C_c] ----
  constexpr int WPT = KS / 2;
  for (int idx = tid; idx < NSPLIT * NT * KS * 32; idx += kThreads) {
    const int ln = idx & 31, rest = idx >> 5;
    const int s = rest % KS, nt = (rest / KS) % NT, sp = rest / (KS * NT);
    const int hh = nt * 8 + (ln >> 2);
    const int wi = (ln & 3) * WPT + (s >> 1);
    const int cb = 8 * wi + 2 * (s & 1);
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    if (hh < d.G) {
      const T* qh = qg + (size_t)hh * d.d_k;
      x[0] = to_f32<T>(qh[chan[cb]]);
      x[1] = to_f32<T>(qh[chan[cb + 4]]);
      x[2] = to_f32<T>(qh[chan[cb + 1]]);
      x[3] = to_f32<T>(qh[chan[cb + 5]]);
    }
    qb[2 * idx] = pack_bf16x2(split_piece(x[0], sp), split_piece(x[1], sp));
    qb[2 * idx + 1] = pack_bf16x2(split_piece(x[2], sp), split_piece(x[3], sp));
  }
  for (int h = tid; h < NT * 8; h += kThreads) {
    float s = 0.f;
    if (h < d.G)
      for (int c = 0; c < d.d_c; ++c) s += to_f32<T>(qg[(size_t)h * d.d_k + chan[c]]);
    qsum[h] = s;
  }
  // ---- a2: M_t = top-k_b of the block scores (K1's output, L2-resident) ----
  // Every CTA of the cluster selects redundantly from identical data, so the
  // candidate list needs no exchange.
  const float* sc = p.scores + (size_t)pair * d.M;
  for (int i = tid; i < m; i += kThreads) bkeys[i] = f2key(sc[i]);
  __syncthreads();
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
  const int lc = nbl * d.B;
  const int ntiles = lc / 16;
  stage_token_index(p, pair, cblk, cb0, nbl, stc, stz);
  if (tid == 0) {
    int nv = 0;
    for (int k = cb0; k < cb1; ++k) nv += min(d.B, n - cblk[k] * d.B);
    ctl.nvalid = nv;
  }
  const float sm2 = d.sm_scale * kLog2e;
  const uint2* qb2 = reinterpret_cast<const uint2*>(qb);
  {  // pass 1: online per-head (max, sum) of L_hj = sm2*(zero*qsum_h + scale*(q~_h . code_j))
    float rm[NT][2], rs[NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i) rm[i][0] = rm[i][1] = -CUDART_INF_F, rs[i][0] = rs[i][1] = 0.f;
    for (int tile = warp; tile < ntiles; tile += kWarps) {
      float acc[NT][4];
      token_tile_mma<KS, NT, NSPLIT>(stc, qb2, tile, acc);
      const int j0 = tile * 16 + r0;
      const int kb = j0 / d.B;
      const int tok0 = cblk[cb0 + kb] * d.B + (j0 - kb * d.B);
      const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
      const float2 z0 = stz[j0], z1 = stz[j0 + 8];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float qs = qsum[nt * 8 + 2 * q4 + e];
          const float l0 = v0 ? sm2 * fmaf(z0.y, qs, z0.x * acc[nt][e]) : -CUDART_INF_F;
          const float l1 = v1 ? sm2 * fmaf(z1.y, qs, z1.x * acc[nt][2 + e]) : -CUDART_INF_F;
          const float mt = fmaxf(l0, l1);
          if (mt != -CUDART_INF_F) {
            const float nm = fmaxf(rm[nt][e], mt);
            rs[nt][e] = rs[nt][e] * exp2f(rm[nt][e] - nm) + exp2f(l0 - nm) + exp2f(l1 - nm);
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
    ctl.hlz[tid] = M + log2f(Z);
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
  for (int tile = warp; tile < ntiles; tile += kWarps) {
    float acc[NT][4];
    token_tile_mma<KS, NT, NSPLIT>(stc, qb2, tile, acc);
    const int j0 = tile * 16 + r0;
    const int kb = j0 / d.B;
    const int tok0 = cblk[cb0 + kb] * d.B + (j0 - kb * d.B);
    const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
    const float2 z0 = stz[j0], z1 = stz[j0 + 8];
    float t0[NT][2], t1[NT][2];
    float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int h = nt * 8 + 2 * q4 + e;
        if (h < d.G) {
          const float qs = qsum[h], lz = ctl.hlz[h];
          t0[nt][e] = sm2 * fmaf(z0.y, qs, z0.x * acc[nt][e]) - lz;
          t1[nt][e] = sm2 * fmaf(z1.y, qs, z1.x * acc[nt][2 + e]) - lz;
        } else {
          t0[nt][e] = t1[nt][e] = -CUDART_INF_F;
        }
        mx0 = fmaxf(mx0, t0[nt][e]);
        mx1 = fmaxf(mx1, t1[nt][e]);
      }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        s0 += exp2f(t0[nt][e] - mx0);
        s1 += exp2f(t1[nt][e] - mx1);
      }
    s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    if (q4 == 0) {
      tkeys[j0] = v0 ? f2key(mx0 + log2f(s0)) : 0u;
      tkeys[j0 + 8] = v1 ? f2key(mx1 + log2f(s1)) : 0u;
    }
  }
  __syncthreads();

  // ---- a4: S_t = top-k_t tokens over the cluster ----
  {
    const int jtot = ctl.jtot;
    const int K = min(d.Kt, jtot);
    const TopK t = radix_topk<true>(tkeys, lc, K, d.Kt >= jtot, cs, rank, ctl.tk);
    int* tout = p.token_ids + (size_t)pair * d.Kt;
    float* sout = p.token_scores ? p.token_scores + (size_t)pair * d.Kt : nullptr;
    const float lnG = logf((float)d.G);
    topk_emit(tkeys, lc, t, ctl.tk, [&](int i, int pos) {
      const int kb = i / d.B;
      tout[pos] = cblk[cb0 + kb] * d.B + (i - kb * d.B);
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
  cluster_sync_all();  // no CTA leaves while its smem may still be read remotely
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
  dim3 grid((unsigned)((p.d.M + kScoreChunk - 1) / kScoreChunk), (unsigned)(p.d.batch * p.d.Hkv), 1);
  block_score_kernel<T, CPL><<<grid, kThreads, 0, st>>>(p);
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
