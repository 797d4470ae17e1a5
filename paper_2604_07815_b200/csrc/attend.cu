// attend.cu -- sparse attention over the selected tokens
// for sm_100a: K3 attend_kernel, one thread-block cluster of cs CTAs per
// (batch, KV-head) pair, each CTA a 1/cs slice of the pair's k_t tokens
// (split-K flash decoding), partials merged over DSMEM with the LSE identity
// (T10).  bf16 GQA with head dim 64/128 runs on tensor cores (mma.sync);
// MLA and fp32 run the generic CUDA-core path (NEXT: tcgen05 for MLA).
#include <math_constants.h>

#include <type_traits>

#include "common.cuh"
#include "params.h"

namespace tls {

struct AttCtl {
  float am[64], al[64];  // per-head partial max / sum, log2 units (read remotely)
};

// --------------------------------------------------------------------------
// Phase E (generic CUDA-core path): partial attention of this CTA over its
// tokens sel[0..tloc) for the G heads of the pair, log2 domain.
// Leaves (am_h, al_h) in ctl and the unnormalised partial o in ao.
// --------------------------------------------------------------------------
template <typename T>
__device__ void phase_attend_generic(const AttendParams& p, int pair, int b, int g, const int* sel, int tloc,
                                     float* aq, float* as, float* ao, AttCtl& ctl) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * p.d.Hq + (size_t)g * p.d.G) * p.d.d_k;
  for (int i = tid; i < p.d.G * p.d.d_k; i += kThreads) aq[i] = to_f32<T>(qg[i]);
  __syncthreads();
  const T* kb = reinterpret_cast<const T*>(p.k_cache) + (size_t)pair * p.d.S * p.d.d_k;
  const T* vb = p.d.mla ? kb : reinterpret_cast<const T*>(p.v_cache) + (size_t)pair * p.d.S * p.d.d_v;
  const int vstride = p.d.mla ? p.d.d_k : p.d.d_v;
  const float sm2 = p.d.sm_scale * kLog2e;
  for (int t = warp; t < tloc; t += kWarps) {
    const T* krow = kb + (size_t)sel[t] * p.d.d_k;
    for (int h = 0; h < p.d.G; ++h) {
      float acc = 0.f;
      for (int e = lane; e < p.d.d_k; e += 32) acc = fmaf(aq[h * p.d.d_k + e], to_f32<T>(krow[e]), acc);
      acc = warp_sum(acc);
      if (lane == 0) as[h * p.tloc_max + t] = acc * sm2;
    }
  }
  __syncthreads();
  for (int h = warp; h < p.d.G; h += kWarps) {
    float mx = -CUDART_INF_F;
    for (int t = lane; t < tloc; t += 32) mx = fmaxf(mx, as[h * p.tloc_max + t]);
    mx = warp_max(mx);
    float l = 0.f;
    for (int t = lane; t < tloc; t += 32) {
      const float e = exp2f(as[h * p.tloc_max + t] - mx);
      as[h * p.tloc_max + t] = e;
      l += e;
    }
    l = warp_sum(l);
    if (lane == 0) {
      ctl.am[h] = mx;
      ctl.al[h] = l;
    }
  }
  __syncthreads();
  for (int idx = tid; idx < p.d.G * p.d.d_v; idx += kThreads) {
    const int h = idx / p.d.d_v, c = idx - h * p.d.d_v;
    float acc = 0.f;
    for (int t = 0; t < tloc; ++t) acc = fmaf(as[h * p.tloc_max + t], to_f32<T>(vb[(size_t)sel[t] * vstride + c]), acc);
    ao[idx] = acc;
  }
}

// --------------------------------------------------------------------------
// Phase E (tensor-core path, bf16 GQA, head dim D): FlashAttention-2 style
// split-K decode over this CTA's tokens sel[0..tloc).  Heads are the M rows of
// mma.sync m16n8k16 (G <= 16, padded), tokens the N / K dimension.  K and V
// rows of a 128-token chunk are gathered into XOR-swizzled shared memory with
// cp.async (16 B per op), read back with ldmatrix (.trans for V); each warp
// owns 16 tokens of the chunk and keeps its own online softmax state; the 8
// warp partials are merged in smem, then the cs CTA partials over DSMEM.
// --------------------------------------------------------------------------
template <int D>
__device__ void phase_attend_mma(const AttendParams& p, int pair, int b, int g, const int* sel, int tloc,
                                 uint8_t* kvbuf, float* ao, AttCtl& ctl) {
  constexpr int TC = kAttnChunk;
  constexpr int CPR = D / 8;  // 16-byte chunks per row
  constexpr int KS = D / 16;  // k-steps of QK^T
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, c2 = 2 * (lane & 3);
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(kvbuf);
  __nv_bfloat16* sV = sK + TC * D;
  const __nv_bfloat16* qg = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b * p.d.Hq + (size_t)g * p.d.G) * D;
  const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_cache) + (size_t)pair * p.d.S * D;
  const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(p.v_cache) + (size_t)pair * p.d.S * D;
  // Q as the A operand (rows = heads; rows >= G are zero)
  uint32_t qa[KS][4];
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int col = kk * 16 + c2;
    qa[kk][0] = r < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + r * D + col) : 0u;
    qa[kk][1] = r + 8 < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + (r + 8) * D + col) : 0u;
    qa[kk][2] = r < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + r * D + col + 8) : 0u;
    qa[kk][3] = r + 8 < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + (r + 8) * D + col + 8) : 0u;
  }
  const float sm2 = p.d.sm_scale * kLog2e;
  float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;
  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;

  for (int c0 = 0; c0 < tloc; c0 += TC) {
    const int nt = min(TC, tloc - c0);
    __syncthreads();  // previous chunk consumed
    for (int i = tid; i < TC * CPR; i += kThreads) {
      const int row = i / CPR, ch = i - row * CPR;
      const bool ok = row < nt;
      const int tok = ok ? sel[c0 + row] : 0;
      const int dst = row * D + ((ch ^ (row & 7)) << 3);
      cp_async16(sK + dst, kb + (size_t)tok * D + ch * 8, ok);
      cp_async16(sV + dst, vb + (size_t)tok * D + ch * 8, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const int tb = warp * 16;
    if (tb < nt) {
      float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int row = tb + ((lane >> 4) << 3) + (lane & 7);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        uint32_t bk[4];
        ldsm_x4(bk, sK + row * D + ((ch ^ (row & 7)) << 3));
        mma_bf16_16816(s[0], qa[kk], bk[0], bk[1]);
        mma_bf16_16816(s[1], qa[kk], bk[2], bk[3]);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int t = tb + j * 8 + c2 + (e & 1);
          s[j][e] = t < nt ? s[j][e] * sm2 : -CUDART_INF_F;
        }
      float x0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
      float x1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
      x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, 1));
      x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, 2));
      x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, 1));
      x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, 2));
      const float n0 = fmaxf(m0, x0), n1 = fmaxf(m1, x1);  // finite: token tb is valid
      const float a0 = exp2f(m0 - n0), a1 = exp2f(m1 - n1);
      float pr[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        pr[j][0] = exp2f(s[j][0] - n0);
        pr[j][1] = exp2f(s[j][1] - n0);
        pr[j][2] = exp2f(s[j][2] - n1);
        pr[j][3] = exp2f(s[j][3] - n1);
      }
      float r0s = pr[0][0] + pr[0][1] + pr[1][0] + pr[1][1];
      float r1s = pr[0][2] + pr[0][3] + pr[1][2] + pr[1][3];
      r0s += __shfl_xor_sync(0xffffffffu, r0s, 1);
      r0s += __shfl_xor_sync(0xffffffffu, r0s, 2);
      r1s += __shfl_xor_sync(0xffffffffu, r1s, 1);
      r1s += __shfl_xor_sync(0xffffffffu, r1s, 2);
      l0 = l0 * a0 + r0s;
      l1 = l1 * a1 + r1s;
      m0 = n0;
      m1 = n1;
#pragma unroll
      for (int j = 0; j < D / 8; ++j) {
        o[j][0] *= a0;
        o[j][1] *= a0;
        o[j][2] *= a1;
        o[j][3] *= a1;
      }
      uint32_t pa[4];
      pa[0] = pack_bf16x2(pr[0][0], pr[0][1]);
      pa[1] = pack_bf16x2(pr[0][2], pr[0][3]);
      pa[2] = pack_bf16x2(pr[1][0], pr[1][1]);
      pa[3] = pack_bf16x2(pr[1][2], pr[1][3]);
#pragma unroll
      for (int jj = 0; jj < D / 16; ++jj) {
        const int row = tb + ((lane >> 3) & 1) * 8 + (lane & 7);
        const int ch = jj * 2 + (lane >> 4);
        uint32_t bv[4];
        ldsm_x4_trans(bv, sV + row * D + ((ch ^ (row & 7)) << 3));
        mma_bf16_16816(o[2 * jj], pa, bv[0], bv[1]);
        mma_bf16_16816(o[2 * jj + 1], pa, bv[2], bv[3]);
      }
    }
  }
  // ---- merge the 8 warp partials (the staging buffer becomes scratch) ----
  __syncthreads();
  float* wo = reinterpret_cast<float*>(kvbuf);  // [warp][G][D]
  float* wml = wo + kWarps * p.d.G * D;           // [warp][16][2]
  if ((lane & 3) == 0) {
    wml[(warp * 16 + r) * 2] = m0;
    wml[(warp * 16 + r) * 2 + 1] = l0;
    wml[(warp * 16 + r + 8) * 2] = m1;
    wml[(warp * 16 + r + 8) * 2 + 1] = l1;
  }
#pragma unroll
  for (int j = 0; j < D / 8; ++j) {
    const int d = j * 8 + c2;
    if (r < p.d.G) {
      wo[(warp * p.d.G + r) * D + d] = o[j][0];
      wo[(warp * p.d.G + r) * D + d + 1] = o[j][1];
    }
    if (r + 8 < p.d.G) {
      wo[(warp * p.d.G + r + 8) * D + d] = o[j][2];
      wo[(warp * p.d.G + r + 8) * D + d + 1] = o[j][3];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < p.d.G * D; idx += kThreads) {
    const int h = idx / D;
    float M = -CUDART_INF_F;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, wml[(w * 16 + h) * 2]);
    float L = 0.f, acc = 0.f;
    if (M != -CUDART_INF_F) {
      for (int w = 0; w < kWarps; ++w) {
        const float mw = wml[(w * 16 + h) * 2];
        const float sc = mw == -CUDART_INF_F ? 0.f : exp2f(mw - M);
        L = fmaf(wml[(w * 16 + h) * 2 + 1], sc, L);
        acc = fmaf(wo[(w * p.d.G + h) * D + (idx - h * D)], sc, acc);
      }
    }
    ao[idx] = acc;
    if (idx - h * D == 0) {
      ctl.am[h] = M;
      ctl.al[h] = L;
    }
  }
}

// Merge the cs partials of the pair (flash-decoding LSE merge, T10) and write
// out / lse.  CTA `rank` writes a 1/cs slice of the G*d_v outputs.
template <typename T>
__device__ void phase_merge(const AttendParams& p, int b, int g, unsigned rank, const float* ao, AttCtl& ctl) {
  const int tid = threadIdx.x;
  const int tot = p.d.G * p.d.d_v;
  const int lo = (int)((long long)tot * rank / p.cs), hi = (int)((long long)tot * (rank + 1) / p.cs);
  T* outg = reinterpret_cast<T*>(p.out) + ((size_t)b * p.d.Hq + (size_t)g * p.d.G) * p.d.d_v;
  for (int idx = lo + tid; idx < hi; idx += kThreads) {
    const int h = idx / p.d.d_v, c = idx - h * p.d.d_v;
    float M = -CUDART_INF_F;
    for (int rr = 0; rr < p.cs; ++rr) M = fmaxf(M, *dsmem(&ctl.am[h], rr));
    float L = 0.f, o = 0.f;
    if (M != -CUDART_INF_F) {
      for (int rr = 0; rr < p.cs; ++rr) {
        const float w = exp2f(*dsmem(&ctl.am[h], rr) - M);
        L = fmaf(*dsmem(&ctl.al[h], rr), w, L);
        o = fmaf(*dsmem(&ao[idx], rr), w, o);
      }
    }
    outg[idx] = from_f32<T>(L > 0.f ? o / L : 0.f);
    if (c == 0 && p.lse != nullptr)
      p.lse[(size_t)b * p.d.Hq + (size_t)g * p.d.G + h] = L > 0.f ? (M + log2f(L)) * kLn2 : -CUDART_INF_F;
  }
}

template <typename T, bool MMA, int D>
__global__ void __launch_bounds__(kThreads, 2) attend_kernel(const __grid_constant__ AttendParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ AttCtl ctl;
  const int tid = threadIdx.x;
  const unsigned rank = blockIdx.x;
  const int cs = p.cs;
  const int pair = blockIdx.y;
  const int b = pair / p.d.Hkv, g = pair - b * p.d.Hkv;
  const int K = min(min(max(p.num_tokens[pair], 0), p.d.Kt), p.tloc_max * cs);
  const int t0 = (int)((long long)K * rank / cs), t1 = (int)((long long)K * (rank + 1) / cs);
  const int tloc = t1 - t0;
  int* sel = reinterpret_cast<int*>(smem + p.off_sel);
  const int* ids = p.token_ids + (size_t)pair * p.d.Kt;
  for (int i = tid; i < tloc; i += kThreads) sel[i] = ids[t0 + i];
  __syncthreads();
  float* ao = reinterpret_cast<float*>(smem + p.off_ao);
  if constexpr (MMA) {
    phase_attend_mma<D>(p, pair, b, g, sel, tloc, smem + p.off_akv, ao, ctl);
  } else {
    phase_attend_generic<T>(p, pair, b, g, sel, tloc, reinterpret_cast<float*>(smem + p.off_aq),
                            reinterpret_cast<float*>(smem + p.off_as), ao, ctl);
  }
  cluster_sync_all();
  phase_merge<T>(p, b, g, rank, ao, ctl);
  cluster_sync_all();  // no CTA leaves while its smem may still be read remotely
}

template <typename T, bool MMA, int D>
static cudaError_t launch_k3(const AttendParams& p, cudaStream_t st) {
  auto kern = attend_kernel<T, MMA, D>;
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

cudaError_t launch_attend(const AttendParams& p, cudaStream_t st) {
  if (p.d.bf16) {
    if (p.mma) return p.d.d_k == 128 ? launch_k3<__nv_bfloat16, true, 128>(p, st)
                                     : launch_k3<__nv_bfloat16, true, 64>(p, st);
    return launch_k3<__nv_bfloat16, false, 0>(p, st);
  }
  return launch_k3<float, false, 0>(p, st);
}

}  // namespace tls
