// index.cu -- index construction (prefill / decode append) and channel
// calibration for AsyncTLS (arXiv 2604.07815), sm_100a.
//
//   build_index  (Fig. 2): per block the channelwise
//                max / min of its valid keys; per token the INT4 code of the
//                channel-projected key (reading U8/U9: per-token asymmetric
//                min/max over the d_c channels, IEEE fp32 RNE, so the codes
//                are a well-defined integer function of the stored keys).
//   calibrate: s_i = (1/G) sum_h max|q_h[i]| * max|k[i]|,
//                top-d_c channels (ties -> lower id), fp64 like the paper's
//                definition leaves it (no rounding choice to make).
#include "common.cuh"
#include "index.h"

#include <math_constants.h>

namespace tls {

// One CTA per (block i, pair).  Blocks before start_block or at / beyond the
// valid length are left untouched.
template <typename T>
__global__ void __launch_bounds__(kThreads) build_index_kernel(const __grid_constant__ IndexParams p) {
  const int i = blockIdx.x + p.start_block;
  const int pair = blockIdx.y;
  const int b = pair / p.Hkv, g = pair - b * p.Hkv;
  const int n = min(max(p.seq_lens[b], 0), p.S);
  const int t0 = i * p.B;
  if (t0 >= n) return;
  const int t1 = min(t0 + p.B, n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const T* K = reinterpret_cast<const T*>(p.k_cache) + (size_t)pair * p.S * p.d_k;
  // k^max_i, k^min_i: exact (max / min of stored values)
  T* bm = reinterpret_cast<T*>(p.block_minmax) + ((size_t)pair * p.M + i) * 2 * p.d_k;
  for (int c = tid; c < p.d_k; c += kThreads) {
    float mx = -CUDART_INF_F, mn = CUDART_INF_F;
    for (int t = t0; t < t1; ++t) {
      const float v = to_f32<T>(K[(size_t)t * p.d_k + c]);
      mx = fmaxf(mx, v);
      mn = fminf(mn, v);
    }
    bm[c] = from_f32<T>(mx);
    bm[p.d_k + c] = from_f32<T>(mn);
  }
  // INT4 token index: x = k_j[C]; zero = min x; scale = (max x - zero)/15;
  // code = scale > 0 ? clamp(rint((x - zero)/scale), 0, 15) : 0.
  const int* chan = p.channels + (size_t)g * p.d_c;
  const int rowbytes = p.d_c / 2;
  uint8_t* cd = p.codes + (size_t)pair * p.S * rowbytes;
  float2* sz = reinterpret_cast<float2*>(p.scale_zero) + (size_t)pair * p.S;
  for (int t = t0 + warp; t < t1; t += kWarps) {
    const T* row = K + (size_t)t * p.d_k;
    float mx = -CUDART_INF_F, mn = CUDART_INF_F;
    for (int c = lane; c < p.d_c; c += 32) {
      const float x = to_f32<T>(row[chan[c]]);
      mx = fmaxf(mx, x);
      mn = fminf(mn, x);
    }
    mx = warp_max(mx);
    mn = warp_min(mn);
    const float zero = mn;
    const float scale = __fdiv_rn(__fsub_rn(mx, zero), 15.0f);
    for (int j = lane; j < rowbytes; j += 32) {
      int code[2] = {0, 0};
      if (scale > 0.f) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float x = to_f32<T>(row[chan[2 * j + e]]);
          const int c = __float2int_rn(__fdiv_rn(__fsub_rn(x, zero), scale));
          code[e] = min(max(c, 0), 15);
        }
      }
      cd[(size_t)t * rowbytes + j] = (uint8_t)(code[0] | (code[1] << 4));
    }
    if (lane == 0) sz[t] = make_float2(scale, zero);
  }
}

// One CTA per KV head g.  Scores in fp64 (smem, d_k <= 1024).
template <typename T>
__global__ void __launch_bounds__(kThreads) calibrate_kernel(const __grid_constant__ CalibParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* s = reinterpret_cast<double*>(smem);
  int* flag = reinterpret_cast<int*>(s + p.d_k);
  const int g = blockIdx.x, tid = threadIdx.x;
  const T* q = reinterpret_cast<const T*>(p.q_cal);
  const T* k = reinterpret_cast<const T*>(p.k_cal) + (size_t)g * p.k_head_stride;
  for (int c = tid; c < p.d_k; c += kThreads) {
    double km = 0.0;
    for (int r = 0; r < p.n_k; ++r) km = fmax(km, fabs((double)to_f32<T>(k[(size_t)r * p.d_k + c])));
    double acc = 0.0;
    for (int h = 0; h < p.G; ++h) {
      double qm = 0.0;
      for (int r = 0; r < p.n_q; ++r)
        qm = fmax(qm, fabs((double)to_f32<T>(q[((size_t)r * p.Hq + (size_t)g * p.G + h) * p.d_k + c])));
      acc += qm * km;
    }
    acc /= (double)p.G;
    s[c] = acc;
    if (p.channel_scores) p.channel_scores[(size_t)g * p.d_k + c] = (float)acc;
  }
  __syncthreads();
  for (int c = tid; c < p.d_k; c += kThreads) {
    int rank = 0;
    for (int c2 = 0; c2 < p.d_k; ++c2) rank += (s[c2] > s[c]) || (s[c2] == s[c] && c2 < c);
    flag[c] = rank < p.d_c;
  }
  __syncthreads();
  for (int c = tid; c < p.d_k; c += kThreads) {
    if (!flag[c]) continue;
    int pos = 0;
    for (int c2 = 0; c2 < c; ++c2) pos += flag[c2];
    p.channels_out[(size_t)g * p.d_c + pos] = c;
  }
}

cudaError_t launch_build_index(const IndexParams& p, bool bf16, cudaStream_t stream) {
  const int nblocks = p.M - p.start_block;
  if (nblocks <= 0) return cudaSuccess;
  dim3 grid((unsigned)nblocks, (unsigned)(p.batch * p.Hkv), 1);
  if (bf16)
    build_index_kernel<__nv_bfloat16><<<grid, kThreads, 0, stream>>>(p);
  else
    build_index_kernel<float><<<grid, kThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_calibrate(const CalibParams& p, bool bf16, cudaStream_t stream) {
  const size_t smem = (size_t)p.d_k * (sizeof(double) + sizeof(int));
  if (bf16)
    calibrate_kernel<__nv_bfloat16><<<p.Hkv, kThreads, smem, stream>>>(p);
  else
    calibrate_kernel<float><<<p.Hkv, kThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace tls
