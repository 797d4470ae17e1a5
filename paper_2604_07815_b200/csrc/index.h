// index.h -- parameter blocks of the index-construction and calibration
// kernels (index.cu), shared with the C ABI layer (api.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace tls {

struct IndexParams {
  int batch, Hkv, d_k, S, B, d_c, M;
  int start_block;
  const void* k_cache;
  const int* seq_lens;
  void* block_minmax;
  uint8_t* codes;
  float* scale_zero;
  const int* channels;
};

struct CalibParams {
  int Hq, Hkv, G, d_k, d_c, n_q, n_k;
  long long k_head_stride;
  const void* q_cal;
  const void* k_cal;
  int* channels_out;
  float* channel_scores;
};

cudaError_t launch_build_index(const IndexParams& p, bool bf16, cudaStream_t stream);
cudaError_t launch_calibrate(const CalibParams& p, bool bf16, cudaStream_t stream);

}  // namespace tls
