// Microbenchmark (diagnostic, not product): TMA bulk-copy streaming rate on B200 for the a1 access pattern
// (contiguous 32 KB tiles as 8 x 4 KB cp.async.bulk copies into a ring of S stages per CTA, one mbarrier per
// copy), vs CTAs per SM and ring depth.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void stream(const uint8_t* src, size_t ntiles, int S, int copy_kb, unsigned* ctr, float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[64];
  __shared__ int tick[16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncopy = 32 / copy_kb;  // copies per 32 KB tile
  if (tid == 0) {
    for (int i = 0; i < S * ncopy; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long ph = 0;  // parity bit per barrier
  auto issue = [&](int st, long t) {
    for (int c = 0; c < ncopy; ++c) {
      uint64_t* b = &bars[st * ncopy + c];
      const uint32_t bytes = copy_kb * 1024;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su(sm + st * 32768 + c * bytes)),
                   "l"(src + t * 32768 + c * bytes), "r"(bytes), "r"(su(b))
                   : "memory");
    }
  };
  if (tid == 0)
    for (int s = 0; s < S; ++s) {
      unsigned t = atomicAdd(ctr, 1u);
      tick[s] = t < ntiles ? (int)t : -1;
      if (t < ntiles) issue(s, t);
    }
  __syncthreads();
  float acc = 0.f;
  for (int k = 0;; ++k) {
    const int st = k % S;
    const int t = tick[st];
    if (t < 0) break;
    // each warp consumes one 4 KB slice
    for (int c = warp; c < 8; c += 8) {
      const int cb = (c * 4) / copy_kb;
      uint64_t* b = &bars[st * ncopy + cb];
      uint32_t done = 0, par = (unsigned)((ph >> (st * ncopy + cb)) & 1);
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(done) : "r"(su(b)), "r"(par) : "memory");
      } while (!done);
      const uint4 v = reinterpret_cast<const uint4*>(sm + st * 32768 + c * 4096)[lane];
      acc += __uint_as_float(v.x & 0x3f800000u);
    }
    for (int c = 0; c < ncopy; ++c) ph ^= 1ull << (st * ncopy + c);
    __syncthreads();
    if (tid == 0) {
      unsigned t2 = atomicAdd(ctr, 1u);
      tick[st] = t2 < ntiles ? (int)t2 : -1;
      if (t2 < ntiles) issue(st, t2);
    }
    __syncthreads();
  }
  if (acc == 12345.f) sink[0] = acc;
}
int main() {
  const size_t bytes = 201850880;  // C3 block summaries
  const size_t ntiles = bytes / 32768;
  uint8_t* src;
  cudaMalloc(&src, bytes + (1 << 20));
  cudaMemset(src, 1, bytes);
  unsigned* ctr;
  cudaMalloc(&ctr, 4);
  float* sink;
  cudaMalloc(&sink, 4);
  uint8_t* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm = 148;
  for (int copy_kb : {4, 8, 32})
    for (int S : {1, 2, 3, 4, 6})
      for (int cps : {1, 2, 3, 4, 6}) {
        size_t smem = (size_t)S * 32768;
        if (smem * cps > 220 * 1024) continue;
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
          cudaMemset(flush, it, 256 << 20);
          cudaMemset(ctr, 0, 4);
          cudaEventRecord(e0);
          stream<<<nsm * cps, 256, smem>>>(src, ntiles, S, copy_kb, ctr, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        printf("copy %2d KB  ring %d  CTAs/SM %d : %7.1f us  %6.0f GB/s %s\n", copy_kb, S, cps, best * 1e3,
               bytes / (best * 1e-3) / 1e9, err ? cudaGetErrorString(err) : ""); fflush(stdout);
      }
  return 0;
}
