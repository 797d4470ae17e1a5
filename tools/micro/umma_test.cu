// Diagnostic (not product): validate hand-built tcgen05 descriptors on sm_100a.
// D[M=128][N] (fp32, TMEM) = A[M][K] . B[N][K]^T, A/B bf16 in shared memory in the canonical
// SWIZZLE_NONE K-major layout (core matrix = 8 rows x 16 B contiguous; LBO = K-adjacent core
// matrices, SBO = M/N-adjacent 8-row groups), or B MN-major (core matrix = 8 K-rows x 16 B of N).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_test umma_test.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm100)
  // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
  return d;
}
// kind::f16 instruction descriptor: D f32, A/B bf16, K-major A, B major per flag, N, M
__host__ __device__ constexpr uint32_t idesc(int M, int N, int b_mn_major, int a_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, int K, int BMN, int M>
__global__ void umma_gemm(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  __shared__ __align__(1024) __nv_bfloat16 sA[M * K];
  __shared__ __align__(1024) __nv_bfloat16 sB[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  // A K-major canonical: element (m, k) at byte ((m/8)*SBO + (k/8)*LBO + (m%8)*16 + (k%8)*2)
  constexpr uint32_t A_LBO = 128, A_SBO = (K / 8) * 128;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const uint32_t off = (m / 8) * A_SBO + (k / 8) * A_LBO + (m % 8) * 16 + (k % 8) * 2;
    sA[off / 2] = A[i];
  }
  uint32_t B_LBO, B_SBO;
  if (BMN == 0) {  // K-major: element (n, k)
    B_LBO = 128;
    B_SBO = (K / 8) * 128;
    for (int i = tid; i < N * K; i += blockDim.x) {
      const int n = i / K, k = i % K;
      const uint32_t off = (n / 8) * B_SBO + (k / 8) * B_LBO + (n % 8) * 16 + (k % 8) * 2;
      sB[off / 2] = B[i];
    }
  } else {  // MN-major: core matrix = 8 k-rows x (8 n-elements = 16 B); n-groups at SBO, k-groups at LBO
    B_SBO = 128;
    B_LBO = (N / 8) * 128;
    for (int i = tid; i < N * K; i += blockDim.x) {
      const int n = i / K, k = i % K;
      const uint32_t off = (k / 8) * B_LBO + (n / 8) * B_SBO + (k % 8) * 16 + (n % 8) * 2;
      sB[off / 2] = B[i];
    }
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su(&tmem_base)),
                 "n"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic smem writes -> async proxy (MMA)
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc(M, N, BMN, 0);
    for (int ks = 0; ks < K / 16; ++ks) {
      // K step of 16 = 2 core-matrix columns: advance by 2*LBO (K-major) ...
      const uint64_t da = sdesc(su(sA) + ks * 2 * A_LBO, A_LBO, A_SBO);
      const uint64_t db = BMN == 0 ? sdesc(su(sB) + ks * 2 * B_LBO, B_LBO, B_SBO)
                                   : sdesc(su(sB) + ks * 2 * B_LBO, B_LBO, B_SBO);  // MN-major: 16 k = 2 LBO groups
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su(&bar))
                 : "memory");
  }
  // wait for the MMAs
  {
    uint32_t done = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                   : "=r"(done) : "r"(su(&bar)) : "memory");
    } while (!done);
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // warp w reads lanes 32w..32w+31 (rows m), 32x32b: thread t of the warp gets lane 32w+t, N columns
  const int warp = tid / 32, lane = tid % 32;
  if (warp < 4) {  // dump all 128 lanes: D[lane][col]
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 8; ++j) D[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(32));
}

template <int N, int K, int BMN, int M = 128>
int run() {
  __nv_bfloat16 *A, *B;
  float* D;
  cudaMallocManaged(&A, M * K * 2);
  cudaMallocManaged(&B, N * K * 2);
  cudaMallocManaged(&D, 128 * N * 4);
  for (int i = 0; i < 128 * N; ++i) D[i] = -12345.f;
  srand(1);
  for (int i = 0; i < M * K; ++i) A[i] = __float2bfloat16((rand() % 17 - 8) / 8.f);
  for (int i = 0; i < N * K; ++i) B[i] = __float2bfloat16((rand() % 17 - 8) / 8.f);
  umma_gemm<N, K, BMN, M><<<1, 128>>>(A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d K=%d BMN=%d: CUDA error %s\n", N, K, BMN, cudaGetErrorString(e));
    return 1;
  }
  if (M == 64) {  // where does row m land? find each row's values among the 128 lanes
    for (int m = 0; m < M; ++m) {
      double ref0 = 0;
      for (int k = 0; k < K; ++k) ref0 += (double)__bfloat162float(A[m * K + k]) * __bfloat162float(B[k]);
      int found = -1;
      for (int l = 0; l < 128; ++l) {
        bool ok = true;
        for (int n = 0; n < N && ok; ++n) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)__bfloat162float(A[m * K + k]) * __bfloat162float(B[n * K + k]);
          ok = fabs(ref - D[l * N + n]) < 1e-3;
        }
        if (ok) { found = l; break; }
      }
      printf("%d->%d ", m, found);
    }
    printf("\n");
    return 0;
  }
  double maxerr = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)__bfloat162float(A[m * K + k]) * __bfloat162float(B[n * K + k]);
      maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
    }
  printf("N=%d K=%d B %s-major: max |err| = %g  (D[0]=%g D[last]=%g)\n", N, K, BMN ? "MN" : "K", maxerr, D[0],
         D[M * N - 1]);
  return maxerr > 1e-3;
}

int main() {
  int bad = 0;
  run<32, 64, 0, 64>();
  bad += run<32, 64, 0>();
  bad += run<32, 128, 0>();
  bad += run<64, 64, 0>();
  bad += run<32, 64, 1>();
  printf(bad ? "FAIL\n" : "ALL OK\n");
  return 0;
}
