// common.cuh -- device helpers shared by the sm_100a kernels of libtls.so.
//
// Nothing here is shared with oracle/ (the fp64 CPU oracle is independent).
#pragma once

#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tls {

namespace cg = cooperative_groups;

constexpr int kThreads = 256;  // every kernel of the decode path runs 8 warps
constexpr int kWarps = kThreads / 32;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// ---------------------------------------------------------------- element I/O
template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// 16-byte streaming load that does not allocate in L1 (data read once).
__device__ __forceinline__ uint4 ldg_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Unpack 16 bytes holding EPC = 16/sizeof(T) elements into fp32.
template <typename T>
__device__ __forceinline__ void unpack16(const uint4& v, float* out);
template <>
__device__ __forceinline__ void unpack16<float>(const uint4& v, float* out) {
  out[0] = __uint_as_float(v.x);
  out[1] = __uint_as_float(v.y);
  out[2] = __uint_as_float(v.z);
  out[3] = __uint_as_float(v.w);
}
template <>
__device__ __forceinline__ void unpack16<__nv_bfloat16>(const uint4& v, float* out) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[2 * i] = __uint_as_float(w[i] << 16);
    out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

// ------------------------------------------------------- order-preserving keys
// Map fp32 -> uint32 so that unsigned comparison equals float comparison;
// -0 is canonicalised to +0 (they tie, as in the fp64 oracle).  Key 0 is
// reserved for "not a candidate" (it is below the key of -inf).
__device__ __forceinline__ uint32_t f2key(float f) {
  f = f + 0.0f;
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// ------------------------------------------------------------ warp / block ops
__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Exclusive scan of one int per thread over the CTA (kThreads threads);
// `scratch` holds >= kWarps + 1 ints.  Returns the exclusive prefix; the CTA
// total is written to *total.  Contains __syncthreads().
__device__ __forceinline__ int block_exclusive_scan(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kWarps ? scratch[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kWarps) scratch[lane] = wi - w;
    if (lane == kWarps - 1) scratch[kWarps] = wi;
  }
  __syncthreads();
  int res = scratch[warp] + inc - v;
  *total = scratch[kWarps];
  __syncthreads();
  return res;
}

// ------------------------------------------------------------------ clusters
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// Address of `p` (a shared-memory variable of this CTA) in CTA `rank` of the cluster.
template <typename P>
__device__ __forceinline__ P* dsmem(P* p, unsigned rank) {
  return cg::this_cluster().map_shared_rank(p, rank);
}

// ------------------------------------------------------------- tensor cores
// Legacy warp-level mma (m16n8k16, bf16 in, fp32 accumulate): D = A*B + D.
__device__ __forceinline__ void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// INT4 nibble pairs -> bf16x2 holding exact integers 0..15.  With
// w = 8 nibbles n0..n7 (n_i = bits 4i..4i+3), nib2bf16(w, s) returns
// bf16x2(n_s, n_{s+4}) for s in 0..3, via the magic 0x4300 (= 128.0 bf16,
// whose last mantissa bit is 1): (0x4300 | n) - 128 = n exactly.
__device__ __forceinline__ uint32_t nib2bf16(uint32_t w, int s) {
  uint32_t x = ((w >> (4 * s)) & 0x000f000fu) | 0x43004300u;
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&x);
  const __nv_bfloat162 magic = __halves2bfloat162(__ushort_as_bfloat16(0x4300), __ushort_as_bfloat16(0x4300));
  v = __hsub2(v, magic);
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace tls

namespace tls {
// ------------------------------------------------------ async copies / ldmatrix
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte global -> shared copy; zero-fills the destination when !valid.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void ldsm_x4(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
}  // namespace tls

namespace tls {
// ------------------------------------------------- mbarrier + TMA bulk copies
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// TMA 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completion counted in bytes on `bar`.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace tls

namespace tls {
// Hardware MUFU approximations (flush-to-zero): relative error ~2^-22, far
// below the parity tolerances, and one instruction each instead of the
// accurate library expansions (exp2f's denormal fix-up, log2f's polynomial).
__device__ __forceinline__ float fexp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float flog2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
}  // namespace tls

namespace tls {
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
}  // namespace tls

namespace tls {
// (a & b) | c in one LOP3 (b, c in registers).
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// Unpack one 32-bit word of 8 INT4 codes n0..n7 into 4 bf16x2 registers
// (n_s, n_{s+4}), s = 0..3, each an exact integer 0..15 (see nib2bf16).
__device__ __forceinline__ void unpack_nibbles8(uint32_t w, uint32_t (&out)[4]) {
  const uint32_t mask = 0x000f000fu, magic = 0x43004300u;
  const __nv_bfloat162 m128 = __halves2bfloat162(__ushort_as_bfloat16(0x4300), __ushort_as_bfloat16(0x4300));
  uint32_t x[4];
  x[0] = lop3_and_or(w, mask, magic);
  x[1] = lop3_and_or(w >> 4, mask, magic);
  x[2] = lop3_and_or(w >> 8, mask, magic);
  x[3] = lop3_and_or(w >> 12, mask, magic);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 v = __hsub2(*reinterpret_cast<__nv_bfloat162*>(&x[i]), m128);
    out[i] = *reinterpret_cast<uint32_t*>(&v);
  }
}
}  // namespace tls

namespace tls {
// Prefetch the 128-byte line holding p into L2 (LSU path; no wait).
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}
// GPU-scope acquire load / relaxed store of a 32-bit flag.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Stage hand-off between the decode-step kernels, which may overlap under
// programmatic dependent launch: thread 0 waits (acquire) until the producer
// published `epoch` for this pair, then orders the async proxy (TMA reads of
// the producer's outputs) after it.  A missing producer traps after ~2 s
// instead of hanging.
__device__ __forceinline__ void wait_ready(const unsigned* flag, unsigned epoch) {
  unsigned spins = 0;
  while (ld_acquire_gpu(flag) != epoch) {
    __nanosleep(128);
    if (++spins > (1u << 24)) __trap();
  }
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
// The same for a per-pair completion count (>= n: done; a count above n --
// e.g. an uninitialised workspace -- is accepted rather than waited on).
__device__ __forceinline__ void wait_count(const unsigned* ctr, unsigned n) {
  unsigned spins = 0;
  while (ld_acquire_gpu(ctr) < n) {
    __nanosleep(128);
    if (++spins > (1u << 24)) __trap();
  }
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
// Let the next kernel in the stream (launched with programmatic stream
// serialization) start its CTAs; its data dependences go through wait_ready.
__device__ __forceinline__ void launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
// TMA bulk prefetch of [src, src + bytes) into L2 (no shared memory, no wait).
__device__ __forceinline__ void tma_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
}  // namespace tls

namespace tls {
// Fixed binning of a ranking key f = log2 alpha~ + log2 G <= log2 G < 6:
// bin 0 holds the largest keys; bins are 1/16 log2 unit wide; monotone
// non-increasing in f (the same fp32 ops everywhere it is evaluated).
__device__ __forceinline__ int key_bin(float f) {
  const float x = (6.0f - f) * 16.0f;
  return x < 0.f ? 0 : (x >= 1023.f ? 1023 : (int)x);
}
}  // namespace tls
