// fused.cu -- the selection kernel of the decode step for sm_100a:
//
//   select_kernel<T, CPL, MODE>, grid (ceil(M / tb), pairs), launched
//   pair-major (blockIdx.x fastest):
//     phase S (every CTA)  a1  s_i = Q+ . k^max_i + Q- . k^min_i over one tile
//                              of <= 32 KB of the pair's block summaries (P:99
//                              via the P:110 identity and linearity of sum_h):
//                              an HBM-streaming GEMV, fp32 scores -> workspace
//     completion           every tile CTA but the pair's last publishes a
//                              flag; the last one (the pair's worker) waits for
//                              them -- only earlier-dispatched CTAs
//     worker (MODE == 1)   a2  M_t = top-k_b blocks, ascending, -1
//                              padded, plus the q-fragment blob and a zeroed key
//                              histogram for the token kernel (select.cu)
//   MODE 0 (tls_block_scores) stops after phase S.
//
// Why the worker lives here: the top-k_b of early pairs runs while later
// pairs' tiles still stream from HBM, instead of as a separate serial launch.
// (A variant that also ran a3-a4 in the worker was measured and dropped: one
// CTA per pair is issue-bound on the token scoring -- ~90 us per pair at C3,
// DESIGN.md §5.)
//
// Citation key: P:n = line n of PAPER.md.  Readings U1..U20: DESIGN.md §3.
#include <math_constants.h>

#include "common.cuh"
#include "fasttopk.cuh"
#include "launch.h"
#include "params.h"
#include "token.cuh"
#include "topk.cuh"
#include "tokensel.cuh"

namespace tls {

// One tile of a1: rows [i0, i0 + nb) of the pair's block summaries.  One
// thread streams the tile into shared memory with one TMA bulk copy per 8-row
// group (each completing on its own single-use mbarrier); warp w scores group
// w as soon as it lands (8 dot products reduced by a transposed butterfly).
// QQ = [Q+ | Q-] (2*d_k fp32), so s_i = QQ . row_i: 1 flop per byte.
template <typename T, int CPL>
__device__ __forceinline__ void score_tile(const FusedParams& p, int pair, int b, int g, int i0, int nb, uint8_t* tile,
                                           float* QQ, uint64_t* bars) {
  constexpr int EPC = 16 / sizeof(T);
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ngrp = (nb + 7) >> 3;
  const int rowbytes = 2 * d.d_k * (int)sizeof(T);
  const uint8_t* src = reinterpret_cast<const uint8_t*>(p.block_minmax) + ((size_t)pair * d.M + i0) * rowbytes;
  if (tid == 0) {
    for (int s = 0; s < ngrp; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
    for (int s = 0; s < ngrp; ++s) {
      const int rows = min(8, nb - 8 * s);
      mbar_arrive_expect_tx(&bars[s], (uint32_t)(rows * rowbytes));
      tma_bulk_g2s(tile + (size_t)s * 8 * rowbytes, src + (size_t)s * 8 * rowbytes, (uint32_t)(rows * rowbytes),
                   &bars[s]);
    }
  }
  if (p.qq != nullptr && !p.qq_local) {
    // QQ of the pair from qq_kernel (PDL primary): the tile copies above are already in flight
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const float* qq = p.qq + (size_t)pair * 2 * d.d_k;
    constexpr int NQ = (32 * CPL * EPC + kThreads - 1) / kThreads;  // QQ holds <= 32 * CPL * EPC floats
    float v[NQ];  // loads batched ahead of the stores (no aliasing chain)
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int c = u * kThreads + tid;
      v[u] = c < 2 * d.d_k ? __ldcg(qq + c) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int c = u * kThreads + tid;
      if (c < 2 * d.d_k) QQ[c] = v[u];
    }
  } else {
    const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * d.Hq + (size_t)g * d.G) * d.d_k;
    for (int c = tid; c < d.d_k; c += kThreads) {
      float qp = 0.f, qn = 0.f;
#pragma unroll 8
      for (int h = 0; h < d.G; ++h) {
        const float v = to_f32<T>(qg[(size_t)h * d.d_k + c]);
        qp += fmaxf(v, 0.f);
        qn += fminf(v, 0.f);
      }
      QQ[c] = qp;
      QQ[d.d_k + c] = qn;
    }
  }
  __syncthreads();  // QQ ready, barriers initialised
  const int nchunk = rowbytes / 16;
  float* out = p.scores + (size_t)pair * p.sstride + i0;
  if constexpr (CPL > 1) {  // wide rows (fp32, MLA): one row per warp step, rows w, w+8, ...
    float qreg[CPL][EPC];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int ch = lane + 32 * c;
#pragma unroll
      for (int e = 0; e < EPC; e += 4) {  // 16-byte loads
        const float4 v = ch < nchunk ? *reinterpret_cast<const float4*>(QQ + ch * EPC + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        qreg[c][e] = v.x;
        qreg[c][e + 1] = v.y;
        qreg[c][e + 2] = v.z;
        qreg[c][e + 3] = v.w;
      }
    }
    for (int r = warp; r < nb; r += kWarps) {
      mbar_wait(&bars[r >> 3], 0);
      const uint4* row = reinterpret_cast<const uint4*>(tile + (size_t)r * rowbytes);
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
      if (lane == 0) out[r] = acc;
    }
    return;
  }
  for (int gq = warp; gq < ngrp; gq += kWarps) {
    float qreg[CPL][EPC];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int ch = lane + 32 * c;
#pragma unroll
      for (int e = 0; e < EPC; ++e) qreg[c][e] = ch < nchunk ? QQ[ch * EPC + e] : 0.f;
    }
    mbar_wait(&bars[gq], 0);
    const int r8 = gq * 8;
    float acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc[u] = 0.f;
      if (r8 + u < nb) {
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
    if ((lane & 3) == 0 && r8 + u < nb) out[r8 + u] = acc[0];
  }
}

// Completion sentinel of the block-score buffer (all-ones bits: a NaN that no
// arithmetic produces; set by tls_workspace_init, restored by every worker).
constexpr uint32_t kScoreSentinel = 0xffffffffu;

// The pair's selection worker (a2): M_t = top-k_b blocks from the pair's
// scores (already converted to keys in smem at off_bkeys), ties -> lower block
// id (U2), written ascending and -1 padded; the scores go back to the sentinel
// and the pair's hand-off flag is published.  Every thread of the CTA calls it; smem holds the worker regions of
// plan_fused.
__device__ __noinline__ void pair_worker(const FusedParams& p, int pair, int m, uint8_t* smem,
                                         TopKCtl& tk, unsigned long long* dbg) {
  const Dims& d = p.d;
  const int tid = threadIdx.x;
#define TLS_STAMP(i) \
  if (dbg && tid == 0) dbg[i] = gtimer();
  uint32_t* bkeys = reinterpret_cast<uint32_t*>(smem + p.off_bkeys);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + p.off_scratch);
  FastTopKCtl& fk = *reinterpret_cast<FastTopKCtl*>(smem + p.off_fk);
  // the hand-off below also certifies qq_kernel's outputs (q fragments, zeroed histogram): when the tile CTAs
  // did not wait for it, the worker does (it has long finished by now)
  if (p.qq != nullptr && p.qq_local) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  TLS_STAMP(3)
  // ---- a2: M_t = top-k_b blocks, ties -> lower block id (U2), ascending ----
  const int K = min(d.Kb, m);
  {
    int* bout = p.block_ids + (size_t)pair * d.Kb;
    __shared__ HistSel hs;
    // one-pass register select (value-linear histogram); else / on an oversized boundary bin the generic
    // range-histogram select (the sample-bracket path measured 2x slower on 1.5k scores)
    bool done = false;
    constexpr int kBlkChunks = 2;  // <= 8 keys per thread (m <= 2048 blocks) within the kernel register budget
    if (K < m && m <= 4 * kBlkChunks * kThreads)
      done = range_topk_select<kBlkChunks>(bkeys, m, K, scratch, fk, tk, hs, [&](int i, int pos) { bout[pos] = i; });
    TLS_STAMP(4)
    if (!done) {
      const TopK t = fast_topk(bkeys, m, K, d.Kb >= m, fk, tk, nullptr);
      topk_emit(bkeys, m, t, tk, [&](int i, int pos) { bout[pos] = i; });
    }
    for (int pos = K + tid; pos < d.Kb; pos += kThreads) bout[pos] = -1;
  }
  if (dbg && tid == 0) dbg[9] = gtimer();  // diagnostics: top-k_b emitted
  TLS_STAMP(1)
  __syncthreads();
  if (tid == 0)  // release store (cumulative over the CTA barrier): block_ids visible (q fragments and the
                  // zeroed histogram: qq_kernel)
    st_release_gpu(p.ready + pair, p.epoch);
  {  // then the pair's scores back to the sentinel for the next call (ordered before it by the stream; after
     // the hand-off so the fence above does not wait for these stores)
    unsigned* sc = reinterpret_cast<unsigned*>(p.scores + (size_t)pair * p.sstride);
    for (int i = tid; i < m; i += kThreads) sc[i] = kScoreSentinel;
  }
  TLS_STAMP(2)
#undef TLS_STAMP
}

struct WorkerCtl {
  TopKCtl tk;
};

// Tile-per-CTA form (fp32, d_k != 128 bf16, MLA): grid (ceil(M / tb), pairs),
// pair-major; every tile CTA but the pair's last publishes a flag, the last
// one waits for them (only earlier-dispatched CTAs) and runs pair_worker.
template <typename T, int CPL, int MODE>
__global__ void __launch_bounds__(kThreads, CPL <= 2 ? 6 : 3) select_kernel(const __grid_constant__ FusedParams p) {
  constexpr int EPC = 16 / sizeof(T);
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(16) float QQ[32 * CPL * EPC];
  __shared__ __align__(8) uint64_t bars[kWarps];
  __shared__ WorkerCtl ctl;
  const Dims& d = p.d;
  const int tid = threadIdx.x;
  const int pair = blockIdx.y;
  if constexpr (MODE != 0) launch_dependents();  // the token kernel may start as CTAs free up
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;  // reading U1
  const int i0 = blockIdx.x * p.tb;
  if (i0 >= m && !(m == 0 && blockIdx.x == 0)) return;
  const unsigned long long t_cta0 = p.dbg ? gtimer() : 0ull;
  const int nb = max(0, min(p.tb, m - i0));
  const int ntiles = max(1, (m + p.tb - 1) / p.tb);  // the pair's last tile CTA is its worker
  if (nb > 0) score_tile<T, CPL>(p, pair, b, g, i0, nb, smem, QQ, bars);
  if constexpr (MODE == 0) return;
  if ((int)blockIdx.x != ntiles - 1) return;  // the scores themselves signal completion (sentinel)
  // ===== the pair's selection worker (the tile buffer is dead from here on) =====
  __syncthreads();  // this CTA's own scores stored
  unsigned long long* dbg = p.dbg ? p.dbg + (size_t)pair * 16 : nullptr;
  if (dbg && tid == 0) {
    dbg[6] = t_cta0;
    dbg[8] = gtimer();  // own tile scored
  }
  // wait for every tile's scores: the buffer holds the sentinel between calls, and the values are
  // the data, so relaxed L2 loads suffice (no flags, no fences in the tile CTAs)
  {
    uint32_t* bkeys = reinterpret_cast<uint32_t*>(smem + p.off_bkeys);
    const unsigned* sc = reinterpret_cast<const unsigned*>(p.scores + (size_t)pair * p.sstride);
    for (int i = tid; i < m; i += kThreads) {
      unsigned v, spins = 0;
      while ((v = ld_relaxed_gpu(sc + i)) == kScoreSentinel) {
        __nanosleep(100);
        if (++spins > (1u << 24)) __trap();
      }
      bkeys[i] = f2key(__uint_as_float(v));
    }
    __syncthreads();
  }
  if (dbg && tid == 0) dbg[0] = gtimer();
  pair_worker(p, pair, m, smem, ctl.tk, dbg);
}

// Per-pair query-side work once per call: QQ = [Q+ | Q-] (fp32, P:110 +
// linearity of sum_h), so that the ceil(M / tb) tile CTAs of a pair do not each
// re-read the pair's G query rows (MLA: 32 x 576 bf16 per tile), and the token
// kernel's q~ fragment blob and zeroed key histogram, off the selection
// worker's critical path.  select_kernel, launched as its PDL secondary, issues
// its tile copies before waiting for it.
template <typename T>
__global__ void __launch_bounds__(kThreads) qq_kernel(const __grid_constant__ FusedParams p) {
  launch_dependents();
  const Dims& d = p.d;
  const int pair = blockIdx.x, b = pair / d.Hkv, g = pair - b * d.Hkv;
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * d.Hq + (size_t)g * d.G) * d.d_k;
  float* qq = p.qq + (size_t)pair * 2 * d.d_k;
  for (int c = threadIdx.x; c < d.d_k; c += kThreads) {
    float qp = 0.f, qn = 0.f;
#pragma unroll 8
    for (int h = 0; h < d.G; ++h) {  // read-only loads: batched ahead of the stores below
      const float v = to_f32<T>(__ldg(qg + (size_t)h * d.d_k + c));
      qp += fmaxf(v, 0.f);
      qn += fminf(v, 0.f);
    }
    qq[c] = qp;
    qq[d.d_k + c] = qn;
  }
  // the token kernel's inputs that do not depend on the scores: the pair's q~ fragments
  // and a zeroed key histogram
  __shared__ float qc[4 * 8 * 128];  // NT * 8 * d_c <= 4096
  const int* ch = p.channels + (size_t)g * d.d_c;
  build_qfrag(d, qg, ch, p.qfrag, pair, qc);
  for (int i = threadIdx.x; i < kKeyBins; i += kThreads) p.khist[(size_t)pair * kKeyBins + i] = 0u;
}

// ============================================================== launchers
int score_cpl(int d_k, size_t elem_bytes) {
  const int nchunk = (int)(2 * d_k * elem_bytes / 16);
  if (nchunk <= 32) return 1;
  if (nchunk <= 64) return 2;
  if (nchunk <= 160) return 5;
  return -1;
}

template <typename T, int CPL, int MODE>
static cudaError_t launch_sel(const FusedParams& p, cudaStream_t st, const LaunchOpts& o) {
  auto kern = select_kernel<T, CPL, MODE>;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, false);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((p.d.M + p.tb - 1) / p.tb), (unsigned)(p.d.batch * p.d.Hkv), 1);
  return launch_ex(kern, grid, kThreads, p.smem_bytes, st, o, 0, p);
}

template <typename T, int CPL>
static cudaError_t dispatch_sel(const FusedParams& p, cudaStream_t st, const LaunchOpts& o) {
  if (p.mode == 0) return launch_sel<T, CPL, 0>(p, st, o);
  return launch_sel<T, CPL, 1>(p, st, o);
}

cudaError_t launch_qq(const FusedParams& p, cudaStream_t st, const LaunchOpts& o) {
  auto kern = p.d.bf16 ? qq_kernel<__nv_bfloat16> : qq_kernel<float>;
  return launch_ex(kern, dim3((unsigned)(p.d.batch * p.d.Hkv)), kThreads, 0, st, o, 0, p);
}

cudaError_t launch_select_fused(const FusedParams& p, cudaStream_t st, const LaunchOpts& o) {
  const int cpl = score_cpl(p.d.d_k, p.d.bf16 ? 2 : 4);
  if (p.d.bf16) {
    if (cpl == 1) return dispatch_sel<__nv_bfloat16, 1>(p, st, o);
    if (cpl == 2) return dispatch_sel<__nv_bfloat16, 2>(p, st, o);
    return dispatch_sel<__nv_bfloat16, 5>(p, st, o);
  }
  if (cpl == 1) return dispatch_sel<float, 1>(p, st, o);
  if (cpl == 2) return dispatch_sel<float, 2>(p, st, o);
  return dispatch_sel<float, 5>(p, st, o);
}

}  // namespace tls
