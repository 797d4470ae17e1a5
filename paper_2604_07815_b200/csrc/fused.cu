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

// ---------------------------------------------------------------------------
// Streaming form of a1 + a2 (bf16 GQA, d_k = 128: 512-byte summary rows) -- OPT-IN (TLS_STREAM_SEL=1):
// measured slower than the tile-per-CTA select_kernel (C3 serialised a1+a2 115 vs 58 us; overlapped step 180 vs
// 128 us: one streamer CTA per SM sustains ~1.4 us per 28 KB stage, ~3 TB/s).
// one persistent CTA per SM streams the block summaries through a ring of
// kRing TMA stages (tb rows each), so that the HBM stream needs one CTA slot
// per SM instead of six and the token kernel -- launched as this kernel's PDL
// secondary, released at once because every streamer starts immediately --
// runs on the other slots while a1 is still streaming.
// Placement: 2 x #SM CTAs are launched (at most two fit an SM by shared
// memory, so every SM receives two); the first to arrive on an SM (per-SM
// word, the call's epoch) streams, the other exits at once and leaves its slot
// to the token kernel.  (148 CTAs alone were packed two per SM onto 75 SMs.)
// Warp specialisation: warp 7 lane 0 produces, warps 0-6 consume.  The
// producer claims tiles from one counter (one claim ahead: each atomic's value
// is read one tile later), waits until a stage is empty (mbarrier, one arrival
// per consumer warp), records the ticket in the stage's slot and issues the
// tile's copies (one TMA bulk copy + mbarrier per 8-row group).  Consumer warp
// w scores row group w of each tile (s_i = Q+ . k^max_i + Q- . k^min_i, P:99
// via P:110 and linearity of sum_h) and arrives on the stage's empty barrier;
// it never waits for the producer's bookkeeping (a per-tile CTA barrier held
// every tile behind it: 2.4 us per 28 KB tile).
// Completion: when a stage comes back empty the producer counts its tile in
// the pair's count of scored tiles (a hint; the scores themselves, against
// the sentinel, are the data).  The CTA that claimed a pair's last tile (by
// index) owns its a2; once the count is complete the producer posts an a2
// marker into the next stage instead of a tile, and when the consumers reach
// it (in ring order) all eight warps run pair_worker together while
// the other stages' copies are in flight.  No CTA waits for another while
// tiles remain, so the streams never fall into lockstep (a "last tile waits
// for the others" rule: 331 us per a1 at C3) and the a2 work does not pile up
// on the slowest CTA (a "last to count runs a2" rule: 412 us).
constexpr int kRing = 4;
constexpr int kPend = 16;          // pending a2 pairs per streamer
constexpr int kEnd = -1;           // stage slot: no more tiles
constexpr int kSkip = -0x7fffffff;  // stage slot: nothing (the producer waits for a2 counts without blocking)

__device__ __forceinline__ void red_relaxed_add_gpu(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 4) stream_select_kernel(const __grid_constant__ FusedParams p) {
  extern __shared__ __align__(128) uint8_t smem[];  // [kRing][tb rows][row] | the a2 worker regions
  __shared__ __align__(8) uint64_t bars[kRing];      // full[stage]: the tile's rows and its pair's QQ landed
  __shared__ __align__(16) float sqq[kRing][256];    // the tile's pair's [Q+ | Q-] per stage
  __shared__ __align__(8) uint64_t empty[kRing];     // stage consumed (kConsumers arrivals)
  __shared__ WorkerCtl ctl;
  __shared__ int s_tick[kRing], s_role;
  launch_dependents();  // the token kernel starts now, on the slots the streamers leave free
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kRow = 2 * 128 * (int)sizeof(T);
  constexpr int kCons = kWarps - 1;  // consumer warps 0..6 (tb <= 56 rows: 7 row groups)
  const int ntile = (d.M + p.tb - 1) / p.tb;
  const int total = d.batch * d.Hkv * ntile;
  unsigned* next = p.sched;           // tile ticket counter
  unsigned* out_ctr = p.sched + 1;    // CTAs out
  unsigned* sm_word = p.sched + 32;   // per SM: epoch of the call whose streamer it hosts
  unsigned long long* dbg = p.dbg ? p.dbg + (size_t)blockIdx.x * 256 : nullptr;  // diagnostics (TLS_DEBUG_BUF)
  struct Tile {
    int pair, tile, i0, nb, ntl, m;
  };
  auto tile_of = [&](int t) {
    Tile r;
    r.pair = t / ntile;
    r.tile = t - r.pair * ntile;
    const int b = r.pair / d.Hkv;
    const int n = min(max(p.seq_lens[b], 0), d.S);
    r.m = (n + d.B - 1) >> d.log2B;  // reading U1
    r.ntl = max(1, (r.m + p.tb - 1) / p.tb);
    r.i0 = r.tile * p.tb;
    r.nb = r.tile < r.ntl ? max(0, min(p.tb, r.m - r.i0)) : -1;  // -1: past the pair's sequence
    return r;
  };
  auto worker = [&](int pair, uint8_t* a2) {  // a2 of a pair whose every tile is scored (all 256 threads);
    // a2: the worker regions -- the stage of the a2 marker's slot, which holds no rows
    const int b = pair / d.Hkv;
    const int n = min(max(p.seq_lens[b], 0), d.S);
    const int m = (n + d.B - 1) >> d.log2B;
    uint32_t* bkeys = reinterpret_cast<uint32_t*>(a2 + p.off_bkeys);
    const unsigned* sc = reinterpret_cast<const unsigned*>(p.scores + (size_t)pair * p.sstride);
    // the scores are the data (a sentinel means not yet visible): 16-byte L2 loads, all issued before any is
    // tested (the row stride is a multiple of 4 floats), then a per-vector re-poll where a sentinel remains
    constexpr int kV = 4;  // vectors per thread per batch
    for (int v0 = 0; v0 * 4 < m; v0 += kV * kThreads) {
      uint4 v[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int vi = v0 + u * kThreads + tid;
        v[u] = vi * 4 < m ? __ldcg(reinterpret_cast<const uint4*>(sc) + vi) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int vi = v0 + u * kThreads + tid;
        if (vi * 4 >= m) continue;
        unsigned spins = 0;
        while ((v[u].x == kScoreSentinel && vi * 4 < m) || (v[u].y == kScoreSentinel && vi * 4 + 1 < m) ||
               (v[u].z == kScoreSentinel && vi * 4 + 2 < m) || (v[u].w == kScoreSentinel && vi * 4 + 3 < m)) {
          __nanosleep(64);
          if (++spins > (1u << 24)) __trap();
          v[u] = __ldcg(reinterpret_cast<const uint4*>(sc) + vi);
        }
        const unsigned w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (vi * 4 + e < m) bkeys[vi * 4 + e] = f2key(__uint_as_float(w[e]));
      }
    }
    if (tid == 0) p.tcount[pair] = 0u;  // reset for the next call (no other user left)
    __syncthreads();
    pair_worker(p, pair, m, a2, ctl.tk, nullptr);
    __syncthreads();  // the worker regions are reused by the next worker
  };
  if (tid == 0) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    s_role = atomicMax(sm_word + smid, p.epoch) < p.epoch;  // the first CTA of this call on this SM streams
    if (s_role) {
      for (int i = 0; i < kRing; ++i) mbar_init(&bars[i], 1);
      for (int i = 0; i < kRing; ++i) mbar_init(&empty[i], kCons);
      mbar_fence_init();
    }
  }
  __syncthreads();
  if (s_role) {
    if (dbg && tid == 0) dbg[0] = gtimer();
    const bool prod = tid == kCons * 32;  // warp 7 lane 0
    // ---- producer state (meaningful in the producer thread only) ----
    __shared__ int pend[kPend];  // pairs whose a2 this CTA owns, oldest first (producer only)
    int npend = 0;
    unsigned seen = 0u;          // the count of pend[0] as read one slot earlier (a hint)
    unsigned eph = 0u;           // empty barriers' phase parities
    unsigned ahead = 0u;         // the ticket claimed one slot ahead
    bool tickets = true, ended = false;
    if (prod) ahead = atomicAdd(next, 1u);
    // post slot j into stage j % kRing: a tile ticket (>= 0), an a2 marker (-2 - pair) or the end (-1)
    auto post_slot = [&](int j) {
      const int st = j % kRing;
      if (j >= kRing) {  // the stage's previous slot is consumed
        mbar_wait(&empty[st], (eph >> st) & 1u);
        eph ^= 1u << st;
      }
      if (ended) return;
      // never block here: a pending pair's tiles may sit in this CTA's own ring, unconsumed
      int post = kEnd;
      for (;;) {
        if (npend > 0) {
          const int pair = pend[0];
          const int m = (min(max(p.seq_lens[pair / d.Hkv], 0), d.S) + d.B - 1) >> d.log2B;
          const unsigned need = (unsigned)max(1, (m + p.tb - 1) / p.tb);
          if (seen >= need) {
            post = -2 - pair;
            for (int i = 1; i < npend; ++i) pend[i - 1] = pend[i];
            --npend;
            seen = 0u;
            break;
          }
        }
        if (tickets && npend < kPend && ahead < (unsigned)total) {
          post = (int)ahead;
          ahead = atomicAdd(next, 1u);
          const Tile r = tile_of(post);
          if (r.nb >= 0 && r.tile == r.ntl - 1) pend[npend++] = r.pair;  // this CTA owns the pair's a2
          break;
        }
        if (ahead >= (unsigned)total) tickets = false;
        if (npend > 0) {  // a count not complete yet: a skip slot (the consumers pass it) and look again
          post = kSkip;
          __nanosleep(200);
        }
        break;  // (npend == 0 and no tickets: the end)
      }
      s_tick[st] = post;
      if (post >= 0) {
        const Tile r = tile_of(post);
        if (r.nb > 0) {  // one bulk copy of the rows and one of the pair's QQ (qq_kernel) per stage
          const uint8_t* src =
              reinterpret_cast<const uint8_t*>(p.block_minmax) + ((size_t)r.pair * d.M + r.i0) * kRow;
          mbar_arrive_expect_tx(&bars[st], (uint32_t)(r.nb * kRow + 2 * 128 * 4));
          tma_bulk_g2s(smem + (size_t)st * p.tb * kRow, src, (uint32_t)(r.nb * kRow), &bars[st]);
          tma_bulk_g2s(sqq[st], p.qq + (size_t)r.pair * 2 * 128, 2 * 128 * 4, &bars[st]);
        } else {
          mbar_arrive(&bars[st]);  // no rows: the slot is posted
        }
      } else {
        mbar_arrive(&bars[st]);  // an a2 marker, a skip or the end
        if (post == kEnd) ended = true;
      }
      if (npend > 0) seen = ld_relaxed_gpu(p.tcount + pend[0]);  // look again at the next slot
    };
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // QQ, q fragments, zeroed histograms (qq_kernel)
    if (prod)
      for (int j = 0; j < kRing - 1; ++j) post_slot(j);
    unsigned cph = 0u;  // consumers: full barriers' phase parities (the same in every consumer thread)
    for (int k = 0;; ++k) {
      const int st = k % kRing;
      if (warp == kCons) {  // the producer posts slot k + kRing - 1 (its stage held slot k - 1)
        if (prod) post_slot(k + kRing - 1);
        __syncwarp();
      }
      if (dbg && tid == 0 && k < 60) dbg[8 + 4 * k] = gtimer();
      mbar_wait(&bars[st], (cph >> st) & 1u);  // slot k is posted (and its rows and QQ landed)
      cph ^= 1u << st;
      const int t = s_tick[st];
      if (t == kEnd) break;
      if (t < 0) {  // an a2 marker or a skip
        if (warp < kCons) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (t != kSkip) worker(-2 - t, smem + (size_t)st * p.tb * kRow);  // ===== a2: all eight warps =====
        continue;
      }
      const Tile r = tile_of(t);
      const int ngrp = r.nb > 0 ? (r.nb + 7) >> 3 : 0;
      if (warp < ngrp) {
        float qreg[8];
        {
          const float4 qa = reinterpret_cast<const float4*>(sqq[st])[lane * 2];
          const float4 qb = reinterpret_cast<const float4*>(sqq[st])[lane * 2 + 1];
          qreg[0] = qa.x, qreg[1] = qa.y, qreg[2] = qa.z, qreg[3] = qa.w;
          qreg[4] = qb.x, qreg[5] = qb.y, qreg[6] = qb.z, qreg[7] = qb.w;
        }
        if (dbg && tid == 0 && k < 60) dbg[9 + 4 * k] = gtimer();
        const uint8_t* tile = smem + (size_t)st * p.tb * kRow;
        const int r8 = warp * 8;
        float acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc[u] = 0.f;
          if (r8 + u < r.nb) {
            float f[8];
            unpack16<T>(reinterpret_cast<const uint4*>(tile + (size_t)(r8 + u) * kRow)[lane], f);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[u] = fmaf(qreg[e], f[e], acc[u]);
          }
        }
        // transposed butterfly: lanes 4u..4u+3 end with the dot product of row u
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
        if ((lane & 3) == 0 && r8 + u < r.nb) p.scores[(size_t)r.pair * p.sstride + r.i0 + r8 + u] = acc[0];
      }
      if (warp < kCons) {
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty[st]);  // this warp is done with the stage
          if (warp == 0 && r.nb >= 0) red_relaxed_add_gpu(p.tcount + r.pair, 1u);  // count the tile (hint)
        }
      }
    }
    if (dbg && tid == 0) {
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      dbg[1] = gtimer();
      dbg[2] = smid;
    }
  }
  if (tid == 0 && atomicAdd(out_ctr, 1u) == gridDim.x - 1) {  // the last CTA out resets the counters
    *next = 0u;
    *out_ctr = 0u;
  }
}

cudaError_t launch_stream_select(const FusedParams& p, int grid, cudaStream_t st, const LaunchOpts& o) {
  auto kern = stream_select_kernel<__nv_bfloat16>;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, false);
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3((unsigned)grid), kThreads, p.smem_bytes, st, o, 0, p);
}

// The worker regions use the stage of the a2 marker's slot, so they must fit one stage.
size_t stream_select_smem(int tb, size_t worker_bytes) {
  return worker_bytes <= (size_t)tb * 512 ? (size_t)kRing * tb * 512 : 0;
}

// Per-pair query-side work once per call: QQ = [Q+ | Q-] (fp32, P:110 +
// linearity of sum_h), so that the ceil(M / tb) tile CTAs of a pair do not each
// re-read the pair's G query rows (MLA: 32 x 576 bf16 per tile), and the token
// kernel's q~ fragment blob and zeroed key histogram, off the selection
// worker's critical path.  select_kernel, launched as its PDL secondary, issues
// its tile copies before waiting for it.
// WIDE (G > 16, e.g. MLA's 32 heads): every head's loads in flight at once; the narrow form keeps 40 registers,
// because qq_kernel co-runs with the select tiles (PDL) and its registers come out of theirs.
template <typename T, bool WIDE>
__global__ void __launch_bounds__(kThreads) qq_kernel(const __grid_constant__ FusedParams p) {
  launch_dependents();
  const Dims& d = p.d;
  const int pair = blockIdx.x, b = pair / d.Hkv, g = pair - b * d.Hkv;
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * d.Hq + (size_t)g * d.G) * d.d_k;
  float* qq = p.qq + (size_t)pair * 2 * d.d_k;
  if (WIDE && sizeof(T) == 2 && (d.d_k & 1) == 0) {
    // bf16: two columns per thread, the loads of up to 32 heads in flight at once (one round trip per 32 heads;
    // a per-head loop of dependent batches cost ~12 round trips at G = 32: MLA qq_kernel 18 us)
    // grid.y CTAs per pair (one per n-tile of 8 heads): CTA y takes QQ column slice y and the q~ fragments of
    // n-tile y, so the latency-bound per-pair work is split four ways (the select tiles wait for the whole grid)
    const uint32_t* q2 = reinterpret_cast<const uint32_t*>(qg);
    const int nq = (int)gridDim.y / 2;  // CTAs y < nq: QQ column slices; y >= nq: the q~ fragments of n-tile y - nq
    const int half = d.d_k >> 1, per = (half + nq - 1) / nq;
    const int cend = (int)blockIdx.y < nq ? min(half, per * ((int)blockIdx.y + 1)) : 0;
    for (int c = per * (int)blockIdx.y + threadIdx.x; c < cend; c += kThreads) {
      float qp0 = 0.f, qn0 = 0.f, qp1 = 0.f, qn1 = 0.f;
      for (int h0 = 0; h0 < d.G; h0 += 32) {
        uint32_t v[32];
#pragma unroll
        for (int h = 0; h < 32; ++h) v[h] = h0 + h < d.G ? __ldg(q2 + (size_t)(h0 + h) * half + c) : 0u;
#pragma unroll
        for (int h = 0; h < 32; ++h) {  // in head order: the same fp32 sums as the per-column loop
          if (h0 + h < d.G) {
            const float a = __uint_as_float(v[h] << 16), b2 = __uint_as_float(v[h] & 0xffff0000u);
            qp0 += fmaxf(a, 0.f);
            qn0 += fminf(a, 0.f);
            qp1 += fmaxf(b2, 0.f);
            qn1 += fminf(b2, 0.f);
          }
        }
      }
      qq[2 * c] = qp0;
      qq[2 * c + 1] = qp1;
      qq[d.d_k + 2 * c] = qn0;
      qq[d.d_k + 2 * c + 1] = qn1;
    }
  } else {
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
  }
  // the token kernel's inputs that do not depend on the scores: the pair's q~ fragments
  // and a zeroed key histogram
  const int ntl = gridDim.y > 1 ? (int)blockIdx.y - (int)gridDim.y / 2 : 0;  // this CTA's n-tile (split form)
  if (gridDim.y > 1 && ntl < 0) return;  // a QQ slice CTA
  __shared__ float qc[4 * 8 * 128];  // NT * 8 * d_c <= 4096
  __shared__ int s_ch[128];          // the channel ids staged once (the q~ gathers below index by them)
  for (int c = threadIdx.x; c < d.d_c; c += kThreads) s_ch[c] = p.channels[(size_t)g * d.d_c + c];
  __syncthreads();
  build_qfrag<WIDE ? 16 : 8>(d, qg, s_ch, p.qfrag, pair, qc, ntl, gridDim.y > 1 ? ntl + 1 : 4);
  if (ntl == 0)
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
  const bool wide = p.d.G > 16;
  auto kern = p.d.bf16 ? (wide ? qq_kernel<__nv_bfloat16, true> : qq_kernel<__nv_bfloat16, false>)
                       : (wide ? qq_kernel<float, true> : qq_kernel<float, false>);
  // wide bf16: one CTA per n-tile of 8 heads (the fp32 / narrow forms: one CTA per pair)
  const unsigned ny = (wide && p.d.bf16 && (p.d.d_k & 1) == 0) ? 2u * ((p.d.G + 7) / 8 <= 2 ? 2u : 4u) : 1u;
  return launch_ex(kern, dim3((unsigned)(p.d.batch * p.d.Hkv), ny), kThreads, 0, st, o, 0, p);
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
