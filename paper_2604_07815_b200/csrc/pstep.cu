// pstep.cu -- the decode step of AsyncTLS (arXiv 2604.07815) as ONE
// persistent kernel with a ticket-ordered work queue, for sm_100a.
//
// Why: the four steps of a pair are a chain of latency-bound stages (two
// exact top-k selections, a softmax normalisation over the pair's candidates)
// between HBM streams.  A kernel per stage can only start once every CTA of
// the previous one has started (the PDL release point), so the stages of the
// step run one after another; one cluster per pair (all four steps in shared
// memory) exposes the whole chain per pair with too few pairs in flight
// (measured: 254 us at C3).  Here every SM runs a few resident
// CTAs that claim work items ("tickets") from one global counter, in an order
// that interleaves the stages of different pairs: while one CTA waits for a
// pair's top-k, the others stream block summaries, token index or K/V rows of
// other pairs.
//
// Work items (one CTA each) per pair p (= (b, g), the independent unit,
// P:118):
//   TILE(p, t)   a1  s_i = Q+ . k^max_i + Q- . k^min_i (P:99 via P:110 and
//                    linearity of sum_h) over tb rows of block summaries (TMA
//                    bulk copies into shared memory, one GEMV dot per row) ->
//                    fp32 scores (workspace, L2).  The pair's last finishing
//                    tile runs a2: M_t = top-k_b blocks, ties -> lower
//                    block id (U2), and publishes it.
//   TOKEN(p, c)  a3  alpha~ over the tokens of candidate blocks
//                    [c cb, (c+1) cb) of M_t (or of the lag-mode guide):
//                    INT4 index staged by TMA, logits on tensor cores
//                    (mma.sync codes x q~), chunk softmax statistics published,
//                    the pair's nch chunks' statistics merged (lz_h), ranking
//                    keys log2 sum_h 2^(L_hj - lz_h) (reading U15) + their
//                    fixed-bin histogram -> workspace.
//   SEL(p)       a4  S_t = top-k_t tokens, ties -> lower token id:
//                    the keys and the histogram by TMA, the register select of
//                    tokensel.cuh; token_ids / token_scores / num_tokens.
//   ATT(p, s)    a5  attention over positions [K s / ns, K (s+1) /
//                    ns) of S_t (K/V rows by cp.async, tensor cores, split-P);
//                    the pair's last finishing slice merges the ns partials
//                    (LSE identity, T10) into out / lse.
// Scheduling: TILE tickets are claimed in pair-major order from one counter;
// every other item enters a ready queue only once its inputs exist (the
// pair's a2 pushes its nch TOKEN items, the last TOKEN runs a4 and pushes the
// ns ATT items).  Each CTA holds at most one reserved queue slot (one
// atomicAdd) and streams TILE items until that slot's entry is published,
// then takes it at its next item boundary -- so no item waits for a producer
// while holding its CTA, except the nch TOKEN siblings of one pair, which
// exchange softmax statistics: a sibling's slot holder is never inside another
// TOKEN item (one reservation per CTA), so it reaches the item after at most
// one TILE.  A TILE item whose CTA has no ready item claims the next TILE
// ticket and issues its TMA copies into the second tile buffer before
// computing its own rows, so every CTA keeps two tiles of block summaries in
// flight while it streams a1.
// Per-pair counters in the workspace are reset by their last user and the
// scheduler words by the last CTA out, so each call leaves the workspace ready
// for the next one (tls_workspace_init once); queue entries carry the call's
// epoch, so entries of an earlier call are never taken for this call's.
//
// Specialisation: bf16 GQA, d_k = d_v = 128, G <= 8, d_c = 32, B = 64 (the
// BASELINE.json GQA configs).  Every other configuration runs the kernel chain
// (fused.cu, select.cu, attend.cu).
//
// Citation key: P:n = line n of PAPER.md.  Readings U1..U20: DESIGN.md §3.
#include <math_constants.h>

#include "common.cuh"
#include "fasttopk.cuh"
#include "launch.h"
#include "params.h"
#include "token.cuh"
#include "tokensel.cuh"
#include "topk.cuh"

namespace tls {

namespace {

constexpr int kD = 128;                     // head dim (d_k = d_v)
constexpr int kRowBytes = 2 * kD * 2;       // one block's [k^max | k^min] row, bf16: 512 B
constexpr int kKS = 2;                      // a3 k-steps: d_c / 16
constexpr int kTPW = 8;                     // a3 16-token tiles per warp (register-resident logits)
constexpr int kTC = 64;                     // a5 tokens per staged chunk
constexpr int kStages = 2;                  // a5 cp.async stages
constexpr float kKeyOff = 64.f;             // a3 ranking-key scale (reading U20)

enum Role : int { kTile = 0, kToken = 1, kSel = 2, kAtt = 3, kExit = 4, kA2 = 5 };

// per-pair counters (PStepParams::ctr, 8 words per pair)
enum Ctr : int { kCtrTiles = 0, kCtrStats = 1, kCtrDone = 2, kCtrAtt = 3 };
// scheduler words (PStepParams::sched)
enum Sched : int { kTileNext = 0, kCtasOut = 1, kRqHead = 2, kRqTail = 3 };  // head: next slot to reserve
constexpr int kBarsPerBuf = 8;  // TILE: one mbarrier per 8-row group of a tile buffer

__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

// thread 0 spins until *p >= v (relaxed loads: an acquire load per spin would invalidate the SM's L1 each
// time), then acquires and orders the async proxy after it.  A hand-off that never comes traps after
// ~seconds; with the diagnostics buffer set (TLS_DEBUG_BUF, host-mapped memory works), a wait still pending
// after ~2^18 spins is reported once at dbg[1 << 20 ..] (tag, observed << 32 | wanted) and keeps waiting.
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned v, unsigned long long* dbg = nullptr,
                                         unsigned long long tag = 0) {
  unsigned spins = 0;
  while (ld_relaxed_gpu(p) < v) {
    __nanosleep(128);
    if (++spins == (1u << 18) && dbg) {
      const unsigned long long slot = atomicAdd(dbg + (1 << 20), 1ull);
      if (slot < 4096) {
        dbg[(1 << 20) + 1 + 2 * slot] = tag;
        dbg[(1 << 20) + 2 + 2 * slot] = ((unsigned long long)ld_relaxed_gpu(p) << 32) | v;
        __threadfence_system();
      }
    }
    if (spins > (1u << 26)) __trap();
  }
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

struct ItemCtl {
  TopKCtl tk;
  int kc, last;
  float wm[kWarps][8], ws[kWarps][8];
  float hlz[8];
  float mw[16][8], minv[8];
};

// ---------------------------------------------------------------------------
// scheduler (thread 0 only)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned pack_item(int role, int sub, int pair) {
  return ((unsigned)role << 29) | ((unsigned)sub << 22) | (unsigned)pair;  // pair < 2^22, sub < 2^7
}
__device__ __forceinline__ void unpack_item(unsigned it, int& role, int& sub, int& pair) {
  role = (int)(it >> 29);
  sub = (int)((it >> 22) & 0x7f);
  pair = (int)(it & 0x3fffff);
}
// Items role x (sub 0 .. n-1) of `pair` enter the ready queue.  Called by thread 0 after a CTA barrier that
// follows every store the items read: the release stores are cumulative over that barrier.
__device__ __forceinline__ void push_items(const PStepParams& p, int role, int pair, int n) {
  const unsigned base = atomicAdd(p.sched + kRqTail, (unsigned)n);
  for (int i = 0; i < n; ++i)
    st_release_u64(p.rq + base + i, ((unsigned long long)p.epoch << 32) | pack_item(role, i, pair));
}
// Ready-queue slots are reserved one at a time per CTA with one atomicAdd (a CAS pop by hundreds of idle CTAs
// serialised every pop: 2.8 ms steps).  A CTA holding slot h streams TILE items until entry h is published
// and takes it at its next item boundary.  Returns true (and the item) once the entry is there.
__device__ __forceinline__ bool slot_ready(const PStepParams& p, int h, unsigned& item) {
  // relaxed poll (an acquire load per poll invalidates the SM's L1 each time), one acquire fence on success
  const unsigned long long e = *reinterpret_cast<volatile const unsigned long long*>(p.rq + h);
  if ((unsigned)(e >> 32) != p.epoch) return false;
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  asm volatile("fence.proxy.async.global;\n" ::: "memory");  // TMA reads of the producer's outputs
  item = (unsigned)e;
  return true;
}
// Claim the next TILE ticket (pair-major), -1 when they are all taken.
__device__ __forceinline__ int claim_tile(const PStepParams& p) {
  if (ld_relaxed_gpu(p.sched + kTileNext) >= (unsigned)p.ntiles_total) return -1;
  const unsigned t = atomicAdd(p.sched + kTileNext, 1u);
  return t < (unsigned)p.ntiles_total ? (int)t : -1;
}

// Rows of TILE ticket t: pair, tile, first row and row count (0: past the pair's sequence, reading U1).
struct TileRef {
  int pair, tile, i0, nb, ntiles, m;
};
__device__ __forceinline__ TileRef tile_ref(const PStepParams& p, int t) {
  TileRef r;
  r.pair = t / p.ntile;
  r.tile = t - r.pair * p.ntile;
  const int b = r.pair / p.d.Hkv;
  const int n = min(max(__ldg(p.seq_lens + b), 0), p.d.S);
  r.m = (n + p.d.B - 1) >> p.d.log2B;
  r.ntiles = max(1, (r.m + p.tb - 1) / p.tb);
  r.i0 = r.tile * p.tb;
  r.nb = r.tile < r.ntiles ? max(0, min(p.tb, r.m - r.i0)) : -1;  // -1: no such tile for this pair
  return r;
}
// Thread 0: TMA bulk copies of a tile's rows into tile buffer `buf` (one mbarrier per 8-row group).
__device__ __forceinline__ void issue_tile(const PStepParams& p, const TileRef& r, uint8_t* smem, uint64_t* bars,
                                           int buf) {
  if (p.dbg) p.dbg[(1 << 19) + 3 * (r.pair * p.ntile + r.tile)] = gtimer();  // diagnostics: issue time
  uint8_t* dst = smem + p.off_tile + (size_t)buf * p.tb * kRowBytes;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(p.block_minmax) + ((size_t)r.pair * p.d.M + r.i0) * kRowBytes;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic accesses of earlier items first
  for (int s = 0; s < (r.nb + 7) >> 3; ++s) {
    const int rows = min(8, r.nb - 8 * s);
    uint64_t* bar = &bars[buf * kBarsPerBuf + s];
    mbar_arrive_expect_tx(bar, (uint32_t)(rows * kRowBytes));
    tma_bulk_g2s(dst + (size_t)s * 8 * kRowBytes, src + (size_t)s * 8 * kRowBytes, (uint32_t)(rows * kRowBytes), bar);
  }
}

// ---------------------------------------------------------------------------
// TILES (streamer CTAs, warp-specialised): warp 0 lane 0 produces, warps 1-7
// consume.  The producer claims TILE tickets (each atomic's value is used one
// tile later), waits until a tile buffer is empty, records the ticket and
// issues the tile's TMA copies (one mbarrier per 8-row group); when a buffer
// it refills held the pair's last tile (by index), the pair's A2 item enters
// the ready queue.  Consumer warp w scores group w - 1 of each tile:
// s_i = Q+ . k^max_i + Q- . k^min_i (P:99 via P:110 and linearity of sum_h),
// then arrives on the buffer's empty barrier.  Barriers: full[b][g] = bars[8b + g],
// empty[b] = bars[16 + b] (7 arrivals).  Used once per launch: their phases
// start at 0 here.
// ---------------------------------------------------------------------------
constexpr uint32_t kScoreSentinel = 0xffffffffu;  // all-ones: a NaN no arithmetic produces
constexpr int kBarEmpty = 16, kBarTok = 18, kBarSel = 19, kNumBars = 20;
constexpr int kConsumers = kWarps - 1;

__device__ __noinline__ void run_tiles(const PStepParams& p, uint8_t* smem, uint64_t* bars, int* s_tick) {
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* QQ = reinterpret_cast<float*>(smem + p.off_qq);
  if (warp == 0) {
    if (lane == 0) {  // ---- producer
      unsigned eph = 0u;         // parity of each empty barrier's current phase
      int held[2] = {-1, -1};    // ticket whose tile sits in each buffer
      unsigned next = atomicAdd(p.sched + kTileNext, 1u);
      for (int k = 0;; ++k) {
        const int b = k & 1;
        if (k >= 2) {
          mbar_wait(&bars[kBarEmpty + b], (eph >> b) & 1u);
          eph ^= 1u << b;
        }
        const int t = next < (unsigned)p.ntiles_total ? (int)next : -1;
        if (t >= 0) next = atomicAdd(p.sched + kTileNext, 1u);
        s_tick[b] = t;
        const TileRef r = tile_ref(p, t >= 0 ? t : 0);
        if (t >= 0 && r.nb > 0) {
          issue_tile(p, r, smem, bars, b);  // arms full[b][0 .. ngrp) with the rows' bytes
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bars[8 * b])) : "memory");
        }
        if (held[b] >= 0) {  // the tile this buffer held is scored: the pair's last tile hands a2 on
          const TileRef rh = tile_ref(p, held[b]);
          if (rh.nb >= 0 && rh.tile == rh.ntiles - 1) push_items(p, kA2, rh.pair, 1);
        }
        held[b] = t;
        if (t < 0) {  // end posted into buffer b; the other buffer's tile, if any, completes last
          const int o = b ^ 1;
          if (held[o] >= 0) {
            mbar_wait(&bars[kBarEmpty + o], (eph >> o) & 1u);
            const TileRef rh = tile_ref(p, held[o]);
            if (rh.nb >= 0 && rh.tile == rh.ntiles - 1) push_items(p, kA2, rh.pair, 1);
          }
          break;
        }
      }
    }
  } else {  // ---- consumers: warp w scores row group w - 1 of each tile
    unsigned cph = 0u;  // parity of each full barrier's current phase (uniform over the consumer warps)
    int qq_pair = -1;
    for (int k = 0;; ++k) {
      const int b = k & 1;
      mbar_wait(&bars[8 * b], (cph >> (8 * b)) & 1u);  // group 0: the ticket is posted (and its rows, if any)
      const int t = s_tick[b];
      if (t < 0) break;
      const TileRef r = tile_ref(p, t);
      const int nb = r.nb, pair = r.pair;
      if (nb > 0 && pair != qq_pair) {  // QQ = [Q+ | Q-] of the pair (fp32): the head-collapsed query
        asm volatile("bar.sync 1, %0;\n" ::"r"(kConsumers * 32) : "memory");  // every warp past the old QQ
        const int b0 = pair / d.Hkv, g = pair - b0 * d.Hkv;
        const int i = tid - 32;
        if (i < kD) {
          const __nv_bfloat16* qg =
              reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b0 * d.Hq + (size_t)g * d.G) * kD;
          float qp = 0.f, qn = 0.f;
          for (int h = 0; h < d.G; ++h) {
            const float v = __bfloat162float(qg[(size_t)h * kD + i]);
            qp += fmaxf(v, 0.f);
            qn += fminf(v, 0.f);
          }
          QQ[i] = qp;
          QQ[kD + i] = qn;
        }
        qq_pair = pair;
        asm volatile("bar.sync 1, %0;\n" ::"r"(kConsumers * 32) : "memory");
      }
      const int ngrp = nb > 0 ? (nb + 7) >> 3 : 0;
      const int gq = warp - 1;
      if (gq < ngrp) {
        const uint8_t* tbuf = smem + p.off_tile + (size_t)b * p.tb * kRowBytes;
        float* out = p.scores + (size_t)pair * d.Ms + r.i0;
        float qreg[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) qreg[e] = QQ[lane * 8 + e];
        if (gq > 0) mbar_wait(&bars[8 * b + gq], (cph >> (8 * b + gq)) & 1u);
        if (p.dbg && gq == 0 && lane == 0) p.dbg[(1 << 19) + 3 * t + 1] = gtimer();  // diagnostics: rows landed
        const int r8 = gq * 8;
        float acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc[u] = 0.f;
          if (r8 + u < nb) {
            float f[8];
            unpack16<__nv_bfloat16>(reinterpret_cast<const uint4*>(tbuf + (size_t)(r8 + u) * kRowBytes)[lane], f);
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
        if ((lane & 3) == 0 && r8 + u < nb) out[r8 + u] = acc[0];
      }
      cph ^= (ngrp > 0 ? (1u << ngrp) - 1u : 1u) << (8 * b);  // the armed groups (group 0 always) consumed
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bars[kBarEmpty + b])) : "memory");
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// A2 (worker): M_t = top-k_b blocks of the pair, ties -> lower block
// id (U2).  The pair's tiles have lower tickets than the one that pushed this
// item, so they are claimed by running streamers that never wait: the scores
// still holding the sentinel arrive.  Restores the sentinel and pushes the
// pair's TOKEN items.
// ---------------------------------------------------------------------------
__device__ __noinline__ void run_a2(const PStepParams& p, int pair, uint8_t* smem, ItemCtl& ctl) {
  const Dims& d = p.d;
  const int tid = threadIdx.x;
  const int b = pair / d.Hkv;
  const int n = min(max(__ldg(p.seq_lens + b), 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;  // reading U1
  uint32_t* bkeys = reinterpret_cast<uint32_t*>(smem + p.off_bkeys);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + p.off_scratch);
  FastTopKCtl& fk = *reinterpret_cast<FastTopKCtl*>(smem + p.off_fk);
  uint32_t* sc = reinterpret_cast<uint32_t*>(p.scores + (size_t)pair * d.Ms);
  if (tid < 32) {  // one warp waits until no score of the pair is the sentinel (relaxed polls, backing off)
    unsigned spins = 0;
    for (int i = tid; i < m;) {
      if (ld_relaxed_gpu(sc + i) != kScoreSentinel) {
        i += 32;
        continue;
      }
      __nanosleep(256);
      if (++spins > (1u << 24)) __trap();
    }
    __syncwarp();
  }
  __syncthreads();
  for (int i = tid; i < m; i += kThreads) {
    bkeys[i] = f2key(__uint_as_float(ld_relaxed_gpu(sc + i)));
    sc[i] = kScoreSentinel;  // restored for the next call (no other reader of this score)
  }
  __syncthreads();
  const int K = min(d.Kb, m);
  int* bout = p.block_ids + (size_t)pair * d.Kb;
  bool done = false;
  __shared__ HistSel hs;
  if (K < m && m <= 4 * 2 * kThreads)
    done = range_topk_select<2>(bkeys, m, K, scratch, fk, ctl.tk, hs, [&](int i, int pos) { bout[pos] = i; });
  if (!done) {
    const TopK tk = fast_topk(bkeys, m, K, d.Kb >= m, fk, ctl.tk, nullptr);
    topk_emit(bkeys, m, tk, ctl.tk, [&](int i, int pos) { bout[pos] = i; });
  }
  for (int q = K + tid; q < d.Kb; q += kThreads) bout[q] = -1;
  __syncthreads();
  if (tid == 0) push_items(p, kToken, pair, p.nch);  // M_t published with the TOKEN items
}

// ---------------------------------------------------------------------------
// TOKEN: a3 over candidate blocks [c cb, (c+1) cb) of the pair (M_t is
// published: the item was pushed by the pair's a2); the pair's last finishing
// TOKEN runs a4 (run_sel) and pushes the pair's ATT items
// ---------------------------------------------------------------------------
__device__ __noinline__ unsigned run_sel(const PStepParams& p, int pair, uint8_t* smem, uint64_t* bars, unsigned bph,
                            ItemCtl& ctl);

__device__ __noinline__ unsigned run_token(const PStepParams& p, int pair, int chunk, uint8_t* smem, uint64_t* bars,
                                           unsigned bph, ItemCtl& ctl, int* ran_sel) {
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q4 = lane & 3, r0 = lane >> 2;
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int G = d.G;
  const int n = min(max(__ldg(p.seq_lens + b), 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;
  unsigned* ctr = p.ctr + (size_t)pair * 8;
  int* cblk = reinterpret_cast<int*>(smem + p.off_cblk);
  uint32_t* qb = reinterpret_cast<uint32_t*>(smem + p.off_qb);
  float* qsum = reinterpret_cast<float*>(smem + p.off_qb + kKS * 256);
  uint32_t* lhist = reinterpret_cast<uint32_t*>(smem + p.off_lhist);
  uint8_t* stc = smem + p.off_stage;
  const int rowb = d.d_c / 2;  // 16 B of codes per token
  float2* stz = reinterpret_cast<float2*>(stc + (size_t)p.cb * d.B * rowb);
  const __nv_bfloat16* qg = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b * d.Hq + (size_t)g * G) * kD;
  if (tid == 0) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // before the stage's TMA writes
  // ---- this chunk's candidate blocks: M_t (ascending, -1 padded) or the lag-mode guide's valid ids ----
  const int c0 = chunk * p.cb;
  if (p.guide == nullptr) {
    if (tid < p.cb) {
      const int k = c0 + tid;
      cblk[tid] = k < p.kb_eff ? __ldcg(p.block_ids + (size_t)pair * d.Kb + k) : -1;
    }
    __syncthreads();
    if (tid == 0) {
      int c = 0;
      while (c < p.cb && cblk[c] >= 0) ++c;
      ctl.kc = c;
    }
  } else {
    const int* gd = p.guide + (size_t)pair * d.Kb;
    const int per = (d.Kb + kThreads - 1) / kThreads;
    const int lo = min(tid * per, d.Kb), hi = min(lo + per, d.Kb);
    int cnt = 0;
    for (int i = lo; i < hi; ++i) cnt += (gd[i] >= 0 && gd[i] < m);
    int total;
    int pos = block_exclusive_scan(cnt, ctl.tk.scan, &total);
    const int kc = min(total, p.kb_eff);
    for (int i = lo; i < hi; ++i)
      if (gd[i] >= 0 && gd[i] < m) {
        if (pos >= c0 && pos < min(c0 + p.cb, kc)) cblk[pos - c0] = gd[i];
        ++pos;
      }
    if (tid == 0) ctl.kc = max(0, min(p.cb, kc - c0));
  }
  __syncthreads();
  const int nbl = ctl.kc;
  if (warp == 0) {
    if (nbl > 0) {  // stage the chunk's INT4 codes and scale/zero rows (TMA bulk, one barrier)
      const uint8_t* cbase = p.codes + (size_t)pair * d.S * rowb;
      const float2* zbase = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * d.S;
      uint32_t bytes = 0;
      for (int k = lane; k < nbl; k += 32) bytes += (uint32_t)(min(d.B, d.S - cblk[k] * d.B) * (rowb + 8));
      bytes = warp_sum_u32(bytes);
      if (lane == 0) mbar_arrive_expect_tx(&bars[kBarTok], bytes);
      __syncwarp();
      for (int k = lane; k < nbl; k += 32) {
        const int blk = cblk[k];
        const int rows = min(d.B, d.S - blk * d.B);
        tma_bulk_g2s(stc + (size_t)k * d.B * rowb, cbase + (size_t)blk * d.B * rowb, rows * rowb, &bars[kBarTok]);
        tma_bulk_g2s(stz + k * d.B, zbase + (size_t)blk * d.B, rows * 8, &bars[kBarTok]);
      }
    }
  } else {  // while the copies fly: q~ fragments and the zeroed local key histogram
    const int* ch = p.channels + (size_t)g * d.d_c;
    const int t = tid - 32;
    if (t < kKS * 32) {  // lane ln, k-step s: head ln >> 2; channels cb, cb+4 | cb+1, cb+5 (token_tile_mma order)
      const int ln = t & 31, s = t >> 5, h = ln >> 2;
      const int cc0 = 8 * (ln & 3) + 2 * s;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (h < G) {
        const int cc[4] = {cc0, cc0 + 4, cc0 + 1, cc0 + 5};
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = __bfloat162float(qg[(size_t)h * kD + __ldg(ch + cc[e])]);
      }
      qb[2 * t] = pack_bf16x2(v[0], v[1]);
      qb[2 * t + 1] = pack_bf16x2(v[2], v[3]);
    } else if (t < kKS * 32 + 8) {  // sum_c q~_h[c]
      const int h = t - kKS * 32;
      float sum = 0.f;
      if (h < G)
        for (int c = 0; c < d.d_c; ++c) sum += __bfloat162float(qg[(size_t)h * kD + __ldg(ch + c)]);
      qsum[h] = sum;
    }
    for (int i = t; i < kKeyBins; i += kThreads - 32) lhist[i] = 0u;
  }
  __syncthreads();
  if (nbl > 0) mbar_wait(&bars[kBarTok], (bph >> kBarTok) & 1u);
  const float sm2 = d.sm_scale * kLog2e;
  float sq[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) sq[e] = sm2 * qsum[2 * q4 + e];
  const uint2* qb2 = reinterpret_cast<const uint2*>(qb);
  const int tshift = d.log2B - 4;
  const int ntiles = nbl << tshift;
  // ---- pass 1: logits of every tile (tile = warp + t * kWarps), per-warp head max ----
  float ev[kTPW][4];
  float hm[2] = {-CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
  for (int t = 0; t < kTPW; ++t) {
    const int tile = warp + t * kWarps;
    if (tile < ntiles) {
      float acc[1][4];
      token_tile_mma<kKS, 1, 1>(stc + (size_t)tile * 16 * rowb, qb2, acc);
      const int blk = cblk[tile >> tshift];
      const int tok0 = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + r0;
      const bool v0 = tok0 < n, v1 = tok0 + 8 < n;
      const float2 z0 = stz[tile * 16 + r0], z1 = stz[tile * 16 + r0 + 8];
      const float s0 = sm2 * z0.x, s1 = sm2 * z1.x;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        ev[t][e] = v0 ? fmaf(s0, acc[0][e], z0.y * sq[e]) : -CUDART_INF_F;
        ev[t][2 + e] = v1 ? fmaf(s1, acc[0][2 + e], z1.y * sq[e]) : -CUDART_INF_F;
        hm[e] = fmaxf(hm[e], fmaxf(ev[t][e], ev[t][2 + e]));
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) ev[t][e] = -CUDART_INF_F;
    }
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) hm[e] = fmaxf(hm[e], __shfl_xor_sync(0xffffffffu, hm[e], o));
    const float mref = hm[e] == -CUDART_INF_F ? 0.f : hm[e];
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < kTPW; ++t) {
      ev[t][e] = fexp2(ev[t][e] - mref);
      ev[t][2 + e] = fexp2(ev[t][2 + e] - mref);
      s += ev[t][e] + ev[t][2 + e];
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (r0 == 0) {
      ctl.wm[warp][2 * q4 + e] = hm[e];
      ctl.ws[warp][2 * q4 + e] = s;
    }
  }
  __syncthreads();
  float* stats = p.stats + (size_t)pair * p.nch * 16;  // [chunk][8 heads][m, s]
  if (tid < 8) {  // the CTA's (max, sum) per head, warps merged in order
    float M = -CUDART_INF_F, S = 0.f;
    if (tid < G)
      for (int w = 0; w < kWarps; ++w) stat_merge(M, S, ctl.wm[w][tid], ctl.ws[w][tid]);
    __stcg(stats + chunk * 16 + 2 * tid, M);
    __stcg(stats + chunk * 16 + 2 * tid + 1, S);
  }
  __syncthreads();
  if (tid == 0) {
    atom_add_acq_rel(ctr + kCtrStats, 1u);
    wait_geq(ctr + kCtrStats, (unsigned)p.nch, p.dbg, ((unsigned long long)pair << 32) | (2u << 16) | chunk);  // all chunks' stats
  }
  __syncthreads();
  if (tid < 8) {  // lz_h = M_h + log2 Z_h over the nch chunks (chunk order: deterministic)
    float M = -CUDART_INF_F, S = 0.f;
    if (tid < G)
      for (int c = 0; c < p.nch; ++c) stat_merge(M, S, __ldcg(stats + c * 16 + 2 * tid), __ldcg(stats + c * 16 + 2 * tid + 1));
    ctl.hlz[tid] = tid < G ? M + flog2(S) : CUDART_INF_F;
  }
  __syncthreads();
  // ---- pass 2: key_j = log2 sum_h 2^(L_hj - lz_h) = log2 (G alpha~_j) of every candidate slot ----
  uint32_t* kout = p.keys + (size_t)pair * p.kb_eff * d.B + ((size_t)c0 << d.log2B);
  {
    float cf[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int h = 2 * q4 + e;
      cf[e] = (h < G && hm[e] != -CUDART_INF_F) ? fexp2(hm[e] - ctl.hlz[h] + kKeyOff) : 0.f;
    }
    const bool bit0 = q4 & 1, bit1 = q4 & 2;
#pragma unroll
    for (int t = 0; t < kTPW; t += 2) {
      if (warp + t * kWarps >= ntiles) break;  // warp-uniform
      const float pa = ev[t][0] * cf[0] + ev[t][1] * cf[1];
      const float pb = ev[t][2] * cf[0] + ev[t][3] * cf[1];
      const float pc = ev[t + 1][0] * cf[0] + ev[t + 1][1] * cf[1];
      const float pd = ev[t + 1][2] * cf[0] + ev[t + 1][3] * cf[1];
      float k1 = bit0 ? pb : pa, k2 = bit0 ? pd : pc;
      k1 += __shfl_xor_sync(0xffffffffu, bit0 ? pa : pb, 1);
      k2 += __shfl_xor_sync(0xffffffffu, bit0 ? pc : pd, 1);
      float mine = bit1 ? k2 : k1;
      mine += __shfl_xor_sync(0xffffffffu, bit1 ? k1 : k2, 2);
      const int tile = warp + (t + (bit1 ? 1 : 0)) * kWarps;
      const int row = r0 + (bit0 ? 8 : 0);
      const int blk = tile < ntiles ? cblk[tile >> tshift] : 0;
      const int tok = (blk << d.log2B) + ((tile & ((1 << tshift) - 1)) << 4) + row;
      const bool v = tile < ntiles && tok < n;
      const float kf = flog2(mine) - kKeyOff;
      if (tile < ntiles) __stcg(kout + tile * 16 + row, v ? f2key(kf) : 0u);
      const int bn = v ? key_bin(kf) : kKeyBins;  // warp-aggregated histogram add
      const unsigned same = __match_any_sync(0xffffffffu, bn);
      if (v && lane == __ffs(same) - 1) atomicAdd(&lhist[bn], (unsigned)__popc(same));
    }
  }
  __syncthreads();
  uint32_t* gh = p.khist + (size_t)pair * kKeyBins;
  for (int i = tid; i < kKeyBins; i += kThreads)
    if (lhist[i]) atomicAdd(&gh[i], lhist[i]);
  __syncthreads();
  const unsigned used = nbl > 0 ? 1u << kBarTok : 0u;
  // keys + histogram counts of this chunk visible (release); the last chunk acquires every chunk's
  if (tid == 0) ctl.last = atom_add_acq_rel(ctr + kCtrDone, 1u) == (unsigned)(p.nch - 1);
  __syncthreads();
  if (!ctl.last) return used;
  if (tid == 0) asm volatile("fence.proxy.async.global;\n" ::: "memory");  // TMA reads of the keys
  *ran_sel = 1;
  return used | run_sel(p, pair, smem, bars, bph, ctl);
}

// ---------------------------------------------------------------------------
// SEL: a4 over the pair's ranking keys, run by the pair's last finishing
// TOKEN item once every chunk's keys are visible; pushes the ATT items.
// Uses mbarrier 1 (the TOKEN stage uses 0).
// ---------------------------------------------------------------------------
__device__ __noinline__ unsigned run_sel(const PStepParams& p, int pair, uint8_t* smem, uint64_t* bars, unsigned bph,
                            ItemCtl& ctl) {
  const Dims& d = p.d;
  const int tid = threadIdx.x;
  const int b = pair / d.Hkv;
  const int n = min(max(__ldg(p.seq_lens + b), 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;
  unsigned* ctr = p.ctr + (size_t)pair * 8;
  uint32_t* skeys = reinterpret_cast<uint32_t*>(smem + p.off_skeys);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + p.off_sscratch);
  uint32_t* shist = reinterpret_cast<uint32_t*>(smem + p.off_shist);
  FastTopKCtl& fk = *reinterpret_cast<FastTopKCtl*>(smem + p.off_sfk);
  int* slist = reinterpret_cast<int*>(smem + p.off_slist);
  int* cblk = reinterpret_cast<int*>(smem + p.off_scblk);
  const uint32_t kbytes = (uint32_t)(p.kb_eff * d.B * 4);
  if (tid == 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the TOKEN item's generic accesses first
    ctr[kCtrDone] = 0u;                                                // reset for the next call (no reader left)
    ctr[kCtrStats] = 0u;
    mbar_arrive_expect_tx(&bars[kBarSel], kbytes + kKeyBins * 4);
    tma_bulk_g2s(shist, p.khist + (size_t)pair * kKeyBins, kKeyBins * 4, &bars[kBarSel]);
    tma_bulk_g2s(skeys, p.keys + (size_t)pair * p.kb_eff * d.B, kbytes, &bars[kBarSel]);
  }
  // candidate blocks in the order the TOKEN items used
  const int* cand = p.guide ? p.guide + (size_t)pair * d.Kb : p.block_ids + (size_t)pair * d.Kb;
  {
    const int per = (d.Kb + kThreads - 1) / kThreads;
    const int lo = min(tid * per, d.Kb), hi = min(lo + per, d.Kb);
    int cnt = 0;
    for (int i = lo; i < hi; ++i) {
      const int c = __ldcg(cand + i);
      cnt += (c >= 0 && c < m);
    }
    int total;
    int pos = block_exclusive_scan(cnt, ctl.tk.scan, &total);
    for (int i = lo; i < hi; ++i) {
      const int c = __ldcg(cand + i);
      if (c >= 0 && c < m && pos < p.kb_eff) cblk[pos++] = c;
    }
    if (tid == 0) ctl.kc = min(total, p.kb_eff);
  }
  __syncthreads();
  const int nslots = ctl.kc << d.log2B;
  mbar_wait(&bars[kBarSel], (bph >> kBarSel) & 1u);
  // the histogram is in shared memory now: zero the pair's global one for the next call
  for (int i = tid; i < kKeyBins; i += kThreads) p.khist[(size_t)pair * kKeyBins + i] = 0u;
  __shared__ HistSel hs;
  int* tout = p.token_ids + (size_t)pair * d.Kt;
  float* sout = p.token_scores ? p.token_scores + (size_t)pair * d.Kt : nullptr;
  const float lnG = logf((float)d.G);
  auto on_k = [&](int) {};
  auto put = [&](int i, int pos) {
    tout[pos] = (cblk[i >> d.log2B] << d.log2B) + (i & (d.B - 1));
    if (sout) sout[pos] = key2f(skeys[i]) * kLn2 - lnG;
  };
  int K;
  if (nslots <= kSelRunMax * kThreads) {
    K = hist_topk_select(skeys, nslots, shist, d.Kt, scratch, fk, ctl.tk, hs, slist, on_k, put);
  } else {
    const HistPlan pl = hist_topk_plan(skeys, nslots, shist, d.Kt, scratch, fk, ctl.tk, hs);
    K = pl.K;
    hist_topk_emit(skeys, nslots, pl, hs, ctl.tk, slist, put);
  }
  for (int q = K + tid; q < d.Kt; q += kThreads) {
    tout[q] = -1;
    if (sout) sout[q] = -CUDART_INF_F;
  }
  if (tid == 0) p.num_tokens[pair] = K;
  __syncthreads();
  if (tid == 0 && p.attend) push_items(p, kAtt, pair, p.ns);  // S_t published with the ATT items
  return 1u << kBarSel;
}

// ---------------------------------------------------------------------------
// ATT: a5 over positions [K s / ns, K (s+1) / ns) of S_t; the last finishing
// slice merges the pair's ns partials
// ---------------------------------------------------------------------------
__device__ __noinline__ void run_att(const PStepParams& p, int pair, int slice, uint8_t* smem, ItemCtl& ctl) {
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int G = d.G;
  unsigned* ctr = p.ctr + (size_t)pair * 8;
  int* sel = reinterpret_cast<int*>(smem + p.off_sel);
  const int K = __ldcg(p.num_tokens + pair);  // S_t is published: the item was pushed after it
  const int t0 = (int)(((long long)K * slice) / p.ns);
  const int tloc = (int)(((long long)K * (slice + 1)) / p.ns) - t0;
  {
    const int* ids = p.token_ids + (size_t)pair * d.Kt + t0;
    const int* sob = p.slot_of_block ? p.slot_of_block + (size_t)pair * d.M : nullptr;
    for (int i = tid; i < tloc; i += kThreads) {
      const int tok = __ldcg(ids + i);
      int row = tok;
      if (sob) {  // block cache: the token's row in the slot arrays (its block must be resident)
        const int sl = __ldcg(sob + (tok >> d.log2B));
        row = sl >= 0 ? (sl << d.log2B) + (tok & (d.B - 1)) : 0;
      }
      sel[i] = row;
    }
  }
  __syncthreads();
  const __nv_bfloat16* qg = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b * d.Hq + (size_t)g * G) * kD;
  const float sm2 = d.sm_scale * kLog2e;
  constexpr int CPR = kD / 8;
  const int r = lane >> 2, q = lane & 3;
  const int tg = warp >> 1, dh = warp & 1;
  uint8_t* U = smem + p.off_kv;
  __nv_bfloat16* sbuf = reinterpret_cast<__nv_bfloat16*>(U);  // [kStages][K kTC*kD | V kTC*kD]
  __nv_bfloat16* pbuf = reinterpret_cast<__nv_bfloat16*>(smem + p.off_pbuf) + warp * 256;  // [hi|lo][8][16]
  const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_cache) + (size_t)pair * p.kv_rows * kD;
  const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(p.v_cache) + (size_t)pair * p.kv_rows * kD;
  const int nchunks = (tloc + kTC - 1) / kTC;
  auto load_chunk = [&](int c, int stage) {
    __nv_bfloat16* sK = sbuf + (size_t)stage * 2 * kTC * kD;
    __nv_bfloat16* sV = sK + kTC * kD;
    const int ntk = min(kTC, tloc - c * kTC);
#pragma unroll
    for (int it = 0; it < (kTC * CPR) / kThreads; ++it) {
      const int i = tid + it * kThreads;
      const int row = i / CPR, chk = i - row * CPR;
      const bool ok = row < ntk;
      const int tok = ok ? sel[c * kTC + row] : 0;
      const int dst = row * kD + ((chk ^ (row & 7)) << 3);
      cp_async16(sK + dst, kb + (size_t)tok * kD + chk * 8, ok);
      cp_async16(sV + dst, vb + (size_t)tok * kD + chk * 8, ok);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int c = 0; c < kStages - 1; ++c) {
    if (c < nchunks) load_chunk(c, c);
    else cp_async_commit();
  }
  uint32_t qf[kD / 16][2];  // Q^T as the B operand (heads >= G: 0)
#pragma unroll
  for (int k = 0; k < kD / 16; ++k) {
    qf[k][0] = r < G ? *reinterpret_cast<const uint32_t*>(qg + r * kD + 16 * k + 2 * q) : 0u;
    qf[k][1] = r < G ? *reinterpret_cast<const uint32_t*>(qg + r * kD + 16 * k + 2 * q + 8) : 0u;
  }
  float mrun[2] = {-CUDART_INF_F, -CUDART_INF_F}, lrun[2] = {0.f, 0.f};  // heads 2q, 2q + 1
  float o[4][4];  // O^T: m-tile mt = dims 64 dh + 16 mt + (r, r + 8), heads (2q, 2q + 1)
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    if (c + kStages - 1 < nchunks) load_chunk(c + kStages - 1, (c + kStages - 1) % kStages);
    else cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncthreads();
    const __nv_bfloat16* sK = sbuf + (size_t)(c % kStages) * 2 * kTC * kD;
    const __nv_bfloat16* sV = sK + kTC * kD;
    const int ntk = min(kTC, tloc - c * kTC);
    const int tb0 = tg * 16;
    if (tb0 < ntk) {
      float s[4] = {0.f, 0.f, 0.f, 0.f};  // S^T (16 tokens x 8 heads) = K Q^T
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) {
        const int row = tb0 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int chk = 2 * k + (lane >> 4);
        uint32_t a[4];
        ldsm_x4(a, sK + row * kD + ((chk ^ (row & 7)) << 3));
        mma_bf16_16816(s, a, qf[k][0], qf[k][1]);
      }
      const bool v0 = tb0 + r < ntk, v1 = tb0 + r + 8 < ntk;
      s[0] = v0 ? s[0] * sm2 : -CUDART_INF_F;
      s[1] = v0 ? s[1] * sm2 : -CUDART_INF_F;
      s[2] = v1 ? s[2] * sm2 : -CUDART_INF_F;
      s[3] = v1 ? s[3] * sm2 : -CUDART_INF_F;
      float x0 = fmaxf(s[0], s[2]), x1 = fmaxf(s[1], s[3]);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, off));
        x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, off));
      }
      // lazy rescaling: the reference max moves only when a score exceeds it by > 8 (log2 units)
      const bool g0 = x0 > mrun[0] + 8.f, g1 = x1 > mrun[1] + 8.f;
      const float n0 = g0 ? x0 : mrun[0], n1 = g1 ? x1 : mrun[1];
      const float a0 = g0 ? fexp2(mrun[0] - n0) : 1.f, a1 = g1 ? fexp2(mrun[1] - n1) : 1.f;
      const float p0 = fexp2(s[0] - n0), p1 = fexp2(s[1] - n1), p2 = fexp2(s[2] - n0), p3 = fexp2(s[3] - n1);
      float r0s = p0 + p2, r1s = p1 + p3;
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        r0s += __shfl_xor_sync(0xffffffffu, r0s, off);
        r1s += __shfl_xor_sync(0xffffffffu, r1s, off);
      }
      lrun[0] = lrun[0] * a0 + r0s;
      lrun[1] = lrun[1] * a1 + r1s;
      mrun[0] = n0;
      mrun[1] = n1;
      if (__any_sync(0xffffffffu, g0 || g1)) {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          o[mt][0] *= a0;
          o[mt][1] *= a1;
          o[mt][2] *= a0;
          o[mt][3] *= a1;
        }
      }
      // P^T as two bf16 pieces (hi + lo) into the B layout: the PV product keeps ~16 bits of P
      const float pv[4] = {p0, p1, p2, p3};
      const int pi[4] = {(2 * q) * 16 + r, (2 * q + 1) * 16 + r, (2 * q) * 16 + r + 8, (2 * q + 1) * 16 + r + 8};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __nv_bfloat16 hi = __float2bfloat16_rn(pv[e]);
        pbuf[pi[e]] = hi;
        pbuf[128 + pi[e]] = __float2bfloat16_rn(pv[e] - __bfloat162float(hi));
      }
      __syncwarp();
      const uint32_t ph0 = *reinterpret_cast<const uint32_t*>(pbuf + r * 16 + 2 * q);
      const uint32_t ph1 = *reinterpret_cast<const uint32_t*>(pbuf + r * 16 + 2 * q + 8);
      const uint32_t pl0 = *reinterpret_cast<const uint32_t*>(pbuf + 128 + r * 16 + 2 * q);
      const uint32_t pl1 = *reinterpret_cast<const uint32_t*>(pbuf + 128 + r * 16 + 2 * q + 8);
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {  // O^T (64 dims x 8 heads) += V^T (dims x 16 tokens) P^T
        const int token = tb0 + (lane & 7) + ((lane >> 4) & 1) * 8;
        const int chk = (dh * 64 + 16 * mt) / 8 + ((lane >> 3) & 1);
        uint32_t a[4];
        ldsm_x4_trans(a, sV + token * kD + ((chk ^ (token & 7)) << 3));
        mma_bf16_16816(o[mt], a, ph0, ph1);
        mma_bf16_16816(o[mt], a, pl0, pl1);
      }
    }
    __syncthreads();  // stage c % kStages consumed before it is refilled
  }
  cp_async_wait<0>();
  // ---- merge the 4 token groups of this CTA (the staging buffers become scratch) ----
  constexpr int WS = kD + 4;
  float* wo = reinterpret_cast<float*>(U);  // [tg][8 heads][WS]
  float* wml = wo + 4 * 8 * WS;             // [tg][8 heads][2]
  if (dh == 0 && r == 0) {
    wml[(tg * 8 + 2 * q) * 2] = mrun[0];
    wml[(tg * 8 + 2 * q) * 2 + 1] = lrun[0];
    wml[(tg * 8 + 2 * q + 1) * 2] = mrun[1];
    wml[(tg * 8 + 2 * q + 1) * 2 + 1] = lrun[1];
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int d0 = dh * 64 + 16 * mt + r;
    wo[(tg * 8 + 2 * q) * WS + d0] = o[mt][0];
    wo[(tg * 8 + 2 * q + 1) * WS + d0] = o[mt][1];
    wo[(tg * 8 + 2 * q) * WS + d0 + 8] = o[mt][2];
    wo[(tg * 8 + 2 * q + 1) * WS + d0 + 8] = o[mt][3];
  }
  __syncthreads();
  const int ngroups = min(4, (min(tloc, kTC) + 15) / 16);  // token groups that saw at least one token
  __nv_bfloat16* outg = reinterpret_cast<__nv_bfloat16*>(p.out) + ((size_t)b * d.Hq + (size_t)g * G) * kD;
  float* po = p.part_o + ((size_t)pair * p.ns + slice) * 8 * kD;
  float* pml = p.part_ml + ((size_t)pair * p.ns + slice) * 16;
  const bool direct = p.ns == 1;
  for (int idx = tid; idx < G * kD; idx += kThreads) {
    const int h = idx / kD, dcol = idx - h * kD;
    float M = -CUDART_INF_F;
    for (int t = 0; t < ngroups; ++t) M = fmaxf(M, wml[(t * 8 + h) * 2]);
    float L = 0.f, acc = 0.f;
    if (M != -CUDART_INF_F) {
      for (int t = 0; t < ngroups; ++t) {
        const float mw = wml[(t * 8 + h) * 2];
        const float sc = mw == -CUDART_INF_F ? 0.f : fexp2(mw - M);
        L = fmaf(wml[(t * 8 + h) * 2 + 1], sc, L);
        acc = fmaf(wo[(t * 8 + h) * WS + dcol], sc, acc);
      }
    }
    if (direct) {
      outg[idx] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
      if (dcol == 0 && p.lse != nullptr)
        p.lse[(size_t)b * d.Hq + (size_t)g * G + h] = L > 0.f ? (M + flog2(L)) * kLn2 : -CUDART_INF_F;
    } else {
      __stcg(po + idx, acc);
      if (dcol == 0) {
        __stcg(pml + 2 * h, M);
        __stcg(pml + 2 * h + 1, L);
      }
    }
  }
  if (direct) return;
  __syncthreads();
  if (tid == 0) ctl.last = atom_add_acq_rel(ctr + kCtrAtt, 1u) == (unsigned)(p.ns - 1);
  __syncthreads();
  if (!ctl.last) return;
  // ---- the pair's last slice: merge the ns partials (flash-decoding LSE identity, T10) ----
  if (tid == 0) ctr[kCtrAtt] = 0u;  // reset for the next call
  const float* po0 = p.part_o + (size_t)pair * p.ns * 8 * kD;
  const float* pm0 = p.part_ml + (size_t)pair * p.ns * 16;
  if (tid < G) {
    float M = -CUDART_INF_F;
    for (int s = 0; s < p.ns; ++s) M = fmaxf(M, __ldcg(pm0 + s * 16 + 2 * tid));
    float L = 0.f;
    for (int s = 0; s < p.ns; ++s) {
      const float ms = __ldcg(pm0 + s * 16 + 2 * tid);
      const float w = (M == -CUDART_INF_F || ms == -CUDART_INF_F) ? 0.f : fexp2(ms - M);
      L = fmaf(__ldcg(pm0 + s * 16 + 2 * tid + 1), w, L);
      ctl.mw[s][tid] = w;
    }
    ctl.minv[tid] = L > 0.f ? 1.f / L : 0.f;
    if (p.lse != nullptr) p.lse[(size_t)b * d.Hq + (size_t)g * G + tid] = L > 0.f ? (M + flog2(L)) * kLn2 : -CUDART_INF_F;
  }
  __syncthreads();
  for (int idx = tid; idx < G * kD; idx += kThreads) {
    const int h = idx / kD;
    float acc = 0.f;
    for (int s = 0; s < p.ns; ++s) acc = fmaf(__ldcg(po0 + (size_t)s * 8 * kD + idx), ctl.mw[s][h], acc);
    outg[idx] = __float2bfloat16_rn(acc * ctl.minv[h]);
  }
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 3) pstep_kernel(const __grid_constant__ PStepParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kNumBars];
  __shared__ ItemCtl ctl;
  __shared__ unsigned s_item;
  __shared__ int s_sel;          // the TOKEN item ran a4
  __shared__ int s_tick[2];      // run_tiles: ticket in each tile buffer (-1: none)
  __shared__ unsigned s_bph;     // parity of the current phase of each mbarrier (initialised once, never re-initialised)
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kNumBars; ++s) mbar_init(&bars[s], s == kBarEmpty || s == kBarEmpty + 1 ? kConsumers : 1);
    mbar_fence_init();
    s_bph = 0u;
  }
  __syncthreads();
  if (blockIdx.x < (unsigned)p.nstream) {  // streamer: a1 until the tickets run out, then a worker
    const unsigned long long t_start = p.dbg ? gtimer() : 0ull;
    run_tiles(p, smem, bars, s_tick);
    if (tid == 0) {
      if (p.dbg) {
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        const unsigned long long slot = atomicAdd(p.dbg + (1 << 20) - 1, 1ull);
        p.dbg[3 * slot] = t_start;
        p.dbg[3 * slot + 1] = gtimer();
        p.dbg[3 * slot + 2] = ((unsigned long long)smid << 32) | ((unsigned)kTile << 24);
      }
    }
  }
  for (;;) {  // worker: reserve the next ready-queue slot, wait for its item, run it
    if (tid == 0) {
      unsigned item = pack_item(kExit, 0, 0);
      const unsigned h = atomicAdd(p.sched + kRqHead, 1u);
      if (h < (unsigned)p.nready) {
        unsigned spins = 0;
        while (!slot_ready(p, (int)h, item)) {
          __nanosleep(256);
          if (++spins > (1u << 26)) __trap();
        }
      }
      s_item = item;
      s_sel = 0;
    }
    __syncthreads();
    const unsigned item = s_item;
    int role, sub, pair;
    unpack_item(item, role, sub, pair);
    if (role == kExit) break;
    const unsigned long long t_start = p.dbg ? gtimer() : 0ull;
    const unsigned bph = s_bph;
    unsigned nbph = bph;
    if (role == kA2) run_a2(p, pair, smem, ctl);
    else if (role == kToken) nbph = bph ^ run_token(p, pair, sub, smem, bars, bph, ctl, &s_sel);
    else run_att(p, pair, sub, smem, ctl);
    __syncthreads();  // shared memory free for the next item; every thread read s_bph
    if (tid == 0) s_bph = nbph;
    if (p.dbg && tid == 0) {  // diagnostics: per item (start, end, smid | role | sub | pair)
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      const unsigned long long slot = atomicAdd(p.dbg + (1 << 20) - 1, 1ull);
      if (slot < (1 << 20) / 3 - 1) {
        const int r = (role == kToken && s_sel) ? kSel : (role == kA2 ? kTile : role);
        p.dbg[3 * slot] = t_start;
        p.dbg[3 * slot + 1] = gtimer();
        p.dbg[3 * slot + 2] = ((unsigned long long)smid << 32) | ((unsigned)r << 24) | ((unsigned)(sub | (role == kA2 ? 0x80 : 0)) << 16) |
                              (unsigned)(pair & 0xffff);
      }
    }
  }
  if (tid == 0 && atom_add_acq_rel(p.sched + kCtasOut, 1u) == gridDim.x - 1) {  // the last CTA out resets
    p.sched[kTileNext] = 0u;
    p.sched[kRqHead] = 0u;
    p.sched[kRqTail] = 0u;
    p.sched[kCtasOut] = 0u;
  }
}

// ============================================================== host side
bool pstep_supported(const Dims& d) {
  return d.bf16 && !d.mla && d.d_k == kD && d.d_v == kD && d.G <= 8 && d.d_c == 32 && d.B == 64 && (d.S % 2) == 0;
}

// Work decomposition, schedule lags and the shared-memory plan (the union of the four roles' regions).
bool plan_pstep(PStepParams& p, int ns_override) {
  const Dims& d = p.d;
  p.pairs = d.batch * d.Hkv;
  p.kb_eff = kb_effective(d);
  p.tb = 56;  // 28 KB of block summaries per TILE: 7 row groups, one per consumer warp
  p.ntile = (d.M + p.tb - 1) / p.tb;
  p.cb = 16;  // 1024 candidate tokens per TOKEN: 8 warps x kTPW tiles x 16
  if (p.cb > p.kb_eff) p.cb = p.kb_eff;
  p.nch = (p.kb_eff + p.cb - 1) / p.cb;
  const int kt = kt_effective(d);
  p.ns = ns_override > 0 ? ns_override : (kt + 255) / 256;  // ~256 selected tokens per ATT
  if (p.ns > 16) p.ns = 16;
  if (p.ns < 1) p.ns = 1;
  const int tok_max = (kt + p.ns - 1) / p.ns;
  if ((size_t)p.kb_eff * d.B > (size_t)kSelRunMax * kThreads) return false;  // SEL: the one-pass register select
  p.ntiles_total = p.pairs * p.ntile;
  p.nready = p.pairs * (1 + p.nch + (p.attend ? p.ns : 0));  // A2, TOKEN x nch, ATT x ns
  if (p.pairs >= (1 << 22) || p.nch > 127 || p.ns > 127) return false;  // queue entry fields
  // shared memory: every role's regions start at 0 (one item at a time per CTA)
  size_t tile_end, tok_end, sel_end, att_end;
  {  // TILE: two tile buffers, QQ; the a2 regions alias the item's own buffer once it is scored
    size_t o = 2 * (size_t)p.tb * kRowBytes;
    p.off_tile = 0;
    p.off_qq = (unsigned)o;
    o = align16(o + 2 * kD * 4);
    size_t w = 0;
    p.off_bkeys = (unsigned)w;
    w = align16(w + (size_t)((d.M + 31) & ~31) * 4);
    p.off_scratch = (unsigned)w;
    w = align16(w + (size_t)kBracketWords * 4);
    p.off_fk = (unsigned)w;
    w = align16(w + sizeof(FastTopKCtl));
    if (w > (size_t)p.tb * kRowBytes) return false;  // a2 regions must fit inside one tile buffer (QQ stays)
    tile_end = o;
  }
  {  // TOKEN: index stage, q~ fragments, candidate ids, local histogram
    size_t o = 0;
    p.off_stage = (unsigned)o;
    o = align16(o + (size_t)p.cb * d.B * (d.d_c / 2 + 8));
    p.off_qb = (unsigned)o;
    o = align16(o + kKS * 256 + 8 * 4);
    p.off_cblk = (unsigned)o;
    o = align16(o + (size_t)p.cb * 4);
    p.off_lhist = (unsigned)o;
    o = align16(o + kKeyBins * 4);
    tok_end = o;
  }
  {  // SEL: keys of every candidate slot, bracket scratch, histogram, FastTopKCtl, selected list, candidates
    size_t o = 0;
    p.off_skeys = (unsigned)o;
    o = align16(o + (size_t)p.kb_eff * d.B * 4);
    p.off_sscratch = (unsigned)o;
    o = align16(o + (size_t)kBracketWords * 4);
    p.off_shist = (unsigned)o;
    o = align16(o + kKeyBins * 4);
    p.off_sfk = (unsigned)o;
    o = align16(o + sizeof(FastTopKCtl));
    p.off_slist = (unsigned)o;
    o = align16(o + (size_t)kt * 4);
    p.off_scblk = (unsigned)o;
    o = align16(o + (size_t)p.kb_eff * 4);
    sel_end = o;
  }
  {  // ATT: K/V stages (then the warp-partial scratch), P buffers, selected rows
    size_t o = 0;
    p.off_kv = (unsigned)o;
    o = align16(o + (size_t)kStages * 2 * kTC * kD * 2);
    p.off_pbuf = (unsigned)o;
    o = align16(o + (size_t)kWarps * 512);
    p.off_sel = (unsigned)o;
    o = align16(o + (size_t)(tok_max + 1) * 4);
    att_end = o;
  }
  size_t mx = tile_end;
  if (tok_end > mx) mx = tok_end;
  if (sel_end > mx) mx = sel_end;
  if (p.attend && att_end > mx) mx = att_end;
  p.smem_bytes = (unsigned)mx;
  return true;
}

// Workspace of the persistent step (bytes) and its carve-up.
size_t pstep_workspace(PStepParams& p, char* ws) {
  const Dims& d = p.d;
  const size_t P = (size_t)p.pairs;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = a256(o + bytes);
    return at;
  };
  const size_t o_sched = take(256);
  const size_t o_rq = take((size_t)p.nready * 8);
  const size_t o_ctr = take(P * 8 * 4);
  const size_t o_scores = take(P * d.Ms * 4);
  const size_t o_keys = take(P * p.kb_eff * d.B * 4);
  const size_t o_khist = take(P * kKeyBins * 4);
  const size_t o_stats = take(P * p.nch * 16 * 4);
  const size_t o_po = take(P * p.ns * 8 * kD * 4);
  const size_t o_pml = take(P * p.ns * 16 * 4);
  if (ws) {
    p.sched = reinterpret_cast<unsigned*>(ws + o_sched);
    p.rq = reinterpret_cast<unsigned long long*>(ws + o_rq);
    p.ctr = reinterpret_cast<unsigned*>(ws + o_ctr);
    p.scores = reinterpret_cast<float*>(ws + o_scores);
    p.keys = reinterpret_cast<uint32_t*>(ws + o_keys);
    p.khist = reinterpret_cast<uint32_t*>(ws + o_khist);
    p.stats = reinterpret_cast<float*>(ws + o_stats);
    p.part_o = reinterpret_cast<float*>(ws + o_po);
    p.part_ml = reinterpret_cast<float*>(ws + o_pml);
  }
  return o;
}

// Resident CTAs per SM of the persistent kernel (the grid is exactly one wave).
int pstep_occupancy(size_t smem) {
  int nb = 0;
  if (prepare_kernel(reinterpret_cast<const void*>(pstep_kernel), smem, false) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pstep_kernel, kThreads, smem) != cudaSuccess) return 0;
  return nb;
}

cudaError_t launch_pstep(const PStepParams& p, int grid, cudaStream_t st) {
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(pstep_kernel), p.smem_bytes, false);
  if (e != cudaSuccess) return e;
  return launch_ex(pstep_kernel, dim3((unsigned)grid, 1, 1), kThreads, p.smem_bytes, st, LaunchOpts{}, 0u, p);
}

}  // namespace tls
