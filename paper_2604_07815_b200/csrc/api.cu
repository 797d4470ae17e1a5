// api.cu -- the C ABI of libtls.so (declared in include/tls.h): argument
// validation, launch planning and dispatch.  No device memory is allocated and
// no global state is kept besides the thread-local error string.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <time.h>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/tls.h"
#include "index.h"
#include "params.h"
#include "fasttopk.cuh"
#include "launch.h"
#include <algorithm>

namespace tls {
cudaError_t launch_select_fused(const FusedParams& p, cudaStream_t st, const LaunchOpts& o);
cudaError_t launch_qq(const FusedParams& p, cudaStream_t st, const LaunchOpts& o);
cudaError_t launch_stream_select(const FusedParams& p, int grid, cudaStream_t st, const LaunchOpts& o);
size_t stream_select_smem(int tb, size_t worker_bytes);
cudaError_t launch_cache_fetch(const CacheFetchParams& p, cudaStream_t st);
cudaError_t launch_block_cache_update(const BlockCacheParams& p, cudaStream_t st);
cudaError_t launch_block_cache_rows(const BlockCacheParams& p, cudaStream_t st);
cudaError_t launch_token_cluster(const SelectParams& p, cudaStream_t st, const LaunchOpts& o);
cudaError_t launch_attend(const AttendParams& p, cudaStream_t st, const LaunchOpts& o);
int score_cpl(int d_k, size_t elem_bytes);
bool select_supported(int d_c, int G);
bool pstep_supported(const Dims& d);
bool plan_pstep(PStepParams& p, int ns_override);
size_t pstep_workspace(PStepParams& p, char* ws);
int pstep_occupancy(size_t smem);
cudaError_t launch_pstep(const PStepParams& p, int grid, cudaStream_t st);
cudaError_t launch_topk_rows(int rows, int n, const float* keys, const int* ids, int k, float* out_keys,
                             int* out_ids, int* out_count, int id_base, const int* lens, int lens_div, int lens_unit,
                             cudaStream_t st);
cudaError_t launch_select_range(int rows, int k, const int* ids, int lo, int hi, int* out_ids, int* out_count,
                                cudaStream_t st);
size_t token_split_smem(const Dims& d);
cudaError_t launch_expand_blocks(const Dims& d, const int* block_ids, const int* seq_lens, int k_out, int* token_ids,
                                 int* num_tokens, cudaStream_t st);
cudaError_t launch_block_iota(const Dims& d, const int* seq_lens, int* block_ids, cudaStream_t st);
cudaError_t launch_token_split(const Dims& d, int mode, const void* q, const int* seq_lens, const uint8_t* codes,
                               const float* scale_zero, const int* channels, const int* block_ids, int P,
                               const float* stats_in, float* stats_out, float* keys_out, int* ids_out, int tok_off,
                               cudaStream_t st);
cudaError_t launch_attn_merge(bool bf16, int P, int rows, int dv, const float* parts_o, const float* parts_lse,
                              void* out, float* lse, cudaStream_t st);
}  // namespace tls

namespace {

thread_local char g_err[512] = "";

tls_status fail(tls_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

tls_status cuda_fail(cudaError_t e, const char* what) {
  return fail(TLS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

size_t elem_bytes(const tls_config* c) { return c->dtype == TLS_BF16 ? 2 : 4; }

constexpr int kMaxSmem = 227 * 1024 - 8 * 1024;  // dynamic budget (static control blocks < 8 KB)

// SM count of the current device (cached per device ordinal).
int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int v = 0;
    cache[dev] = (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) ? v : 148;
  }
  return cache[dev];
}

constexpr int kSMs = 148;

// Shape / hyper-parameter checks shared by every call.
tls_status check_config(const tls_config* c) {
  if (!c) return fail(TLS_ERR_INPUT, "cfg is NULL");
  if (c->batch < 1) return fail(TLS_ERR_INPUT, "batch must be >= 1 (got %d)", c->batch);
  if (c->dtype != TLS_BF16 && c->dtype != TLS_FP32) return fail(TLS_ERR_CONFIG, "unknown dtype %d", c->dtype);
  if (c->layout != TLS_GQA && c->layout != TLS_MLA) return fail(TLS_ERR_CONFIG, "unknown layout %d", c->layout);
  if (c->num_q_heads < 1 || c->num_kv_heads < 1 || c->d_k < 1 || c->d_v < 1 || c->max_seq_len < 1)
    return fail(TLS_ERR_DIM, "heads, widths and max_seq_len must be >= 1");
  if (c->num_q_heads % c->num_kv_heads)
    return fail(TLS_ERR_DIM, "num_q_heads (%d) %% num_kv_heads (%d) != 0", c->num_q_heads, c->num_kv_heads);
  if (c->layout == TLS_MLA) {
    if (c->num_kv_heads != 1) return fail(TLS_ERR_DIM, "MLA has one shared latent KV head (P:73)");
    if (c->d_v > c->d_k) return fail(TLS_ERR_DIM, "MLA needs d_v <= d_k (V = K[..., :d_v])");
  }
  if (c->block_size < 1) return fail(TLS_ERR_CONFIG, "block_size must be >= 1");
  if (c->d_c < 1 || c->d_c > c->d_k || (c->d_c & 1)) return fail(TLS_ERR_CONFIG, "d_c must be even and in [1, d_k]");
  if (c->top_blocks < 1 || c->top_tokens < 1) return fail(TLS_ERR_CONFIG, "top_blocks and top_tokens must be >= 1");
  if (!(c->sm_scale > 0.f) || c->sm_scale > 1e30f) return fail(TLS_ERR_CONFIG, "sm_scale must be positive and finite");
  // What the kernels implement.
  const size_t eb = elem_bytes(c);
  if ((c->d_k * eb) % 16 || (c->d_v * eb) % 16)
    return fail(TLS_ERR_UNSUPPORTED, "d_k and d_v rows must be multiples of 16 bytes");
  const int G = c->num_q_heads / c->num_kv_heads;
  if (G > 32) return fail(TLS_ERR_UNSUPPORTED, "at most 32 query heads per KV head");
  if (c->d_c % 32 || c->d_c > 128 || !tls::select_supported(c->d_c, G))
    return fail(TLS_ERR_UNSUPPORTED, "d_c must be 32, 64 or 128");
  if (c->block_size < 16 || c->block_size > 1024 || (c->block_size & (c->block_size - 1)))
    return fail(TLS_ERR_UNSUPPORTED, "block_size must be a power of two in [16, 1024]");
  if ((long long)c->batch * c->num_kv_heads > 65535) return fail(TLS_ERR_UNSUPPORTED, "batch*num_kv_heads > 65535");
  if (tls::score_cpl(c->d_k, eb) < 0) return fail(TLS_ERR_UNSUPPORTED, "d_k too large for the block-score kernel");
  return TLS_OK;
}

tls::Dims dims_of(const tls_config* c) {
  tls::Dims d;
  memset(&d, 0, sizeof(d));
  d.batch = c->batch;
  d.Hq = c->num_q_heads;
  d.Hkv = c->num_kv_heads;
  d.G = c->num_q_heads / c->num_kv_heads;
  d.d_k = c->d_k;
  d.d_v = c->d_v;
  d.S = c->max_seq_len;
  d.B = c->block_size;
  d.d_c = c->d_c;
  d.Kb = c->top_blocks;
  d.Kt = c->top_tokens;
  d.M = (c->max_seq_len + c->block_size - 1) / c->block_size;
  d.sm_scale = c->sm_scale;
  d.mla = c->layout == TLS_MLA;
  d.bf16 = c->dtype == TLS_BF16;
  d.log2B = 0;
  while ((1 << d.log2B) < c->block_size) ++d.log2B;
  d.Ms = (d.M + 3) & ~3;
  return d;
}

// Diagnostics only: TLS_DEBUG_BUF=<hex device address> makes K2 and K3 write
// per-CTA %globaltimer stamps there (K2 at [pair*8+chunk]*8, K3 at 65536*8 +
// pair*8).  Unset in normal use.
unsigned long long* env_debug_buf() {
  const char* e = getenv("TLS_DEBUG_BUF");
  return e ? reinterpret_cast<unsigned long long*>(strtoull(e, nullptr, 16)) : nullptr;
}

int env_cluster() {
  const char* env = getenv("TLS_CLUSTER");
  return (env && atoi(env) > 0) ? atoi(env) : 0;
}

// The persistent step kernel (pstep.cu: one launch, work items of every stage of every pair claimed from a
// ticket queue) for the configurations it supports; false: the kernel chain runs instead.  TLS_CLUSTER
// (tuning / tests) sets its attention slices per pair; TLS_PSTEP="L1,L2,L3" (tuning) its schedule lags.
bool pstep_plan(const tls_config* c, int do_attend, tls::PStepParams& sp) {
  memset(&sp, 0, sizeof(sp));
  sp.d = dims_of(c);
  const char* e = getenv("TLS_PSTEP");  // opt-in while it is slower than the chain
  if (!tls::pstep_supported(sp.d) || e == nullptr) return false;
  sp.attend = do_attend;
  const int env = env_cluster();
  if (env > 16) return false;
  return tls::plan_pstep(sp, env) && (int)sp.smem_bytes <= kMaxSmem;
}

tls_status plan_select(const tls_config* c, tls::SelectParams& p) {
  memset(&p, 0, sizeof(p));
  p.d = dims_of(c);
  // TLS_K2_FORM (A/B and tests): "cluster" = the cluster forms even where token_pair_kernel fits; "1" / "2" =
  // token_pair_kernel with that many CTAs per pair
  const char* e = getenv("TLS_K2_FORM");
  tls::plan_select(p, !e ? 0 : (e[0] == 'c' ? -1 : (e[0] == '1' ? 1 : (e[0] == '2' ? 2 : (e[0] == '4' ? 4 : 0)))));
  if ((int)p.smem_bytes > kMaxSmem) return fail(TLS_ERR_UNSUPPORTED, "token-kernel shared-memory plan does not fit");
  return TLS_OK;
}

// K3 cluster size: one CTA per pair once the pairs cover the SMs; else split
// the pair's tokens.  TLS_CLUSTER overrides (tuning / tests).
tls_status plan_attend(const tls_config* c, tls::AttendParams& p, int select, int attend) {
  memset(&p, 0, sizeof(p));
  p.d = dims_of(c);
  p.select = select;
  p.attend = attend;
  p.mma = c->dtype == TLS_BF16 && c->layout == TLS_GQA && c->d_k == c->d_v && (c->d_k == 64 || c->d_k == 128) &&
          p.d.G <= 16;
  if (c->dtype == TLS_BF16 && c->layout == TLS_MLA && c->d_k == 576 && c->d_v == 512 && p.d.G <= 32) p.mma = 2;
  const long long pairs = (long long)c->batch * c->num_kv_heads;
  const int kt = tls::kt_effective(p.d);
  int cs = env_cluster();
  if (!attend) cs = 1;  // selection only: one CTA per pair
  if (p.mma == 2 && attend) {  // MLA on tcgen05 (attend.cu attend_mla_tc_kernel)
    const char* e = getenv("TLS_MLA_TC");  // opt-in ("1"): slower than the mma.sync kernel so far
    // one wave of CTAs (one per SM), each with >= 128 selected tokens
    int c2 = cs;
    if (!c2) {
      c2 = 1;
      while (c2 < 16 && pairs * c2 * 2 <= (long long)num_sms() && (kt + 2 * c2 - 1) / (2 * c2) >= 128) c2 *= 2;
    }
    if (e && e[0] == '1') {
      p.mma = 3;
      p.mla_tc = 64;
      p.cs = c2;
      tls::plan_attend(p, sizeof(tls::FastTopKCtl));
      if ((int)p.smem_bytes <= kMaxSmem) return TLS_OK;
      p.mma = 2;  // does not fit: the mma.sync kernel
    }
  }
  if (!cs) {
    // split a pair's tokens over more CTAs only while the whole grid stays one wave of
    // co-resident CTAs (MLA: one 117 KB CTA per SM; GQA mma: two) and each CTA keeps >= 64
    // tokens (measured, C4: cs 4 -> 62 us, cs 8 -> 113 us; C2: cs 2 best)
    const int per_sm = p.mma == 2 ? 1 : 2;
    const int sms = num_sms();
    cs = 1;
    while (cs < 16 && pairs * cs * 2 <= (long long)sms * per_sm && (kt + 2 * cs - 1) / (2 * cs) >= 64) cs *= 2;
  }
  // more CTAs per pair first (shorter selected-token lists per CTA); MLA falls back to its 32-token staging
  // only when no cluster size fits the 64-token one
  for (const int tc : {64, 32}) {
    p.mla_tc = tc;
    for (int c = cs; c <= 16; c *= 2) {
      p.cs = c;
      tls::plan_attend(p, sizeof(tls::FastTopKCtl));
      if ((int)p.smem_bytes <= kMaxSmem) return TLS_OK;
    }
    if (p.mma != 2) break;
  }
  return fail(TLS_ERR_UNSUPPORTED, "attention shared-memory plan does not fit");
}

tls_status check_index(const tls_index* idx) {
  if (!idx || !idx->block_minmax || !idx->codes || !idx->scale_zero || !idx->channels)
    return fail(TLS_ERR_INPUT, "index buffers must be non-NULL");
  if (!aligned16(idx->block_minmax) || !aligned16(idx->codes) || !aligned16(idx->scale_zero))
    return fail(TLS_ERR_INPUT, "index buffers must be 16-byte aligned");
  return TLS_OK;
}

// ---- live per-kernel timing (tls_timing_enable / tls_timing_read) ----
constexpr int kMarks = 4;  // select_kernel | token_cluster_kernel | attend_kernel
struct KernelTimer {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // kMarks per recorded call
  size_t used = 0;              // events recorded so far
  cudaEvent_t next() {
    if (used == ev.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      ev.push_back(e);
    }
    return ev[used++];
  }
  void mark(cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e = next();
    if (e) cudaEventRecord(e, st);
  }
};
KernelTimer g_timer;

// Sub-batch pipeline.  Pairs are independent, so the batch can be cut
// into ns contiguous sub-batches whose four-kernel chains run on ns internal
// streams: the HBM-streaming block-score kernel (K1) of one sub-batch then
// overlaps the latency-bound selection / attention kernels of another.  K1
// launches carry the lowest scheduling priority and K1b/K2/K3 the highest, so
// whenever an SM frees up the block scheduler places the dependent chain's
// CTAs first and K1's CTAs fill the rest.  The result is bit-identical to
// ns = 1 (every kernel's arithmetic is per pair).  TLS_NSPLIT overrides the
// heuristic (tuning / tests).
int n_split(const tls_config* c) {
  int ns = 1;
  const char* e = getenv("TLS_NSPLIT");
  if (e && atoi(e) > 0) ns = atoi(e);
  if (ns > 8) ns = 8;
  if (ns > c->batch) ns = c->batch;
  if (c->max_seq_len & 1) ns = 1;  // keep every sub-batch's scale/zero rows 16-byte aligned
  return ns < 1 ? 1 : ns;
}

tls_config sub_config(const tls_config* c, int ns, int s, int* b0) {
  tls_config sc = *c;
  const int lo = (int)((long long)c->batch * s / ns), hi = (int)((long long)c->batch * (s + 1) / ns);
  sc.batch = hi - lo;
  *b0 = lo;
  return sc;
}

// Selection mode: select_kernel does a1-a2, then the cluster token kernel
// (a3) and the attention kernel's top-k_t prologue (a4).  (A mode 2 that ran
// a1-a4 in select_kernel was measured and dropped.)
int fused_mode(const tls_config*) { return 1; }

// Bytes of block summaries per select_kernel CTA (TLS_TILE_KB overrides; tuning).
// Block-summary rows per K1 tile CTA: <= 64 rows (8 TMA groups of 8 rows, one
// mbarrier per warp), 32 KB of rows by default (C4 measured: 32 KB 129.9 us/step,
// 64 KB 133.6, 96 KB 132.9, 128 KB 153.2).  Tuning: env TLS_TILE_KB (4..192).
int score_tile_rows(int rowbytes) {
  const char* e = getenv("TLS_TILE_KB");
  const int kb = e ? atoi(e) : 0;
  const int bytes = (kb >= 4 && kb <= 192) ? kb * 1024 : tls::kScoreTileBytes;
  return std::min(64, bytes / rowbytes);
}

struct ChainPlan {
  int mode;
  int stream_sel;  // a1 + a2 by the persistent streaming kernel (one CTA per SM, TMA ring)
  tls::FusedParams fp;
  tls::SelectParams sp;  // mode 1
  tls::AttendParams ap;  // do_attend, or mode 1
  tls::SelectWs w;
  size_t att_ws;
  size_t total;
};

tls_status plan_chain(const tls_config* cfg, int do_attend, ChainPlan& c) {
  memset(&c, 0, sizeof(c));
  c.mode = fused_mode(cfg);
  c.fp.d = dims_of(cfg);
  c.fp.mode = c.mode;
  c.fp.tb = score_tile_rows(2 * cfg->d_k * (int)elem_bytes(cfg));
  if (c.fp.tb < 1) return fail(TLS_ERR_UNSUPPORTED, "block summary row larger than the K1 tile");
  tls::plan_fused(c.fp, sizeof(tls::FastTopKCtl));
  if ((int)c.fp.smem_bytes > kMaxSmem) return fail(TLS_ERR_UNSUPPORTED, "selection-kernel shared-memory plan does not fit");
  {  // bf16 GQA with 512-byte summary rows: the streaming select kernel (fused.cu stream_select_kernel)
    const char* e = getenv("TLS_STREAM_SEL");  // opt-in experiment ("1"): slower, DESIGN.md §5.1
    c.stream_sel = c.mode == 1 && cfg->dtype == TLS_BF16 && cfg->layout == TLS_GQA && cfg->d_k == 128 &&
                   e != nullptr && e[0] == '1';
    if (c.stream_sel) {
      const size_t worker = c.fp.off_fk + tls::align16(sizeof(tls::FastTopKCtl));
      c.fp.tb = 56;  // 28 KB stages: 7 row groups (warps 0-6)
      c.fp.smem_bytes = (unsigned)tls::stream_select_smem(c.fp.tb, worker);
      if (c.fp.smem_bytes == 0) {  // the a2 worker regions (M-sized key list) do not fit one stage
        c.stream_sel = 0;
        c.fp.tb = score_tile_rows(2 * cfg->d_k * (int)elem_bytes(cfg));
        tls::plan_fused(c.fp, sizeof(tls::FastTopKCtl));
      }
    }
  }
  tls_status s = TLS_OK;
  if (c.mode == 1) {
    s = plan_select(cfg, c.sp);
    if (s) return s;
  }
  c.w = tls::select_workspace(c.fp.d);
  c.att_ws = 0;
  if (c.mode == 1 || do_attend) {
    s = plan_attend(cfg, c.ap, c.mode == 1, do_attend);
    if (s) return s;
    if (do_attend) c.att_ws = tls::attend_workspace_bytes(c.ap.d, c.ap.cs);
  }
  c.total = tls::a256(c.w.total + c.att_ws);
  return TLS_OK;
}

// Workspace of one (sub-)batch chain.
tls_status chain_workspace(const tls_config* cfg, int do_attend, size_t* bytes) {
  ChainPlan c;
  tls_status s = plan_chain(cfg, do_attend, c);
  if (s) return s;
  *bytes = c.total;
  return TLS_OK;
}

tls_status step_workspace(const tls_config* cfg, int do_attend, size_t* bytes) {
  tls::PStepParams sk;
  if (pstep_plan(cfg, do_attend, sk)) {
    *bytes = tls::pstep_workspace(sk, nullptr);
    return TLS_OK;
  }
  const int ns = n_split(cfg);
  size_t tot = 0;
  for (int s = 0; s < ns; ++s) {
    int b0;
    const tls_config sc = sub_config(cfg, ns, s, &b0);
    size_t w;
    tls_status st = chain_workspace(&sc, do_attend, &w);
    if (st) return st;
    tot += w;
  }
  *bytes = tot;
  return TLS_OK;
}

struct StepPtrs {
  const void* q;
  const void* k_cache;
  const void* v_cache;
  const int32_t* seq_lens;
  tls_index idx;
  const int32_t* guide;
  int32_t* block_ids;
  int32_t* token_ids;
  int32_t* num_tokens;
  float* token_scores;
  void* out;
  float* lse;
  const int32_t* slot_of_block;  // block cache (tls_decode_block_cache): K/V rows via the slot map, else NULL
  long long kv_rows;             // rows per pair of k_cache / v_cache (max_seq_len, or capacity * block_size)
  int pair0;                     // first pair of this (sub-)batch (diagnostic stamps only)
};

// The pointers of sub-batch [b0, b0 + n) (row-major layouts of tls.h).
StepPtrs offset_ptrs(const tls_config* c, const StepPtrs& a, int b0) {
  const size_t eb = elem_bytes(c), B0 = (size_t)b0, Hkv = (size_t)c->num_kv_heads, S = (size_t)c->max_seq_len;
  const size_t M = (S + c->block_size - 1) / c->block_size;
  StepPtrs r = a;
  auto adv = [](const void* p, size_t bytes) -> const char* {
    return p ? static_cast<const char*>(p) + bytes : nullptr;
  };
  r.q = adv(a.q, B0 * c->num_q_heads * c->d_k * eb);
  const size_t R = (size_t)a.kv_rows;
  r.k_cache = adv(a.k_cache, B0 * Hkv * R * c->d_k * eb);
  r.v_cache = adv(a.v_cache, B0 * Hkv * R * c->d_v * eb);
  r.slot_of_block = a.slot_of_block ? a.slot_of_block + B0 * Hkv * M : nullptr;
  r.seq_lens = a.seq_lens + b0;
  r.idx.block_minmax = const_cast<char*>(adv(a.idx.block_minmax, B0 * Hkv * M * 2 * c->d_k * eb));
  r.idx.codes = a.idx.codes + B0 * Hkv * S * (c->d_c / 2);
  r.idx.scale_zero = a.idx.scale_zero + B0 * Hkv * S * 2;
  r.guide = a.guide ? a.guide + B0 * Hkv * c->top_blocks : nullptr;
  r.block_ids = a.block_ids + B0 * Hkv * c->top_blocks;
  r.token_ids = a.token_ids + B0 * Hkv * c->top_tokens;
  r.num_tokens = a.num_tokens + B0 * Hkv;
  r.token_scores = a.token_scores ? a.token_scores + B0 * Hkv * c->top_tokens : nullptr;
  r.out = a.out ? const_cast<char*>(adv(a.out, B0 * c->num_q_heads * c->d_v * eb)) : nullptr;
  r.lse = a.lse ? a.lse + B0 * c->num_q_heads : nullptr;
  r.pair0 = a.pair0 + b0 * c->num_kv_heads;
  return r;
}

// Enqueue one chain for the pairs of `cfg` on stream st: select_kernel (a1-a2,
// or a1-a4 in mode 2), then in mode 1 the cluster token kernel (a3), then the
// attention kernel (a4 prologue in mode 1 + a5 when do_attend).  Arguments
// were validated by run_step.
std::atomic<unsigned> g_epoch{1u};

tls_status enqueue_chain(const tls_config* cfg, const StepPtrs& a, char* ws, int do_attend, cudaStream_t st,
                         const tls::LaunchOpts& lo_k1, const tls::LaunchOpts& lo_dep_in, bool timed) {
  ChainPlan c;
  tls_status s = plan_chain(cfg, do_attend, c);
  if (s) return s;
  // per-pair hand-off value of this call (never 0: consumers reset the flags to 0)
  unsigned epoch = g_epoch.fetch_add(1u);
  if (epoch == 0u) epoch = g_epoch.fetch_add(1u);
  // the token and attention kernels start under PDL unless events sit between the launches
  tls::LaunchOpts lo_dep = lo_dep_in;
  lo_dep.pdl = (!timed || !g_timer.on) && getenv("TLS_NO_PDL") == nullptr;
  tls::FusedParams& fp = c.fp;
  fp.sstride = fp.d.Ms;
  fp.q = a.q;
  fp.seq_lens = a.seq_lens;
  fp.block_minmax = a.idx.block_minmax;
  fp.channels = a.idx.channels;
  fp.scores = reinterpret_cast<float*>(ws + c.w.scores);
  fp.khist = reinterpret_cast<uint32_t*>(ws + c.w.khist);
  fp.qfrag = reinterpret_cast<uint8_t*>(ws + c.w.qfrag);
  fp.block_ids = a.block_ids;
  fp.ready = reinterpret_cast<unsigned*>(ws + c.w.ready_b);
  fp.tcount = reinterpret_cast<unsigned*>(ws + c.w.tcount);
  fp.sched = reinterpret_cast<unsigned*>(ws + c.w.sched);
  fp.epoch = epoch;
  fp.dbg = env_debug_buf();
  unsigned long long* dbg0 = fp.dbg;
  if (fp.dbg) fp.dbg += (size_t)a.pair0 * 16;
  fp.qq = reinterpret_cast<float*>(ws + c.w.qq);
  // small query groups (GQA, G * d_k <= 512 elements): every tile CTA forms QQ itself (the same fp32 ops as
  // qq_kernel, so the same bits) and starts streaming without waiting for qq_kernel (A/B: C2 79.0 -> 77.2 us;
  // at C3, G = 8, the per-tile work cost more than the wait: 127.4 -> 128.5)
  fp.qq_local = (cfg->layout == TLS_GQA && fp.d.G * cfg->d_k <= 512) ? 1 : 0;
  if (timed) g_timer.mark(st);
  cudaError_t e = tls::launch_qq(fp, st, lo_k1);
  if (e != cudaSuccess) return cuda_fail(e, "qq_kernel launch");
  tls::LaunchOpts lo_sel = lo_k1;
  lo_sel.pdl = lo_dep.pdl;  // select_kernel streams its tiles while qq_kernel finishes
  if (c.stream_sel) {
    const int tiles = cfg->batch * cfg->num_kv_heads * ((fp.d.M + fp.tb - 1) / fp.tb);
    // two CTAs per SM are launched; one per SM streams (the other exits at once: placement, fused.cu)
    (void)tiles;
    e = tls::launch_stream_select(fp, 2 * num_sms(), st, lo_sel);
    if (e != cudaSuccess) return cuda_fail(e, "stream_select_kernel launch");
  } else {
    e = tls::launch_select_fused(fp, st, lo_sel);
    if (e != cudaSuccess) return cuda_fail(e, "select_kernel launch");
  }
  if (timed) g_timer.mark(st);
  tls::SelectParams& sp = c.sp;
  if (c.mode == 1) {
    sp.q = a.q;
    sp.seq_lens = a.seq_lens;
    sp.scores = fp.scores;
    sp.codes = a.idx.codes;
    sp.scale_zero = a.idx.scale_zero;
    sp.channels = a.idx.channels;
    sp.guide = a.guide;
    sp.block_ids = a.block_ids;
    sp.keys = reinterpret_cast<uint32_t*>(ws + c.w.keys);
    sp.khist = fp.khist;
    sp.qfrag = fp.qfrag;
    sp.ready_in = fp.ready;
    sp.ready_out = reinterpret_cast<unsigned*>(ws + c.w.ready_t);
    sp.epoch = epoch;
    sp.dbg = dbg0 ? dbg0 + 65536 * 16 + (size_t)a.pair0 * 64 : nullptr;
    e = tls::launch_token_cluster(sp, st, lo_dep);
    if (e != cudaSuccess) return cuda_fail(e, "token_cluster_kernel launch");
  }
  if (timed) g_timer.mark(st);
  if (c.mode == 1 || do_attend) {
    tls::AttendParams& ap = c.ap;
    ap.q = a.q;
    ap.k_cache = a.k_cache;
    ap.v_cache = cfg->layout == TLS_MLA ? nullptr : a.v_cache;
    ap.kv_rows = a.kv_rows;
    ap.slot_of_block = a.slot_of_block;
    ap.seq_lens = a.seq_lens;
    ap.cand = a.guide ? a.guide : a.block_ids;
    ap.keys = sp.keys;
    ap.khist = sp.khist;
    ap.dbg = dbg0 ? dbg0 + 65536 * 24 + (size_t)a.pair0 * 8 : nullptr;
    ap.ready_in = c.mode == 1 ? sp.ready_out : nullptr;
    ap.ready_count = sp.nch;
    ap.epoch = epoch;
    ap.token_ids = a.token_ids;
    ap.num_tokens = a.num_tokens;
    ap.token_scores = a.token_scores;
    ap.out = a.out;
    ap.lse = a.lse;
    const size_t pairs = (size_t)cfg->batch * cfg->num_kv_heads;
    ap.part_o = reinterpret_cast<float*>(ws + c.w.total);
    ap.part_ml = reinterpret_cast<float*>(ws + c.w.total + tls::a256(pairs * ap.cs * ap.d.G * ap.d.d_v * 4));
    e = tls::launch_attend(ap, st, lo_dep);
    if (e != cudaSuccess) return cuda_fail(e, "attend_kernel launch");
  }
  if (timed) g_timer.mark(st);
  return TLS_OK;
}

// Internal streams / events of the sub-batch pipeline, per thread and device
// (created on first use, never destroyed: the library allocates no device
// memory, these are scheduling handles only).
struct Pipeline {
  int device = -1;
  cudaStream_t streams[8] = {};
  cudaEvent_t fork = nullptr, join[8] = {};
  int prio_lo = 0, prio_hi = 0;
};
thread_local Pipeline g_pipe[16];

tls_status pipeline_for_device(Pipeline** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 16) return fail(TLS_ERR_UNSUPPORTED, "device ordinal %d >= 16", dev);
  Pipeline& p = g_pipe[dev];
  if (p.device != dev) {
    e = cudaDeviceGetStreamPriorityRange(&p.prio_lo, &p.prio_hi);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetStreamPriorityRange");
    for (int i = 0; i < 8; ++i) {
      e = cudaStreamCreateWithFlags(&p.streams[i], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.join[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "pipeline stream/event creation");
    }
    e = cudaEventCreateWithFlags(&p.fork, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "pipeline event creation");
    p.device = dev;
  }
  *out = &p;
  return TLS_OK;
}

tls_status run_step(const tls_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                    const int32_t* seq_lens, const tls_index* idx, const int32_t* guide, int32_t* block_ids,
                    int32_t* token_ids, int32_t* num_tokens, float* token_scores, void* out, float* lse,
                    void* workspace, size_t workspace_bytes, int do_attend, cudaStream_t st,
                    const int32_t* slot_of_block = nullptr, long long kv_rows = 0) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!q || !aligned16(q)) return fail(TLS_ERR_INPUT, "q must be a non-NULL 16-byte aligned device pointer");
  if (!seq_lens || !block_ids || !token_ids || !num_tokens)
    return fail(TLS_ERR_INPUT, "seq_lens, block_ids, token_ids and num_tokens are required");
  s = check_index(idx);
  if (s) return s;
  if (do_attend) {
    if (!k_cache || !aligned16(k_cache)) return fail(TLS_ERR_INPUT, "k_cache must be a 16-byte aligned device pointer");
    if (cfg->layout == TLS_GQA && (!v_cache || !aligned16(v_cache)))
      return fail(TLS_ERR_INPUT, "GQA needs a 16-byte aligned v_cache");
    if (!out) return fail(TLS_ERR_INPUT, "out is required");
  }
  size_t need = 0;
  s = step_workspace(cfg, do_attend, &need);
  if (s) return s;
  if (!workspace || workspace_bytes < need || !aligned16(workspace))
    return fail(TLS_ERR_WORKSPACE, "workspace must be >= %zu bytes, 16-byte aligned (got %zu)", need, workspace_bytes);
  const StepPtrs all = {q, k_cache, v_cache, seq_lens, *idx, guide, block_ids, token_ids, num_tokens,
                        token_scores, out, lse, slot_of_block, kv_rows > 0 ? kv_rows : cfg->max_seq_len, 0};
  if (g_timer.on && g_timer.used % kMarks != 0) g_timer.used -= g_timer.used % kMarks;  // drop a partial record
  tls::PStepParams sk;
  if (pstep_plan(cfg, do_attend, sk)) {  // one launch: every stage of every pair (opt-in, TLS_PSTEP)
    if (guide != nullptr || slot_of_block != nullptr)
      return fail(TLS_ERR_UNSUPPORTED, "the persistent step kernel (TLS_PSTEP) has no lag / block-cache mode");
    tls::pstep_workspace(sk, static_cast<char*>(workspace));
    unsigned epoch = g_epoch.fetch_add(1u);
    if (epoch == 0u) epoch = g_epoch.fetch_add(1u);
    sk.epoch = epoch;
    sk.q = q;
    sk.seq_lens = seq_lens;
    sk.block_minmax = idx->block_minmax;
    sk.codes = idx->codes;
    sk.scale_zero = idx->scale_zero;
    sk.channels = idx->channels;
    sk.guide = guide;
    sk.k_cache = k_cache;
    sk.v_cache = v_cache;
    sk.kv_rows = kv_rows > 0 ? kv_rows : cfg->max_seq_len;
    sk.slot_of_block = slot_of_block;
    sk.block_ids = block_ids;
    sk.token_ids = token_ids;
    sk.num_tokens = num_tokens;
    sk.token_scores = token_scores;
    sk.out = out;
    sk.lse = lse;
    sk.dbg = env_debug_buf();
    const int occ = tls::pstep_occupancy(sk.smem_bytes);
    if (occ < 1) return fail(TLS_ERR_UNSUPPORTED, "persistent step kernel does not fit on an SM");
    const int grid = num_sms() * occ;
    sk.nstream = num_sms();  // one streamer per SM (the first wave places blockIdx 0..SMs-1 on distinct SMs)
    g_timer.mark(st);
    cudaError_t e = tls::launch_pstep(sk, grid, st);
    if (e != cudaSuccess) return cuda_fail(e, "pstep_kernel launch");
    for (int k = 1; k < kMarks; ++k) g_timer.mark(st);  // one launch: slot 0 holds the whole step
    return TLS_OK;
  }
  char* ws = static_cast<char*>(workspace);
  const int ns = n_split(cfg);
  if (ns == 1) return enqueue_chain(cfg, all, ws, do_attend, st, tls::LaunchOpts{}, tls::LaunchOpts{}, true);
  Pipeline* pl = nullptr;
  s = pipeline_for_device(&pl);
  if (s) return s;
  // per-kernel timing is not defined for overlapped chains: the record spans the whole step
  g_timer.mark(st);
  cudaError_t e = cudaEventRecord(pl->fork, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord(fork)");
  tls::LaunchOpts lo_k1, lo_dep;
  lo_k1.use_prio = lo_dep.use_prio = 1;
  lo_k1.prio = pl->prio_lo;
  lo_dep.prio = pl->prio_hi;
  for (int i = 0; i < ns; ++i) {
    e = cudaStreamWaitEvent(pl->streams[i], pl->fork, 0);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent(fork)");
    int b0;
    const tls_config sc = sub_config(cfg, ns, i, &b0);
    size_t w;
    s = chain_workspace(&sc, do_attend, &w);
    if (s) return s;
    s = enqueue_chain(&sc, offset_ptrs(cfg, all, b0), ws, do_attend, pl->streams[i], lo_k1, lo_dep, false);
    if (s) return s;
    ws += w;
    e = cudaEventRecord(pl->join[i], pl->streams[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, pl->join[i], 0);
    if (e != cudaSuccess) return cuda_fail(e, "pipeline join");
  }
  for (int k = 1; k < kMarks; ++k) g_timer.mark(st);
  return TLS_OK;
}

tls_status run_attend(const tls_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                      const int32_t* token_ids, const int32_t* num_tokens, void* out, float* lse, void* workspace,
                      size_t workspace_bytes, cudaStream_t st, int out_f32 = 0) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!q || !aligned16(q)) return fail(TLS_ERR_INPUT, "q must be a non-NULL 16-byte aligned device pointer");
  if (!token_ids || !num_tokens || !out) return fail(TLS_ERR_INPUT, "token_ids, num_tokens and out are required");
  if (!k_cache || !aligned16(k_cache)) return fail(TLS_ERR_INPUT, "k_cache must be a 16-byte aligned device pointer");
  if (cfg->layout == TLS_GQA && (!v_cache || !aligned16(v_cache)))
    return fail(TLS_ERR_INPUT, "GQA needs a 16-byte aligned v_cache");
  tls::AttendParams ap;
  s = plan_attend(cfg, ap, 0, 1);
  if (s) return s;
  const size_t need = tls::attend_workspace_bytes(ap.d, ap.cs);
  if (!workspace || workspace_bytes < need || !aligned16(workspace))
    return fail(TLS_ERR_WORKSPACE, "attention workspace must be >= %zu bytes, 16-byte aligned (got %zu)", need,
                workspace_bytes);
  ap.q = q;
  ap.k_cache = k_cache;
  ap.v_cache = cfg->layout == TLS_MLA ? nullptr : v_cache;
  ap.kv_rows = cfg->max_seq_len;
  ap.token_ids = const_cast<int32_t*>(token_ids);
  ap.num_tokens = const_cast<int32_t*>(num_tokens);
  ap.out = out;
  ap.out_f32 = out_f32;
  ap.lse = lse;
  const size_t pairs = (size_t)cfg->batch * cfg->num_kv_heads;
  ap.part_o = static_cast<float*>(workspace);
  ap.part_ml = reinterpret_cast<float*>(static_cast<char*>(workspace) +
                                        tls::a256(pairs * ap.cs * ap.d.G * ap.d.d_v * 4));
  cudaError_t e = tls::launch_attend(ap, st, tls::LaunchOpts{});
  if (e != cudaSuccess) return cuda_fail(e, "attend_kernel launch");
  return TLS_OK;
}

size_t attend_ws(const tls_config* cfg, int select) {
  tls::AttendParams ap;
  if (plan_attend(cfg, ap, select, 1) != TLS_OK) return (size_t)-1;
  return tls::attend_workspace_bytes(ap.d, ap.cs);
}

}  // namespace

extern "C" {

tls_status tls_calibrate_channels(const tls_config* cfg, const void* q_cal, int32_t n_q, const void* k_cal,
                                  int32_t n_k, int64_t k_head_stride, int32_t* channels_out, float* channel_scores,
                                  tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (n_q < 1 || n_k < 1) return fail(TLS_ERR_INPUT, "empty calibration set (n_q=%d, n_k=%d)", n_q, n_k);
  if (!q_cal || !k_cal || !channels_out) return fail(TLS_ERR_INPUT, "q_cal, k_cal and channels_out are required");
  if (cfg->d_k > 8192) return fail(TLS_ERR_UNSUPPORTED, "d_k too large for calibration");
  tls::CalibParams p;
  p.Hq = cfg->num_q_heads;
  p.Hkv = cfg->num_kv_heads;
  p.G = cfg->num_q_heads / cfg->num_kv_heads;
  p.d_k = cfg->d_k;
  p.d_c = cfg->d_c;
  p.n_q = n_q;
  p.n_k = n_k;
  p.k_head_stride = k_head_stride;
  p.q_cal = q_cal;
  p.k_cal = k_cal;
  p.channels_out = channels_out;
  p.channel_scores = channel_scores;
  cudaError_t e = tls::launch_calibrate(p, cfg->dtype == TLS_BF16, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "calibrate kernel launch");
  return TLS_OK;
}

tls_status tls_build_index(const tls_config* cfg, const void* k_cache, const int32_t* seq_lens, int32_t start_token,
                           const tls_index* idx, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  s = check_index(idx);
  if (s) return s;
  if (!k_cache || !seq_lens) return fail(TLS_ERR_INPUT, "k_cache and seq_lens are required");
  if (start_token < 0 || start_token >= cfg->max_seq_len)
    return fail(TLS_ERR_INPUT, "start_token %d outside [0, max_seq_len)", start_token);
  tls::IndexParams p;
  p.batch = cfg->batch;
  p.Hkv = cfg->num_kv_heads;
  p.d_k = cfg->d_k;
  p.S = cfg->max_seq_len;
  p.B = cfg->block_size;
  p.d_c = cfg->d_c;
  p.M = (cfg->max_seq_len + cfg->block_size - 1) / cfg->block_size;
  p.start_block = start_token / cfg->block_size;
  p.k_cache = k_cache;
  p.seq_lens = seq_lens;
  p.block_minmax = idx->block_minmax;
  p.codes = idx->codes;
  p.scale_zero = idx->scale_zero;
  p.channels = idx->channels;
  cudaError_t e = tls::launch_build_index(p, cfg->dtype == TLS_BF16, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "build_index kernel launch");
  return TLS_OK;
}

tls_status tls_block_scores(const tls_config* cfg, const void* q, const int32_t* seq_lens,
                            const void* block_minmax, float* scores, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!q || !aligned16(q)) return fail(TLS_ERR_INPUT, "q must be a non-NULL 16-byte aligned device pointer");
  if (!seq_lens || !block_minmax || !scores || !aligned16(block_minmax))
    return fail(TLS_ERR_INPUT, "seq_lens, block_minmax (16-byte aligned) and scores are required");
  tls::FusedParams fp;
  memset(&fp, 0, sizeof(fp));
  fp.d = dims_of(cfg);
  fp.mode = 0;
  fp.tb = score_tile_rows(2 * cfg->d_k * (int)elem_bytes(cfg));
  if (fp.tb < 1) return fail(TLS_ERR_UNSUPPORTED, "block summary row larger than the K1 tile");
  tls::plan_fused(fp, sizeof(tls::FastTopKCtl));
  fp.sstride = fp.d.M;
  fp.q = q;
  fp.seq_lens = seq_lens;
  fp.block_minmax = block_minmax;
  fp.scores = scores;
  cudaError_t e = tls::launch_select_fused(fp, (cudaStream_t)stream, tls::LaunchOpts{});
  if (e != cudaSuccess) return cuda_fail(e, "select_kernel launch");
  return TLS_OK;
}

// ---- sequence-split decode (seqsplit.cu)
tls_status tls_topk_rows(int32_t rows, int32_t n, const float* keys, const int32_t* ids, int32_t k,
                         float* out_keys, int32_t* out_ids, int32_t* out_count, tls_stream_t stream) {
  if (rows < 1 || n < 1 || k < 1) return fail(TLS_ERR_INPUT, "rows, n and k must be >= 1");
  if (!keys || !ids || !out_keys || !out_ids) return fail(TLS_ERR_INPUT, "keys, ids, out_keys, out_ids are required");
  cudaError_t e = tls::launch_topk_rows(rows, n, keys, ids, k, out_keys, out_ids, out_count, 0, nullptr, 1, 1,
                                        (cudaStream_t)stream);
  return e == cudaSuccess ? TLS_OK : cuda_fail(e, "topk_rows_kernel launch");
}

tls_status tls_block_topk(const tls_config* cfg, const float* scores, const int32_t* seq_lens, int32_t block_offset,
                          float* out_scores, int32_t* out_block_ids, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!scores || !seq_lens || !out_scores || !out_block_ids)
    return fail(TLS_ERR_INPUT, "scores, seq_lens, out_scores and out_block_ids are required");
  if (block_offset < 0) return fail(TLS_ERR_INPUT, "block_offset must be >= 0");
  const tls::Dims d = dims_of(cfg);
  cudaError_t e = tls::launch_topk_rows(cfg->batch * cfg->num_kv_heads, d.M, scores, nullptr, cfg->top_blocks,
                                        out_scores, out_block_ids, nullptr, block_offset, seq_lens, cfg->num_kv_heads,
                                        cfg->block_size, (cudaStream_t)stream);
  return e == cudaSuccess ? TLS_OK : cuda_fail(e, "topk_rows_kernel launch");
}

tls_status tls_select_range(int32_t rows, int32_t k, const int32_t* ids, int32_t lo, int32_t hi,
                            int32_t* out_ids, int32_t* out_count, tls_stream_t stream) {
  if (rows < 1 || k < 1 || lo > hi) return fail(TLS_ERR_INPUT, "rows, k >= 1 and lo <= hi required");
  if (!ids || !out_ids) return fail(TLS_ERR_INPUT, "ids and out_ids are required");
  cudaError_t e = tls::launch_select_range(rows, k, ids, lo, hi, out_ids, out_count, (cudaStream_t)stream);
  return e == cudaSuccess ? TLS_OK : cuda_fail(e, "select_range_kernel launch");
}

tls_status tls_expand_blocks(const tls_config* cfg, const int32_t* block_ids, const int32_t* seq_lens,
                             int32_t k_out, int32_t* token_ids, int32_t* num_tokens, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!block_ids || !seq_lens || !token_ids || !num_tokens || k_out < 1)
    return fail(TLS_ERR_INPUT, "block_ids, seq_lens, token_ids, num_tokens and k_out >= 1 are required");
  if (cfg->top_blocks > 1024) return fail(TLS_ERR_UNSUPPORTED, "top_blocks > 1024");
  cudaError_t e = tls::launch_expand_blocks(dims_of(cfg), block_ids, seq_lens, k_out, token_ids, num_tokens,
                                            (cudaStream_t)stream);
  return e == cudaSuccess ? TLS_OK : cuda_fail(e, "expand_blocks_kernel launch");
}

tls_status tls_block_iota(const tls_config* cfg, const int32_t* seq_lens, int32_t* block_ids, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!seq_lens || !block_ids) return fail(TLS_ERR_INPUT, "seq_lens and block_ids are required");
  cudaError_t e = tls::launch_block_iota(dims_of(cfg), seq_lens, block_ids, (cudaStream_t)stream);
  return e == cudaSuccess ? TLS_OK : cuda_fail(e, "block_iota_kernel launch");
}

namespace {
tls_status token_split(const tls_config* cfg, int mode, const void* q, const int32_t* seq_lens, const tls_index* idx,
                       const int32_t* block_ids, int32_t n_parts, const float* stats_in, float* stats_out,
                       float* keys, int32_t* token_ids, int32_t token_offset, cudaStream_t st) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!q || !seq_lens || !idx || !idx->codes || !idx->scale_zero || !idx->channels || !block_ids)
    return fail(TLS_ERR_INPUT, "q, seq_lens, the token index and block_ids are required");
  const tls::Dims d = dims_of(cfg);
  if (tls::token_split_smem(d) > (size_t)kMaxSmem) return fail(TLS_ERR_UNSUPPORTED, "q~ of the group too large");
  if (mode == 0 && !stats_out) return fail(TLS_ERR_INPUT, "stats is required");
  if (mode == 1 && (n_parts < 1 || !stats_in || !keys || !token_ids))
    return fail(TLS_ERR_INPUT, "n_parts >= 1, stats_parts, keys and token_ids are required");
  cudaError_t e = tls::launch_token_split(d, mode, q, seq_lens, idx->codes, idx->scale_zero, idx->channels,
                                          block_ids, n_parts, stats_in, stats_out, keys, token_ids, token_offset, st);
  return e == cudaSuccess ? TLS_OK : cuda_fail(e, "token_split_kernel launch");
}
}  // namespace

tls_status tls_token_stats(const tls_config* cfg, const void* q, const int32_t* seq_lens, const tls_index* idx,
                           const int32_t* block_ids, float* stats, tls_stream_t stream) {
  return token_split(cfg, 0, q, seq_lens, idx, block_ids, 1, nullptr, stats, nullptr, nullptr, 0,
                     (cudaStream_t)stream);
}

tls_status tls_token_keys(const tls_config* cfg, const void* q, const int32_t* seq_lens, const tls_index* idx,
                          const int32_t* block_ids, int32_t n_parts, const float* stats_parts,
                          int32_t token_offset, float* keys, int32_t* token_ids, tls_stream_t stream) {
  return token_split(cfg, 1, q, seq_lens, idx, block_ids, n_parts, stats_parts, nullptr, keys, token_ids,
                     token_offset, (cudaStream_t)stream);
}

tls_status tls_attn_merge(const tls_config* cfg, int32_t n_parts, const float* parts_out, const float* parts_lse,
                          void* out, float* lse, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (n_parts < 1 || !parts_out || !parts_lse || !out)
    return fail(TLS_ERR_INPUT, "n_parts >= 1, parts_out, parts_lse and out are required");
  cudaError_t e = tls::launch_attn_merge(cfg->dtype == TLS_BF16, n_parts, cfg->batch * cfg->num_q_heads, cfg->d_v,
                                         parts_out, parts_lse, out, lse, (cudaStream_t)stream);
  return e == cudaSuccess ? TLS_OK : cuda_fail(e, "attn_merge_kernel launch");
}

tls_status tls_select(const tls_config* cfg, const void* q, const int32_t* seq_lens, const tls_index* idx,
                      const int32_t* guide_block_ids, int32_t* block_ids, int32_t* token_ids, int32_t* num_tokens,
                      float* token_scores, void* workspace, size_t workspace_bytes, tls_stream_t stream) {
  return run_step(cfg, q, nullptr, nullptr, seq_lens, idx, guide_block_ids, block_ids, token_ids, num_tokens,
                  token_scores, nullptr, nullptr, workspace, workspace_bytes, 0, (cudaStream_t)stream);
}

tls_status tls_sparse_attend(const tls_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                             const int32_t* token_ids, const int32_t* num_tokens, void* out, float* lse,
                             void* workspace, size_t workspace_bytes, tls_stream_t stream) {
  return run_attend(cfg, q, k_cache, v_cache, token_ids, num_tokens, out, lse, workspace, workspace_bytes,
                    (cudaStream_t)stream);
}

tls_status tls_sparse_attend_f32(const tls_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                                 const int32_t* token_ids, const int32_t* num_tokens, float* out, float* lse,
                                 void* workspace, size_t workspace_bytes, tls_stream_t stream) {
  return run_attend(cfg, q, k_cache, v_cache, token_ids, num_tokens, out, lse, workspace, workspace_bytes,
                    (cudaStream_t)stream, 1);
}

tls_status tls_decode(const tls_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                      const int32_t* seq_lens, const tls_index* idx, const int32_t* guide_block_ids,
                      int32_t* block_ids, int32_t* token_ids, int32_t* num_tokens, float* token_scores, void* out,
                      float* lse, void* workspace, size_t workspace_bytes, tls_stream_t stream) {
  return run_step(cfg, q, k_cache, v_cache, seq_lens, idx, guide_block_ids, block_ids, token_ids, num_tokens,
                  token_scores, out, lse, workspace, workspace_bytes, 1, (cudaStream_t)stream);
}

tls_status tls_decode_block_cache(const tls_config* cfg, const void* q, const int32_t* seq_lens, const tls_index* idx,
                                  const int32_t* guide_block_ids, const tls_block_cache* cache, int32_t* block_ids,
                                  int32_t* token_ids, int32_t* num_tokens, float* token_scores, void* out,
                                  float* lse, void* workspace, size_t workspace_bytes, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!cache || !cache->k_slots || !cache->slot_of_block || !cache->block_of_slot)
    return fail(TLS_ERR_INPUT, "block cache buffers must be non-NULL");
  if (cfg->layout == TLS_GQA && !cache->v_slots) return fail(TLS_ERR_INPUT, "GQA needs v_slots");
  if (cache->capacity < 1) return fail(TLS_ERR_CONFIG, "block cache capacity must be >= 1");
  // only the lag-mode candidates M_{t-1} are guaranteed resident: M_t is fetched after this step
  if (!guide_block_ids) return fail(TLS_ERR_INPUT, "tls_decode_block_cache needs guide_block_ids (M_{t-1}, P:373)");
  return run_step(cfg, q, cache->k_slots, cache->v_slots, seq_lens, idx, guide_block_ids, block_ids, token_ids,
                  num_tokens, token_scores, out, lse, workspace, workspace_bytes, 1, (cudaStream_t)stream,
                  cache->slot_of_block, (long long)cache->capacity * cfg->block_size);
}

size_t tls_workspace_bytes(const tls_config* cfg, int32_t which) {
  if (check_config(cfg) != TLS_OK || which < 0 || which > 2) return (size_t)-1;
  if (which == 1) return attend_ws(cfg, 0);
  size_t w = 0;
  if (step_workspace(cfg, which == 2, &w) != TLS_OK) return (size_t)-1;
  return w;
}

tls_status tls_workspace_init(const tls_config* cfg, int32_t which, void* workspace, size_t workspace_bytes,
                              tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (which < 0 || which > 2) return fail(TLS_ERR_INPUT, "which must be 0, 1 or 2");
  const size_t need = tls_workspace_bytes(cfg, which);
  if (need == (size_t)-1) return fail(TLS_ERR_CONFIG, "invalid configuration");
  if (!workspace || workspace_bytes < need) return fail(TLS_ERR_WORKSPACE, "workspace must be >= %zu bytes", need);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(workspace, 0, need, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  tls::PStepParams sk;
  if (which == 1) return TLS_OK;  // counters start at 0
  if (pstep_plan(cfg, which == 2, sk)) {  // counters start at 0, block scores as the completion sentinel
    tls::pstep_workspace(sk, static_cast<char*>(workspace));
    e = cudaMemsetAsync(sk.scores, 0xff, (size_t)sk.pairs * sk.d.Ms * 4, st);
    return e == cudaSuccess ? TLS_OK : cuda_fail(e, "cudaMemsetAsync");
  }
  // every chain's block-score buffer starts as the completion sentinel (fused.cu kScoreSentinel)
  char* ws = static_cast<char*>(workspace);
  const int ns = n_split(cfg);
  for (int i = 0; i < ns; ++i) {
    int b0;
    const tls_config sc = sub_config(cfg, ns, i, &b0);
    ChainPlan c;
    s = plan_chain(&sc, which == 2, c);
    if (s) return s;
    e = cudaMemsetAsync(ws + c.w.scores, 0xff, (size_t)sc.batch * sc.num_kv_heads * c.fp.d.Ms * 4, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
    ws += c.total;
  }
  return TLS_OK;
}

tls_status tls_cache_fetch(const tls_config* cfg, const void* k_host, const void* v_host, const int32_t* token_ids,
                           const int32_t* num_tokens, const tls_token_cache* cache, int32_t* slot_ids,
                           int32_t* miss_count, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!cache || !cache->k_slots || !cache->slot_of_token || !cache->token_of_slot)
    return fail(TLS_ERR_INPUT, "cache buffers must be non-NULL");
  if (cfg->layout == TLS_GQA && (!cache->v_slots || !v_host)) return fail(TLS_ERR_INPUT, "GQA needs v_host and v_slots");
  if (!k_host || !token_ids || !num_tokens || !slot_ids)
    return fail(TLS_ERR_INPUT, "k_host, token_ids, num_tokens and slot_ids are required");
  if (cache->capacity < cfg->top_tokens)
    return fail(TLS_ERR_CONFIG, "cache capacity (%d) must be >= top_tokens (%d)", cache->capacity, cfg->top_tokens);
  // the host caches must be reachable from the device (pinned + mapped, or managed / device memory)
  const void* dk = nullptr;
  const void* dv = nullptr;
  for (int i = 0; i < 2; ++i) {
    const void* h = i == 0 ? k_host : v_host;
    if (!h) continue;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, h);
    if (e != cudaSuccess || at.devicePointer == nullptr)
      return fail(TLS_ERR_INPUT, "k_host / v_host must be pinned, device-mapped host memory (cudaHostAlloc mapped)");
    (i == 0 ? dk : dv) = at.devicePointer;
  }
  tls::CacheFetchParams p;
  memset(&p, 0, sizeof(p));
  p.d = dims_of(cfg);
  p.capacity = cache->capacity;
  p.bitmap_words = (cfg->max_seq_len + 31) / 32;
  const size_t smem = (size_t)p.bitmap_words * 4 + (size_t)p.capacity * 4 + (size_t)cfg->top_tokens * 4;
  if ((int)smem > kMaxSmem) return fail(TLS_ERR_UNSUPPORTED, "cache_fetch shared-memory plan does not fit");
  p.k_host = static_cast<const uint8_t*>(dk);
  p.v_host = cfg->layout == TLS_GQA ? static_cast<const uint8_t*>(dv) : nullptr;
  p.token_ids = token_ids;
  p.num_tokens = num_tokens;
  p.k_slots = static_cast<uint8_t*>(cache->k_slots);
  p.v_slots = cfg->layout == TLS_GQA ? static_cast<uint8_t*>(cache->v_slots) : nullptr;
  p.slot_of_token = cache->slot_of_token;
  p.token_of_slot = cache->token_of_slot;
  p.slot_ids = slot_ids;
  p.miss_count = miss_count;
  cudaError_t e = tls::launch_cache_fetch(p, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "cache_fetch_kernel launch");
  return TLS_OK;
}

static tls_status host_device_ptr(const void* h, const void** dptr) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, h);
  if (e != cudaSuccess || at.devicePointer == nullptr)
    return fail(TLS_ERR_INPUT, "k_host / v_host must be pinned, device-mapped host memory (cudaHostAlloc mapped)");
  *dptr = at.devicePointer;
  return TLS_OK;
}

static tls_status check_block_cache(const tls_config* cfg, const tls_block_cache* cache) {
  if (!cache || !cache->k_slots || !cache->slot_of_block || !cache->block_of_slot)
    return fail(TLS_ERR_INPUT, "block cache buffers must be non-NULL");
  if (cfg->layout == TLS_GQA && !cache->v_slots) return fail(TLS_ERR_INPUT, "GQA needs v_slots");
  if (cache->capacity < 2 * cfg->top_blocks)
    return fail(TLS_ERR_CONFIG, "block cache capacity (%d) must be >= 2 * top_blocks (%d)", cache->capacity,
                2 * cfg->top_blocks);
  return TLS_OK;
}

tls_status tls_block_cache_update(const tls_config* cfg, const void* k_host, const void* v_host,
                                  const int32_t* keep_block_ids, const int32_t* block_ids,
                                  const tls_block_cache* cache, int32_t* miss_count, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if ((s = check_block_cache(cfg, cache))) return s;
  if (!k_host || !block_ids) return fail(TLS_ERR_INPUT, "k_host and block_ids are required");
  if (cfg->layout == TLS_GQA && !v_host) return fail(TLS_ERR_INPUT, "GQA needs v_host");
  tls::BlockCacheParams p;
  memset(&p, 0, sizeof(p));
  p.d = dims_of(cfg);
  const void* dk = nullptr;
  const void* dv = nullptr;
  if ((s = host_device_ptr(k_host, &dk))) return s;
  if (cfg->layout == TLS_GQA && (s = host_device_ptr(v_host, &dv))) return s;
  p.capacity = cache->capacity;
  p.bitmap_words = (p.d.M + 31) / 32;
  const size_t smem = (size_t)p.bitmap_words * 4 + (size_t)p.capacity * 4 + (size_t)cfg->top_blocks * 4;
  if ((int)smem > kMaxSmem) return fail(TLS_ERR_UNSUPPORTED, "block cache shared-memory plan does not fit");
  p.k_host = static_cast<const uint8_t*>(dk);
  p.v_host = cfg->layout == TLS_GQA ? static_cast<const uint8_t*>(dv) : nullptr;
  p.keep_ids = keep_block_ids;
  p.block_ids = block_ids;
  p.k_slots = static_cast<uint8_t*>(cache->k_slots);
  p.v_slots = cfg->layout == TLS_GQA ? static_cast<uint8_t*>(cache->v_slots) : nullptr;
  p.slot_of_block = cache->slot_of_block;
  p.block_of_slot = cache->block_of_slot;
  p.miss_count = miss_count;
  cudaError_t e = tls::launch_block_cache_update(p, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "block_cache_update_kernel launch");
  return TLS_OK;
}

tls_status tls_block_cache_rows(const tls_config* cfg, const int32_t* token_ids, const int32_t* num_tokens,
                                const tls_block_cache* cache, int32_t* slot_rows, int32_t* absent,
                                tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if ((s = check_block_cache(cfg, cache))) return s;
  if (!token_ids || !num_tokens || !slot_rows) return fail(TLS_ERR_INPUT, "token_ids, num_tokens, slot_rows required");
  tls::BlockCacheParams p;
  memset(&p, 0, sizeof(p));
  p.d = dims_of(cfg);
  p.capacity = cache->capacity;
  p.slot_of_block = cache->slot_of_block;
  p.block_of_slot = cache->block_of_slot;
  p.token_ids = token_ids;
  p.num_tokens = num_tokens;
  p.slot_rows = slot_rows;
  p.absent = absent;
  cudaError_t e = tls::launch_block_cache_rows(p, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "block_cache_rows_kernel launch");
  return TLS_OK;
}

int32_t tls_launch_count(const tls_config* cfg, int32_t which) {
  if (check_config(cfg) != TLS_OK) return -1;
  tls::PStepParams sk;
  if ((which == 0 || which == 2) && pstep_plan(cfg, which == 2, sk)) return 1;  // pstep_kernel
  const int mode = fused_mode(cfg), ns = n_split(cfg);
  switch (which) {
    case 0: return ns * (mode == 2 ? 1 : 4);  // qq, select, token and attend (selection prologue only) kernels
    case 1: return 1;                         // attend_kernel
    case 2: return ns * (mode == 2 ? 2 : 4);  // qq, select, token and attend kernels
    case 3: return 1;  // build_index_kernel
    case 4: return 1;  // calibrate_kernel
    default: return -1;
  }
}

int32_t tls_select_mode(const tls_config* cfg) {
  if (check_config(cfg) != TLS_OK) return -1;
  tls::PStepParams sk;
  if (pstep_plan(cfg, 1, sk)) return 3;  // the persistent step kernel
  return fused_mode(cfg);
}

int32_t tls_cluster_size(const tls_config* cfg, int32_t which) {
  if (check_config(cfg) != TLS_OK || which < 0 || which > 5) return -1;
  if (which == 5) {  // the token kernel's form: 1 / 4 token_pair_kernel with 1 / 2 CTAs per pair, 2 register
                     // cluster, 3 two-pass cluster
    tls::SelectParams sp;
    if (fused_mode(cfg) != 1 || plan_select(cfg, sp) != TLS_OK) return -1;
    return sp.pairk == 1 ? 1 : (sp.pairk == 2 ? 4 : (sp.pairk == 4 ? 5 : (sp.pairk >= 8 ? 6 : (sp.tpw > 0 ? 2 : 3))));
  }
  if (which == 3 || which == 4) {  // tls_sparse_attend's attention plan
    tls::AttendParams ap;
    if (plan_attend(cfg, ap, 0, 1) != TLS_OK) return -1;
    if (which == 4) return ap.mma == 3 ? 3 : (ap.mma ? 2 : 1);  // tcgen05 | mma.sync | CUDA cores
    return cfg->layout == TLS_MLA ? ap.mla_tc : 0;             // MLA tokens per staged chunk
  }
  tls::PStepParams sk;
  if (which != 1 && pstep_plan(cfg, 1, sk)) return sk.ns;  // attention slices per pair
  tls::AttendParams ap;
  return plan_attend(cfg, ap, which != 1, which != 0) == TLS_OK ? ap.cs : -1;
}

tls_status tls_timing_enable(int32_t n_calls) {
  if (n_calls < 0) return fail(TLS_ERR_INPUT, "n_calls must be >= 0");
  g_timer.used = 0;
  if (n_calls == 0) {
    cudaDeviceSynchronize();
    for (cudaEvent_t e : g_timer.ev) cudaEventDestroy(e);
    g_timer.ev.clear();
    g_timer.on = false;
    return TLS_OK;
  }
  while (g_timer.ev.size() < (size_t)n_calls * kMarks) {
    cudaEvent_t e;
    cudaError_t err = cudaEventCreate(&e);
    if (err != cudaSuccess) return cuda_fail(err, "cudaEventCreate");
    g_timer.ev.push_back(e);
  }
  g_timer.on = true;
  return TLS_OK;
}

tls_status tls_timing_read(double* ms_sum, int64_t* calls) {
  if (!ms_sum || !calls) return fail(TLS_ERR_INPUT, "ms_sum and calls are required");
  const size_t n = g_timer.used / kMarks;
  for (int k = 0; k < kMarks - 1; ++k) ms_sum[k] = 0.0;
  for (size_t c = 0; c < n; ++c) {
    for (int k = 0; k < kMarks - 1; ++k) {
      cudaEvent_t a = g_timer.ev[c * kMarks + k], b = g_timer.ev[c * kMarks + k + 1];
      cudaError_t err = cudaEventSynchronize(b);
      if (err != cudaSuccess) return cuda_fail(err, "cudaEventSynchronize");
      float ms = 0.f;
      err = cudaEventElapsedTime(&ms, a, b);
      if (err != cudaSuccess) return cuda_fail(err, "cudaEventElapsedTime");
      ms_sum[k] += ms;
    }
  }
  *calls = (int64_t)n;
  g_timer.used = 0;
  return TLS_OK;
}

const char* tls_status_string(tls_status status) {
  switch (status) {
    case TLS_OK: return "TLS_OK";
    case TLS_ERR_DIM: return "TLS_ERR_DIM";
    case TLS_ERR_CONFIG: return "TLS_ERR_CONFIG";
    case TLS_ERR_INPUT: return "TLS_ERR_INPUT";
    case TLS_ERR_WORKSPACE: return "TLS_ERR_WORKSPACE";
    case TLS_ERR_UNSUPPORTED: return "TLS_ERR_UNSUPPORTED";
    case TLS_ERR_CUDA: return "TLS_ERR_CUDA";
  }
  return "TLS_ERR_UNKNOWN";
}

const char* tls_last_error(void) { return g_err; }

const char* tls_version(void) { return "tls-b200 0.1 (sm_100a)"; }

}  // extern "C"
