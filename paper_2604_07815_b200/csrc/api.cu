// api.cu -- the C ABI of libtls.so (declared in include/tls.h): argument
// validation, launch planning and dispatch.  No device memory is allocated and
// no global state is kept besides the thread-local error string.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "../../include/tls.h"
#include "decode.h"

#include "index.h"

namespace tls {
cudaError_t launch_decode(const DecodeParams& p, bool bf16, cudaStream_t stream);
int decode_cpl(int d_k, size_t elem_bytes);
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

constexpr int kMaxSmem = 227 * 1024 - 8 * 1024;  // dynamic budget (static Ctl ~5 KB)

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
  if (c->d_c % 32 || c->d_c > 128) return fail(TLS_ERR_UNSUPPORTED, "d_c must be a multiple of 32 and <= 128");
  if (c->block_size % 16 || c->block_size > 1024) return fail(TLS_ERR_UNSUPPORTED, "block_size must be a multiple of 16, <= 1024");
  const int G = c->num_q_heads / c->num_kv_heads;
  if (G > 64) return fail(TLS_ERR_UNSUPPORTED, "at most 64 query heads per KV head");
  if ((long long)c->batch * c->num_kv_heads > 65535) return fail(TLS_ERR_UNSUPPORTED, "batch*num_kv_heads > 65535");
  if (tls::decode_cpl(c->d_k, eb) < 0) return fail(TLS_ERR_UNSUPPORTED, "d_k too large for the block-score kernel");
  return TLS_OK;
}

void fill_dims(const tls_config* c, tls::DecodeParams& p) {
  memset(&p, 0, sizeof(p));
  p.batch = c->batch;
  p.Hq = c->num_q_heads;
  p.Hkv = c->num_kv_heads;
  p.G = c->num_q_heads / c->num_kv_heads;
  p.d_k = c->d_k;
  p.d_v = c->d_v;
  p.S = c->max_seq_len;
  p.B = c->block_size;
  p.d_c = c->d_c;
  p.Kb = c->top_blocks;
  p.Kt = c->top_tokens;
  p.M = (c->max_seq_len + c->block_size - 1) / c->block_size;
  p.sm_scale = c->sm_scale;
  p.mla = c->layout == TLS_MLA;
  p.nsplit = c->dtype == TLS_BF16 ? 1 : 3;
}

// Cluster size (CTAs per pair): enough CTAs to cover the 148 SMs a few times,
// and a shared-memory footprint that fits.  TLS_CLUSTER overrides (tuning).
tls_status plan(const tls_config* c, tls::DecodeParams& p, int do_select, int do_attend) {
  fill_dims(c, p);
  p.do_select = do_select;
  p.do_attend = do_attend;
  const long long pairs = (long long)c->batch * c->num_kv_heads;
  int cs = 1;
  const char* env = getenv("TLS_CLUSTER");
  if (env && atoi(env) > 0) {
    cs = atoi(env);
  } else {
    while (cs < 8 && pairs * cs < 4 * 148) cs *= 2;
  }
  for (;; cs *= 2) {
    if (cs > 16) return fail(TLS_ERR_UNSUPPORTED, "shared-memory plan does not fit even with 16 CTAs per pair");
    p.cs = cs;
    tls::plan_decode_smem(p, elem_bytes(c));
    if ((int)p.smem_bytes <= kMaxSmem) break;
  }
  return TLS_OK;
}

tls_status check_index(const tls_index* idx) {
  if (!idx || !idx->block_minmax || !idx->codes || !idx->scale_zero || !idx->channels)
    return fail(TLS_ERR_INPUT, "index buffers must be non-NULL");
  if (!aligned16(idx->block_minmax) || !aligned16(idx->codes) || !aligned16(idx->scale_zero))
    return fail(TLS_ERR_INPUT, "index buffers must be 16-byte aligned");
  return TLS_OK;
}

tls_status run_decode(const tls_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                      const int32_t* seq_lens, const tls_index* idx, const int32_t* guide, int32_t* block_ids,
                      int32_t* token_ids, int32_t* num_tokens, float* token_scores, void* out, float* lse,
                      int do_select, int do_attend, tls_stream_t stream) {
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!q || !aligned16(q)) return fail(TLS_ERR_INPUT, "q must be a non-NULL 16-byte aligned device pointer");
  if (!token_ids || !num_tokens) return fail(TLS_ERR_INPUT, "token_ids and num_tokens are required");
  tls::DecodeParams p;
  s = plan(cfg, p, do_select, do_attend);
  if (s) return s;
  if (do_select) {
    s = check_index(idx);
    if (s) return s;
    if (!seq_lens || !block_ids) return fail(TLS_ERR_INPUT, "seq_lens and block_ids are required");
    p.block_minmax = idx->block_minmax;
    p.codes = idx->codes;
    p.scale_zero = idx->scale_zero;
    p.channels = idx->channels;
  }
  if (do_attend) {
    if (!k_cache || !aligned16(k_cache)) return fail(TLS_ERR_INPUT, "k_cache must be a 16-byte aligned device pointer");
    if (cfg->layout == TLS_GQA && (!v_cache || !aligned16(v_cache)))
      return fail(TLS_ERR_INPUT, "GQA needs a 16-byte aligned v_cache");
    if (!out) return fail(TLS_ERR_INPUT, "out is required");
  }
  if (!seq_lens) return fail(TLS_ERR_INPUT, "seq_lens is required");
  p.q = q;
  p.k_cache = k_cache;
  p.v_cache = cfg->layout == TLS_MLA ? nullptr : v_cache;
  p.seq_lens = seq_lens;
  p.guide = guide;
  p.block_ids = block_ids;
  p.token_ids = token_ids;
  p.num_tokens = num_tokens;
  p.token_scores = token_scores;
  p.out = out;
  p.lse = lse;
  cudaError_t e = tls::launch_decode(p, cfg->dtype == TLS_BF16, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "decode kernel launch");
  return TLS_OK;
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

tls_status tls_select(const tls_config* cfg, const void* q, const int32_t* seq_lens, const tls_index* idx,
                      const int32_t* guide_block_ids, int32_t* block_ids, int32_t* token_ids, int32_t* num_tokens,
                      float* token_scores, void* workspace, size_t workspace_bytes, tls_stream_t stream) {
  (void)workspace;
  (void)workspace_bytes;
  return run_decode(cfg, q, nullptr, nullptr, seq_lens, idx, guide_block_ids, block_ids, token_ids, num_tokens,
                    token_scores, nullptr, nullptr, 1, 0, stream);
}

tls_status tls_sparse_attend(const tls_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                             const int32_t* token_ids, const int32_t* num_tokens, void* out, float* lse,
                             void* workspace, size_t workspace_bytes, tls_stream_t stream) {
  (void)workspace;
  (void)workspace_bytes;
  // seq_lens is not needed by attention; pass a dummy non-NULL pointer check-free path.
  tls_status s = check_config(cfg);
  if (s) return s;
  if (!q || !aligned16(q)) return fail(TLS_ERR_INPUT, "q must be a non-NULL 16-byte aligned device pointer");
  if (!token_ids || !num_tokens || !out) return fail(TLS_ERR_INPUT, "token_ids, num_tokens and out are required");
  if (!k_cache || !aligned16(k_cache)) return fail(TLS_ERR_INPUT, "k_cache must be a 16-byte aligned device pointer");
  if (cfg->layout == TLS_GQA && (!v_cache || !aligned16(v_cache)))
    return fail(TLS_ERR_INPUT, "GQA needs a 16-byte aligned v_cache");
  tls::DecodeParams p;
  s = plan(cfg, p, 0, 1);
  if (s) return s;
  p.q = q;
  p.k_cache = k_cache;
  p.v_cache = cfg->layout == TLS_MLA ? nullptr : v_cache;
  p.seq_lens = num_tokens;  // read only to clamp; attention does not use it
  p.token_ids = const_cast<int32_t*>(token_ids);
  p.num_tokens = const_cast<int32_t*>(num_tokens);
  p.out = out;
  p.lse = lse;
  cudaError_t e = tls::launch_decode(p, cfg->dtype == TLS_BF16, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "attend kernel launch");
  return TLS_OK;
}

tls_status tls_decode(const tls_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                      const int32_t* seq_lens, const tls_index* idx, const int32_t* guide_block_ids,
                      int32_t* block_ids, int32_t* token_ids, int32_t* num_tokens, float* token_scores, void* out,
                      float* lse, void* workspace, size_t workspace_bytes, tls_stream_t stream) {
  (void)workspace;
  (void)workspace_bytes;
  return run_decode(cfg, q, k_cache, v_cache, seq_lens, idx, guide_block_ids, block_ids, token_ids, num_tokens,
                    token_scores, out, lse, 1, 1, stream);
}

size_t tls_workspace_bytes(const tls_config* cfg, int32_t which) {
  if (check_config(cfg) != TLS_OK || which < 0 || which > 2) return (size_t)-1;
  return 0;  // every intermediate lives in (distributed) shared memory
}

int32_t tls_launch_count(const tls_config* cfg, int32_t which) {
  if (check_config(cfg) != TLS_OK) return -1;
  switch (which) {
    case 0:
    case 1:
    case 2:
    case 3:
    case 4:
      return 1;
    default:
      return -1;
  }
}

int32_t tls_cluster_size(const tls_config* cfg, int32_t which) {
  if (check_config(cfg) != TLS_OK || which < 0 || which > 2) return -1;
  tls::DecodeParams p;
  if (plan(cfg, p, which != 1, which != 0) != TLS_OK) return -1;
  return p.cs;
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
