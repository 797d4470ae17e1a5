// seqsplit.cu -- kernels of the sequence-split decode step:
// one very long sequence whose KV cache (and index) is split along the
// sequence over P ranks, each rank holding a contiguous, block-aligned token
// range.  The step stays EXACT -- the same M_t, S_t and output as the
// unsplit operator -- because every global decision is assembled from local
// pieces that contain it:
//   * top-k_b: the global top-k_b blocks are among the union of the
//     ranks' local top-k_b  ->  tls_topk_rows over the gathered candidates;
//   * alpha~: the softmax over the candidates J = union of the ranks'
//     candidates needs per-head (max, sum) over all of J  ->  tls_token_stats
//     per rank, gathered, merged inside tls_token_keys (LSE identity);
//   * top-k_t: as for blocks  ->  tls_topk_rows twice;
//   * attention: softmax over S_t split by rank  ->  per-rank partial
//     (o, lse) merged by tls_attn_merge (LSE identity, T10).
// The collectives between these calls (all_gather over NCCL) are issued by the
// Python layer (paper_2604_07815_b200/seqsplit.py); these kernels never
// communicate.  Citation key: P:n = line n of PAPER.md; readings U*: DESIGN.md §3.
#include <math_constants.h>

#include "common.cuh"
#include "params.h"

namespace tls {

namespace {

constexpr int kT = 256;  // threads per CTA

template <typename T>
__device__ __forceinline__ T store_as(float v);
template <>
__device__ __forceinline__ float store_as<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 store_as<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// exclusive scan of one value per thread over the CTA (kT threads); total in *tot
__device__ __forceinline__ int cta_exclusive_scan(int v, int* sh, int* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kT / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kT / 32) sh[lane] = w;  // inclusive per-warp totals
  }
  __syncthreads();
  const int base = warp > 0 ? sh[warp - 1] : 0;
  *tot = sh[kT / 32 - 1];
  __syncthreads();
  return base + x - v;
}

// Composite ranking key: larger key first, equal keys -> lower id first (U2); 0 = not a candidate.
__device__ __forceinline__ unsigned long long composite(float key, int id) {
  return id < 0 ? 0ull : ((unsigned long long)f2key(key) << 32) | (unsigned)(~(unsigned)id);
}

// ---------------------------------------------------------------------------
// Exact top-k of each row of (key, id) pairs, ids ascending within the row
// (-1 = empty entry).  Output: the k selected pairs in ascending id order,
// -1 / -inf padded, and the count min(k, #entries).  The k-th largest
// composite key is found by an 8-pass byte radix select; selection is then
// "composite >= that key" (composites are unique), compacted in input order.
// ---------------------------------------------------------------------------
// Implicit ids (ids == NULL): entry i of row r has id id_base + i and exists
// iff i < ceil(lens[r / lens_div] / lens_unit) (a rank's block scores).
struct RowIds {
  const int* ids;
  int n, id_base, lens_div, lens_unit;
  const int* lens;
  __device__ __forceinline__ int nv(size_t row) const {
    return ids ? n : min(n, (max(lens[row / lens_div], 0) + lens_unit - 1) / lens_unit);
  }
  __device__ __forceinline__ int at(size_t row, int i, int nvr) const {
    return ids ? ids[row * n + i] : (i < nvr ? id_base + i : -1);
  }
};

__global__ void __launch_bounds__(kT) topk_rows_kernel(int n, const float* __restrict__ keys, RowIds rid, int k,
                                                       float* out_keys, int* out_ids, int* out_count) {
  __shared__ unsigned hist[256];
  __shared__ int sh[32];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_rem;
  const int tid = threadIdx.x;
  const size_t row = blockIdx.x;
  const float* kr = keys + row * n;
  const int nvr = rid.nv(row);
  auto id_at = [&](int i) { return rid.at(row, i, nvr); };
  int nvalid = 0;
  for (int i = tid; i < n; i += kT) nvalid += id_at(i) >= 0;
  int tot;
  cta_exclusive_scan(nvalid, sh, &tot);
  const int kk = min(k, tot);
  if (tid == 0) {
    s_prefix = 0ull;
    s_rem = kk;
  }
  __syncthreads();
  unsigned long long mask = 0ull;
  if (kk > 0) {
    for (int pass = 7; pass >= 0; --pass) {
      const int sft = 8 * pass;
      for (int i = tid; i < 256; i += kT) hist[i] = 0u;
      __syncthreads();
      const unsigned long long pre = s_prefix;
      for (int i = tid; i < n; i += kT) {
        const unsigned long long c = composite(kr[i], id_at(i));
        if (c != 0ull && (c & mask) == pre) atomicAdd(&hist[(unsigned)(c >> sft) & 0xffu], 1u);
      }
      __syncthreads();
      if (tid == 0) {  // the bin holding the rem-th largest among the prefix-matching keys
        int rem = s_rem, bsel = 0;
        for (int b = 255; b >= 0; --b) {
          const int h = (int)hist[b];
          if (rem <= h) {
            bsel = b;
            break;
          }
          rem -= h;
        }
        s_rem = rem;
        s_prefix = pre | ((unsigned long long)bsel << sft);
      }
      mask |= 0xffull << sft;
      __syncthreads();
    }
  }
  const unsigned long long thr = kk > 0 ? s_prefix : ~0ull;  // the kk-th largest composite
  // ordered compaction: thread t owns the contiguous slice [t*n/kT, (t+1)*n/kT)
  const int lo = (int)((long long)n * tid / kT), hi = (int)((long long)n * (tid + 1) / kT);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += composite(kr[i], id_at(i)) >= thr && id_at(i) >= 0;
  int pos = cta_exclusive_scan(cnt, sh, &tot);
  float* ok = out_keys + row * k;
  int* oi = out_ids + row * k;
  for (int i = lo; i < hi; ++i)
    if (id_at(i) >= 0 && composite(kr[i], id_at(i)) >= thr) {
      ok[pos] = kr[i];
      oi[pos] = id_at(i);
      ++pos;
    }
  for (int q = kk + tid; q < k; q += kT) {
    ok[q] = -CUDART_INF_F;
    oi[q] = -1;
  }
  if (tid == 0 && out_count) out_count[row] = kk;
}

// ---------------------------------------------------------------------------
// Ids of each row (ascending, -1 padded, `k` per row) inside [lo, hi), shifted
// by -lo, compacted in order, -1 padded; count of each row.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) select_range_kernel(int k, const int* __restrict__ ids, int lo, int hi,
                                                          int* out_ids, int* out_count) {
  __shared__ int sh[32];
  const int tid = threadIdx.x;
  const size_t row = blockIdx.x;
  const int* ir = ids + row * k;
  int* o = out_ids + row * k;
  const int a = (int)((long long)k * tid / kT), b = (int)((long long)k * (tid + 1) / kT);
  int cnt = 0;
  for (int i = a; i < b; ++i) cnt += ir[i] >= lo && ir[i] < hi;
  int tot;
  int pos = cta_exclusive_scan(cnt, sh, &tot);
  for (int i = a; i < b; ++i)
    if (ir[i] >= lo && ir[i] < hi) o[pos++] = ir[i] - lo;
  for (int q = tot + tid; q < k; q += kT) o[q] = -1;
  if (tid == 0 && out_count) out_count[row] = tot;
}

// ---------------------------------------------------------------------------
// The comparison operators of the paper:
// expand_blocks -- Quest's token set: every token (below the sequence length)
//   of the selected blocks, ascending (block ids ascending, -1 padded).
// block_iota -- DS's candidate blocks: every block of the sequence.
// One CTA per pair.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) expand_blocks_kernel(Dims d, const int* __restrict__ block_ids,
                                                           const int* __restrict__ seq_lens, int k_out,
                                                           int* token_ids, int* num_tokens) {
  __shared__ int sh[32];
  __shared__ int s_pre[1024 + 1];
  const int pair = blockIdx.x, b = pair / d.Hkv;
  const int n = min(max(seq_lens[b], 0), d.S);
  const int* bl = block_ids + (size_t)pair * d.Kb;
  int* out = token_ids + (size_t)pair * k_out;
  // tokens per selected block (ascending ids: the output is the concatenation in block order)
  int total = 0;
  for (int base = 0; base < d.Kb; base += kT) {
    const int i = base + threadIdx.x;
    const int blk = i < d.Kb ? bl[i] : -1;
    const int cnt = blk >= 0 ? max(0, min(d.B, n - blk * d.B)) : 0;
    int tot;
    const int pos = cta_exclusive_scan(cnt, sh, &tot);
    if (i < d.Kb && i < 1024) s_pre[i] = total + pos;
    total += tot;
  }
  if (threadIdx.x == 0) s_pre[min(d.Kb, 1024)] = total;
  __syncthreads();
  const int kk = min(total, k_out);
  for (int i = 0; i < min(d.Kb, 1024); ++i) {  // block i's tokens, one per thread
    const int blk = bl[i];
    if (blk < 0) break;
    const int c = s_pre[i + 1] - s_pre[i];
    for (int r = threadIdx.x; r < c; r += kT)
      if (s_pre[i] + r < kk) out[s_pre[i] + r] = blk * d.B + r;
  }
  for (int q = kk + threadIdx.x; q < k_out; q += kT) out[q] = -1;
  if (threadIdx.x == 0) num_tokens[pair] = kk;
}

__global__ void __launch_bounds__(kT) block_iota_kernel(Dims d, const int* __restrict__ seq_lens, int* block_ids) {
  const int pair = blockIdx.x, b = pair / d.Hkv;
  const int m = (min(max(seq_lens[b], 0), d.S) + d.B - 1) / d.B;  // reading U1
  for (int i = threadIdx.x; i < d.Kb; i += kT) block_ids[(size_t)pair * d.Kb + i] = i < m ? i : -1;
}

// ---------------------------------------------------------------------------
// a3 on a rank's candidate blocks (block_ids: local block ids, ascending, -1
// padded, k_b per pair) -- one CTA per pair.  Logits in log2 units
// (reading U10: sm_scale = 1/sqrt(d)):
//   L_hj = sm_scale log2(e) (zero_j sum_c q~_h[c] + scale_j sum_c q~_h[c] code_jc),  q~_h = q_h[C].
// mode 0 (tls_token_stats): per head M_h = max_j L_hj, Z_h = sum_j 2^(L_hj - M_h)
//   over this rank's candidates -> stats[pair][h] = (M_h, Z_h) ((-inf, 0) if none).
// mode 1 (tls_token_keys): lz_h = M_h + log2 Z_h merged over the P ranks' stats
//   (gathered [P][pairs][G][2]); for every candidate slot (block k, row r):
//   key = ln alpha~_j = ln((1/G) sum_h 2^(L_hj - lz_h))  (reading U15), id = j + tok_off;
//   slots past the candidates or the sequence: (-inf, -1).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kT) token_split_kernel(Dims d, int mode, const T* __restrict__ q,
                                                         const int* __restrict__ seq_lens,
                                                         const uint8_t* __restrict__ codes,
                                                         const float* __restrict__ scale_zero,
                                                         const int* __restrict__ channels,
                                                         const int* __restrict__ block_ids, int P,
                                                         const float* __restrict__ stats_in, float* stats_out,
                                                         float* keys_out, int* ids_out, int tok_off) {
  extern __shared__ float smem_f[];
  __shared__ float red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pair = blockIdx.x;
  const int b = pair / d.Hkv, g = pair - b * d.Hkv;
  const int G = d.G, DC = d.d_c;
  const int n = min(max(seq_lens[b], 0), d.S);
  float* qt = smem_f;              // [G][DC]
  float* qs = qt + G * DC;         // [G] sum_c q~_h[c]
  float* lz = qs + G;              // [G]
  int* blk = reinterpret_cast<int*>(lz + G);  // [Kb]
  const T* qg = q + ((size_t)b * d.Hq + (size_t)g * G) * d.d_k;
  for (int i = tid; i < G * DC; i += kT) {
    const int h = i / DC, c = i - h * DC;
    qt[i] = to_f32(qg[(size_t)h * d.d_k + channels[(size_t)g * DC + c]]);
  }
  for (int i = tid; i < d.Kb; i += kT) blk[i] = block_ids[(size_t)pair * d.Kb + i];
  __syncthreads();
  for (int h = warp; h < G; h += kT / 32) {
    float s = 0.f;
    for (int c = lane; c < DC; c += 32) s += qt[h * DC + c];
    s = warp_sum(s);
    if (lane == 0) qs[h] = s;
  }
  if (mode == 1 && tid < G) {  // lz_h over the P ranks (LSE merge, chunk order: deterministic)
    float M = -CUDART_INF_F, Z = 0.f;
    for (int r = 0; r < P; ++r) {
      const float* st = stats_in + (((size_t)r * gridDim.x + pair) * G + tid) * 2;
      const float m2 = st[0], z2 = st[1];
      const float nm = fmaxf(M, m2);
      if (nm == -CUDART_INF_F) continue;
      Z = (M == -CUDART_INF_F ? 0.f : Z * exp2f(M - nm)) + (m2 == -CUDART_INF_F ? 0.f : z2 * exp2f(m2 - nm));
      M = nm;
    }
    lz[tid] = Z > 0.f ? M + log2f(Z) : CUDART_INF_F;
  }
  __syncthreads();
  int kc = 0;
  while (kc < d.Kb && blk[kc] >= 0) ++kc;
  const int nslots = kc * d.B;
  const int rowb = DC / 2;
  const float sm2 = d.sm_scale * 1.4426950408889634f;
  auto logit = [&](int h, int j, const uint8_t* cj, float2 sz) {
    float acc = 0.f;
    for (int c2 = 0; c2 < rowb; ++c2) {
      const unsigned byte = cj[c2];
      acc = fmaf(qt[h * DC + 2 * c2], (float)(byte & 15u), acc);
      acc = fmaf(qt[h * DC + 2 * c2 + 1], (float)(byte >> 4), acc);
    }
    return sm2 * fmaf(sz.x, acc, sz.y * qs[h]);
  };
  const uint8_t* cbase = codes + (size_t)pair * d.S * rowb;
  const float2* zbase = reinterpret_cast<const float2*>(scale_zero) + (size_t)pair * d.S;
  if (mode == 0) {
    for (int h = 0; h < G; ++h) {
      float mx = -CUDART_INF_F;
      for (int s = tid; s < nslots; s += kT) {
        const int j = blk[s / d.B] * d.B + (s % d.B);
        if (j < n) mx = fmaxf(mx, logit(h, j, cbase + (size_t)j * rowb, zbase[j]));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) red[warp] = mx;
      __syncthreads();
      float M = -CUDART_INF_F;
      for (int w = 0; w < kT / 32; ++w) M = fmaxf(M, red[w]);
      __syncthreads();
      float z = 0.f;
      if (M != -CUDART_INF_F)
        for (int s = tid; s < nslots; s += kT) {
          const int j = blk[s / d.B] * d.B + (s % d.B);
          if (j < n) z += exp2f(logit(h, j, cbase + (size_t)j * rowb, zbase[j]) - M);
        }
      z = warp_sum(z);
      if (lane == 0) red[warp] = z;
      __syncthreads();
      if (tid == 0) {
        float Z = 0.f;
        for (int w = 0; w < kT / 32; ++w) Z += red[w];
        stats_out[((size_t)pair * G + h) * 2] = M;
        stats_out[((size_t)pair * G + h) * 2 + 1] = Z;
      }
      __syncthreads();
    }
    return;
  }
  const float lnG = logf((float)G);
  const size_t nout = (size_t)d.Kb * d.B;
  for (int s = tid; s < (int)nout; s += kT) {
    float key = -CUDART_INF_F;
    int id = -1;
    if (s < nslots) {
      const int j = blk[s / d.B] * d.B + (s % d.B);
      if (j < n) {
        float acc = 0.f;
        for (int h = 0; h < G; ++h)
          if (lz[h] != CUDART_INF_F) acc += exp2f(logit(h, j, cbase + (size_t)j * rowb, zbase[j]) - lz[h]);
        key = logf(acc) - lnG;
        id = j + tok_off;
      }
    }
    keys_out[(size_t)pair * nout + s] = key;
    ids_out[(size_t)pair * nout + s] = id;
  }
}

// ---------------------------------------------------------------------------
// LSE merge of P partial attention results (T10): for every query head
// row r: lse = log sum_p exp(lse_p), out = sum_p exp(lse_p - lse) o_p.
// Partials with lse_p = -inf (no selected token on that rank) weigh 0.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kT) attn_merge_kernel(int P, int rows, int dv, const float* __restrict__ parts_o,
                                                        const float* __restrict__ parts_lse, T* out, float* lse) {
  const int r = blockIdx.x;
  float M = -CUDART_INF_F;
  for (int p = 0; p < P; ++p) M = fmaxf(M, parts_lse[(size_t)p * rows + r]);
  float L = 0.f;
  for (int p = 0; p < P; ++p) {
    const float lp = parts_lse[(size_t)p * rows + r];
    if (lp != -CUDART_INF_F) L += expf(lp - M);
  }
  const float tot = M == -CUDART_INF_F ? -CUDART_INF_F : M + logf(L);
  for (int c = threadIdx.x; c < dv; c += kT) {
    float acc = 0.f;
    for (int p = 0; p < P; ++p) {
      const float lp = parts_lse[(size_t)p * rows + r];
      if (lp != -CUDART_INF_F) acc = fmaf(expf(lp - tot), parts_o[((size_t)p * rows + r) * dv + c], acc);
    }
    out[(size_t)r * dv + c] = store_as<T>(acc);
  }
  if (threadIdx.x == 0 && lse) lse[r] = tot;
}

}  // namespace

cudaError_t launch_topk_rows(int rows, int n, const float* keys, const int* ids, int k, float* out_keys,
                             int* out_ids, int* out_count, int id_base, const int* lens, int lens_div, int lens_unit,
                             cudaStream_t st) {
  RowIds rid{ids, n, id_base, lens_div, lens_unit, lens};
  topk_rows_kernel<<<rows, kT, 0, st>>>(n, keys, rid, k, out_keys, out_ids, out_count);
  return cudaGetLastError();
}

cudaError_t launch_select_range(int rows, int k, const int* ids, int lo, int hi, int* out_ids, int* out_count,
                                cudaStream_t st) {
  select_range_kernel<<<rows, kT, 0, st>>>(k, ids, lo, hi, out_ids, out_count);
  return cudaGetLastError();
}

cudaError_t launch_expand_blocks(const Dims& d, const int* block_ids, const int* seq_lens, int k_out, int* token_ids,
                                 int* num_tokens, cudaStream_t st) {
  expand_blocks_kernel<<<d.batch * d.Hkv, kT, 0, st>>>(d, block_ids, seq_lens, k_out, token_ids, num_tokens);
  return cudaGetLastError();
}

cudaError_t launch_block_iota(const Dims& d, const int* seq_lens, int* block_ids, cudaStream_t st) {
  block_iota_kernel<<<d.batch * d.Hkv, kT, 0, st>>>(d, seq_lens, block_ids);
  return cudaGetLastError();
}

size_t token_split_smem(const Dims& d) { return ((size_t)d.G * d.d_c + 2 * d.G) * 4 + (size_t)d.Kb * 4; }

cudaError_t launch_token_split(const Dims& d, int mode, const void* q, const int* seq_lens, const uint8_t* codes,
                               const float* scale_zero, const int* channels, const int* block_ids, int P,
                               const float* stats_in, float* stats_out, float* keys_out, int* ids_out, int tok_off,
                               cudaStream_t st) {
  const size_t smem = token_split_smem(d);
  const int pairs = d.batch * d.Hkv;
  if (d.bf16) {
    cudaError_t e = cudaFuncSetAttribute(token_split_kernel<__nv_bfloat16>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    token_split_kernel<__nv_bfloat16><<<pairs, kT, smem, st>>>(
        d, mode, static_cast<const __nv_bfloat16*>(q), seq_lens, codes, scale_zero, channels, block_ids, P,
        stats_in, stats_out, keys_out, ids_out, tok_off);
  } else {
    cudaError_t e =
        cudaFuncSetAttribute(token_split_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    token_split_kernel<float><<<pairs, kT, smem, st>>>(d, mode, static_cast<const float*>(q), seq_lens, codes,
                                                       scale_zero, channels, block_ids, P, stats_in, stats_out,
                                                       keys_out, ids_out, tok_off);
  }
  return cudaGetLastError();
}

cudaError_t launch_attn_merge(bool bf16, int P, int rows, int dv, const float* parts_o, const float* parts_lse,
                              void* out, float* lse, cudaStream_t st) {
  if (bf16)
    attn_merge_kernel<__nv_bfloat16><<<rows, kT, 0, st>>>(P, rows, dv, parts_o, parts_lse,
                                                          static_cast<__nv_bfloat16*>(out), lse);
  else
    attn_merge_kernel<float><<<rows, kT, 0, st>>>(P, rows, dv, parts_o, parts_lse, static_cast<float*>(out), lse);
  return cudaGetLastError();
}

}  // namespace tls
