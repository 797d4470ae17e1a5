// offload.cu -- GPU side of the KV-offload engine (AsyncTLS §4.2, P:358-383;
// SURVEY.md §8(f) f1) for sm_100a.
//
// The full K/V cache stays in pinned, device-mapped host memory.  Each pair
// owns a GPU token cache of `capacity` slots.  After a selection S_t
// (tls_select), cache_fetch_kernel makes every selected token resident:
//   * tokens of S_t already resident are hits (the step-to-step temporal
//     locality of the selection);
//   * slots holding tokens outside S_t are evicted (the cache keeps the
//     current selection, the token-granular form of C_{t+1} = M_t);
//   * every miss is copied from host memory into a freed slot by a zero-copy
//     gather (16-byte loads through the mapped pointer, one warp per row);
// and writes slot_ids, the cache rows of S_t in selection order, so the
// attention kernel (attend.cu) runs unchanged over the slot array.
//
// One CTA per pair.  Free slots and misses are compacted with block scans in
// slot / selection order, so the cache state is deterministic.
#include <math_constants.h>

#include "common.cuh"
#include "launch.h"
#include "params.h"
#include "topk.cuh"

namespace tls {

__global__ void __launch_bounds__(kThreads) cache_fetch_kernel(const __grid_constant__ CacheFetchParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ TopKCtl tk;
  __shared__ int s_nfree, s_nmiss;
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pair = blockIdx.x;
  const int C = p.capacity;
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem);               // [bitmap_words] selected-token set
  int* freelist = reinterpret_cast<int*>(smem + (size_t)p.bitmap_words * 4);  // [capacity]
  int* misspos = freelist + C;                                          // [Kt] positions of misses
  const int K = min(max(p.num_tokens[pair], 0), min(d.Kt, C));
  const int* tids = p.token_ids + (size_t)pair * d.Kt;
  int* sot = p.slot_of_token + (size_t)pair * d.S;
  int* tos = p.token_of_slot + (size_t)pair * C;
  int* sid = p.slot_ids + (size_t)pair * d.Kt;
  // 1. the selected set as a bitmap over the pair's tokens
  for (int i = tid; i < p.bitmap_words; i += kThreads) bitmap[i] = 0u;
  __syncthreads();
  for (int pos = tid; pos < K; pos += kThreads) {
    const int t = tids[pos];
    if (t >= 0 && t < d.S) atomicOr(&bitmap[t >> 5], 1u << (t & 31));
  }
  __syncthreads();
  // 2. evict slots whose token left the selection; free slots in slot order
  {
    const int per = (C + kThreads - 1) / kThreads;
    const int lo = min(tid * per, C), hi = min(lo + per, C);
    int cnt = 0;
    for (int s = lo; s < hi; ++s) {
      const int t = tos[s];
      const bool keep = t >= 0 && t < d.S && ((bitmap[t >> 5] >> (t & 31)) & 1u);
      if (!keep) {
        if (t >= 0 && t < d.S) sot[t] = -1;
        tos[s] = -1;
        ++cnt;
      }
    }
    int total;
    int pos = block_exclusive_scan(cnt, tk.scan, &total);
    for (int s = lo; s < hi; ++s)
      if (tos[s] < 0) freelist[pos++] = s;
    if (tid == 0) s_nfree = total;
  }
  __syncthreads();
  // 3. hits keep their slot; misses (in selection order) take free slots in order
  {
    const int per = (K + kThreads - 1) / kThreads;
    const int lo = min(tid * per, K), hi = min(lo + per, K);
    int cnt = 0;
    for (int pos = lo; pos < hi; ++pos) {
      const int t = tids[pos];
      const int s = (t >= 0 && t < d.S) ? sot[t] : 0;
      if (t >= 0 && t < d.S && s < 0) ++cnt;
      else sid[pos] = s;
    }
    int total;
    int m = block_exclusive_scan(cnt, tk.scan, &total);
    for (int pos = lo; pos < hi; ++pos) {
      const int t = tids[pos];
      if (t >= 0 && t < d.S && sot[t] < 0) misspos[m++] = pos;
    }
    if (tid == 0) s_nmiss = total;
  }
  __syncthreads();
  const int nmiss = min(s_nmiss, s_nfree);  // capacity >= Kt guarantees nmiss <= nfree
  for (int i = tid; i < nmiss; i += kThreads) {
    const int pos = misspos[i], t = tids[pos], s = freelist[i];
    sid[pos] = s;
    sot[t] = s;
    tos[s] = t;
  }
  for (int pos = K + tid; pos < d.Kt; pos += kThreads) sid[pos] = 0;  // past num_tokens: unused
  if (tid == 0 && p.miss_count) p.miss_count[pair] = nmiss;
  __syncthreads();
  // 4. zero-copy gather of the missed rows: host (mapped) -> slot, one warp per row, 16-byte lanes
  const size_t eb = d.bf16 ? 2 : 4;
  const int kq = (int)(d.d_k * eb / 16), vq = (int)(d.d_v * eb / 16);  // 16-byte words per row
  const size_t kv_pair_k = (size_t)pair * d.S * d.d_k * eb, kv_pair_v = (size_t)pair * d.S * d.d_v * eb;
  for (int i = warp; i < nmiss; i += kWarps) {
    const int t = tids[misspos[i]], s = freelist[i];
    const uint4* ksrc = reinterpret_cast<const uint4*>(p.k_host + kv_pair_k + (size_t)t * d.d_k * eb);
    uint4* kdst = reinterpret_cast<uint4*>(p.k_slots + ((size_t)pair * C + s) * d.d_k * eb);
    for (int w = lane; w < kq; w += 32) kdst[w] = ksrc[w];
    if (p.v_host != nullptr) {
      const uint4* vsrc = reinterpret_cast<const uint4*>(p.v_host + kv_pair_v + (size_t)t * d.d_v * eb);
      uint4* vdst = reinterpret_cast<uint4*>(p.v_slots + ((size_t)pair * C + s) * d.d_v * eb);
      for (int w = lane; w < vq; w += 32) vdst[w] = vsrc[w];
    }
  }
}

cudaError_t launch_cache_fetch(const CacheFetchParams& p, cudaStream_t st) {
  const size_t smem = (size_t)p.bitmap_words * 4 + (size_t)p.capacity * 4 + (size_t)p.d.Kt * 4;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(cache_fetch_kernel), smem, false);
  if (e != cudaSuccess) return e;
  return launch_ex(cache_fetch_kernel, dim3((unsigned)(p.d.batch * p.d.Hkv)), kThreads, smem, st, LaunchOpts{}, 0, p);
}

// ---------------------------------------------------------------------------
// Block-granular cache: after step t's selection, make the blocks
// of M_t resident while keeping M_{t-1} (still read by step t's attention):
// slots whose block is in neither set are freed (slot order), missing blocks of
// M_t take free slots in M_t order (deterministic), and their B rows of K and V
// are copied from host memory by a zero-copy gather, a warp per row.  Meant to
// run on a side stream, overlapped with the attention of step t; the next
// step's token selection is confined to M_t (lag mode), so it only reads
// resident blocks.  One CTA per pair.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) block_cache_update_kernel(const __grid_constant__ BlockCacheParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ TopKCtl tk;
  __shared__ int s_nfree, s_nmiss;
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pair = blockIdx.x;
  const int C = p.capacity;
  uint32_t* keep = reinterpret_cast<uint32_t*>(smem);  // [bitmap_words] M_{t-1} u M_t
  int* freelist = reinterpret_cast<int*>(smem + (size_t)p.bitmap_words * 4);  // [capacity]
  int* missblk = freelist + C;                                            // [Kb]
  const int* ids = p.block_ids + (size_t)pair * d.Kb;
  const int* kids = p.keep_ids ? p.keep_ids + (size_t)pair * d.Kb : nullptr;
  int* sob = p.slot_of_block + (size_t)pair * d.M;
  int* bos = p.block_of_slot + (size_t)pair * C;
  for (int i = tid; i < p.bitmap_words; i += kThreads) keep[i] = 0u;
  __syncthreads();
  for (int k = tid; k < d.Kb; k += kThreads) {
    const int a = ids[k];
    if (a >= 0 && a < d.M) atomicOr(&keep[a >> 5], 1u << (a & 31));
    if (kids) {
      const int b = kids[k];
      if (b >= 0 && b < d.M) atomicOr(&keep[b >> 5], 1u << (b & 31));
    }
  }
  __syncthreads();
  {  // free every slot whose block is in neither set, in slot order
    const int per = (C + kThreads - 1) / kThreads;
    const int lo = min(tid * per, C), hi = min(lo + per, C);
    int cnt = 0;
    for (int s = lo; s < hi; ++s) {
      const int b = bos[s];
      const bool kept = b >= 0 && b < d.M && ((keep[b >> 5] >> (b & 31)) & 1u);
      if (!kept) {
        if (b >= 0 && b < d.M) sob[b] = -1;
        bos[s] = -1;
        ++cnt;
      }
    }
    int total;
    int pos = block_exclusive_scan(cnt, tk.scan, &total);
    for (int s = lo; s < hi; ++s)
      if (bos[s] < 0) freelist[pos++] = s;
    if (tid == 0) s_nfree = total;
  }
  __syncthreads();
  {  // blocks of M_t that are not resident, in M_t order
    const int per = (d.Kb + kThreads - 1) / kThreads;
    const int lo = min(tid * per, d.Kb), hi = min(lo + per, d.Kb);
    int cnt = 0;
    for (int k = lo; k < hi; ++k) {
      const int a = ids[k];
      cnt += (a >= 0 && a < d.M && sob[a] < 0);
    }
    int total;
    int m = block_exclusive_scan(cnt, tk.scan, &total);
    for (int k = lo; k < hi; ++k) {
      const int a = ids[k];
      if (a >= 0 && a < d.M && sob[a] < 0) missblk[m++] = a;
    }
    if (tid == 0) s_nmiss = total;
  }
  __syncthreads();
  const int nmiss = min(s_nmiss, s_nfree);  // capacity >= 2 Kb guarantees nmiss <= nfree
  for (int i = tid; i < nmiss; i += kThreads) {
    const int a = missblk[i], s = freelist[i];
    sob[a] = s;
    bos[s] = a;
  }
  if (tid == 0 && p.miss_count) p.miss_count[pair] = nmiss;
  // zero-copy gather of the missing blocks: B rows each, one warp per row, 16-byte lanes
  const size_t eb = d.bf16 ? 2 : 4;
  const int kq = (int)(d.d_k * eb / 16), vq = (int)(d.d_v * eb / 16);
  const size_t kpair = (size_t)pair * d.S * d.d_k * eb, vpair = (size_t)pair * d.S * d.d_v * eb;
  const size_t kslot = (size_t)pair * C * d.B * d.d_k * eb, vslot = (size_t)pair * C * d.B * d.d_v * eb;
  for (int r = warp; r < nmiss * d.B; r += kWarps) {
    const int i = r >> d.log2B, j = r & (d.B - 1);
    const int t = (missblk[i] << d.log2B) + j;
    if (t >= d.S) continue;
    const int row = (freelist[i] << d.log2B) + j;
    const uint4* ks = reinterpret_cast<const uint4*>(p.k_host + kpair + (size_t)t * d.d_k * eb);
    uint4* kd = reinterpret_cast<uint4*>(p.k_slots + kslot + (size_t)row * d.d_k * eb);
    for (int w = lane; w < kq; w += 32) kd[w] = ks[w];
    if (p.v_host != nullptr) {
      const uint4* vs = reinterpret_cast<const uint4*>(p.v_host + vpair + (size_t)t * d.d_v * eb);
      uint4* vd = reinterpret_cast<uint4*>(p.v_slots + vslot + (size_t)row * d.d_v * eb);
      for (int w = lane; w < vq; w += 32) vd[w] = vs[w];
    }
  }
}

// Cache rows of the selected tokens: row = slot_of_block[t / B] * B + t % B.
__global__ void __launch_bounds__(kThreads) block_cache_rows_kernel(const __grid_constant__ BlockCacheParams p) {
  const Dims& d = p.d;
  const int pair = blockIdx.x, tid = threadIdx.x;
  const int K = min(max(p.num_tokens[pair], 0), d.Kt);
  const int* tids = p.token_ids + (size_t)pair * d.Kt;
  const int* sob = p.slot_of_block + (size_t)pair * d.M;
  int* rows = p.slot_rows + (size_t)pair * d.Kt;
  int bad = 0;
  for (int i = tid; i < d.Kt; i += kThreads) {
    int r = 0;
    if (i < K) {
      const int t = tids[i];
      const int s = (t >= 0 && t < d.S) ? sob[t >> d.log2B] : -1;
      if (s >= 0) r = (s << d.log2B) + (t & (d.B - 1));
      else ++bad;
    }
    rows[i] = r;
  }
  if (p.absent) {
    __shared__ int s_bad;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    if (bad) atomicAdd(&s_bad, bad);
    __syncthreads();
    if (tid == 0) p.absent[pair] = s_bad;
  }
}

cudaError_t launch_block_cache_update(const BlockCacheParams& p, cudaStream_t st) {
  const size_t smem = (size_t)p.bitmap_words * 4 + (size_t)p.capacity * 4 + (size_t)p.d.Kb * 4;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(block_cache_update_kernel), smem, false);
  if (e != cudaSuccess) return e;
  return launch_ex(block_cache_update_kernel, dim3((unsigned)(p.d.batch * p.d.Hkv)), kThreads, smem, st, LaunchOpts{},
                   0, p);
}

cudaError_t launch_block_cache_rows(const BlockCacheParams& p, cudaStream_t st) {
  return launch_ex(block_cache_rows_kernel, dim3((unsigned)(p.d.batch * p.d.Hkv)), kThreads, 0, st, LaunchOpts{}, 0, p);
}

}  // namespace tls
