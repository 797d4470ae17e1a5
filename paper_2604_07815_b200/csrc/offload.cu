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

}  // namespace tls
