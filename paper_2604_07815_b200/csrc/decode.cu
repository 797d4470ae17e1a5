// decode.cu -- the decode-step hot path of AsyncTLS two-level sparse attention
// (arXiv 2604.07815) for sm_100a: one thread-block CLUSTER per
// (batch element, KV head) pair, cs CTAs per pair, all five steps in one
// launch with no HBM round trip for intermediates.
//
//   phase A  block scores  s_i = Q+ . k^max_i + Q- . k^min_i
//            each CTA streams a 1/cs slice of the pair's block index
//   phase B  top-k_b blocks: cluster-wide radix select; histograms
//            merged through distributed shared memory (DSMEM)
//   phase C  token scores over the candidate blocks: INT4 codes x
//            the channel-projected query on tensor cores (mma.sync bf16), the
//            per-head softmax normalisers merged over the cluster, ranking key
//            log2 alpha~_j = log2 sum_h exp2(l_hj - lz_h)  (reading U15)
//   phase D  top-k_t tokens: cluster radix select again
//   phase E  split-K sparse attention over the selected tokens,
//            per-CTA partial (max, sum, o) merged through DSMEM
//
// Citation key: P:n = line n of PAPER.md.  Readings U1..U18: DESIGN.md §3.
#include "common.cuh"
#include "decode.h"

#include <math_constants.h>

namespace tls {

struct Ctl {
  uint32_t hist[2][256];  // radix histograms, double-buffered (read remotely)
  uint32_t tot[256];      // cluster-summed histogram
  int scan[kWarps + 2];
  int xc[4][2];           // per top-k call: (count > thr, count == thr)  (read remotely)
  int dig, krem, bincnt;  // radix pass result
  int r_take, r_off, r_total;
  int nvalid;             // valid candidate tokens of this CTA (read remotely)
  int kc, jtot;
  float hm[64], hz[64];   // per-head local max / sum (read remotely)
  float hlz[64];          // per-head log2 normaliser M_h + log2 Z_h
  float am[64], al[64];   // attention partial max / sum (read remotely)
};

struct TopK {
  uint32_t thr;
  int take_eq;
  int offset;
  int total;
  bool eq_mode;
};

// --------------------------------------------------------------------------
// Cluster-wide exact top-k with the lower-index tie rule (readings U2-U4).
// Every CTA holds `nloc` keys (larger = better, 0 = not a candidate) in smem;
// the global order of elements is (CTA rank, local index), which equals
// ascending block / token id.  K must not exceed the number of nonzero keys
// unless take_all.  Selected set = {k > thr} plus, in eq_mode, the first
// `take_eq` elements with k == thr of this CTA.
// --------------------------------------------------------------------------
__device__ TopK cluster_topk(const uint32_t* keys, int nloc, int K, bool take_all, int cs, unsigned rank,
                             Ctl& ctl, int call) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t prefix = 0, mask = 0, thr = 0;
  int krem = K;
  bool eq_mode = false;
  if (!take_all) {
    bool done = false;
    for (int pass = 0; pass < 4 && !done; ++pass) {
      const int shift = 24 - 8 * pass, buf = pass & 1;
      for (int i = tid; i < 256; i += kThreads) ctl.hist[buf][i] = 0;
      __syncthreads();
      for (int base = 0; base < nloc; base += kThreads) {
        const int i = base + tid;
        const uint32_t k = i < nloc ? keys[i] : 0u;
        const bool cand = k != 0u && (k & mask) == prefix;
        const uint32_t digit = cand ? ((k >> shift) & 255u) : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        if (cand && lane == __ffs(peers) - 1) atomicAdd(&ctl.hist[buf][digit], (uint32_t)__popc(peers));
      }
      cluster_sync_all();
      if (tid < 256) {
        uint32_t s = 0;
        for (int rr = 0; rr < cs; ++rr) s += *dsmem(&ctl.hist[buf][tid], rr);
        ctl.tot[tid] = s;
      }
      __syncthreads();
      if (warp == 0) {
        int c[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          c[j] = (int)ctl.tot[255 - 8 * lane - j];
          sum += c[j];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const int excl = incl - sum;
        if (excl < krem && krem <= incl) {
          int above = excl;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (above + c[j] >= krem) {
              ctl.dig = 255 - 8 * lane - j;
              ctl.krem = krem - above;
              ctl.bincnt = c[j];
              break;
            }
            above += c[j];
          }
        }
      }
      __syncthreads();
      prefix |= (uint32_t)ctl.dig << shift;
      mask |= 0xffu << shift;
      krem = ctl.krem;
      if (krem == ctl.bincnt) {  // the whole bin is taken: select k >= prefix
        done = true;
        thr = prefix ? prefix - 1u : 0u;
      }
    }
    if (!done) {
      thr = prefix;
      eq_mode = true;
    }
  }
  // Per-CTA counts -> ranks' offsets.
  int gt = 0, eq = 0;
  for (int i = tid; i < nloc; i += kThreads) {
    const uint32_t k = keys[i];
    gt += k > thr;
    eq += (eq_mode && k == thr);
  }
  int gtot, etot;
  block_exclusive_scan(gt, ctl.scan, &gtot);
  block_exclusive_scan(eq, ctl.scan, &etot);
  if (tid == 0) {
    ctl.xc[call][0] = gtot;
    ctl.xc[call][1] = etot;
  }
  cluster_sync_all();
  if (tid == 0) {
    int eq_before = 0, off = 0, total = 0, my_take = 0;
    for (int rr = 0; rr < cs; ++rr) {
      const int* x = dsmem(&ctl.xc[call][0], rr);
      const int g = x[0], e = x[1];
      int take = 0;
      if (eq_mode) take = min(max(krem - eq_before, 0), e);
      eq_before += e;
      const int s = g + take;
      if (rr < (int)rank) off += s;
      if (rr == (int)rank) my_take = take;
      total += s;
    }
    ctl.r_take = my_take;
    ctl.r_off = off;
    ctl.r_total = total;
  }
  __syncthreads();
  TopK r;
  r.thr = thr;
  r.eq_mode = eq_mode;
  r.take_eq = ctl.r_take;
  r.offset = ctl.r_off;
  r.total = ctl.r_total;
  __syncthreads();
  return r;
}

// Emit this CTA's selected elements in local-index order: f(local_index, out_pos).
template <class F>
__device__ void topk_emit(const uint32_t* keys, int nloc, const TopK& t, Ctl& ctl, F f) {
  const int tid = threadIdx.x;
  const int per = (nloc + kThreads - 1) / kThreads;
  const int b = min(tid * per, nloc), e = min(b + per, nloc);
  int eqc = 0;
  if (t.eq_mode)
    for (int i = b; i < e; ++i) eqc += keys[i] == t.thr;
  int tot;
  const int eqbase = block_exclusive_scan(eqc, ctl.scan, &tot);
  int selc = 0, eqs = eqbase;
  for (int i = b; i < e; ++i) {
    const uint32_t k = keys[i];
    bool s = k > t.thr;
    if (t.eq_mode && k == t.thr) s = (eqs++ < t.take_eq);
    selc += s;
  }
  int pos = t.offset + block_exclusive_scan(selc, ctl.scan, &tot);
  eqs = eqbase;
  for (int i = b; i < e; ++i) {
    const uint32_t k = keys[i];
    bool s = k > t.thr;
    if (t.eq_mode && k == t.thr) s = (eqs++ < t.take_eq);
    if (s) f(i, pos++);
  }
}

// --------------------------------------------------------------------------
// Phase A: block scores of blocks [i0, i1) of this pair (P:99 via P:110).
// QQ = [Q+ (d_k) | Q- (d_k)] in fp32; a block's summary row is
// [k^max (d_k) | k^min (d_k)], so s_i = QQ . row_i (a GEMV, HBM-bound).
// --------------------------------------------------------------------------
template <typename T, int CPL>
__device__ void phase_block_scores(const DecodeParams& p, int pair, int i0, int i1, const float* QQ,
                                   uint32_t* bkeys) {
  constexpr int EPC = 16 / sizeof(T);
  constexpr int U = CPL == 1 ? 4 : (CPL == 2 ? 2 : 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nchunk = 2 * p.d_k / EPC;
  float qreg[CPL][EPC];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int ch = lane + 32 * c;
#pragma unroll
    for (int e = 0; e < EPC; ++e) qreg[c][e] = ch < nchunk ? QQ[ch * EPC + e] : 0.f;
  }
  const T* bm = reinterpret_cast<const T*>(p.block_minmax) + (size_t)pair * p.M * 2 * p.d_k;
  for (int i = i0 + warp * U; i < i1; i += kWarps * U) {
    uint4 v[U][CPL];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int ch = lane + 32 * c;
        if (i + u < i1 && ch < nchunk)
          v[u][c] = ldg_stream16(bm + (size_t)(i + u) * 2 * p.d_k + (size_t)ch * EPC);
        else
          v[u][c] = make_uint4(0u, 0u, 0u, 0u);
      }
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[u] = 0.f;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        float f[EPC];
        unpack16<T>(v[u][c], f);
#pragma unroll
        for (int e = 0; e < EPC; ++e) acc[u] = fmaf(qreg[c][e], f[e], acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = warp_sum(acc[u]);
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u < i1) bkeys[i + u - i0] = f2key(acc[u]);
    }
  }
}

// bf16 piece `sp` of x: x ~= hi + mid + lo (sp = 0, 1, 2), each exact in bf16.
__device__ __forceinline__ float split_piece(float x, int sp) {
  float hi = __bfloat162float(__float2bfloat16_rn(x));
  if (sp == 0) return hi;
  float r1 = x - hi;
  float mid = __bfloat162float(__float2bfloat16_rn(r1));
  if (sp == 1) return mid;
  return __bfloat162float(__float2bfloat16_rn(r1 - mid));
}

// --------------------------------------------------------------------------
// Phase C: token logits of this CTA's candidate blocks cblk[c0 .. c0+nbl)
// (P:129-133).  Logit (log2 units):
//   L_hj = sm_scale*log2e * (zero_j * sum_c q_h[C_c] + scale_j * sum_c q_h[C_c]*code_jc)
// the code contraction on tensor cores: A = codes (16 tokens x 16 channels,
// nibbles -> exact bf16), B = query heads (16 channels x 8 heads, bf16, fp32
// queries split in 3 bf16 pieces).  The K order of the MMA is a permutation
// of the channels, applied identically to A and B.
// --------------------------------------------------------------------------
__device__ void phase_token_logits(const DecodeParams& p, int pair, int n, const int* cblk, int c0, int nbl,
                                   const uint32_t* qb, const float* qsum, float* logits) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q4 = lane & 3, r0 = lane >> 2;
  const int tpb = p.B / 16;
  const int ntiles = nbl * tpb;
  const int rowbytes = p.d_c / 2;
  const uint8_t* cbase = p.codes + (size_t)pair * p.S * rowbytes;
  const float2* szbase = reinterpret_cast<const float2*>(p.scale_zero) + (size_t)pair * p.S;
  const float sm2 = p.sm_scale * kLog2e;
  const uint2* qb2 = reinterpret_cast<const uint2*>(qb);
  for (int tile = warp; tile < ntiles; tile += kWarps) {
    const int kb = tile / tpb;
    const int rowoff = (tile - kb * tpb) * 16;
    const int blk = cblk[c0 + kb];
    const int tok0 = blk * p.B + rowoff + r0, tok1 = tok0 + 8;
    const bool v0 = tok0 < n, v1 = tok1 < n;
    uint32_t w0[4] = {0u, 0u, 0u, 0u}, w1[4] = {0u, 0u, 0u, 0u};
    const uint32_t* rp0 = reinterpret_cast<const uint32_t*>(cbase + (size_t)tok0 * rowbytes) + q4 * p.wpt;
    const uint32_t* rp1 = reinterpret_cast<const uint32_t*>(cbase + (size_t)tok1 * rowbytes) + q4 * p.wpt;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u < p.wpt) {
        if (v0) w0[u] = __ldg(rp0 + u);
        if (v1) w1[u] = __ldg(rp1 + u);
      }
    }
    const float2 sz0 = v0 ? __ldg(szbase + tok0) : make_float2(0.f, 0.f);
    const float2 sz1 = v1 ? __ldg(szbase + tok1) : make_float2(0.f, 0.f);
    uint32_t a[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (s < p.ksteps) {
        const int u = s >> 1, sel = 2 * (s & 1);
        a[s][0] = nib2bf16(w0[u], sel);
        a[s][1] = nib2bf16(w1[u], sel);
        a[s][2] = nib2bf16(w0[u], sel + 1);
        a[s][3] = nib2bf16(w1[u], sel + 1);
      }
    }
    const int jl = tile * 16 + r0;
    for (int nt = 0; nt < p.nt; ++nt) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (s < p.ksteps) {
          for (int sp = 0; sp < p.nsplit; ++sp) {
            const uint2 bb = qb2[((sp * p.nt + nt) * p.ksteps + s) * 32 + lane];
            mma_bf16_16816(acc, a[s], bb.x, bb.y);
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int h = nt * 8 + 2 * q4 + e;
        if (h < p.G) {
          const float qs = qsum[h];
          logits[h * p.ls + jl] = v0 ? sm2 * fmaf(sz0.y, qs, sz0.x * acc[e]) : -CUDART_INF_F;
          logits[h * p.ls + jl + 8] = v1 ? sm2 * fmaf(sz1.y, qs, sz1.x * acc[2 + e]) : -CUDART_INF_F;
        }
      }
    }
  }
}

// --------------------------------------------------------------------------
// Phase E (generic CUDA-core path): partial attention of this CTA over its
// tokens sel[0..tloc) for the G heads of the pair, log2 domain.
// Leaves (am_h, al_h) in ctl and the unnormalised partial o in ao.
// --------------------------------------------------------------------------
template <typename T>
__device__ void phase_attend_generic(const DecodeParams& p, int pair, int b, int g, const int* sel, int tloc,
                                     float* aq, float* as, float* ao, Ctl& ctl) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * p.Hq + (size_t)g * p.G) * p.d_k;
  for (int i = tid; i < p.G * p.d_k; i += kThreads) aq[i] = to_f32<T>(qg[i]);
  __syncthreads();
  const T* kb = reinterpret_cast<const T*>(p.k_cache) + (size_t)pair * p.S * p.d_k;
  const T* vb = p.mla ? kb : reinterpret_cast<const T*>(p.v_cache) + (size_t)pair * p.S * p.d_v;
  const int vstride = p.mla ? p.d_k : p.d_v;
  const float sm2 = p.sm_scale * kLog2e;
  for (int t = warp; t < tloc; t += kWarps) {
    const T* krow = kb + (size_t)sel[t] * p.d_k;
    for (int h = 0; h < p.G; ++h) {
      float acc = 0.f;
      for (int e = lane; e < p.d_k; e += 32) acc = fmaf(aq[h * p.d_k + e], to_f32<T>(krow[e]), acc);
      acc = warp_sum(acc);
      if (lane == 0) as[h * p.tloc_max + t] = acc * sm2;
    }
  }
  __syncthreads();
  for (int h = warp; h < p.G; h += kWarps) {
    float mx = -CUDART_INF_F;
    for (int t = lane; t < tloc; t += 32) mx = fmaxf(mx, as[h * p.tloc_max + t]);
    mx = warp_max(mx);
    float l = 0.f;
    for (int t = lane; t < tloc; t += 32) {
      const float e = exp2f(as[h * p.tloc_max + t] - mx);
      as[h * p.tloc_max + t] = e;
      l += e;
    }
    l = warp_sum(l);
    if (lane == 0) {
      ctl.am[h] = mx;
      ctl.al[h] = l;
    }
  }
  __syncthreads();
  for (int idx = tid; idx < p.G * p.d_v; idx += kThreads) {
    const int h = idx / p.d_v, c = idx - h * p.d_v;
    float acc = 0.f;
    for (int t = 0; t < tloc; ++t) acc = fmaf(as[h * p.tloc_max + t], to_f32<T>(vb[(size_t)sel[t] * vstride + c]), acc);
    ao[idx] = acc;
  }
}

// Merge the cs partials of the pair (flash-decoding LSE merge, T10) and write
// out / lse.  CTA `rank` writes a 1/cs slice of the G*d_v outputs.
template <typename T>
__device__ void phase_merge(const DecodeParams& p, int b, int g, unsigned rank, const float* ao, Ctl& ctl) {
  const int tid = threadIdx.x;
  const int tot = p.G * p.d_v;
  const int lo = (int)((long long)tot * rank / p.cs), hi = (int)((long long)tot * (rank + 1) / p.cs);
  T* outg = reinterpret_cast<T*>(p.out) + ((size_t)b * p.Hq + (size_t)g * p.G) * p.d_v;
  for (int idx = lo + tid; idx < hi; idx += kThreads) {
    const int h = idx / p.d_v, c = idx - h * p.d_v;
    float M = -CUDART_INF_F;
    for (int rr = 0; rr < p.cs; ++rr) M = fmaxf(M, *dsmem(&ctl.am[h], rr));
    float L = 0.f, o = 0.f;
    if (M != -CUDART_INF_F) {
      for (int rr = 0; rr < p.cs; ++rr) {
        const float w = exp2f(*dsmem(&ctl.am[h], rr) - M);
        L = fmaf(*dsmem(&ctl.al[h], rr), w, L);
        o = fmaf(*dsmem(&ao[idx], rr), w, o);
      }
    }
    outg[idx] = from_f32<T>(L > 0.f ? o / L : 0.f);
    if (c == 0 && p.lse != nullptr)
      p.lse[(size_t)b * p.Hq + (size_t)g * p.G + h] = L > 0.f ? (M + log2f(L)) * kLn2 : -CUDART_INF_F;
  }
}

template <typename T, int CPL>
__global__ void __launch_bounds__(kThreads) tls_decode_kernel(const __grid_constant__ DecodeParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Ctl ctl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rank = blockIdx.x;  // cluster = the cs CTAs of blockIdx.y
  const int cs = p.cs;
  const int pair = blockIdx.y;
  const int b = pair / p.Hkv, g = pair - b * p.Hkv;
  const int n = p.do_select ? min(max(p.seq_lens[b], 0), p.S) : 0;
  const int m = (n + p.B - 1) / p.B;  // reading U1: ceil, partial last block
  int* sel = reinterpret_cast<int*>(smem + p.off_sel);
  int* cblk = reinterpret_cast<int*>(smem + p.off_cblk);
  int katt = 0;  // tokens the cluster attends (fused mode)

  if (p.do_select) {
    float* QQ = reinterpret_cast<float*>(smem + p.off_qq);
    uint32_t* bkeys = reinterpret_cast<uint32_t*>(smem + p.off_bkeys);
    uint32_t* qb = reinterpret_cast<uint32_t*>(smem + p.off_qb);
    float* qsum = reinterpret_cast<float*>(smem + p.off_qsum);
    float* logits = reinterpret_cast<float*>(smem + p.off_logits);
    uint32_t* tkeys = reinterpret_cast<uint32_t*>(smem + p.off_tkeys);
    const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * p.Hq + (size_t)g * p.G) * p.d_k;
    const int* chan = p.channels + (size_t)g * p.d_c;

    // ---- query-side preparation (Q+-, bf16 query fragments, qsum) ----
    for (int c = tid; c < p.d_k; c += kThreads) {
      float qp = 0.f, qn = 0.f;
      for (int h = 0; h < p.G; ++h) {
        const float v = to_f32<T>(qg[(size_t)h * p.d_k + c]);
        qp += fmaxf(v, 0.f);
        qn += fminf(v, 0.f);
      }
      QQ[c] = qp;
      QQ[p.d_k + c] = qn;
    }
    const int nqb = p.nsplit * p.nt * p.ksteps * 32;
    for (int idx = tid; idx < nqb; idx += kThreads) {
      const int ln = idx & 31, rest = idx >> 5;
      const int s = rest % p.ksteps, nt = (rest / p.ksteps) % p.nt, sp = rest / (p.ksteps * p.nt);
      const int hh = nt * 8 + (ln >> 2);
      const int wi = (ln & 3) * p.wpt + (s >> 1);
      const int cb = 8 * wi + 2 * (s & 1);
      float x[4] = {0.f, 0.f, 0.f, 0.f};
      if (hh < p.G) {
        const T* qh = qg + (size_t)hh * p.d_k;
        x[0] = to_f32<T>(qh[chan[cb]]);
        x[1] = to_f32<T>(qh[chan[cb + 4]]);
        x[2] = to_f32<T>(qh[chan[cb + 1]]);
        x[3] = to_f32<T>(qh[chan[cb + 5]]);
      }
      qb[2 * idx] = pack_bf16x2(split_piece(x[0], sp), split_piece(x[1], sp));
      qb[2 * idx + 1] = pack_bf16x2(split_piece(x[2], sp), split_piece(x[3], sp));
    }
    for (int h = tid; h < p.nt * 8; h += kThreads) {
      float s = 0.f;
      if (h < p.G)
        for (int c = 0; c < p.d_c; ++c) s += to_f32<T>(qg[(size_t)h * p.d_k + chan[c]]);
      qsum[h] = s;
    }
    __syncthreads();

    // ---- phase A: block scores of this CTA's slice ----
    const int i0 = (int)((long long)m * rank / cs), i1 = (int)((long long)m * (rank + 1) / cs);
    phase_block_scores<T, CPL>(p, pair, i0, i1, QQ, bkeys);
    __syncthreads();

    // ---- phase B: M_t = top-k_b blocks ----
    {
      const int K = min(p.Kb, m);
      const TopK t = cluster_topk(bkeys, i1 - i0, K, p.Kb >= m, cs, rank, ctl, 0);
      int* bout = p.block_ids + (size_t)pair * p.Kb;
      const bool sync_mode = p.guide == nullptr;
      topk_emit(bkeys, i1 - i0, t, ctl, [&](int i, int pos) {
        bout[pos] = i0 + i;
        if (sync_mode)
          for (int rr = 0; rr < cs; ++rr) *dsmem(&cblk[pos], rr) = i0 + i;
      });
      if (rank == 0)
        for (int pos = t.total + tid; pos < p.Kb; pos += kThreads) bout[pos] = -1;
      if (sync_mode) {
        if (tid == 0) ctl.kc = t.total;
      } else {
        // one-step-lag mode: candidates = guide blocks (ascending, -1 padded)
        const int* gd = p.guide + (size_t)pair * p.Kb;
        const int per = (p.Kb + kThreads - 1) / kThreads;
        const int lo = min(tid * per, p.Kb), hi = min(lo + per, p.Kb);
        int cnt = 0;
        for (int i = lo; i < hi; ++i) cnt += (gd[i] >= 0 && gd[i] < m);
        int total;
        int pos = block_exclusive_scan(cnt, ctl.scan, &total);
        for (int i = lo; i < hi; ++i)
          if (gd[i] >= 0 && gd[i] < m) cblk[pos++] = gd[i];
        if (tid == 0) ctl.kc = total;
      }
      cluster_sync_all();  // cblk complete in every CTA
    }

    // ---- phase C: token logits + per-head softmax normalisers ----
    const int kc = ctl.kc;
    const int cb0 = (int)((long long)kc * rank / cs), cb1 = (int)((long long)kc * (rank + 1) / cs);
    const int nbl = cb1 - cb0;
    const int lc = nbl * p.B;
    phase_token_logits(p, pair, n, cblk, cb0, nbl, qb, qsum, logits);
    if (tid == 0) {
      int nv = 0;
      for (int k = cb0; k < cb1; ++k) nv += min(p.B, n - cblk[k] * p.B);
      ctl.nvalid = nv;
    }
    __syncthreads();
    for (int h = warp; h < p.G; h += kWarps) {
      float mx = -CUDART_INF_F;
      for (int j = lane; j < lc; j += 32) mx = fmaxf(mx, logits[h * p.ls + j]);
      mx = warp_max(mx);
      if (lane == 0) ctl.hm[h] = mx;
    }
    cluster_sync_all();
    if (tid < p.G) {
      float M = -CUDART_INF_F;
      for (int rr = 0; rr < cs; ++rr) M = fmaxf(M, *dsmem(&ctl.hm[tid], rr));
      ctl.hlz[tid] = M;
    }
    if (tid == 32) {
      int jt = 0;
      for (int rr = 0; rr < cs; ++rr) jt += *dsmem(&ctl.nvalid, rr);
      ctl.jtot = jt;
    }
    __syncthreads();
    for (int h = warp; h < p.G; h += kWarps) {
      const float M = ctl.hlz[h];
      float z = 0.f;
      if (M != -CUDART_INF_F)
        for (int j = lane; j < lc; j += 32) z += exp2f(logits[h * p.ls + j] - M);
      z = warp_sum(z);
      if (lane == 0) ctl.hz[h] = z;
    }
    cluster_sync_all();
    if (tid < p.G) {
      float Z = 0.f;
      for (int rr = 0; rr < cs; ++rr) Z += *dsmem(&ctl.hz[tid], rr);
      ctl.hlz[tid] = ctl.hlz[tid] + log2f(Z);
    }
    __syncthreads();
    // ranking key: log2 alpha~_j + log2 G = log2 sum_h exp2(L_hj - lz_h)  (U15)
    for (int j = tid; j < lc; j += kThreads) {
      if (logits[j] == -CUDART_INF_F) {
        tkeys[j] = 0u;
        continue;
      }
      float mx = -CUDART_INF_F;
      for (int h = 0; h < p.G; ++h) mx = fmaxf(mx, logits[h * p.ls + j] - ctl.hlz[h]);
      float s = 0.f;
      for (int h = 0; h < p.G; ++h) s += exp2f(logits[h * p.ls + j] - ctl.hlz[h] - mx);
      tkeys[j] = f2key(mx + log2f(s));
    }
    __syncthreads();

    // ---- phase D: S_t = top-k_t tokens ----
    {
      const int jtot = ctl.jtot;
      const int K = min(p.Kt, jtot);
      katt = K;
      const TopK t = cluster_topk(tkeys, lc, K, p.Kt >= jtot, cs, rank, ctl, 1);
      int* tout = p.token_ids + (size_t)pair * p.Kt;
      float* sout = p.token_scores ? p.token_scores + (size_t)pair * p.Kt : nullptr;
      const float lnG = logf((float)p.G);
      const bool fused = p.do_attend != 0;
      topk_emit(tkeys, lc, t, ctl, [&](int i, int pos) {
        const int kb = i / p.B;
        const int tok = cblk[cb0 + kb] * p.B + (i - kb * p.B);
        tout[pos] = tok;
        if (sout) sout[pos] = key2f(tkeys[i]) * kLn2 - lnG;
        if (fused) {
          int rr = (int)(((long long)pos * cs) / K);
          while (rr + 1 < cs && (long long)K * (rr + 1) / cs <= pos) ++rr;
          while (rr > 0 && (long long)K * rr / cs > pos) --rr;
          *dsmem(&sel[pos - (int)((long long)K * rr / cs)], rr) = tok;
        }
      });
      if (rank == 0) {
        for (int pos = K + tid; pos < p.Kt; pos += kThreads) {
          tout[pos] = -1;
          if (sout) sout[pos] = -CUDART_INF_F;
        }
        if (tid == 0) p.num_tokens[pair] = K;
      }
    }
    if (p.do_attend) cluster_sync_all();  // sel lists complete; select smem dead
  }

  if (p.do_attend) {
    int K = katt;
    if (!p.do_select) K = min(max(p.num_tokens[pair], 0), p.Kt);
    const int t0 = (int)((long long)K * rank / cs), t1 = (int)((long long)K * (rank + 1) / cs);
    const int tloc = t1 - t0;
    if (!p.do_select) {
      const int* ids = p.token_ids + (size_t)pair * p.Kt;
      for (int i = tid; i < tloc; i += kThreads) sel[i] = ids[t0 + i];
      __syncthreads();
    }
    float* aq = reinterpret_cast<float*>(smem + p.off_aq);
    float* as = reinterpret_cast<float*>(smem + p.off_as);
    float* ao = reinterpret_cast<float*>(smem + p.off_ao);
    phase_attend_generic<T>(p, pair, b, g, sel, tloc, aq, as, ao, ctl);
    cluster_sync_all();
    phase_merge<T>(p, b, g, rank, ao, ctl);
  }
  cluster_sync_all();  // no CTA leaves while its smem may still be read remotely
}

// ---------------------------------------------------------------- launcher
template <typename T, int CPL>
static cudaError_t launch_t(const DecodeParams& p, cudaStream_t stream) {
  auto kern = tls_decode_kernel<T, CPL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  if (p.cs > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)p.cs, (unsigned)(p.batch * p.Hkv), 1);
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.dynamicSmemBytes = p.smem_bytes;
  lc.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, kern, p);
}

// CPL = 16-byte chunks per lane of one block-summary row (2*d_k elements).
int decode_cpl(int d_k, size_t elem_bytes) {
  const int nchunk = (int)(2 * d_k * elem_bytes / 16);
  if (nchunk <= 32) return 1;
  if (nchunk <= 64) return 2;
  if (nchunk <= 160) return 5;
  return -1;
}

cudaError_t launch_decode(const DecodeParams& p, bool bf16, cudaStream_t stream) {
  const int cpl = decode_cpl(p.d_k, bf16 ? 2 : 4);
  if (bf16) {
    if (cpl == 1) return launch_t<__nv_bfloat16, 1>(p, stream);
    if (cpl == 2) return launch_t<__nv_bfloat16, 2>(p, stream);
    return launch_t<__nv_bfloat16, 5>(p, stream);
  }
  if (cpl == 1) return launch_t<float, 1>(p, stream);
  if (cpl == 2) return launch_t<float, 2>(p, stream);
  return launch_t<float, 5>(p, stream);
}

}  // namespace tls
