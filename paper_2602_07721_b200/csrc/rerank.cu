// Stage II on the GPU: RSQ-IP rerank (a5) and final top-k (a6) — PAPER §4.1.3 Eq. 8-10, §4.2.2 (2),
// P:409-425, P:482-486, P:526 ("fused reranking kernel (gather+unpack+score)").
//
// rerank_cpt_kernel  a thread pair per candidate, CPT candidates per pair: each thread gathers half of the
//                    candidate's record (32 B of 4-bit codes + its 8 weights: fp32 w' = w/||sign*L[idx]||, or fp16
//                    with a per-key exponent) and decodes each nibble through a per-query table
//                    T[j][nibble] = sign*L[idx]*q~_j in shared memory: est = ||q|| sum_b w'_b sum_j T[8b+j][nib].
// topk_cl_kernel     per (sequence, query head) a thread-block cluster: local bucket-select top-k per CTA, sorted
//                    lists exchanged over DSMEM, global ranks by binary search; with ATTEND the gather and
//                    attention of the selected rows and of the hot rows (the latter before the dependency wait).
// topk_kernel        single-CTA variant for segmented (> 8 x 16384) candidate lists; merge_kernel merges
//                    per-segment / per-rank lists by MSB-first radix select on (ord(est) << 32 | id), so ties in
//                    est go to the larger id.
#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace pkv {
namespace {

constexpr int SEL_STRIDE = 4 + 4 * MAX_CHUNKS;
constexpr int RR_THREADS = 256;

// Two threads per candidate: the even thread decodes subspaces 0-7 (coordinates 0..63), the odd thread
// subspaces 8-15. Table row of coordinate c lives at physical row 2*(c mod 64) + c/64, so at every step the
// even lanes read an even row and the odd lanes the adjacent odd row: with 16-word rows the two halves use
// disjoint 16-bank halves (no conflicts), and the half offset (64 B) folds into the LOP3 that extracts the
// nibble address, so a lookup is SHF + LOP3 + LDS [reg + imm] + FADD.
constexpr int RT_ROWS = D;

// CPT candidates per thread pair (candidate tile of PER_CTA*CPT per CTA): the per-CTA work (table staging,
// pointers) is amortised over CPT candidates and their record loads are all in flight before the lookups.
// W16: records of 96 bytes with fp16 weights h_b and a per-key exponent E in their sign bits (encode.cu):
// each thread of the pair reads its 32 B of nibbles + 16 B of halves and decodes E from its own 8 halves.
template <int CPT, bool W16, int OCC = 6>
__global__ void __launch_bounds__(RR_THREADS, OCC) rerank_cpt_kernel(const uint8_t* __restrict__ rec, const int32_t* cand,
                                                                 const int32_t* sel, const float* rtab,
                                                                 const float* qnorm, int64_t cap, int n_q, int n_kv,
                                                                 int G, int64_t cand_stride, int64_t id_offset,
                                                                 float* est_out) {
  constexpr int RB = W16 ? 96 : REC;  // record stride
  __shared__ __align__(16) float T[RT_ROWS * 16];
  phase_mark(K_RERANK, 0);
  pdl_trigger();
  pdl_wait();
  phase_mark(K_RERANK, 1);
  cta_mark(K_RERANK, 1);
  const int h = blockIdx.y, b = blockIdx.z;
  const int g = h / G;
  const int64_t bhq = (int64_t)b * n_q + h;
  constexpr int PER_CTA = RR_THREADS / 2;
  constexpr int TILE = PER_CTA * CPT;
  const int32_t* cd = cand + bhq * cand_stride;
  const int C_local = sel[bhq * SEL_STRIDE + 2];
  // candidate tiles blockIdx.x, blockIdx.x + gridDim.x, ...: the grid is capped at the resident CTA count, so the
  // query table below is staged once per CTA, not once per tile (at 1M tokens: 205 tiles per head)
  int tile = blockIdx.x;
  int32_t cid[CPT];
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const int pos = tile * TILE + (threadIdx.x >> 1) + u * PER_CTA;
    cid[u] = pos < cand_stride ? cd[pos] : 0;  // speculative (inside the capacity); used only if pos < C_local
  }
  const float4* tsrc = reinterpret_cast<const float4*>(rtab + bhq * D * 16);
  float4 tv[D * 4 / RR_THREADS];
#pragma unroll
  for (int u = 0; u < D * 4 / RR_THREADS; ++u) tv[u] = tsrc[threadIdx.x + u * RR_THREADS];
  const float qn = qnorm[bhq];
  if (tile * TILE >= C_local) return;
#pragma unroll
  for (int u = 0; u < D * 4 / RR_THREADS; ++u) {  // coordinate c -> physical row 2(c%64)+c/64
    const int i = threadIdx.x + u * RR_THREADS;
    const int c = i >> 2;
    reinterpret_cast<float4*>(T)[(2 * (c & 63) + (c >> 6)) * 4 + (i & 3)] = tv[u];
  }
  const int half = threadIdx.x & 1;
  const uint8_t* rec_bh = rec + ((int64_t)b * n_kv + g) * cap * RB + 32 * half;
  float* eo = est_out + bhq * cand_stride;
  const char* Tb = reinterpret_cast<const char*>(T);
  const uint32_t hoff = half ? 64u : 0u;
  bool staged = false;
  for (; tile * TILE < C_local; tile += gridDim.x) {
  const int pos0 = tile * TILE + (threadIdx.x >> 1);
  // each thread's 32 B of nibbles and 32 B of weights (fp32) in one 256-bit load each: every request is a
  // whole sector (two 16-byte halves from two instructions would each fetch the sector from L2)
  u32x8 cr[CPT], wr[CPT];
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
#pragma unroll
    for (int i = 0; i < 8; ++i) cr[u].w[i] = wr[u].w[i] = 0u;
    if (pos0 + u * PER_CTA < C_local) {
      const uint8_t* r = rec_bh + ((int64_t)cid[u] - id_offset) * RB;
      cr[u] = ldg_nc_v8_early(r);
      if (W16) {
        const uint4 hv = ldg_nc_v4_early(r + 64 - 16 * half);  // halves of subspaces 8*half .. 8*half+7
        wr[u].w[0] = hv.x;
        wr[u].w[1] = hv.y;
        wr[u].w[2] = hv.z;
        wr[u].w[3] = hv.w;
      } else {
        wr[u] = ldg_nc_v8_early(r + 64);  // w' of subspaces 8*half .. 8*half+7 (r includes 32*half)
      }
    }
  }
  // the next tile's candidate ids, in flight during this tile's lookups
  const int nxt = tile + gridDim.x;
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const int pos = nxt * TILE + (threadIdx.x >> 1) + u * PER_CTA;
    cid[u] = (nxt * TILE < C_local && pos < cand_stride) ? cd[pos] : 0;
  }
  if (!staged) {
    __syncthreads();
    staged = true;
  }
  phase_mark(K_RERANK, 2);
  float est[CPT];
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const uint32_t* cw = cr[u].w;
    uint32_t ww[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ww[i] = wr[u].w[i];
    float escale = 1.f;
    if (W16) {
      const uint32_t h4[4] = {wr[u].w[0], wr[u].w[1], wr[u].w[2], wr[u].w[3]};
      uint32_t e8 = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) e8 |= (((h4[i] >> 15) & 1u) << (2 * i)) | (((h4[i] >> 31) & 1u) << (2 * i + 1));
      escale = __int_as_float((127 + (int)(int8_t)e8) << 23);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h4[i]));
        ww[2 * i] = __float_as_uint(fabsf(f.x));
        ww[2 * i + 1] = __float_as_uint(fabsf(f.y));
      }
    }
    float e = 0.f;
#pragma unroll
    for (int sb = 0; sb < 8; ++sb) {
      float dot = *reinterpret_cast<const float*>(Tb + (8 * sb) * 128 + (((cw[sb] << 2) & 0x3cu) | hoff));
#pragma unroll
      for (int j = 1; j < 8; ++j) {
        const uint32_t off = (cw[sb] >> (4 * j - 2)) & 0x3cu;
        dot += *reinterpret_cast<const float*>(Tb + (8 * sb + j) * 128 + (off | hoff));
      }
      e = fmaf(__uint_as_float(ww[sb]), dot, e);
    }
    est[u] = W16 ? e * escale : e;
  }
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const float e = est[u] + __shfl_xor_sync(0xffffffffu, est[u], 1);
    const int pos = pos0 + u * PER_CTA;
    if (!half && pos < C_local) eo[pos] = e * qn;
  }
  }  // tiles
  phase_mark(K_RERANK, 3);
  cta_mark(K_RERANK, 0);
}

// Long lists, balanced per SM (fp32 weights, one candidate per thread pair): a flat grid of exactly (resident CTAs
// per SM) x (SMs) CTAs, CTA c taking the contiguous range [c*NT/grid, (c+1)*NT/grid) of the NT = heads x tiles
// flattened (head, 128-candidate tile) space — every SM holds the same number of CTAs with the same number of
// tiles. rerank_cpt_kernel's grid of 27 CTAs per head puts 6 CTAs on some SMs and 5 on others (864 over 148 x 6
// slots) and those SMs finish ~20% apart at 1M. A CTA spans at most a few heads; the query table is restaged at
// each head change. Same decode as rerank_cpt_kernel (the identical instruction sequence): same bits.
template <int OCC>
__global__ void __launch_bounds__(RR_THREADS, OCC) rerank_flat_kernel(const uint8_t* __restrict__ rec, const int32_t* cand,
                                                                  const int32_t* sel, const float* rtab,
                                                                  const float* qnorm, int64_t cap, int n_q, int n_kv,
                                                                  int G, int64_t cand_stride, int64_t id_offset,
                                                                  float* est_out, int tiles_per_head, int64_t n_tiles,
                                                                  float alpha) {
  __shared__ __align__(16) float T[RT_ROWS * 16];
  phase_mark(K_RERANK, 0);
  pdl_trigger();
  pdl_wait();
  phase_mark(K_RERANK, 1);
  cta_mark(K_RERANK, 1);
  constexpr int TILE = RR_THREADS / 2;
  // range of CTA c: equal shares (alpha = 0), or shares ~ 1 / (1 + alpha c / P) — CTAs with higher linear ids run
  // slower when all of them compete for the SM (measured at 1M, see DESIGN), so they get fewer tiles:
  // f(c) = NT ln(1 + alpha c / P) / ln(1 + alpha)
  auto edge = [&](int x) -> int64_t {
    if (x >= (int)gridDim.x) return n_tiles;
    if (alpha <= 0.f) return (int64_t)x * n_tiles / gridDim.x;
    return (int64_t)((double)n_tiles * log1p((double)alpha * x / gridDim.x) / log1p((double)alpha));
  };
  const int64_t f0 = edge(blockIdx.x), f1 = edge(blockIdx.x + 1);
  const int half = threadIdx.x & 1;
  const char* Tb = reinterpret_cast<const char*>(T);
  const uint32_t hoff = half ? 64u : 0u;
  auto cid_of = [&](int64_t f) -> int32_t {  // candidate id of this thread pair in flattened tile f (0 if none)
    if (f >= f1) return 0;
    const int bhq = (int)f / tiles_per_head, tile = (int)f - bhq * tiles_per_head;  // 32-bit: < 2^31 tiles
    const int64_t pos = (int64_t)tile * TILE + (threadIdx.x >> 1);
    return pos < cand_stride ? cand[(int64_t)bhq * cand_stride + pos] : 0;
  };
  int32_t cid = cid_of(f0);
  int cur = -1;  // head whose table is staged
  int C_local = 0;
  float qn = 0.f;
  const uint8_t* rec_bh = nullptr;
  float* eo = nullptr;
  for (int64_t f = f0; f < f1; ++f) {
    const int bhq = (int)f / tiles_per_head, tile = (int)f - bhq * tiles_per_head;
    if (bhq != cur) {  // uniform over the CTA
      __syncthreads();  // every thread is done with the previous head's table
      const float4* tsrc = reinterpret_cast<const float4*>(rtab + (int64_t)bhq * D * 16);
#pragma unroll
      for (int u = 0; u < D * 4 / RR_THREADS; ++u) {
        const int i = threadIdx.x + u * RR_THREADS;
        const int c = i >> 2;
        reinterpret_cast<float4*>(T)[(2 * (c & 63) + (c >> 6)) * 4 + (i & 3)] = tsrc[i];
      }
      cur = bhq;
      const int b = bhq / n_q, h = bhq - b * n_q;
      C_local = sel[(int64_t)bhq * SEL_STRIDE + 2];
      qn = qnorm[bhq];
      rec_bh = rec + ((int64_t)b * n_kv + h / G) * cap * REC + 32 * half;
      eo = est_out + (int64_t)bhq * cand_stride;
      __syncthreads();
    }
    const int pos = tile * TILE + (threadIdx.x >> 1);
    u32x8 cr, wr;
#pragma unroll
    for (int i = 0; i < 8; ++i) cr.w[i] = wr.w[i] = 0u;
    if (pos < C_local) {
      const uint8_t* r = rec_bh + ((int64_t)cid - id_offset) * REC;
      cr = ldg_nc_v8_early(r);
      wr = ldg_nc_v8_early(r + 64);
    }
    cid = cid_of(f + 1);  // the next tile's candidate ids, in flight during this tile's lookups
    if (f == f0) phase_mark(K_RERANK, 2);
    const uint32_t* cw = cr.w;
    float e = 0.f;
#pragma unroll
    for (int sb = 0; sb < 8; ++sb) {
      float dot = *reinterpret_cast<const float*>(Tb + (8 * sb) * 128 + (((cw[sb] << 2) & 0x3cu) | hoff));
#pragma unroll
      for (int j = 1; j < 8; ++j) {
        const uint32_t off = (cw[sb] >> (4 * j - 2)) & 0x3cu;
        dot += *reinterpret_cast<const float*>(Tb + (8 * sb + j) * 128 + (off | hoff));
      }
      e = fmaf(__uint_as_float(wr.w[sb]), dot, e);
    }
    const float et = e + __shfl_xor_sync(0xffffffffu, e, 1);
    if (!half && pos < C_local) eo[pos] = et * qn;
  }
  phase_mark(K_RERANK, 3);
  cta_mark(K_RERANK, 0);
}

// GQA-union rerank: one record read per (key, KV head) for the union of the group's candidate
// lists. A half-warp per record, lane = subspace b: the lane reads the record's 4-byte nibble word and weight of
// its subspace (a half-warp reads the 128-byte record in two fully used 64-byte pieces), decodes each nibble to
// the signed level sign*L[idx] (16-entry smem table: distinct entries sit in distinct banks) and accumulates it
// against its 8 rotated query coordinates of every query head of the group (registers, loaded once per CTA):
// est_h = ||q_h|| sum_b w'_b sum_j v_{b,j} q~_{h,b,j}, the 16 subspace partials of the G <= 4 heads reduced
// with one reduce-scatter over the half-warp (5 shuffles), est_h written at the key's position in head h's list.
constexpr int UR_THREADS = 256;
#ifndef PKV_UR_PER
#define PKV_UR_PER 4
#endif
constexpr int UR_PER = PKV_UR_PER;                     // records per half-warp in flight
constexpr int UR_TILE = (UR_THREADS / 16) * UR_PER;   // records per CTA iteration

template <bool W16>
__global__ void __launch_bounds__(UR_THREADS) rerank_union_kernel(const uint8_t* __restrict__ rec, const int32_t* uid,
                                                                   const int32_t* upos, const unsigned int* ucount,
                                                                   const float* qrot, const float* qnorm, DevCfg cfg,
                                                                   int64_t cap, int n_q, int n_kv, int G,
                                                                   int64_t ustride, int64_t cand_stride,
                                                                   float* est_out) {
  constexpr int RB = W16 ? 96 : REC;
  __shared__ float sLv[16];  // nibble (sign << 3 | idx) -> sign * L[idx]
  const int g = blockIdx.y, b = blockIdx.z;
  const int64_t bg = (int64_t)b * n_kv + g;
  const int sb = threadIdx.x & 15, hw = threadIdx.x >> 4, hsel = sb >> 2;
  if (threadIdx.x < 16) {
    const float L = cfg.levels[threadIdx.x & 7];
    sLv[threadIdx.x] = (threadIdx.x & 8) ? L : -L;
  }
  pdl_trigger();
  pdl_wait();
  float qv[GMAX][8];
#pragma unroll
  for (int hh = 0; hh < GMAX; ++hh) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), c = a;
    if (hh < G) {
      const float4* qp = reinterpret_cast<const float4*>(qrot + ((int64_t)b * n_q + g * G + hh) * D + 8 * sb);
      a = qp[0];
      c = qp[1];
    }
    qv[hh][0] = a.x; qv[hh][1] = a.y; qv[hh][2] = a.z; qv[hh][3] = a.w;
    qv[hh][4] = c.x; qv[hh][5] = c.y; qv[hh][6] = c.z; qv[hh][7] = c.w;
  }
  const float qn = hsel < G ? qnorm[(int64_t)b * n_q + g * G + hsel] : 0.f;
  float* eo = est_out + ((int64_t)b * n_q + g * G + (hsel < G ? hsel : 0)) * cand_stride;
  const int64_t n_u = ucount[bg];
  __syncthreads();
  const uint8_t* rb = rec + bg * cap * RB;
  const int32_t* ub = uid + bg * ustride;
  const int32_t* pb = upos + bg * ustride * 4 + hsel;
  const bool b3 = (sb & 8) != 0, b2 = (sb & 4) != 0;
  for (int64_t u0 = (int64_t)blockIdx.x * UR_TILE + hw; u0 < n_u; u0 += (int64_t)gridDim.x * UR_TILE) {
    int key[UR_PER], pos[UR_PER];
    uint32_t cw[UR_PER], wb[UR_PER];
#pragma unroll
    for (int i = 0; i < UR_PER; ++i) {
      const int64_t u = u0 + 16 * i;
      key[i] = u < n_u ? ub[u] : -1;
      pos[i] = (u < n_u && (sb & 3) == 0) ? pb[4 * u] : -1;
    }
#pragma unroll
    for (int i = 0; i < UR_PER; ++i) {
      cw[i] = 0u;
      wb[i] = 0u;
      if (key[i] >= 0) {
        const uint8_t* r = rb + (int64_t)key[i] * RB;
        cw[i] = __ldg(reinterpret_cast<const uint32_t*>(r) + sb);
        wb[i] = W16 ? (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(r + 64) + sb)
                    : __ldg(reinterpret_cast<const uint32_t*>(r + 64) + sb);
      }
    }
#pragma unroll
    for (int i = 0; i < UR_PER; ++i) {
      float d[GMAX] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float v = sLv[(cw[i] >> (4 * j)) & 15u];
#pragma unroll
        for (int hh = 0; hh < GMAX; ++hh) d[hh] = fmaf(v, qv[hh][j], d[hh]);
      }
      float w, escale = 1.f;
      if (W16) {  // E: bit (b mod 8) in the sign bit of h_b (encode.cu); lanes 0-7 of the half-warp hold bits 0-7
        const uint32_t m = __ballot_sync(0xffffffffu, (wb[i] >> 15) & 1u);
        const int e8 = (int)(int8_t)((m >> (threadIdx.x & 16)) & 0xffu);
        escale = __int_as_float((127 + e8) << 23);
        w = __half2float(__ushort_as_half((unsigned short)(wb[i] & 0x7fffu)));
      } else {
        w = __uint_as_float(wb[i]);
      }
#pragma unroll
      for (int hh = 0; hh < GMAX; ++hh) d[hh] *= w;
      // reduce-scatter over the half-warp: afterwards lane b holds the sum of head b >> 2
      float k0 = b3 ? d[2] : d[0], k1 = b3 ? d[3] : d[1];
      k0 += __shfl_xor_sync(0xffffffffu, b3 ? d[0] : d[2], 8);
      k1 += __shfl_xor_sync(0xffffffffu, b3 ? d[1] : d[3], 8);
      float k = b2 ? k1 : k0;
      k += __shfl_xor_sync(0xffffffffu, b2 ? k0 : k1, 4);
      k += __shfl_xor_sync(0xffffffffu, k, 2);
      k += __shfl_xor_sync(0xffffffffu, k, 1);
      if (pos[i] >= 0) eo[pos[i]] = k * qn * escale;
    }
  }
}

// ---------------------------------------------------------------- radix top-k
constexpr int TK_THREADS = 1024;
constexpr int TK_CACHE = 12288;  // composite keys cached in (dynamic) smem when the list is short enough
constexpr int TK_SMEM = 16384 * 8;  // >= BS_CACHE * (4 + 4) and TK_CACHE * 8

struct CandSrc {  // unsharded: est/cand arrays of one (b, h); count from sel
  const float* est;
  const int32_t* idx;
  __device__ __forceinline__ unsigned long long key(int i) const {
    return ((unsigned long long)ord_f32(est[i]) << 32) | (uint32_t)idx[i];
  }
};
struct MergeSrc {  // sharded merge: P lists of k entries with stride
  const float* est;
  const int32_t* idx;
  int k;
  int64_t rank_stride;
  __device__ __forceinline__ unsigned long long key(int i) const {
    const int r = i / k, j = i % k;
    const int id = idx[r * rank_stride + j];
    if (id < 0) return 0ull;  // padding: never selected (excluded from counts)
    return ((unsigned long long)ord_f32(est[r * rank_stride + j]) << 32) | (uint32_t)id;
  }
};

template <class Src>
__device__ void radix_topk(const Src& src, int count, int k, int32_t* out_idx, float* out_est,
                           int cache_cap = TK_CACHE) {
  extern __shared__ unsigned long long cache[];  // [cache_cap] (aliases the caller's dynamic smem)
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long win[MAX_TOPK];
  __shared__ unsigned long long prefix_s;
  __shared__ int need_s, done_s, nvalid_s, wcount;
  const int tid = threadIdx.x;
  const bool cached = count <= cache_cap;
  int nv = 0;
  if (tid == 0) {
    nvalid_s = 0;
    wcount = 0;
  }
  __syncthreads();
  for (int i = tid; i < count; i += blockDim.x) {
    const unsigned long long kk = src.key(i);
    if (cached) cache[i] = kk;
    nv += (kk != 0ull);
  }
  atomicAdd(&nvalid_s, nv);
  __syncthreads();
  const int kv = min(k, nvalid_s);
  if (tid == 0) {
    prefix_s = 0ull;
    need_s = kv;
    done_s = (kv == 0);
  }
  __syncthreads();
  for (int shift = 56; shift >= 0; shift -= 8) {
    if (done_s) break;
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const unsigned long long hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
    const unsigned long long pre = prefix_s;
    for (int i = tid; i < count; i += blockDim.x) {
      const unsigned long long kk = cached ? cache[i] : src.key(i);
      if (kk != 0ull && (kk & hmask) == pre) atomicAdd(&hist[(kk >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l covers digits 255-8l .. 248-8l (descending)
      const unsigned int need = (unsigned int)need_s;  // read by every lane before the owner lane updates it
      unsigned int c[8], s = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        c[e] = hist[255 - 8 * tid - e];
        s += c[e];
      }
      unsigned int inc = s;
#pragma unroll
      for (int x = 1; x < 32; x <<= 1) {
        const unsigned int o = __shfl_up_sync(0xffffffffu, inc, x);
        if (tid >= x) inc += o;
      }
      const unsigned int before = inc - s;
      const bool mine = before < need && inc >= need;
      __syncwarp();  // all lanes have read need_s / prefix_s (independent thread scheduling)
      if (mine) {
        unsigned int cum = before;
        for (int e = 0; e < 8; ++e) {
          if (cum + c[e] >= need) {
            const unsigned int d = 255u - 8u * tid - e;
            prefix_s = pre | ((unsigned long long)d << shift);
            need_s = (int)(need - cum);
            done_s = (need - cum == c[e]);  // whole bucket taken: threshold = bucket floor
            break;
          }
          cum += c[e];
        }
      }
    }
    __syncthreads();
  }
  const unsigned long long kth = prefix_s;  // k-th largest composite key (or its bucket floor)
  if (kv > 0) {
    for (int i = tid; i < count; i += blockDim.x) {
      const unsigned long long kk = cached ? cache[i] : src.key(i);
      if (kk != 0ull && kk >= kth) {
        const int slot = atomicAdd(&wcount, 1);
        if (slot < MAX_TOPK) win[slot] = kk;
      }
    }
  }
  __syncthreads();
  int npow = 1;
  while (npow < kv) npow <<= 1;
  for (int i = kv + tid; i < npow; i += blockDim.x) win[i] = 0ull;
  __syncthreads();
  // bitonic sort descending
  for (int kk2 = 2; kk2 <= npow; kk2 <<= 1) {
    for (int j = kk2 >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < npow; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const bool desc = (i & kk2) == 0;
          const unsigned long long a = win[i], c = win[p];
          if (desc ? (a < c) : (a > c)) {
            win[i] = c;
            win[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < k; i += blockDim.x) {
    if (i < kv) {
      const unsigned long long kk = win[i];
      out_idx[i] = (int32_t)(uint32_t)(kk & 0xffffffffull);
      out_est[i] = unord_f32((uint32_t)(kk >> 32));
    } else {
      out_idx[i] = -1;
      out_est[i] = -INFINITY;
    }
  }
}

// Value-range bucket select (no sort over C): min/max of the estimates, a 2048-bin histogram of
// floor((est - min) * 2048 / (max - min)) (monotone in est, so bins partition the order), the boundary bin
// holding the k-th largest, and an exact (est, id) selection inside that bin only; the final order comes from
// rank counting over the k winners (composite keys are unique). Falls back to the radix select when the
// list does not fit the smem cache or the boundary bin is larger than its buffer.
constexpr int BS_BINS = 2048;
constexpr int BS_BND = 1024;
constexpr int BS_THREADS = 512;
constexpr int BS_CACHE = 16384;  // estimates cached in dynamic smem (64 KB)

__device__ __forceinline__ unsigned long long ckey(float e, int id) {
  return ((unsigned long long)ord_f32(e) << 32) | (uint32_t)id;
}

// Top-k of the `count` (estimate, id) pairs at es / ids, written in order to oi / oe (k entries, -1 padded).
__device__ __forceinline__ void topk_select(const float* es, const int32_t* ids, int count,
                                            int k, int32_t* oi, float* oe) {
  extern __shared__ float ecache[];  // [BS_CACHE] estimates, then [BS_CACHE] ids
  int32_t* icache = reinterpret_cast<int32_t*>(ecache + BS_CACHE);
  __shared__ unsigned int hist[BS_BINS];
  __shared__ unsigned long long win[MAX_TOPK];
  __shared__ unsigned long long bnd[BS_BND];
  __shared__ float red_mn[BS_THREADS / 32], red_mx[BS_THREADS / 32];
  __shared__ unsigned int wsum[BS_THREADS / 32];
  __shared__ int s_bstar, s_need, s_wc, s_bc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = BS_THREADS / 32;
  const int kv = min(k, count);
  phase_mark(K_TOPK, 2);
  if (count > BS_CACHE) {  // long lists (1M-token contexts): radix select straight from global memory
    CandSrc src{es, ids};
    radix_topk(src, count, k, oi, oe);
    return;
  }
  float mn = INFINITY, mx = -INFINITY;
  for (int i0 = 0; i0 < count; i0 += 16 * BS_THREADS) {  // 16 estimates + 16 ids in flight per thread
    float ev[16];
    int32_t iv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u * BS_THREADS + tid;
      ev[u] = i < count ? es[i] : 0.f;
      iv[u] = i < count ? ids[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u * BS_THREADS + tid;
      if (i < count) {
        ecache[i] = ev[u];
        icache[i] = iv[u];
        mn = fminf(mn, ev[u]);
        mx = fmaxf(mx, ev[u]);
      }
    }
  }
#pragma unroll
  for (int x = 16; x > 0; x >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, x));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, x));
  }
  if (lane == 0) {
    red_mn[warp] = mn;
    red_mx[warp] = mx;
  }
  for (int i = tid; i < BS_BINS; i += BS_THREADS) hist[i] = 0u;
  if (tid == 0) {
    s_wc = 0;
    s_bc = 0;
    s_bstar = -1;
    s_need = 0;
  }
  __syncthreads();
  mn = red_mn[lane % NW];
  mx = red_mx[lane % NW];
#pragma unroll
  for (int x = 16; x > 0; x >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, x));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, x));
  }
  phase_mark(K_TOPK, 3);
  const float range = mx - mn;
  const float scale = (range > 0.f) ? (float)BS_BINS / range : 0.f;
  auto bin_of = [&](float e) -> int { return min(BS_BINS - 1, (int)((e - mn) * scale)); };
  if (count > kv) {
    for (int i = tid; i < count; i += BS_THREADS) atomicAdd(&hist[bin_of(ecache[i])], 1u);
    __syncthreads();
    // thread t owns bins [2048 - 4(t+1), 2048 - 4t) (descending order); block suffix scan
    constexpr int PER = BS_BINS / BS_THREADS;
    unsigned int c[PER], sum = 0;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      c[e] = hist[BS_BINS - 1 - PER * tid - e];
      sum += c[e];
    }
    unsigned int inc = sum;
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) {
      const unsigned int o = __shfl_up_sync(0xffffffffu, inc, x);
      if (lane >= x) inc += o;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    unsigned int wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += wsum[w];
    const unsigned int before = wbase + inc - sum;
    if (before < (unsigned)kv && before + sum >= (unsigned)kv) {
      unsigned int cum = before;
#pragma unroll
      for (int e = 0; e < PER; ++e) {
        if (cum + c[e] >= (unsigned)kv) {
          s_bstar = BS_BINS - 1 - PER * tid - e;
          s_need = kv - (int)cum;
          break;
        }
        cum += c[e];
      }
    }
  }
  __syncthreads();
  phase_mark(K_TOPK, 4);
  const int bstar = s_bstar;
  if (bstar >= 0 && (int)hist[bstar] > BS_BND) {  // boundary bin too large (massive ties): exact radix
    CandSrc src{es, ids};
    radix_topk(src, count, k, oi, oe);
    return;
  }
  for (int i = tid; i < count; i += BS_THREADS) {
    const float e = ecache[i];
    const int bb = (bstar < 0) ? BS_BINS : bin_of(e);
    if (bb > bstar) win[atomicAdd(&s_wc, 1)] = ckey(e, icache[i]);
    else if (bb == bstar) bnd[atomicAdd(&s_bc, 1)] = ckey(e, icache[i]);
  }
  __syncthreads();
  phase_mark(K_TOPK, 5);
  const int nb = s_bc, need = s_need, wc = s_wc;
  // exact selection inside the boundary bin by rank counting (keys are unique)
  for (int i = tid; i < nb; i += BS_THREADS) {
    const unsigned long long x = bnd[i];
    int r = 0;
    for (int j2 = 0; j2 < nb; ++j2) r += bnd[j2] > x;
    if (r < need) win[wc + r] = x;
  }
  __syncthreads();
  phase_mark(K_TOPK, 6);
  // final order by rank counting over the kv winners: 4 threads per winner, each counting a quarter
  __shared__ int rk[MAX_TOPK];
  for (int i = tid; i < kv; i += BS_THREADS) rk[i] = 0;
  __syncthreads();
  {
    const int per = (kv + 3) / 4;
    for (int e = tid; e < 4 * kv; e += BS_THREADS) {
      const int i = e % kv, part = e / kv;
      const unsigned long long x = win[i];
      int r = 0;
      const int j1 = min(kv, (part + 1) * per);
      for (int j2 = part * per; j2 < j1; ++j2) r += win[j2] > x;
      if (r) atomicAdd(&rk[i], r);
    }
  }
  __syncthreads();
  for (int i = tid; i < kv; i += BS_THREADS) {
    const unsigned long long x = win[i];
    const int r = rk[i];
    oi[r] = (int32_t)(uint32_t)(x & 0xffffffffull);
    oe[r] = unord_f32((uint32_t)(x >> 32));
  }
  for (int i = kv + tid; i < k; i += BS_THREADS) {
    oi[i] = -1;
    oe[i] = -INFINITY;
  }
}


struct AttendEpi {  // gather + attention over the selected rows and the hot rows
  const void* q;
  const void* K;
  const void* V;
  int64_t sb, sh, st;
  float scale;
  const void* K_hot;      // hot rows attended in this kernel (may be null): row t of (b, h) at
  const void* V_hot;      //   K_hot + ((b*n_kv + h)*hot_rows + t)*D
  int n_hot;
  int hot_rows;
  void* out;
  float* lse;
  int G;
  float* out_f32;         // optional fp32 copy of out (pkv_index_set_debug_output), may be null
};

// Grid (n_q, batch, nseg). nseg == 1: the whole candidate list of a head, output at out_idx + bhq*out_stride.
// nseg > 1 (very long lists, e.g. 1M-token contexts): CTA z takes candidates [z*seg_len, (z+1)*seg_len) and
// writes its local top-k to slot z of out (slot stride seg_stride), to be merged by merge_kernel.
template <bool ATTEND, bool SELECT = true>
__global__ void __launch_bounds__(BS_THREADS) topk_kernel(const float* est, const int32_t* cand,
                                                           const int32_t* sel, int n_q,
                                                           int64_t cand_stride, int k, int out_stride,
                                                           int32_t* out_idx, float* out_est, AttendEpi ep,
                                                           int64_t seg_stride, int seg_len) {
  phase_mark(K_TOPK, 0);
  pdl_trigger();
  pdl_wait();
  phase_mark(K_TOPK, 1);
  if (SELECT) {
    const int h = blockIdx.x, b = blockIdx.y, z = blockIdx.z;
    const int64_t bhq = (int64_t)b * n_q + h;
    const int total = sel[bhq * SEL_STRIDE + 2];
    const int begin = gridDim.z > 1 ? min(total, z * seg_len) : 0;
    const int count = gridDim.z > 1 ? max(0, min(seg_len, total - begin)) : total;
    topk_select(est + bhq * cand_stride + begin, cand + bhq * cand_stride + begin, count, k,
                out_idx + z * seg_stride + bhq * out_stride, out_est + z * seg_stride + bhq * out_stride);
  }
  if constexpr (ATTEND) {
    __syncthreads();  // out_idx of this head written by this CTA
    extern __shared__ float ecache[];
    float* sm_o = ecache;                       // [16][128]
    float* sm_ml = ecache + 16 * D;             // [16][2]
    const int h = blockIdx.x, b = blockIdx.y;
    const int g = h / ep.G;
    const int n_kv = n_q / ep.G;
    const int64_t bhq = (int64_t)b * n_q + h;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NW = BS_THREADS / 32;
    const float qscale = ep.scale * 1.4426950408889634f;
    const uint2 qraw = ldg_v2(static_cast<const uint16_t*>(ep.q) + bhq * D + 4 * lane);
    const float q0 = bf16_lo(qraw.x) * qscale, q1 = bf16_hi(qraw.x) * qscale;
    const float q2 = bf16_lo(qraw.y) * qscale, q3 = bf16_hi(qraw.y) * qscale;
    const int32_t* oi = out_idx + bhq * out_stride;  // (ATTEND is only launched with nseg == 1)
    const uint16_t* Kb = static_cast<const uint16_t*>(ep.K) + (int64_t)b * ep.sb + (int64_t)g * ep.sh + 4 * lane;
    const uint16_t* Vb = static_cast<const uint16_t*>(ep.V) + (int64_t)b * ep.sb + (int64_t)g * ep.sh + 4 * lane;
    float m = -INFINITY, l = 0.f, o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
    constexpr int RB = 8;
    // rows of this head: the n_hot hot rows (sink + local + buffer) then the k retrieved rows
    const uint16_t* Khb = static_cast<const uint16_t*>(ep.K_hot) + ((int64_t)b * n_kv + g) * ep.hot_rows * D + 4 * lane;
    const uint16_t* Vhb = static_cast<const uint16_t*>(ep.V_hot) + ((int64_t)b * n_kv + g) * ep.hot_rows * D + 4 * lane;
    const int nrows = ep.n_hot + k;
    for (int r0 = warp; r0 < nrows; r0 += NW * RB) {
      int id[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int r = r0 + u * NW;
        id[u] = (r < ep.n_hot) ? r : (r < nrows ? oi[r - ep.n_hot] : -1);
      }
      uint2 kr[RB], vr[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int r = r0 + u * NW;
        kr[u] = make_uint2(0, 0);
        vr[u] = make_uint2(0, 0);
        if (r < ep.n_hot) {
          kr[u] = ldg_v2(Khb + (int64_t)r * D);
          vr[u] = ldg_v2(Vhb + (int64_t)r * D);
        } else if (id[u] >= 0) {
          kr[u] = ldg_v2(Kb + (int64_t)id[u] * ep.st);
          vr[u] = ldg_v2(Vb + (int64_t)id[u] * ep.st);
        }
      }
      float x[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u)
        x[u] = bf16_lo(kr[u].x) * q0 + bf16_hi(kr[u].x) * q1 + bf16_lo(kr[u].y) * q2 + bf16_hi(kr[u].y) * q3;
#pragma unroll
      for (int xm = 16; xm > 0; xm >>= 1) {
#pragma unroll
        for (int u = 0; u < RB; ++u) x[u] += __shfl_xor_sync(0xffffffffu, x[u], xm);
      }
      float mx = m;
#pragma unroll
      for (int u = 0; u < RB; ++u)
        if (id[u] >= 0) mx = fmaxf(mx, x[u]);
      if (mx == -INFINITY) continue;
      const float c = exp2f(m - mx);
      l *= c;
      o0 *= c;
      o1 *= c;
      o2 *= c;
      o3 *= c;
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        if (id[u] >= 0) {
          const float pu = exp2f(x[u] - mx);
          l += pu;
          o0 = fmaf(pu, bf16_lo(vr[u].x), o0);
          o1 = fmaf(pu, bf16_hi(vr[u].x), o1);
          o2 = fmaf(pu, bf16_lo(vr[u].y), o2);
          o3 = fmaf(pu, bf16_hi(vr[u].y), o3);
        }
      }
      m = mx;
    }
    phase_mark(K_TOPK, 8);
    sm_o[warp * D + 4 * lane] = o0;
    sm_o[warp * D + 4 * lane + 1] = o1;
    sm_o[warp * D + 4 * lane + 2] = o2;
    sm_o[warp * D + 4 * lane + 3] = o3;
    if (lane == 0) {
      sm_ml[2 * warp] = m;
      sm_ml[2 * warp + 1] = l;
    }
    __syncthreads();
    if (threadIdx.x < D) {
      const int d = threadIdx.x;
      float M = -INFINITY;
      for (int w = 0; w < NW; ++w) M = fmaxf(M, sm_ml[2 * w]);
      float L = 0.f, O = 0.f;
      if (M != -INFINITY) {
        for (int w = 0; w < NW; ++w) {
          const float mw = sm_ml[2 * w];
          if (mw == -INFINITY) continue;
          const float cw = exp2f(mw - M);
          L += cw * sm_ml[2 * w + 1];
          O += cw * sm_o[w * D + d];
        }
      }
      const float o = L > 0.f ? O / L : 0.f;
      static_cast<__nv_bfloat16*>(ep.out)[bhq * D + d] = __float2bfloat16_rn(o);
      if (ep.out_f32) ep.out_f32[bhq * D + d] = o;
      if (ep.lse && d == 0) ep.lse[bhq] = L > 0.f ? (M + log2f(L)) * 0.6931471805599453f : -INFINITY;
    }

  phase_mark(K_TOPK, 9);    (void)n_kv;
  }
}

// ---------------------------------------------------------------- cluster top-k (+ gather/attention)
// One thread-block cluster of R CTAs per (sequence, query head). CTA r owns candidates [r*per, (r+1)*per)
// (per = ceil(count/R)), caches them in shared memory and selects their local top-k with the value-range
// bucket select (exact, composite keys), sorted descending by split rank counting. The global top-k is contained
// in the union of the R local lists, so after one cluster barrier every CTA copies its peers' lists (at most
// R*k*8 bytes of distributed shared memory — DSMEM bandwidth is ~20 B/clk per SM, so only these short lists
// cross it) and ranks its own entries: global rank = local index + #peer entries greater, one binary search per
// (entry, peer list) pair, all in parallel. The CTA writes its entries
// with rank < k to out[rank] and, when ATTEND, gathers and attends those rows (the hot rows r*per .. (r+1)*per were attended before the dependency wait, seeding the
// online-softmax state), sending one (m, l, o) partial to CTA 0, which merges the
// R partials (log2 domain) after the second and last cluster barrier.
constexpr int CL_MAX = 8;
constexpr int CL_PARTS = 8;  // threads counting one local entry's rank within the CTA's list
constexpr int CL_SLICE = 16384;  // candidates per CTA (est + id cached: 8 B each)

struct SmemCand {  // radix fallback source: the CTA's cached slice
  const float* est;
  const int32_t* idx;
  __device__ __forceinline__ unsigned long long key(int i) const { return ckey(est[i], idx[i]); }
};

template <bool ATTEND>
__global__ void __launch_bounds__(BS_THREADS) topk_cl_kernel(const float* est, const int32_t* cand,
                                                              const int32_t* sel, int n_q,
                                                              int64_t cand_stride, int k, int out_stride,
                                                              int32_t* out_idx, float* out_est, AttendEpi ep,
                                                              int slice_cap) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int NW = BS_THREADS / 32;
  // dynamic: [slice_cap] estimates + [slice_cap] ids; after the local select: the peers' lists, then the
  // per-warp attention partials
  extern __shared__ float ecache[];
  int32_t* icache = reinterpret_cast<int32_t*>(ecache + slice_cap);
  __shared__ unsigned int hist[BS_BINS];
  __shared__ unsigned long long win[MAX_TOPK];
  __shared__ unsigned long long lst[MAX_TOPK];  // local top-k, descending (read by the peers)
  __shared__ unsigned long long bnd[BS_BND];
  int* rk = reinterpret_cast<int*>(hist);  // [MAX_TOPK] local ranks (the histogram is dead by then)
  __shared__ float cpart[CL_MAX][PART];  // CTA 0: the cluster's attention partials
  __shared__ float red_mn[NW], red_mx[NW];
  __shared__ unsigned int wsum[NW];
  __shared__ int s_wc, s_bc, s_bstar, s_need, s_bcount, s_kl;
  const int R = (int)cl.num_blocks(), r = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = blockIdx.y, b = blockIdx.z;
  const int64_t bhq = (int64_t)b * n_q + h;
  phase_mark(K_TOPK, 0);
  pdl_trigger();
  float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
  // online-softmax state of this warp (log2 domain); seeded with hot rows before the wait
  float am = -INFINITY, al = 0.f, ao0 = 0.f, ao1 = 0.f, ao2 = 0.f, ao3 = 0.f;
  if constexpr (ATTEND) {  // the query is an input of the layer, complete before the retrieval chain started
    const float qscale = ep.scale * 1.4426950408889634f;
    const uint2 qraw = ldg_v2(static_cast<const uint16_t*>(ep.q) + bhq * D + 4 * lane);
    q0 = bf16_lo(qraw.x) * qscale;
    q1 = bf16_hi(qraw.x) * qscale;
    q2 = bf16_lo(qraw.y) * qscale;
    q3 = bf16_hi(qraw.y) * qscale;
    // Hot rows (sink + local + buffer) do not depend on the retrieval: CTA r of the cluster attends
    // rows [r*per, (r+1)*per) of its head's KV group while the rerank kernel is still draining.
    if (ep.n_hot > 0) {
      const int Rr = (int)cl.num_blocks(), rr = (int)cl.block_rank();
      const int per = (ep.n_hot + Rr - 1) / Rr;
      const int r0 = rr * per, r1 = min(ep.n_hot, r0 + per);
      const int64_t hb = ((int64_t)b * (n_q / ep.G) + h / ep.G) * ep.hot_rows * D + 4 * lane;
      const uint16_t* Kh = static_cast<const uint16_t*>(ep.K_hot) + hb;
      const uint16_t* Vh = static_cast<const uint16_t*>(ep.V_hot) + hb;
      constexpr int HB2 = 4;
      for (int j0 = r0 + warp; j0 < r1; j0 += NW * HB2) {
        uint2 kr[HB2], vr[HB2];
#pragma unroll
        for (int u = 0; u < HB2; ++u) {
          const int r = j0 + u * NW;
          kr[u] = vr[u] = make_uint2(0, 0);
          if (r < r1) {
            kr[u] = ldg_v2(Kh + (int64_t)r * D);
            vr[u] = ldg_v2(Vh + (int64_t)r * D);
          }
        }
        float x[HB2];
#pragma unroll
        for (int u = 0; u < HB2; ++u)
          x[u] = bf16_lo(kr[u].x) * q0 + bf16_hi(kr[u].x) * q1 + bf16_lo(kr[u].y) * q2 + bf16_hi(kr[u].y) * q3;
#pragma unroll
        for (int xm = 16; xm > 0; xm >>= 1) {
#pragma unroll
          for (int u = 0; u < HB2; ++u) x[u] += __shfl_xor_sync(0xffffffffu, x[u], xm);
        }
        float mxx = am;
#pragma unroll
        for (int u = 0; u < HB2; ++u)
          if (j0 + u * NW < r1) mxx = fmaxf(mxx, x[u]);
        const float c = exp2f(am - mxx);
        al *= c;
        ao0 *= c;
        ao1 *= c;
        ao2 *= c;
        ao3 *= c;
#pragma unroll
        for (int u = 0; u < HB2; ++u) {
          if (j0 + u * NW < r1) {
            const float pu = exp2f(x[u] - mxx);
            al += pu;
            ao0 = fmaf(pu, bf16_lo(vr[u].x), ao0);
            ao1 = fmaf(pu, bf16_hi(vr[u].x), ao1);
            ao2 = fmaf(pu, bf16_lo(vr[u].y), ao2);
            ao3 = fmaf(pu, bf16_hi(vr[u].y), ao3);
          }
        }
        am = mxx;
      }
    }
  }
  pdl_wait();
  phase_mark(K_TOPK, 1);
  const int count = sel[bhq * SEL_STRIDE + 2];
  const int kv = min(k, count);
  const int per = (count + R - 1) / R;
  const int lo = min(count, r * per), n_loc = min(count, lo + per) - lo;
  const int kl = min(k, n_loc);
  const float* es = est + bhq * cand_stride;
  const int32_t* ids = cand + bhq * cand_stride;
  int32_t* oi = out_idx + bhq * out_stride;
  float* oe = out_est + bhq * out_stride;
  // ---- 1. cache the slice, min / max
  float mn = INFINITY, mx = -INFINITY;
  for (int i0 = 0; i0 < n_loc; i0 += 16 * BS_THREADS) {  // 16 per thread: an 8K slice (1M) in one round trip
    float ev[16];
    int32_t iv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u * BS_THREADS + tid;
      ev[u] = i < n_loc ? es[lo + i] : 0.f;
      iv[u] = i < n_loc ? ids[lo + i] : 0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u * BS_THREADS + tid;
      if (i < n_loc) {
        ecache[i] = ev[u];
        icache[i] = iv[u];
        mn = fminf(mn, ev[u]);
        mx = fmaxf(mx, ev[u]);
      }
    }
  }
#pragma unroll
  for (int x = 16; x > 0; x >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, x));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, x));
  }
  if (lane == 0) {
    red_mn[warp] = mn;
    red_mx[warp] = mx;
  }
  for (int i = tid; i < BS_BINS; i += BS_THREADS) hist[i] = 0u;
  if (tid == 0) {
    s_wc = 0;
    s_bc = 0;
    s_bstar = -1;
    s_need = 0;
    s_bcount = 0;
  }
  __syncthreads();
  mn = red_mn[lane % NW];
  mx = red_mx[lane % NW];
#pragma unroll
  for (int x = 16; x > 0; x >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, x));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, x));
  }
  phase_mark(K_TOPK, 2);
  const float range = mx - mn;
  const float scale = (range > 0.f) ? (float)BS_BINS / range : 0.f;
  auto bin_of = [&](float e) -> int { return min(BS_BINS - 1, (int)((e - mn) * scale)); };

  // ---- 2. local boundary bin (the kl-th largest) by a 2048-bin histogram
  if (n_loc > kl) {
    for (int i = tid; i < n_loc; i += BS_THREADS) atomicAdd(&hist[bin_of(ecache[i])], 1u);
    __syncthreads();
    constexpr int PER = BS_BINS / BS_THREADS;  // thread t owns bins [2048 - 4(t+1), 2048 - 4t)
    unsigned int c[PER], sum = 0;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      c[e] = hist[BS_BINS - 1 - PER * tid - e];
      sum += c[e];
    }
    unsigned int inc = sum;
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) {
      const unsigned int o = __shfl_up_sync(0xffffffffu, inc, x);
      if (lane >= x) inc += o;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    unsigned int wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += wsum[w];
    const unsigned int before = wbase + inc - sum;
    if (before < (unsigned)kl && before + sum >= (unsigned)kl) {
      unsigned int cum = before;
#pragma unroll
      for (int e = 0; e < PER; ++e) {
        if (cum + c[e] >= (unsigned)kl) {
          s_bstar = BS_BINS - 1 - PER * tid - e;
          s_need = kl - (int)cum;
          s_bcount = (int)c[e];
          break;
        }
        cum += c[e];
      }
    }
    __syncthreads();
  }
  phase_mark(K_TOPK, 3);
  const int bstar = s_bstar;
  if (s_bcount > BS_BND) {  // massive ties in one bin: exact radix select over the cached slice
    int32_t* tix = reinterpret_cast<int32_t*>(bnd);
    float* tes = reinterpret_cast<float*>(bnd) + MAX_TOPK;
    radix_topk(SmemCand{ecache, icache}, n_loc, kl, tix, tes, 0);
    __syncthreads();
    for (int i = tid; i < kl; i += BS_THREADS) lst[i] = ckey(tes[i], tix[i]);
  } else {
    // ---- 3. partition: above the boundary bin -> win, inside it -> bnd. Two passes over the cached slice: the
    // per-warp counts, one scan of them, then every warp writes at its own offsets (no contended atomics;
    // deterministic order)
    __shared__ int pw_w[NW], pw_b[NW];
    int cw = 0, cb = 0;
    for (int i0 = 0; i0 < n_loc; i0 += BS_THREADS) {
      const int i = i0 + tid;
      const int bb = i < n_loc ? ((bstar < 0) ? BS_BINS : bin_of(ecache[i])) : -2;
      cw += __popc(__ballot_sync(0xffffffffu, i < n_loc && bb > bstar));
      cb += __popc(__ballot_sync(0xffffffffu, i < n_loc && bb == bstar));
    }
    if (lane == 0) {
      pw_w[warp] = cw;
      pw_b[warp] = cb;
    }
    __syncthreads();
    int basew = 0, baseb = 0, totw = 0, totb = 0;
    for (int w = 0; w < NW; ++w) {
      basew += w < warp ? pw_w[w] : 0;
      baseb += w < warp ? pw_b[w] : 0;
      totw += pw_w[w];
      totb += pw_b[w];
    }
    if (tid == 0) {
      s_wc = totw;
      s_bc = totb;
    }
    const unsigned below = (1u << lane) - 1u;
    for (int i0 = 0; i0 < n_loc; i0 += BS_THREADS) {
      const int i = i0 + tid;
      float e = 0.f;
      int bb = -2;
      if (i < n_loc) {
        e = ecache[i];
        bb = (bstar < 0) ? BS_BINS : bin_of(e);
      }
      const unsigned mw = __ballot_sync(0xffffffffu, i < n_loc && bb > bstar);
      const unsigned mb = __ballot_sync(0xffffffffu, i < n_loc && bb == bstar);
      if ((mw >> lane) & 1u) win[basew + __popc(mw & below)] = ckey(e, icache[i]);
      if ((mb >> lane) & 1u) bnd[baseb + __popc(mb & below)] = ckey(e, icache[i]);
      basew += __popc(mw);
      baseb += __popc(mb);
    }
    __syncthreads();
    phase_mark(K_TOPK, 12);
    // ---- 4. exact selection inside the boundary bin (keys are unique): the local top-kl, in no order
    const int wc = s_wc, nb = s_bc, need = s_need;
    for (int i = tid; i < nb; i += BS_THREADS) {
      const unsigned long long x = bnd[i];
      int rr = 0;
      for (int j2 = 0; j2 < nb; ++j2) rr += bnd[j2] > x;
      if (rr < need) win[wc + rr] = x;
    }
    __syncthreads();
    phase_mark(K_TOPK, 13);
    // local order (descending) by split rank counting: CL_PARTS threads per entry, kl/CL_PARTS comparisons each
    for (int i = tid; i < kl; i += BS_THREADS) rk[i] = 0;  // rk aliases the histogram (dead since step 2)
    __syncthreads();
    const int seg = (kl + CL_PARTS - 1) / CL_PARTS;
    for (int e = tid; e < CL_PARTS * kl; e += BS_THREADS) {
      const int i = e % kl, part = e / kl;
      const unsigned long long x = win[i];
      int rr = 0;
      const int j1 = min(kl, (part + 1) * seg);
      for (int j2 = part * seg; j2 < j1; ++j2) rr += win[j2] > x;
      if (rr) atomicAdd(&rk[i], rr);
    }
    __syncthreads();
    for (int i = tid; i < kl; i += BS_THREADS) lst[rk[i]] = win[i];
  }
  if (tid == 0) s_kl = kl;
  phase_mark(K_TOPK, 4);
  cl.sync();  // #1: every CTA's local list is published
  phase_mark(K_TOPK, 5);

  // ---- 5. all R lists side by side (peers' over DSMEM, this CTA's own), then the global rank of each local
  // entry x: rank(x) = #{entries > x in the R lists} (composite keys are unique) = its local index + one binary
  // search per peer list. The rank-indexed slots win[0..kv) receive this CTA's winners.
  constexpr unsigned long long EMPTY = ~0ull;  // no candidate key has id 0xffffffff
  unsigned long long* plist = reinterpret_cast<unsigned long long*>(ecache);  // [R][k]
  __shared__ int pk[CL_MAX];
  if (tid < R) pk[tid] = (tid == r) ? kl : *cl.map_shared_rank(&s_kl, tid);
  __syncthreads();
  for (int e = tid; e < R * k; e += BS_THREADS) {  // one element per thread: all DSMEM reads in flight at once
    const int pr = e / k, i = e - pr * k;
    if (i < pk[pr]) plist[e] = (pr == r) ? lst[i] : *cl.map_shared_rank(lst + i, pr);
  }
  for (int i = tid; i < kl; i += BS_THREADS) rk[i] = 0;  // (the histogram it aliases is dead)
  for (int i = tid; i < kv; i += BS_THREADS) win[i] = EMPTY;
  __syncthreads();
  phase_mark(K_TOPK, 6);
  for (int e = tid; e < kl * R; e += BS_THREADS) {  // thread (entry i, list pr): binary search, all in parallel
    const int i = e % kl, pr = e / kl;
    const unsigned long long x = lst[i];
    int c = i;  // own list: sorted descending, so i entries are greater
    if (pr != r) {
      const unsigned long long* L = plist + pr * k;
      int a = 0, z = pk[pr];  // number of entries > x in the descending list L[0..pk)
      while (a < z) {
        const int m = (a + z) >> 1;
        if (L[m] > x) a = m + 1;
        else z = m;
      }
      c = a;
    }
    if (c) atomicAdd(&rk[i], c);
  }
  __syncthreads();
  phase_mark(K_TOPK, 14);
  for (int i = tid; i < kl; i += BS_THREADS) {
    const int rank = rk[i];
    if (rank < kv) {
      const unsigned long long x = lst[i];
      oi[rank] = (int32_t)(uint32_t)(x & 0xffffffffull);
      oe[rank] = unord_f32((uint32_t)(x >> 32));
      win[rank] = x;
    }
  }
  if (r == 0)
    for (int i = kv + tid; i < k; i += BS_THREADS) {
      oi[i] = -1;
      oe[i] = -INFINITY;
    }
  __syncthreads();
  // this CTA's winners compacted in rank order into bnd[0..nwin) (ordered ballot compaction over the slots)
  int nwin = 0;
  for (int t0 = 0; t0 < kv; t0 += BS_THREADS) {
    const int t = t0 + tid;
    const bool f = t < kv && win[t] != EMPTY;
    const unsigned mk = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[warp] = __popc(mk);
    __syncthreads();
    int before = nwin, tot = 0;
    for (int w = 0; w < NW; ++w) {
      const int c = (int)wsum[w];
      before += w < warp ? c : 0;
      tot += c;
    }
    if (f) bnd[before + __popc(mk & ((1u << lane) - 1u))] = win[t];
    nwin += tot;
    __syncthreads();
  }
  phase_mark(K_TOPK, 7);

  if constexpr (ATTEND) {
    // ---- 6. attention over this CTA's winners bnd[0..nwin), continuing the hot-row state
    const int g = h / ep.G;
    const uint16_t* Kb = static_cast<const uint16_t*>(ep.K) + (int64_t)b * ep.sb + (int64_t)g * ep.sh + 4 * lane;
    const uint16_t* Vb = static_cast<const uint16_t*>(ep.V) + (int64_t)b * ep.sb + (int64_t)g * ep.sh + 4 * lane;
    float m = am, l = al, o0 = ao0, o1 = ao1, o2 = ao2, o3 = ao3;  // continues the hot-row state
    constexpr int RB = 4;
    for (int j0 = warp; j0 < nwin; j0 += NW * RB) {
      int id[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int j = j0 + u * NW;
        id[u] = j < nwin ? (int)(uint32_t)(bnd[j] & 0xffffffffull) : -1;
      }
      uint2 kr[RB], vr[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        kr[u] = make_uint2(0, 0);
        vr[u] = make_uint2(0, 0);
        if (id[u] >= 0) {
          kr[u] = ldg_v2(Kb + (int64_t)id[u] * ep.st);
          vr[u] = ldg_v2(Vb + (int64_t)id[u] * ep.st);
        }
      }
      float x[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u)
        x[u] = bf16_lo(kr[u].x) * q0 + bf16_hi(kr[u].x) * q1 + bf16_lo(kr[u].y) * q2 + bf16_hi(kr[u].y) * q3;
#pragma unroll
      for (int xm = 16; xm > 0; xm >>= 1) {
#pragma unroll
        for (int u = 0; u < RB; ++u) x[u] += __shfl_xor_sync(0xffffffffu, x[u], xm);
      }
      float mxx = m;
#pragma unroll
      for (int u = 0; u < RB; ++u)
        if (id[u] >= 0) mxx = fmaxf(mxx, x[u]);
      const float c = exp2f(m - mxx);
      l *= c;
      o0 *= c;
      o1 *= c;
      o2 *= c;
      o3 *= c;
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        if (id[u] >= 0) {
          const float pu = exp2f(x[u] - mxx);
          l += pu;
          o0 = fmaf(pu, bf16_lo(vr[u].x), o0);
          o1 = fmaf(pu, bf16_hi(vr[u].x), o1);
          o2 = fmaf(pu, bf16_lo(vr[u].y), o2);
          o3 = fmaf(pu, bf16_hi(vr[u].y), o3);
        }
      }
      m = mxx;
    }
    phase_mark(K_TOPK, 8);
    float* sm_o = ecache + 2 * CL_MAX * k;         // [NW][D] (after the peers' lists)
    float* sm_ml = sm_o + NW * D;                  // [NW][2]
    sm_o[warp * D + 4 * lane] = o0;
    sm_o[warp * D + 4 * lane + 1] = o1;
    sm_o[warp * D + 4 * lane + 2] = o2;
    sm_o[warp * D + 4 * lane + 3] = o3;
    if (lane == 0) {
      sm_ml[2 * warp] = m;
      sm_ml[2 * warp + 1] = l;
    }
    __syncthreads();
    if (tid < D) {
      const int d = tid;
      float M = -INFINITY;
      for (int w = 0; w < NW; ++w) M = fmaxf(M, sm_ml[2 * w]);
      float L = 0.f, O = 0.f;
      if (M != -INFINITY) {
        for (int w = 0; w < NW; ++w) {
          const float mw = sm_ml[2 * w];
          if (mw == -INFINITY) continue;
          const float cw = exp2f(mw - M);
          L = fmaf(cw, sm_ml[2 * w + 1], L);
          O = fmaf(cw, sm_o[w * D + d], O);
        }
      }
      float* cp = cl.map_shared_rank(&cpart[r][0], 0);
      if (d == 0) {
        cp[0] = M;
        cp[1] = L;
      }
      cp[2 + d] = O;
    }
  }
  phase_mark(K_TOPK, 9);
  cl.sync();  // #2: no CTA reads a peer's shared memory past this point; CTA 0 holds the R partials
  phase_mark(K_TOPK, 10);
  if constexpr (ATTEND) {
    if (r == 0 && tid < D) {
      const int d = tid;
      float M = -INFINITY;
      for (int pr = 0; pr < R; ++pr) M = fmaxf(M, cpart[pr][0]);
      float L = 0.f, O = 0.f;
      if (M != -INFINITY) {
        for (int pr = 0; pr < R; ++pr) {
          if (cpart[pr][0] == -INFINITY) continue;
          const float c = exp2f(cpart[pr][0] - M);
          L = fmaf(c, cpart[pr][1], L);
          O = fmaf(c, cpart[pr][2 + d], O);
        }
      }
      const float o = L > 0.f ? O / L : 0.f;
      static_cast<__nv_bfloat16*>(ep.out)[bhq * D + d] = __float2bfloat16_rn(o);
      if (ep.out_f32) ep.out_f32[bhq * D + d] = o;
      if (ep.lse && d == 0) ep.lse[bhq] = L > 0.f ? (M + log2f(L)) * 0.6931471805599453f : -INFINITY;
    }
  }
  phase_mark(K_TOPK, 11);
}

__global__ void __launch_bounds__(TK_THREADS) merge_kernel(const float* all_est,
                                                            const int32_t* all_idx, int P, int64_t rank_stride,
                                                            int n_q, int k, int32_t* out_idx, float* out_est,
                                                            int out_stride) {
  const int h = blockIdx.x, b = blockIdx.y;
  const int64_t bhq = (int64_t)b * n_q + h;
  MergeSrc src{all_est + bhq * MAX_TOPK, all_idx + bhq * MAX_TOPK, k, rank_stride};
  radix_topk(src, P * k, k, out_idx + bhq * out_stride, out_est + bhq * out_stride);
}

// ---------------------------------------------------------------- sharded: fused top-k + attention exchange
// SURVEY §8(f3) "fusing T+A": instead of all-gathering the local top-k lists, merging, then computing and
// all-gathering attention partials over the owned winners (two exchanges), every rank ships, per query head,
// its local top-k entries together with what the attention needs from them — the logit x_j = <q, k_j>/sqrt(D)
// (log2 domain) and the value row v_j — plus its hot-row partial (last rank). After ONE all-gather every rank
// merges the P*k entries (same radix select on (est, id) as the unfused merge: identical top-k) and attends the
// selected entries' (x, v) directly, merging the hot partials: replicated output, one collective less.
// Slot of one (rank, sequence, head), in 32-bit words: [k x (est, id, x, 0)] [k x 64 words of bf16 v] [m, l, o[128]].
struct TASrc {  // merge source: P ranks x k entries, entries 4 words apart
  const uint32_t* base;
  int k;
  int64_t rank_stride;
  __device__ __forceinline__ unsigned long long key(int i) const {
    const int r = i / k, j = i % k;
    const uint32_t* e = base + r * rank_stride + 4 * j;
    if ((int32_t)e[1] < 0) return 0ull;  // padding: never selected
    return ((unsigned long long)ord_f32(__uint_as_float(e[0])) << 32) | e[1];
  }
};

__host__ __device__ constexpr int64_t ta_slot_words(int k) { return ((int64_t)68 * k + PART + 3) / 4 * 4; }

// Grid (n_q, batch), 256 threads: pack this rank's local top-k (lidx/lest, stride MAX_TOPK) into its slots.
__global__ void __launch_bounds__(256) ta_pack_kernel(const int32_t* lidx, const float* lest, int k, int n_q, int G,
                                                      const uint16_t* q, const uint16_t* K, const uint16_t* V,
                                                      int64_t sb, int64_t sh, int64_t st, float scale, int64_t off,
                                                      const uint16_t* K_hot, const uint16_t* V_hot, int n_hot,
                                                      uint32_t* msg, int64_t SW) {
  __shared__ float sm_o[8][D], sm_ml[8][2];
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x, b = blockIdx.y, g = h / G, n_kv = n_q / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bhq = (int64_t)b * n_q + h;
  uint32_t* slot = msg + bhq * SW;
  const float qs = scale * 1.4426950408889634f;
  const uint2 qr = ldg_v2(q + bhq * D + 4 * lane);
  const float q0 = bf16_lo(qr.x) * qs, q1 = bf16_hi(qr.x) * qs, q2 = bf16_lo(qr.y) * qs, q3 = bf16_hi(qr.y) * qs;
  const uint16_t* Kb = K + (int64_t)b * sb + (int64_t)g * sh + 4 * lane;
  const uint16_t* Vb = V + (int64_t)b * sb + (int64_t)g * sh + 4 * lane;
  for (int j = warp; j < k; j += 8) {
    const int32_t id = lidx[bhq * MAX_TOPK + j];
    float x = 0.f;
    if (id >= 0) {
      const uint2 kr = ldg_v2(Kb + (id - off) * st);
      const uint2 vr = ldg_v2(Vb + (id - off) * st);
      x = bf16_lo(kr.x) * q0 + bf16_hi(kr.x) * q1 + bf16_lo(kr.y) * q2 + bf16_hi(kr.y) * q3;
#pragma unroll
      for (int xm = 16; xm > 0; xm >>= 1) x += __shfl_xor_sync(0xffffffffu, x, xm);
      reinterpret_cast<uint2*>(slot + 4 * k + 64 * j)[lane] = vr;
    }
    if (lane == 0) {
      slot[4 * j] = __float_as_uint(id >= 0 ? lest[bhq * MAX_TOPK + j] : -INFINITY);
      slot[4 * j + 1] = (uint32_t)id;
      slot[4 * j + 2] = __float_as_uint(x);
      slot[4 * j + 3] = 0u;
    }
  }
  // hot-row partial of this head (n_hot = 0 except on the last rank)
  float m = -INFINITY, l = 0.f, o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
  const uint16_t* Kh = K_hot + ((int64_t)b * n_kv + g) * n_hot * D + 4 * lane;
  const uint16_t* Vh = V_hot + ((int64_t)b * n_kv + g) * n_hot * D + 4 * lane;
  for (int r = warp; r < n_hot; r += 8) {
    const uint2 kr = ldg_v2(Kh + (int64_t)r * D), vr = ldg_v2(Vh + (int64_t)r * D);
    float x = bf16_lo(kr.x) * q0 + bf16_hi(kr.x) * q1 + bf16_lo(kr.y) * q2 + bf16_hi(kr.y) * q3;
#pragma unroll
    for (int xm = 16; xm > 0; xm >>= 1) x += __shfl_xor_sync(0xffffffffu, x, xm);
    const float mx = fmaxf(m, x), c = exp2f(m - mx), p = exp2f(x - mx);
    l = l * c + p;
    o0 = fmaf(p, bf16_lo(vr.x), o0 * c);
    o1 = fmaf(p, bf16_hi(vr.x), o1 * c);
    o2 = fmaf(p, bf16_lo(vr.y), o2 * c);
    o3 = fmaf(p, bf16_hi(vr.y), o3 * c);
    m = mx;
  }
  sm_o[warp][4 * lane] = o0;
  sm_o[warp][4 * lane + 1] = o1;
  sm_o[warp][4 * lane + 2] = o2;
  sm_o[warp][4 * lane + 3] = o3;
  if (lane == 0) {
    sm_ml[warp][0] = m;
    sm_ml[warp][1] = l;
  }
  __syncthreads();
  if (threadIdx.x < D) {
    const int d = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < 8; ++w) M = fmaxf(M, sm_ml[w][0]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY)
      for (int w = 0; w < 8; ++w) {
        if (sm_ml[w][0] == -INFINITY) continue;
        const float c = exp2f(sm_ml[w][0] - M);
        L = fmaf(c, sm_ml[w][1], L);
        O = fmaf(c, sm_o[w][d], O);
      }
    float* hp = reinterpret_cast<float*>(slot + 68 * k);
    if (d == 0) {
      hp[0] = M;
      hp[1] = L;
    }
    hp[2 + d] = O;
  }
}

// Grid (n_q, batch), TK_THREADS: merge the P ranks' entries into the global top-k (radix select on (est, id), as
// merge_kernel) and attend the selected entries' (x, v) plus the P hot partials.
__global__ void __launch_bounds__(TK_THREADS) ta_merge_kernel(const uint32_t* msg, int P, int64_t rank_stride,
                                                              int64_t SW, int n_q, int k, int32_t* out_idx,
                                                              float* out_est, void* out, float* lse,
                                                              float* out_f32) {
  constexpr int NW = TK_THREADS / 32;
  __shared__ float sm_o[NW][D], sm_ml[NW][2];
  __shared__ unsigned long long s_kth;
  const int h = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bhq = (int64_t)b * n_q + h;
  pdl_trigger();
  pdl_wait();
  int32_t* oi = out_idx + bhq * k;
  float* oe = out_est + bhq * k;
  radix_topk(TASrc{msg + bhq * SW, k, rank_stride}, P * k, k, oi, oe);
  __syncthreads();
  if (threadIdx.x == 0) {
    int kv = 0;
    while (kv < k && oi[kv] >= 0) ++kv;
    s_kth = kv > 0 ? ckey(oe[kv - 1], oi[kv - 1]) : ~0ull;  // the k-th largest composite key (none: select none)
  }
  __syncthreads();
  const unsigned long long kth = s_kth;
  float m = -INFINITY, l = 0.f, o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
  for (int e = warp; e < P * k; e += NW) {
    const int r = e / k, j = e - r * k;
    const uint32_t* slot = msg + r * rank_stride + bhq * SW;
    const int32_t id = (int32_t)slot[4 * j + 1];
    if (id < 0 || ckey(__uint_as_float(slot[4 * j]), id) < kth) continue;  // warp-uniform
    const float x = __uint_as_float(slot[4 * j + 2]);
    const uint2 vr = reinterpret_cast<const uint2*>(slot + 4 * k + 64 * j)[lane];
    const float mx = fmaxf(m, x), c = exp2f(m - mx), p = exp2f(x - mx);
    l = l * c + p;
    o0 = fmaf(p, bf16_lo(vr.x), o0 * c);
    o1 = fmaf(p, bf16_hi(vr.x), o1 * c);
    o2 = fmaf(p, bf16_lo(vr.y), o2 * c);
    o3 = fmaf(p, bf16_hi(vr.y), o3 * c);
    m = mx;
  }
  sm_o[warp][4 * lane] = o0;
  sm_o[warp][4 * lane + 1] = o1;
  sm_o[warp][4 * lane + 2] = o2;
  sm_o[warp][4 * lane + 3] = o3;
  if (lane == 0) {
    sm_ml[warp][0] = m;
    sm_ml[warp][1] = l;
  }
  __syncthreads();
  if (threadIdx.x < D) {
    const int d = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < NW; ++w) M = fmaxf(M, sm_ml[w][0]);
    for (int r = 0; r < P; ++r) M = fmaxf(M, reinterpret_cast<const float*>(msg + r * rank_stride + bhq * SW + 68 * k)[0]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < NW; ++w) {
        if (sm_ml[w][0] == -INFINITY) continue;
        const float c = exp2f(sm_ml[w][0] - M);
        L = fmaf(c, sm_ml[w][1], L);
        O = fmaf(c, sm_o[w][d], O);
      }
      for (int r = 0; r < P; ++r) {
        const float* hp = reinterpret_cast<const float*>(msg + r * rank_stride + bhq * SW + 68 * k);
        if (hp[0] == -INFINITY) continue;
        const float c = exp2f(hp[0] - M);
        L = fmaf(c, hp[1], L);
        O = fmaf(c, hp[2 + d], O);
      }
    }
    const float o = L > 0.f ? O / L : 0.f;
    static_cast<__nv_bfloat16*>(out)[bhq * D + d] = __float2bfloat16_rn(o);
    if (out_f32) out_f32[bhq * D + d] = o;
    if (lse && d == 0) lse[bhq] = L > 0.f ? (M + log2f(L)) * 0.6931471805599453f : -INFINITY;
  }
}

__global__ void dbg_cand_kernel(const int32_t* __restrict__ cand, const float* __restrict__ est,
                                const int32_t* __restrict__ sel, int n_q, int64_t cand_stride, int64_t C,
                                int32_t* dbg_cand, float* dbg_est) {
  const int h = blockIdx.y, b = blockIdx.z;
  const int64_t bhq = (int64_t)b * n_q + h;
  const int cl = sel[bhq * SEL_STRIDE + 2];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < C; i += (int64_t)gridDim.x * blockDim.x) {
    if (dbg_cand) dbg_cand[bhq * C + i] = i < cl ? cand[bhq * cand_stride + i] : -1;
    if (dbg_est) dbg_est[bhq * C + i] = i < cl ? est[bhq * cand_stride + i] : 0.f;
  }
}

}  // namespace

// Cluster size for the top-k of C_cap candidates per head: enough CTAs to fill the SMs once (at most 8),
// and enough that each slice fits CL_SLICE. 0: too long for one cluster (segmented top-k + merge instead).
static int topk_cluster(const pkv_index* ix, int64_t C_cap, int* slice) {
  const int64_t heads = (int64_t)ix->cfg.n_q_heads * ix->batch;
  int R = (int)std::max<int64_t>(1, std::min<int64_t>(CL_MAX, ix->num_sms / heads));
  static const int r_env = [] {  // PKV_CL_R=1..8: cluster size override (A/B only; results are identical)
    const char* e = getenv("PKV_CL_R");
    return e ? atoi(e) : 0;
  }();
  if (C_cap < 1) C_cap = 1;
  // long lists: 8-CTA clusters once a 4-CTA slice would exceed 8192 candidates (1M: 184.0 vs 191.6 us/layer;
  // 6-CTA clusters measured 194.6 — they tile the GPCs poorly); short lists keep 4 (128K: 42.7 vs 48.4 with 8)
  if (R < CL_MAX && (C_cap + R - 1) / R > 8192) R = CL_MAX;
  if (r_env >= 1 && r_env <= CL_MAX) R = r_env;
  while (R < CL_MAX && (C_cap + R - 1) / R > CL_SLICE) ++R;
  if ((C_cap + R - 1) / R > CL_SLICE) return 0;
  *slice = (int)((C_cap + R - 1) / R);
  return R;
}

static size_t topk_cluster_smem(int slice, int k) {
  // max(candidate cache, peers' lists [CL_MAX][k] u64 + per-warp attention partials)
  const size_t need = (size_t)slice * 8, lists = (size_t)CL_MAX * k * 8 + (size_t)(BS_THREADS / 32) * (D + 2) * 4;
  return need > lists ? need : lists;
}

// Segments of a list too long for one cluster: ceil(C/BS_CACHE) (each cached in smem), at most SEG_SLOTS; beyond
// that the segments grow and topk_select streams them from global memory (radix path).
int topk_segments(int64_t C_cap) {
  if (C_cap <= (int64_t)CL_MAX * CL_SLICE) return 1;
  return (int)std::min<int64_t>(SEG_SLOTS, (C_cap + BS_CACHE - 1) / BS_CACHE);
}

cudaError_t init_rerank_attrs() {
  cudaError_t e = cudaFuncSetAttribute(topk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TK_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(topk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TK_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(topk_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TK_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(topk_cl_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SLICE * 8);
  if (e != cudaSuccess) return e;
  static_assert(CL_SLICE * 8 >= CL_MAX * MAX_TOPK * 8 + (BS_THREADS / 32) * (D + 2) * 4, "cluster top-k smem");
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(topk_cl_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SLICE * 8);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(ta_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TK_SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TK_SMEM);
}

// Read at every call (tests switch it); select and rerank of one step read it back to back.
bool union_rerank() {
  const char* e = getenv("PKV_RERANK");
  return e && std::string(e) == "union";
}

// Share skew of the flat rerank grid (PKV_RR_ALPHA overrides; 0 = equal ranges). 1M, same box, 200-step graphs:
// alpha 0 185.7-185.9, 0.7 179.5, 1.0 181.2-181.3, 1.4 182.1, 2.0 183.3 us/layer (another box: 0 183.1-183.8,
// 0.7 180.8). With equal ranges the CTA end times grow with the linear id (101.6 -> 120.2 us at 1M, independent of
// which tiles a CTA holds: a permuted id -> range map keeps the spread with the id), so the SMs idle through a tail.
static float rr_alpha() {
  static const float a = [] {
    const char* e = getenv("PKV_RR_ALPHA");
    return e ? (float)atof(e) : 0.7f;
  }();
  return a;
}

cudaError_t launch_rerank(const pkv_index* ix, int64_t C_cap, int64_t id_offset, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  if (union_rerank()) {
    static int occ = 0;
    if (!occ) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rerank_union_kernel<false>, UR_THREADS, 0) !=
              cudaSuccess || occ < 1)
        occ = 1;
    }
    const int64_t bk = (int64_t)ix->batch * ix->cfg.n_kv_heads;
    const int64_t most = std::min<int64_t>((int64_t)ix->dcfg.G * C_cap, ix->n);  // union size bound
    const int64_t tiles = std::max<int64_t>(1, (most + UR_TILE - 1) / UR_TILE);
    const int64_t persist = std::max<int64_t>(1, (int64_t)ix->num_sms * occ / bk);
    const dim3 grid((unsigned)std::min(tiles, persist), ix->cfg.n_kv_heads, ix->batch);
    ProfScope p_(K_RERANK, stream);
    auto kern = ix->dcfg.w16 ? rerank_union_kernel<true> : rerank_union_kernel<false>;
    return pdl_launch(kern, grid, dim3(UR_THREADS), 0, stream, (const uint8_t*)ix->rec, (const int32_t*)ws->uid,
                      (const int32_t*)ws->upos, (const unsigned int*)ws->ucount, (const float*)ws->qrot,
                      (const float*)ws->qnorm, ix->dcfg, ix->cap, ix->cfg.n_q_heads, ix->cfg.n_kv_heads, ix->dcfg.G,
                      ws->cap, ws->cap, ws->est);
  }
  static const int cpt_env = [] {  // candidates per thread pair (PKV_RR_CPT=1|2|4; default by list length)
    const char* e = getenv("PKV_RR_CPT");
    return e ? atoi(e) : 0;
  }();
  // one candidate per thread pair measured best at every size (1M: 186.7 vs 192.6 us/layer with 2)
  const int cpt = (cpt_env == 1 || cpt_env == 2 || cpt_env == 4) ? cpt_env : 1;
  const int64_t per = (int64_t)(RR_THREADS / 2) * cpt;
  // Register budget: 32 registers (8 CTAs = 2048 threads per SM) for short lists, where the whole list is
  // in flight in one wave (128K: 42.9 vs 43.8 us/layer); 40 (6 CTAs) for long lists that loop over tiles
  // (1M: 194.0 vs 197.1). PKV_RR_OCC=6|8 forces one (A/B).
  static const int occ_env = [] {
    const char* e = getenv("PKV_RR_OCC");
    return e ? atoi(e) : 0;
  }();
  const bool occ8 = (cpt <= 2) && (occ_env == 8 || (occ_env != 6 && C_cap <= 16384));
  auto kern = ix->dcfg.w16 ? (cpt == 1 ? rerank_cpt_kernel<1, true> : cpt == 2 ? rerank_cpt_kernel<2, true>
                                                                              : rerank_cpt_kernel<4, true>)
                           : (cpt == 1 ? rerank_cpt_kernel<1, false> : cpt == 2 ? rerank_cpt_kernel<2, false>
                                                                               : rerank_cpt_kernel<4, false>);
  if (occ8) kern = ix->dcfg.w16 ? (cpt == 1 ? rerank_cpt_kernel<1, true, 8> : rerank_cpt_kernel<2, true, 8>)
                                : (cpt == 1 ? rerank_cpt_kernel<1, false, 8> : rerank_cpt_kernel<2, false, 8>);
  // at most the resident CTA count per (sequence, query head): longer lists loop over tiles inside the CTA
  static int occ_cache[2][2][5] = {};
  int& occ = occ_cache[occ8 ? 1 : 0][ix->dcfg.w16 ? 1 : 0][cpt];
  if (!occ) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, RR_THREADS, 0) != cudaSuccess || occ < 1) occ = 1;
  }
  const int64_t tiles = std::max<int64_t>(1, (C_cap + per - 1) / per);
  const int64_t persist = std::max<int64_t>(1, (int64_t)ix->num_sms * occ / ((int64_t)ix->batch * ix->cfg.n_q_heads));
  // capped only when the tiles exceed two full waves: a short list (128K: 31 tiles per head vs 27 resident CTAs)
  // runs one CTA per tile, a long one (1M: 205+) loops over tiles in resident CTAs
  static const int flat_env = [] {  // PKV_RR_FLAT=0|1: force the per-head / the flat balanced grid (A/B)
    const char* e = getenv("PKV_RR_FLAT");
    return e ? atoi(e) : -1;
  }();
  // long lists, fp32 weights, one candidate per pair: the SM-balanced flat grid once every CTA loops over >= 8
  // tiles (1M: ~15 per CTA, 181.1-181.3 vs 182.3-182.7 us/layer same box; 32K bs 8, ~4.5 per CTA: 85.0 vs 82.7-83.0
  // — too few tiles to amortise the table restaging at head changes)
  auto fk = occ8 ? rerank_flat_kernel<8> : rerank_flat_kernel<6>;
  static int focc[2] = {0, 0};
  int& o = focc[occ8 ? 1 : 0];
  if (!o && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fk, RR_THREADS, 0) != cudaSuccess || o < 1)) o = 1;
  const int64_t heads = (int64_t)ix->batch * ix->cfg.n_q_heads;
  const int64_t n_tiles = heads * tiles;
  const int64_t ctas = std::min<int64_t>(n_tiles, (int64_t)ix->num_sms * o);
  const bool flat = !ix->dcfg.w16 && cpt == 1 && (flat_env == 1 || (flat_env != 0 && n_tiles >= 8 * ctas));
  if (flat) {
    ProfScope p_(K_RERANK, stream);
    return pdl_launch(fk, dim3((unsigned)ctas), dim3(RR_THREADS), 0, stream, (const uint8_t*)ix->rec,
                      (const int32_t*)ws->cand, (const int32_t*)ws->sel, (const float*)ws->rtab,
                      (const float*)ws->qnorm, ix->cap, ix->cfg.n_q_heads, ix->cfg.n_kv_heads, ix->dcfg.G, ws->cap,
                      id_offset, ws->est, (int)tiles, n_tiles, rr_alpha());
  }
  const dim3 grid((unsigned)(tiles > 2 * persist ? persist : tiles), ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_RERANK, stream);
  return pdl_launch(kern, grid, dim3(RR_THREADS), 0, stream, (const uint8_t*)ix->rec, (const int32_t*)ws->cand,
                    (const int32_t*)ws->sel, (const float*)ws->rtab, (const float*)ws->qnorm, ix->cap,
                    ix->cfg.n_q_heads, ix->cfg.n_kv_heads, ix->dcfg.G, ws->cap, id_offset, ws->est);
}

cudaError_t launch_topk(const pkv_index* ix, int64_t C_cap, int k, int32_t* out_idx, float* out_est,
                        int out_stride, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  C_cap = std::min<int64_t>(C_cap, ws->cap);  // a head's list never exceeds the workspace capacity (sharded: global C)
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_TOPK, stream);
  AttendEpi ep{};
  int slice = 0;
  const int R = topk_cluster(ix, C_cap, &slice);
  if (R > 0)
    return pdl_launch_cluster(topk_cl_kernel<false>, dim3(R, ix->cfg.n_q_heads, ix->batch), dim3(BS_THREADS),
                              topk_cluster_smem(slice, k), stream, R, (const float*)ws->est, (const int32_t*)ws->cand,
                              (const int32_t*)ws->sel, ix->cfg.n_q_heads, ws->cap, k, out_stride, out_idx, out_est,
                              ep, slice);
  const int nseg = topk_segments(C_cap);
  if (nseg > 1) {  // long candidate lists: per-segment top-k into the segment slots, then the merge kernel
    if (nseg > ws->seg_slots) return cudaErrorInvalidValue;  // the workspace holds seg_slots lists per head
    const size_t slot = (size_t)ix->batch * ix->cfg.n_q_heads * MAX_TOPK;
    const int seg_len = (int)((C_cap + nseg - 1) / nseg);
    dim3 g3(ix->cfg.n_q_heads, ix->batch, nseg);
    cudaError_t e = pdl_launch(topk_kernel<false>, g3, dim3(BS_THREADS), TK_SMEM, stream, (const float*)ws->est,
                               (const int32_t*)ws->cand, (const int32_t*)ws->sel, ix->cfg.n_q_heads, ws->cap, k,
                               MAX_TOPK, ws->seg_idx, ws->seg_est, ep, (int64_t)slot, seg_len);
    if (e != cudaSuccess) return e;
    return launch_topk_merge_strided(ix, nseg, k, ws->seg_est, ws->seg_idx, out_idx, out_est, out_stride, stream);
  }
  return pdl_launch(topk_kernel<false>, grid, dim3(BS_THREADS), TK_SMEM, stream, (const float*)ws->est,
                    (const int32_t*)ws->cand, (const int32_t*)ws->sel, ix->cfg.n_q_heads, ws->cap, k, out_stride,
                    out_idx, out_est, ep, (int64_t)0, 0);
}

cudaError_t launch_topk_attend(const pkv_index* ix, int64_t C_cap, int k, int32_t* out_idx, float* out_est, const void* q,
                               const void* K, const void* V, int64_t sb, int64_t sh, int64_t st, float scale,
                               const void* K_hot, const void* V_hot, int n_hot,
                               int hot_rows, void* out, float* lse, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_TOPK, stream);
  AttendEpi ep{q, K, V, sb, sh, st, scale, K_hot, V_hot, n_hot, hot_rows, out, lse, ix->dcfg.G, ix->dbg_out_f32};
  int slice = 0;
  const int R = topk_cluster(ix, C_cap, &slice);
  if (R > 0)
    return pdl_launch_cluster(topk_cl_kernel<true>, dim3(R, ix->cfg.n_q_heads, ix->batch), dim3(BS_THREADS),
                              topk_cluster_smem(slice, k), stream, R, (const float*)ws->est, (const int32_t*)ws->cand,
                              (const int32_t*)ws->sel, ix->cfg.n_q_heads, ws->cap, k, k, out_idx, out_est, ep,
                              slice);
  return pdl_launch(topk_kernel<true>, grid, dim3(BS_THREADS), TK_SMEM, stream, (const float*)ws->est,
                    (const int32_t*)ws->cand, (const int32_t*)ws->sel, ix->cfg.n_q_heads, ws->cap, k, k, out_idx,
                    out_est, ep, (int64_t)0, 0);
}

cudaError_t launch_topk_merge(const pkv_index* ix, int P, int k, const float* all_est, const int32_t* all_idx,
                              int64_t rank_stride, int32_t* out_idx, float* out_est, cudaStream_t stream) {
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_MERGE, stream);
  merge_kernel<<<grid, TK_THREADS, TK_SMEM, stream>>>(all_est, all_idx, P, rank_stride, ix->cfg.n_q_heads, k,
                                                out_idx, out_est, k);
  return cudaGetLastError();
}

cudaError_t launch_topk_attend_rows(const pkv_index* ix, int k, const int32_t* idx, const void* q, const void* K,
                                    const void* V, int64_t sb, int64_t sh, int64_t st, float scale,
                                    const void* K_hot, const void* V_hot, int n_hot, int hot_rows, void* out,
                                    float* lse, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_ATTEND, stream);
  AttendEpi ep{q, K, V, sb, sh, st, scale, K_hot, V_hot, n_hot, hot_rows, out, lse, ix->dcfg.G, ix->dbg_out_f32};
  return pdl_launch(topk_kernel<true, false>, grid, dim3(BS_THREADS), TK_SMEM, stream, (const float*)ws->est,
                    (const int32_t*)ws->cand, (const int32_t*)ws->sel, ix->cfg.n_q_heads, ws->cap, k, k,
                    const_cast<int32_t*>(idx), (float*)nullptr, ep, (int64_t)0, 0);
}

cudaError_t launch_topk_merge_strided(const pkv_index* ix, int P, int k, const float* all_est, const int32_t* all_idx,
                                      int32_t* out_idx, float* out_est, int out_stride, cudaStream_t stream) {
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_MERGE, stream);
  merge_kernel<<<grid, TK_THREADS, TK_SMEM, stream>>>(all_est, all_idx, P,
                                                (int64_t)ix->batch * ix->cfg.n_q_heads * MAX_TOPK,
                                                ix->cfg.n_q_heads, k, out_idx, out_est, out_stride);
  return cudaGetLastError();
}

int64_t ta_slot(int k) { return ta_slot_words(k); }

cudaError_t launch_ta_pack(const pkv_index* ix, const int32_t* lidx, const float* lest, int k, const void* q,
                           const void* K, const void* V, int64_t sb, int64_t sh, int64_t st, float scale, int64_t off,
                           const void* K_hot, const void* V_hot, int n_hot, uint32_t* msg, cudaStream_t stream) {
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_ATTEND, stream);
  return pdl_launch(ta_pack_kernel, grid, dim3(256), 0, stream, lidx, lest, k, ix->cfg.n_q_heads, ix->dcfg.G,
                    static_cast<const uint16_t*>(q), static_cast<const uint16_t*>(K), static_cast<const uint16_t*>(V),
                    sb, sh, st, scale, off, static_cast<const uint16_t*>(K_hot), static_cast<const uint16_t*>(V_hot),
                    n_hot, msg, ta_slot_words(k));
}

cudaError_t launch_ta_merge(const pkv_index* ix, const uint32_t* msg, int P, int k, int32_t* out_idx, float* out_est,
                            void* out, float* lse, cudaStream_t stream) {
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_MERGE, stream);
  const int64_t SW = ta_slot_words(k);
  return pdl_launch(ta_merge_kernel, grid, dim3(TK_THREADS), TK_SMEM, stream, msg, P,
                    (int64_t)ix->batch * ix->cfg.n_q_heads * SW, SW, ix->cfg.n_q_heads, k, out_idx, out_est, out, lse,
                    ix->dbg_out_f32);
}

cudaError_t launch_dbg_cand(const pkv_index* ix, int64_t C, int32_t* dbg_cand, float* dbg_est, cudaStream_t stream) {
  if (C <= 0) return cudaSuccess;
  dim3 grid((unsigned)((C + 255) / 256 < 64 ? (C + 255) / 256 : 64), ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_DEBUG, stream);
  dbg_cand_kernel<<<grid, 256, 0, stream>>>(ix->ws->cand, ix->ws->est, ix->ws->sel, ix->cfg.n_q_heads, ix->ws->cap, C,
                                            dbg_cand, dbg_est);
  return cudaGetLastError();
}

cudaError_t set_phase_rerank(unsigned long long* p) { return set_phase_ptr_tu(p); }

}  // namespace pkv
