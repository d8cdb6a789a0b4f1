// Stage II on the GPU: RSQ-IP rerank (a5) and final top-k (a6) — PAPER §4.1.3 Eq. 8-10, §4.2.2 (2),
// P:409-425, P:482-486, P:526 ("fused reranking kernel (gather+unpack+score)").
//
// rerank_kernel  one thread per candidate: gathers the key's 128-byte record (64 B of 4-bit codes + 16 fp32
//                w' = w/||sign*L[idx]||), decodes each nibble through a per-query table
//                T[j][nibble] = sign*L[idx]*q~_j held in shared memory (all lanes read the same 16-word row j,
//                which spans 16 distinct banks: conflict-free), est = ||q|| sum_b w'_b sum_j T[8b+j][nib].
// topk_kernel    per (sequence, query head): MSB-first radix select (8-bit digits) on the 64-bit composite key
//                (order-preserving fp32 bits of est << 32 | id), so ties in est go to the larger id;
//                the k winners are then bitonic-sorted descending. Also used to merge the ranks' local top-k
//                lists when sequence-sharded.
#include "common.cuh"

namespace pkv {
namespace {

constexpr int SEL_STRIDE = 4 + 4 * MAX_CHUNKS;
constexpr int RR_THREADS = 256;

__global__ void __launch_bounds__(RR_THREADS) rerank_kernel(const uint8_t* __restrict__ rec, const int32_t* __restrict__ cand,
                                                             const int32_t* __restrict__ sel,
                                                             const float* __restrict__ rtab,
                                                             const float* __restrict__ qnorm, int64_t cap, int n_q,
                                                             int n_kv, int G, int64_t cand_stride, int64_t id_offset,
                                                             float* __restrict__ est_out) {
  __shared__ float T[D * 16];
  const int h = blockIdx.y, b = blockIdx.z;
  const int g = h / G;
  const int64_t bhq = (int64_t)b * n_q + h;
  const int C_local = sel[bhq * SEL_STRIDE + 2];
  if ((int64_t)blockIdx.x * RR_THREADS >= C_local) return;
  const float* tsrc = rtab + bhq * D * 16;
  for (int i = threadIdx.x; i < D * 16; i += RR_THREADS) T[i] = tsrc[i];
  __syncthreads();
  const float qn = qnorm[bhq];
  const uint8_t* rec_bh = rec + ((int64_t)b * n_kv + g) * cap * REC;
  const int32_t* cd = cand + bhq * cand_stride;
  float* eo = est_out + bhq * cand_stride;
  for (int pos = blockIdx.x * RR_THREADS + threadIdx.x; pos < C_local; pos += gridDim.x * RR_THREADS) {
    const int64_t t = (int64_t)cd[pos] - id_offset;
    const uint8_t* r = rec_bh + t * REC;
    uint4 c4[4], w4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c4[i] = ldg_nc_v4(r + 16 * i);
#pragma unroll
    for (int i = 0; i < 4; ++i) w4[i] = ldg_nc_v4(r + 64 + 16 * i);
    const uint32_t cw[16] = {c4[0].x, c4[0].y, c4[0].z, c4[0].w, c4[1].x, c4[1].y, c4[1].z, c4[1].w,
                             c4[2].x, c4[2].y, c4[2].z, c4[2].w, c4[3].x, c4[3].y, c4[3].z, c4[3].w};
    const uint32_t ww[16] = {w4[0].x, w4[0].y, w4[0].z, w4[0].w, w4[1].x, w4[1].y, w4[1].z, w4[1].w,
                             w4[2].x, w4[2].y, w4[2].z, w4[2].w, w4[3].x, w4[3].y, w4[3].z, w4[3].w};
    float est = 0.f;
#pragma unroll
    for (int sb = 0; sb < NB; ++sb) {
      float dot = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t nib = (cw[sb] >> (4 * j)) & 15u;
        dot += T[(8 * sb + j) * 16 + nib];
      }
      est = fmaf(__uint_as_float(ww[sb]), dot, est);
    }
    eo[pos] = est * qn;
  }
}

// ---------------------------------------------------------------- radix top-k
constexpr int TK_THREADS = 1024;
constexpr int TK_CACHE = 12288;  // composite keys cached in (dynamic) smem when the list is short enough
constexpr int TK_SMEM = TK_CACHE * 8;

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
__device__ void radix_topk(const Src& src, int count, int k, int32_t* out_idx, float* out_est) {
  extern __shared__ unsigned long long cache[];  // [TK_CACHE]
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long win[MAX_TOPK];
  __shared__ unsigned long long prefix_s;
  __shared__ int need_s, done_s, nvalid_s, wcount;
  const int tid = threadIdx.x;
  const bool cached = count <= TK_CACHE;
  int nv = 0;
  if (tid == 0) {
    nvalid_s = 0;
    wcount = 0;
  }
  __syncthreads();
  for (int i = tid; i < count; i += TK_THREADS) {
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
    for (int i = tid; i < 256; i += TK_THREADS) hist[i] = 0u;
    __syncthreads();
    const unsigned long long hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
    const unsigned long long pre = prefix_s;
    for (int i = tid; i < count; i += TK_THREADS) {
      const unsigned long long kk = cached ? cache[i] : src.key(i);
      if (kk != 0ull && (kk & hmask) == pre) atomicAdd(&hist[(kk >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l covers digits 255-8l .. 248-8l (descending)
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
      const unsigned int need = (unsigned int)need_s;
      const bool mine = before < need && inc >= need;
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
    for (int i = tid; i < count; i += TK_THREADS) {
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
  for (int i = kv + tid; i < npow; i += TK_THREADS) win[i] = 0ull;
  __syncthreads();
  // bitonic sort descending
  for (int kk2 = 2; kk2 <= npow; kk2 <<= 1) {
    for (int j = kk2 >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < npow; i += TK_THREADS) {
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
  for (int i = tid; i < k; i += TK_THREADS) {
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

__global__ void __launch_bounds__(TK_THREADS) topk_kernel(const float* __restrict__ est, const int32_t* __restrict__ cand,
                                                           const int32_t* __restrict__ sel, int n_q,
                                                           int64_t cand_stride, int k, int out_stride,
                                                           int32_t* out_idx, float* out_est) {
  const int h = blockIdx.x, b = blockIdx.y;
  const int64_t bhq = (int64_t)b * n_q + h;
  const int count = sel[bhq * SEL_STRIDE + 2];
  CandSrc src{est + bhq * cand_stride, cand + bhq * cand_stride};
  radix_topk(src, count, k, out_idx + bhq * out_stride, out_est + bhq * out_stride);
}

__global__ void __launch_bounds__(TK_THREADS) merge_kernel(const float* __restrict__ all_est,
                                                            const int32_t* __restrict__ all_idx, int P, int batch,
                                                            int n_q, int k, int32_t* out_idx, float* out_est) {
  const int h = blockIdx.x, b = blockIdx.y;
  const int64_t bhq = (int64_t)b * n_q + h;
  MergeSrc src{all_est + bhq * MAX_TOPK, all_idx + bhq * MAX_TOPK, k, (int64_t)batch * n_q * MAX_TOPK};
  radix_topk(src, P * k, k, out_idx + bhq * k, out_est + bhq * k);
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

cudaError_t init_rerank_attrs() {
  cudaError_t e = cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TK_SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TK_SMEM);
}

cudaError_t launch_rerank(const pkv_index* ix, int64_t C_cap, int64_t id_offset, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  int64_t tiles = (C_cap + RR_THREADS - 1) / RR_THREADS;
  if (tiles < 1) tiles = 1;
  dim3 grid((unsigned)tiles, ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_RERANK, stream);
  rerank_kernel<<<grid, RR_THREADS, 0, stream>>>(ix->rec, ws->cand, ws->sel, ws->rtab, ws->qnorm, ix->cap,
                                                 ix->cfg.n_q_heads, ix->cfg.n_kv_heads, ix->dcfg.G, ws->cap,
                                                 id_offset, ws->est);
  return cudaGetLastError();
}

cudaError_t launch_topk(const pkv_index* ix, int64_t C_cap, int k, int32_t* out_idx, float* out_est,
                        int out_stride, cudaStream_t stream) {
  (void)C_cap;
  const Workspace* ws = ix->ws;
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_TOPK, stream);
  topk_kernel<<<grid, TK_THREADS, TK_SMEM, stream>>>(ws->est, ws->cand, ws->sel, ix->cfg.n_q_heads, ws->cap, k, out_stride,
                                               out_idx, out_est);
  return cudaGetLastError();
}

cudaError_t launch_topk_merge(const pkv_index* ix, int P, int k, const float* all_est, const int32_t* all_idx,
                              int32_t* out_idx, float* out_est, cudaStream_t stream) {
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_MERGE, stream);
  merge_kernel<<<grid, TK_THREADS, TK_SMEM, stream>>>(all_est, all_idx, P, ix->batch, ix->cfg.n_q_heads, k, out_idx,
                                                out_est);
  return cudaGetLastError();
}

cudaError_t launch_dbg_cand(const pkv_index* ix, int64_t C, int32_t* dbg_cand, float* dbg_est, cudaStream_t stream) {
  if (C <= 0) return cudaSuccess;
  dim3 grid((unsigned)((C + 255) / 256 < 64 ? (C + 255) / 256 : 64), ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_DEBUG, stream);
  dbg_cand_kernel<<<grid, 256, 0, stream>>>(ix->ws->cand, ix->ws->est, ix->ws->sel, ix->cfg.n_q_heads, ix->ws->cap, C,
                                            dbg_cand, dbg_est);
  return cudaGetLastError();
}

}  // namespace pkv
