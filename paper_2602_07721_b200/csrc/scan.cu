// Stage I on the GPU: collision scan (a3) and bucket_topk (a4) — PAPER §4.2.2 (1).
//
// scan_kernel      every key of every KV head: score = sum_b LUT_b[id_b], 4 query heads per KV head packed as
//                  bytes of one u32 (max score 96 < 128, no carries). Reads 16 B of centroid ids per key.
//                  Lookup table in shared memory, 64 tables interleaved (word = c*64 + t, table t serves
//                  subspace t mod 16): lane L at step i reads subspace (L+i) mod 16 from table L+i, so the 32
//                  lanes of a warp hit 32 distinct banks for ANY ids (conflict-free). The encoder stores key t's
//                  id row rotated by t mod 16 bytes, so byte i of the row is that subspace; one PRMT builds the
//                  smem address (id byte -> bits 8..15, table offset -> bits 0..7). Per-warp score histograms
//                  in shared memory; per-chunk totals to global (deterministic, no global atomics).
// threshold_kernel s* = max{s : #(score >= s) >= C} per query head from the histograms, ties in the s* bucket
//                  handed out newest first (AMB-12), per-chunk output offsets.
// compact_kernel   writes the candidate ids (score > s*, plus each chunk's share of newest s* ties).
#include "common.cuh"

namespace pkv {
namespace {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_WARPS = SCAN_THREADS / 32;
constexpr int LUT_WORDS = NC * 64;                 // 64 KB
constexpr int SCAN_SMEM = LUT_WORDS * 4 + SCAN_WARPS * GMAX * HB * 4;
constexpr int SCAN_UNROLL = 4;

template <int RES, bool FAST>
__device__ __forceinline__ uint32_t lut_load(uint32_t addr, uint32_t lut_base) {
  uint32_t v;
  if (FAST) {
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(RES));
  } else {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr + lut_base));
  }
  return v;
}

template <int RES, bool FAST>
__device__ __forceinline__ void scan_loop(const uint8_t* __restrict__ ids_bh, uint32_t* __restrict__ scores_bh,
                                          uint32_t* hist_w, int64_t t_begin, int64_t t_end, int G,
                                          uint32_t lut_base) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t p[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) p[i] = (uint32_t)(lane + i) * 4u;
  for (int64_t base = t_begin + (int64_t)warp * 32; base < t_end; base += (int64_t)SCAN_WARPS * 32 * SCAN_UNROLL) {
    uint4 row[SCAN_UNROLL];
#pragma unroll
    for (int u = 0; u < SCAN_UNROLL; ++u) {
      const int64_t t = base + (int64_t)u * SCAN_WARPS * 32 + lane;
      if (t < t_end) row[u] = ldg_nc_v4(ids_bh + t * NB);
      else row[u] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < SCAN_UNROLL; ++u) {
      const int64_t t = base + (int64_t)u * SCAN_WARPS * 32 + lane;
      const uint32_t wds[4] = {row[u].x, row[u].y, row[u].z, row[u].w};
      uint32_t acc = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t a = prmt(wds[i >> 2], p[i], 0x5504u | ((uint32_t)(i & 3) << 4));
        acc += lut_load<RES, FAST>(a, lut_base);
      }
      if (t < t_end) {
        scores_bh[t] = acc;
        for (int hh = 0; hh < G; ++hh) atomicAdd(&hist_w[hh * HB + ((acc >> (8 * hh)) & 0xffu)], 1u);
      }
    }
  }
}

template <int RES>
__global__ void __launch_bounds__(SCAN_THREADS, 1)
    scan_kernel(const uint8_t* __restrict__ ids, const uint32_t* __restrict__ lut_g, uint32_t* __restrict__ scores,
                uint32_t* __restrict__ chunk_hist, int64_t cap, int64_t n, int64_t chunk, int G) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* lut = smem;
  uint32_t* hist = smem + LUT_WORDS;
  const int bh = blockIdx.y, j = blockIdx.x;
  const int64_t t_begin = (int64_t)j * chunk;
  const int64_t t_end = min(n, t_begin + chunk);
  // expand the compact table [c][16] into 4 interleaved replicas: word c*64 + s + 16 r
  const uint32_t* lg = lut_g + (int64_t)bh * NC * NB;
  for (int i = threadIdx.x; i < NC * NB; i += SCAN_THREADS) {
    const int c = i >> 4, s = i & 15;
    const uint32_t v = lg[i];
#pragma unroll
    for (int r = 0; r < 4; ++r) lut[c * 64 + s + 16 * ((r + (c & 1)) & 3)] = v;
  }
  for (int i = threadIdx.x; i < SCAN_WARPS * GMAX * HB; i += SCAN_THREADS) hist[i] = 0u;
  __syncthreads();
  const uint32_t lut_base = (uint32_t)__cvta_generic_to_shared(lut);
  const uint8_t* ids_bh = ids + (int64_t)bh * cap * NB;
  uint32_t* scores_bh = scores + (int64_t)bh * cap;
  uint32_t* hist_w = hist + (threadIdx.x >> 5) * GMAX * HB;
  if (lut_base == (uint32_t)RES) scan_loop<RES, true>(ids_bh, scores_bh, hist_w, t_begin, t_end, G, lut_base);
  else scan_loop<RES, false>(ids_bh, scores_bh, hist_w, t_begin, t_end, G, lut_base);
  __syncthreads();
  uint32_t* out = chunk_hist + ((int64_t)bh * MAX_CHUNKS + j) * GMAX * HB;
  for (int i = threadIdx.x; i < GMAX * HB; i += SCAN_THREADS) {
    uint32_t s = 0;
    for (int w = 0; w < SCAN_WARPS; ++w) s += hist[w * GMAX * HB + i];
    out[i] = s;
  }
}

// sel layout per (b, q head): [0] s*, [1] gt_local, [2] C_local, [3] take_local,
// then per chunk j: [4+4j] gt_off, [+1] tie_off, [+2] take_j, [+3] eq_j
constexpr int SEL_STRIDE = 4 + 4 * MAX_CHUNKS;

__global__ void __launch_bounds__(HB) threshold_kernel(const uint32_t* __restrict__ chunk_hist,
                                                        const uint32_t* __restrict__ all_hist, int P, int rank,
                                                        int nchunks, int n_q, int n_kv, int G, int batch,
                                                        int64_t C, int32_t* __restrict__ sel) {
  __shared__ uint32_t tot[HB], loc[HB];
  __shared__ int s_star_s, take_local_s, gt_local_s;
  __shared__ int gt_j[MAX_CHUNKS], eq_j[MAX_CHUNKS];
  const int h = blockIdx.x, b = blockIdx.y;
  const int g = h / G, hh = h % G;
  const int bin = threadIdx.x;
  const uint32_t* ch = chunk_hist + ((int64_t)(b * n_kv + g) * MAX_CHUNKS) * GMAX * HB + hh * HB;
  uint32_t l = 0;
  for (int j = 0; j < nchunks; ++j) l += ch[(int64_t)j * GMAX * HB + bin];
  loc[bin] = l;
  uint32_t t = l;
  if (P > 1) {
    t = 0;
    for (int r = 0; r < P; ++r) t += all_hist[(((int64_t)r * batch + b) * n_q + h) * HB + bin];
  }
  tot[bin] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t ge = 0;
    int s_star = HB;  // C == 0: nothing selected
    if (C > 0) {
      for (int s = HB - 1; s >= 0; --s) {
        if (ge + tot[s] >= C) { s_star = s; break; }
        ge += tot[s];
      }
    }
    int64_t need = (s_star < HB) ? C - ge : 0;
    // ties: newest rank first
    if (P > 1 && s_star < HB) {
      for (int r = P - 1; r > rank; --r) {
        need -= all_hist[(((int64_t)r * batch + b) * n_q + h) * HB + s_star];
        if (need < 0) need = 0;
      }
    }
    int64_t eq_local = (s_star < HB) ? loc[s_star] : 0;
    int64_t take_local = need < eq_local ? need : eq_local;
    int64_t gt_local = 0;
    for (int s = s_star + 1; s < HB; ++s) gt_local += loc[s];
    s_star_s = s_star;
    take_local_s = (int)take_local;
    gt_local_s = (int)gt_local;
  }
  __syncthreads();
  const int s_star = s_star_s;
  for (int j = threadIdx.x; j < nchunks; j += blockDim.x) {
    const uint32_t* cj = ch + (int64_t)j * GMAX * HB;
    uint32_t gsum = 0;
    for (int s = s_star + 1; s < HB; ++s) gsum += cj[s];
    gt_j[j] = (int)gsum;
    eq_j[j] = (s_star < HB) ? (int)cj[s_star] : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* o = sel + ((int64_t)b * n_q + h) * SEL_STRIDE;
    o[0] = s_star;
    o[1] = gt_local_s;
    o[2] = gt_local_s + take_local_s;
    o[3] = take_local_s;
    int run = 0;
    for (int j = 0; j < nchunks; ++j) {
      o[4 + 4 * j] = run;
      run += gt_j[j];
    }
    int rem = take_local_s, toff = gt_local_s;
    for (int j = nchunks - 1; j >= 0; --j) {
      const int take = rem < eq_j[j] ? rem : eq_j[j];
      o[4 + 4 * j + 1] = toff;
      o[4 + 4 * j + 2] = take;
      o[4 + 4 * j + 3] = eq_j[j];
      toff += take;
      rem -= take;
    }
  }
}

constexpr int CMP_THREADS = 1024;

__global__ void __launch_bounds__(CMP_THREADS) compact_kernel(const uint32_t* __restrict__ scores,
                                                               const int32_t* __restrict__ sel, int64_t cap,
                                                               int64_t n, int64_t chunk, int n_q, int n_kv, int G,
                                                               int64_t id_offset, int64_t cand_stride,
                                                               int32_t* __restrict__ cand) {
  __shared__ uint32_t wtot[32][2 * GMAX];
  __shared__ uint32_t wexc[32][2 * GMAX];
  __shared__ uint32_t ttot[2 * GMAX];
  __shared__ int prm[GMAX][5];
  const int bh = blockIdx.y, j = blockIdx.x;
  const int b = bh / n_kv, g = bh % n_kv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t_begin = (int64_t)j * chunk;
  const int64_t t_end = min(n, t_begin + chunk);
  if (threadIdx.x < G) {
    const int32_t* o = sel + ((int64_t)b * n_q + g * G + threadIdx.x) * SEL_STRIDE;
    prm[threadIdx.x][0] = o[0];
    prm[threadIdx.x][1] = o[4 + 4 * j];
    prm[threadIdx.x][2] = o[4 + 4 * j + 1];
    prm[threadIdx.x][3] = o[4 + 4 * j + 2];
    prm[threadIdx.x][4] = o[4 + 4 * j + 3];
  }
  __syncthreads();
  uint32_t run_gt[GMAX] = {0, 0, 0, 0}, run_eq[GMAX] = {0, 0, 0, 0};
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t* sc = scores + (int64_t)bh * cap;
  for (int64_t base = t_begin; base < t_end; base += CMP_THREADS) {
    const int64_t t = base + threadIdx.x;
    const uint32_t s = (t < t_end) ? sc[t] : 0xffffffffu;
    bool fgt[GMAX], feq[GMAX];
    uint32_t pre[2 * GMAX];
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) {
      const int sv = (int)((s >> (8 * hh)) & 0xffu);
      const bool valid = (t < t_end) && hh < G;
      fgt[hh] = valid && sv > prm[hh < G ? hh : 0][0];
      feq[hh] = valid && sv == prm[hh < G ? hh : 0][0];
      const uint32_t mg = __ballot_sync(0xffffffffu, fgt[hh]);
      const uint32_t me = __ballot_sync(0xffffffffu, feq[hh]);
      pre[2 * hh] = __popc(mg & lt_mask);
      pre[2 * hh + 1] = __popc(me & lt_mask);
      if (lane == 0) {
        wtot[warp][2 * hh] = __popc(mg);
        wtot[warp][2 * hh + 1] = __popc(me);
      }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int k = 0; k < 2 * GMAX; ++k) {
        const uint32_t v = wtot[lane][k];
        uint32_t inc = v;
#pragma unroll
        for (int x = 1; x < 32; x <<= 1) {
          const uint32_t o = __shfl_up_sync(0xffffffffu, inc, x);
          if (lane >= x) inc += o;
        }
        wexc[lane][k] = inc - v;
        if (lane == 31) ttot[k] = inc;
      }
    }
    __syncthreads();
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) {
      if (hh >= G) break;
      const int h = g * G + hh;
      int32_t* cd = cand + ((int64_t)b * n_q + h) * cand_stride;
      if (fgt[hh]) {
        const uint32_t pos = prm[hh][1] + run_gt[hh] + wexc[warp][2 * hh] + pre[2 * hh];
        cd[pos] = (int32_t)(t + id_offset);
      }
      if (feq[hh]) {
        const uint32_t asc = run_eq[hh] + wexc[warp][2 * hh + 1] + pre[2 * hh + 1];
        const int from_end = prm[hh][4] - 1 - (int)asc;
        if (from_end < prm[hh][3]) cd[prm[hh][2] + from_end] = (int32_t)(t + id_offset);
      }
      run_gt[hh] += ttot[2 * hh];
      run_eq[hh] += ttot[2 * hh + 1];
    }
    __syncthreads();
  }
}

__global__ void dbg_scores_kernel(const uint32_t* __restrict__ scores, int64_t cap, int64_t n, int n_q, int n_kv,
                                  int G, uint8_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int bh = blockIdx.y;
  if (t >= n) return;
  const int b = bh / n_kv, g = bh % n_kv;
  const uint32_t s = scores[(int64_t)bh * cap + t];
  for (int hh = 0; hh < G; ++hh) out[((int64_t)b * n_q + g * G + hh) * n + t] = (uint8_t)(s >> (8 * hh));
}

}  // namespace

cudaError_t init_scan_attrs() {
  cudaError_t e = cudaFuncSetAttribute(scan_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAN_SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(scan_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAN_SMEM);
}

ScanPlan plan_scan(const pkv_index* ix, int64_t n) {
  ScanPlan p;
  const int units = ix->batch * ix->cfg.n_kv_heads;
  int target = (ix->num_sms + units - 1) / units;  // ~1 CTA per SM (1024 threads, ~113 KB smem)
  int64_t chunk = (n + target - 1) / target;
  if (chunk < 2048) chunk = 2048;
  chunk = (chunk + 31) / 32 * 32;
  int nch = (int)((n + chunk - 1) / chunk);
  if (nch > MAX_CHUNKS) {
    chunk = ((n + MAX_CHUNKS - 1) / MAX_CHUNKS + 31) / 32 * 32;
    nch = (int)((n + chunk - 1) / chunk);
  }
  if (nch < 1) nch = 1;
  p.nchunks = nch;
  p.chunk = chunk;
  return p;
}

cudaError_t launch_scan(const pkv_index* ix, int64_t n, const ScanPlan& plan, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(plan.nchunks, ix->batch * ix->cfg.n_kv_heads);
  cudaError_t e;
  if (ix->smem_reserved == 1024) {
    ProfScope p_(K_SCAN, stream);
    scan_kernel<1024><<<grid, SCAN_THREADS, SCAN_SMEM, stream>>>(ix->ids, ws->lut, ws->scores, ws->chunk_hist,
                                                                  ix->cap, n, plan.chunk, ix->dcfg.G);
  } else {
    ProfScope p_(K_SCAN, stream);
    scan_kernel<0><<<grid, SCAN_THREADS, SCAN_SMEM, stream>>>(ix->ids, ws->lut, ws->scores, ws->chunk_hist,
                                                               ix->cap, n, plan.chunk, ix->dcfg.G);
  }
  e = cudaGetLastError();
  return e;
}

cudaError_t launch_threshold(const pkv_index* ix, const ScanPlan& plan, const uint32_t* all_hist, int P, int rank,
                             int64_t C, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_THRESHOLD, stream);
  threshold_kernel<<<grid, HB, 0, stream>>>(ws->chunk_hist, all_hist, P, rank, plan.nchunks, ix->cfg.n_q_heads,
                                            ix->cfg.n_kv_heads, ix->dcfg.G, ix->batch, C, ws->sel);
  return cudaGetLastError();
}

cudaError_t launch_compact(const pkv_index* ix, int64_t n, const ScanPlan& plan, int64_t id_offset,
                           int64_t cand_stride, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(plan.nchunks, ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_COMPACT, stream);
  compact_kernel<<<grid, CMP_THREADS, 0, stream>>>(ws->scores, ws->sel, ix->cap, n, plan.chunk, ix->cfg.n_q_heads,
                                                   ix->cfg.n_kv_heads, ix->dcfg.G, id_offset, cand_stride,
                                                   ws->cand);
  return cudaGetLastError();
}

cudaError_t launch_dbg_scores(const pkv_index* ix, int64_t n, uint8_t* out, cudaStream_t stream) {
  dim3 grid((unsigned)((n + 255) / 256), ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_DEBUG, stream);
  dbg_scores_kernel<<<grid, 256, 0, stream>>>(ix->ws->scores, ix->cap, n, ix->cfg.n_q_heads, ix->cfg.n_kv_heads,
                                              ix->dcfg.G, out);
  return cudaGetLastError();
}

__global__ void head_hist_kernel(const uint32_t* __restrict__ chunk_hist, int nchunks, int n_q, int n_kv, int G,
                                 uint32_t* __restrict__ out) {
  const int h = blockIdx.x, b = blockIdx.y, bin = threadIdx.x;
  const int g = h / G, hh = h % G;
  const uint32_t* ch = chunk_hist + ((int64_t)(b * n_kv + g) * MAX_CHUNKS) * GMAX * HB + hh * HB;
  uint32_t s = 0;
  for (int j = 0; j < nchunks; ++j) s += ch[(int64_t)j * GMAX * HB + bin];
  out[((int64_t)b * n_q + h) * HB + bin] = s;
}

cudaError_t launch_head_hist(const pkv_index* ix, const ScanPlan& plan, uint32_t* head_hist_out,
                             cudaStream_t stream) {
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_HEADHIST, stream);
  head_hist_kernel<<<grid, HB, 0, stream>>>(ix->ws->chunk_hist, plan.nchunks, ix->cfg.n_q_heads,
                                            ix->cfg.n_kv_heads, ix->dcfg.G, head_hist_out);
  return cudaGetLastError();
}

}  // namespace pkv
