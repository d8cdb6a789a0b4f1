// Inverted-list collision variant (the "collision processing scales with rho*n" formulation of
// P:531): instead of streaming all 16 centroid ids of every key (16 B per key, 16 lookups), the index keeps,
// per chunk of POST_CHUNK keys and per subspace, the chunk's keys bucketed by centroid id (u16 offsets, a
// counting sort), and a query visits only the buckets of its probed centroids: for every subspace s and
// centroid c whose packed lookup word (4 query heads' bonuses) is non-zero, one shared-memory atomic add of
// that word per key of the bucket. The packed scores are the dense scan's exactly (integer adds commute), and
// the kernel writes the same scores and cumulative per-chunk histograms, so the select kernel is unchanged.
//
// postings_build_kernel  grid (chunks, batch*n_kv): per subspace a 256-bin histogram, its exclusive scan
//                        (bucket offsets, u16 [257]) and the scatter of the keys' chunk offsets.
// postings_scan_kernel   grid (chunks, batch*n_kv), 1024 threads: zero the chunk's scores in shared memory,
//                        visit the probed buckets (each thread takes 4 of the 4096 (subspace, centroid) pairs,
//                        postings read 8 at a time), then scores + histograms as the dense scan's epilogue.
#include "common.cuh"

namespace pkv {
namespace {

constexpr int PS_THREADS = 1024;
constexpr int PS_WARPS = PS_THREADS / 32;

__global__ void __launch_bounds__(256) postings_build_kernel(const uint8_t* __restrict__ ids, int64_t cap, int64_t n,
                                                             int64_t chunk0, uint16_t* post_off, uint16_t* post_key) {
  __shared__ unsigned int hist[NC];
  __shared__ unsigned int cur[NC];
  const int j = (int)chunk0 + blockIdx.x, bh = blockIdx.y;
  const int64_t t0 = (int64_t)j * POST_CHUNK;
  const int len = (int)min((int64_t)POST_CHUNK, n - t0);
  const int64_t nchunk_cap = (cap + POST_CHUNK - 1) / POST_CHUNK;
  const uint8_t* idr = ids + ((int64_t)bh * cap + t0) * NB;
  uint16_t* off = post_off + ((int64_t)bh * nchunk_cap + j) * NB * (NC + 1);
  uint16_t* keys = post_key + ((int64_t)bh * nchunk_cap + j) * NB * POST_CHUNK;
  for (int s = 0; s < NB; ++s) {
    for (int c = threadIdx.x; c < NC; c += blockDim.x) hist[c] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const int64_t t = t0 + i;
      atomicAdd(&hist[idr[(int64_t)i * NB + ((s - (int)(t & 15)) & 15)]], 1u);  // rows are stored rotated
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of 256 bins, 8 per lane
      const int lane = threadIdx.x;
      unsigned int v[8], sum = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[e] = hist[8 * lane + e];
        sum += v[e];
      }
      unsigned int inc = sum;
#pragma unroll
      for (int x = 1; x < 32; x <<= 1) {
        const unsigned int o = __shfl_up_sync(0xffffffffu, inc, x);
        if (lane >= x) inc += o;
      }
      unsigned int run = inc - sum;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        off[s * (NC + 1) + 8 * lane + e] = (uint16_t)run;
        cur[8 * lane + e] = run;
        run += v[e];
      }
      if (lane == 31) off[s * (NC + 1) + NC] = (uint16_t)run;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const int64_t t = t0 + i;
      const int c = idr[(int64_t)i * NB + ((s - (int)(t & 15)) & 15)];
      keys[s * POST_CHUNK + atomicAdd(&cur[c], 1u)] = (uint16_t)i;  // order inside a bucket is immaterial
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(PS_THREADS, 1) postings_scan_kernel(const uint16_t* post_off, const uint16_t* post_key,
                                                                      const uint32_t* lut_g, uint32_t* scores,
                                                                      uint32_t* chunk_hist, int64_t cap, int64_t sstride,
                                                                      int64_t n) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* sc = smem;                       // [POST_CHUNK] packed scores of the chunk
  uint32_t* hist = smem + POST_CHUNK;        // [PS_WARPS][GMAX][HB]
  const int j = blockIdx.x, bh = blockIdx.y;
  const int64_t t0 = (int64_t)j * POST_CHUNK;
  const int len = (int)min((int64_t)POST_CHUNK, n - t0);
  const int64_t nchunk_cap = (cap + POST_CHUNK - 1) / POST_CHUNK;
  const uint16_t* off = post_off + ((int64_t)bh * nchunk_cap + j) * NB * (NC + 1);
  const uint16_t* keys = post_key + ((int64_t)bh * nchunk_cap + j) * NB * POST_CHUNK;
  pdl_trigger();
  for (int i = threadIdx.x; i < POST_CHUNK; i += PS_THREADS) sc[i] = 0u;
  for (int i = threadIdx.x; i < PS_WARPS * GMAX * HB; i += PS_THREADS) hist[i] = 0u;
  __syncthreads();
  pdl_wait();  // lookup table comes from qprep
  const uint8_t* lb = reinterpret_cast<const uint8_t*>(lut_g + (int64_t)bh * NC * NB);  // [hh][s][c] bonus bytes
  // each thread: (s, c) pairs p = tid + 1024 u, s = p % 16, c = p / 16; word = the 4 query heads' bonus bytes
  uint32_t w[NC * NB / PS_THREADS];
#pragma unroll
  for (int u = 0; u < NC * NB / PS_THREADS; ++u) {
    const int p = threadIdx.x + u * PS_THREADS, s = p & 15, c = p >> 4;
    w[u] = 0u;
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) w[u] |= (uint32_t)lb[(hh * NB + s) * NC + c] << (8 * hh);
  }
#pragma unroll
  for (int u = 0; u < NC * NB / PS_THREADS; ++u) {
    if (w[u] == 0u) continue;
    const int p = threadIdx.x + u * PS_THREADS, s = p & 15, c = p >> 4;
    const int a = off[s * (NC + 1) + c], z = off[s * (NC + 1) + c + 1];
    const uint16_t* kb = keys + s * POST_CHUNK;
    int i = a;
    for (; i < z && (i & 7); ++i) atomicAdd(&sc[kb[i]], w[u]);
    for (; i + 8 <= z; i += 8) {  // 8 postings per 16-byte load
      const uint4 v = *reinterpret_cast<const uint4*>(kb + i);
      const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        atomicAdd(&sc[vv[e] & 0xffffu], w[u]);
        atomicAdd(&sc[vv[e] >> 16], w[u]);
      }
    }
    for (; i < z; ++i) atomicAdd(&sc[kb[i]], w[u]);
  }
  __syncthreads();
  // scores to global + per-warp histograms (the dense scan's epilogue)
  uint32_t* out_sc = scores + (int64_t)bh * sstride + t0;
  uint32_t* hist_w = hist + (threadIdx.x >> 5) * GMAX * HB;
  for (int i = threadIdx.x; i < len; i += PS_THREADS) {
    const uint32_t acc = sc[i];
    out_sc[i] = acc;
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) atomicAdd(&hist_w[hh * HB + prmt(acc, 0u, 0x4440u | (uint32_t)hh)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < GMAX * HB; i += PS_THREADS) {
    uint32_t s2 = 0;
    for (int w2 = 0; w2 < PS_WARPS; ++w2) s2 += hist[w2 * GMAX * HB + i];
    hist[i] = s2;
  }
  __syncthreads();
  uint32_t* outh = chunk_hist + ((int64_t)bh * MAX_CHUNKS + j) * GMAX * HB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < GMAX) {  // cumulative counts #(score >= s), lane l owns bins 4l..4l+3
    uint32_t v[4], tot = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[e] = hist[warp * HB + 4 * lane + e];
      tot += v[e];
    }
    uint32_t inc = tot;
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) {
      const uint32_t o = __shfl_down_sync(0xffffffffu, inc, x);
      if (lane + x < 32) inc += o;
    }
    uint32_t run = inc - tot;
#pragma unroll
    for (int e = 3; e >= 0; --e) {
      run += v[e];
      outh[warp * HB + 4 * lane + e] = run;
    }
  }
}

}  // namespace

constexpr int PS_SMEM = POST_CHUNK * 4 + PS_WARPS * GMAX * HB * 4;

cudaError_t init_postings_attrs() {
  return cudaFuncSetAttribute(postings_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PS_SMEM);
}

cudaError_t launch_postings_build(const pkv_index* ix, int64_t chunk0, int64_t chunk1, cudaStream_t stream) {
  if (chunk1 <= chunk0) return cudaSuccess;
  dim3 grid((unsigned)(chunk1 - chunk0), ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_ENCODE, stream);
  postings_build_kernel<<<grid, 256, 0, stream>>>(ix->ids, ix->cap, ix->n, chunk0, ix->post_off, ix->post_key);
  return cudaGetLastError();
}

cudaError_t launch_postings_scan(const pkv_index* ix, int64_t n, int64_t sstride, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid((unsigned)((n + POST_CHUNK - 1) / POST_CHUNK), ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_SCAN, stream);
  return pdl_launch(postings_scan_kernel, grid, dim3(PS_THREADS), PS_SMEM, stream, (const uint16_t*)ix->post_off,
                    (const uint16_t*)ix->post_key, (const uint32_t*)ws->lut, ws->scores, ws->chunk_hist, ix->cap,
                    sstride, n);
}

}  // namespace pkv
