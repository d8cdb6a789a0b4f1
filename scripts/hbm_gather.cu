// Gather roofline for the rerank (a5): how fast can B200 read 128-byte records at sparse, ascending positions
// (a candidate list in key order) from HBM? Records of 128 B, a buffer of 8 KV heads x n keys, density = C / n.
//   dense  : every record (streaming reference)
//   sparse : each of 32 "query heads" reads C sorted random records of its KV head (h / 4), two threads per
//            record (32 B + 32 B each, like rerank_cpt_kernel), grid capped at the resident CTA count
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hbm_gather scripts/hbm_gather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

struct u32x8 { uint32_t w[8]; };
__device__ __forceinline__ u32x8 ld8(const void* p) {
  u32x8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
                 "=r"(r.w[7]) : "l"(p));
  return r;
}

template <int CPT>
__global__ void __launch_bounds__(256) gather(const uint8_t* rec, const int* cand, int64_t n, int C, int G, unsigned* out) {
  const int h = blockIdx.y;
  const uint8_t* rb = rec + (int64_t)(h / G) * n * 128 + 32 * (threadIdx.x & 1);
  const int* cd = cand + (int64_t)h * C;
  uint32_t acc = 0;
  for (int tile = blockIdx.x; tile * 128 * CPT < C; tile += gridDim.x) {
    u32x8 a[CPT], b[CPT];
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
      const int pos = tile * 128 * CPT + u * 128 + (threadIdx.x >> 1);
      if (pos < C) {
        const uint8_t* r = rb + (int64_t)cd[pos] * 128;
        a[u] = ld8(r);
        b[u] = ld8(r + 64);
      } else {
        for (int i = 0; i < 8; ++i) a[u].w[i] = b[u].w[i] = 0;
      }
    }
#pragma unroll
    for (int u = 0; u < CPT; ++u)
      for (int i = 0; i < 8; ++i) acc += a[u].w[i] ^ b[u].w[i];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int n_kv = 8, n_q = 32, G = 4;
  for (int64_t n : {130800LL, 1048304LL}) {
    uint8_t* rec;
    CK(cudaMalloc(&rec, (size_t)n_kv * n * 128));
    CK(cudaMemset(rec, 1, (size_t)n_kv * n * 128));
    uint8_t* flush;
    CK(cudaMalloc(&flush, 512ull << 20));
    unsigned* dout;
    CK(cudaMalloc(&dout, 4));
    for (double dens : {0.06, 0.05, 1.0}) {
      const int C = (int)(dens * n);
      std::vector<int> ids((size_t)n_q * C);
      std::mt19937 rng(5);
      std::vector<int> perm(n);
      for (int h = 0; h < n_q; ++h) {
        for (int64_t i = 0; i < n; ++i) perm[i] = (int)i;
        if (dens < 1.0) {
          for (int i = 0; i < C; ++i) std::swap(perm[i], perm[i + rng() % (n - i)]);
          std::sort(perm.begin(), perm.begin() + C);
        }
        std::copy(perm.begin(), perm.begin() + C, ids.begin() + (size_t)h * C);
      }
      int* dids;
      CK(cudaMalloc(&dids, ids.size() * 4));
      CK(cudaMemcpy(dids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice));
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      int occ;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather<2>, 256, 0));
      const int tiles = (C + 255) / 256;
      const int gx = std::min(tiles, std::max(1, sms * occ / n_q));
      float best = 1e30f;
      for (int it = 0; it < 8; ++it) {
        CK(cudaMemsetAsync(flush, it, 512ull << 20));  // evict L2
        CK(cudaEventRecord(a));
        gather<2><<<dim3(gx, n_q), 256>>>(rec, dids, n, C, G, dout);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, ms);
      }
      const double bytes = (double)n_q * C * 128;
      printf("n=%lld density=%.2f C=%d pairs=%d alg_MB=%.1f us=%.2f alg_GBs=%.1f\n", (long long)n, dens, C, n_q * C,
             bytes / 1e6, best * 1e3, bytes / (best * 1e-3) / 1e9);
      CK(cudaFree(dids));
    }
    CK(cudaFree(rec));
    CK(cudaFree(flush));
  }
  return 0;
}
