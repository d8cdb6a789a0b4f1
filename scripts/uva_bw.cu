// Host-link roofline for the 1M-token configuration ("Host link ... measure it"): how fast can a
// kernel read pinned, mapped host memory through UVA?
//   stream   : every byte of a 256 MB mapped buffer read once by a full grid (16-byte loads) — peak UVA read rate
//   gather   : R random rows of 512 B (K row 256 B + V row 256 B, like the attention gather), one warp per row,
//              8 bytes per lane per half-row, all rows issued at once — the shape of a 1M decode step's fetch
//   memcpy   : cudaMemcpyAsync of 256 MB pinned host -> device (copy-engine DMA), for reference
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o uva_bw scripts/uva_bw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void stream_read(const uint4* __restrict__ p, size_t n16, unsigned* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = p[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void gather_rows(const uint16_t* __restrict__ K, const uint16_t* __restrict__ V, const int* __restrict__ ids,
                            int R, unsigned* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= R) return;
  const int64_t row = ids[warp];
  const uint2 k = *reinterpret_cast<const uint2*>(K + row * 128 + 4 * lane);
  const uint2 v = *reinterpret_cast<const uint2*>(V + row * 128 + 4 * lane);
  const uint32_t acc = k.x ^ k.y ^ v.x ^ v.y;
  if (acc == 0x12345678u) out[0] = acc;
}

// one instruction per row: lanes 0-15 read the K row (16 B each), lanes 16-31 the V row
__global__ void gather_rows_v4(const uint16_t* __restrict__ K, const uint16_t* __restrict__ V,
                               const int* __restrict__ ids, int R, unsigned* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= R) return;
  const int64_t row = ids[warp];
  const uint16_t* src = (lane < 16 ? K : V) + row * 128 + 8 * (lane & 15);
  const uint4 v = *reinterpret_cast<const uint4*>(src);
  const uint32_t acc = v.x ^ v.y ^ v.z ^ v.w;
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t bytes = 256ull << 20;
  void *hbuf, *dbuf;
  CK(cudaHostAlloc(&hbuf, 2 * bytes, cudaHostAllocMapped));
  for (size_t i = 0; i < 2 * bytes / 4; i += 1024) reinterpret_cast<uint32_t*>(hbuf)[i] = (uint32_t)i;
  CK(cudaMalloc(&dbuf, bytes));
  unsigned* dout;
  CK(cudaMalloc(&dout, 4));
  void* dh;
  CK(cudaHostGetDevicePointer(&dh, hbuf, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float ms;
  // stream
  for (int it = 0; it < 3; ++it) {
    CK(cudaEventRecord(a));
    stream_read<<<sms * 8, 256>>>((const uint4*)dh, bytes / 16, dout);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
  }
  printf("uva_stream_read_GBs %.1f\n", bytes / (ms * 1e-3) / 1e9);
  // memcpy
  for (int it = 0; it < 3; ++it) {
    CK(cudaEventRecord(a));
    CK(cudaMemcpyAsync(dbuf, hbuf, bytes, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
  }
  printf("memcpy_h2d_GBs %.1f\n", bytes / (ms * 1e-3) / 1e9);
  // gather: K and V halves of the mapped buffer, rows of 256 B each
  const int nrows = (int)(bytes / 256);
  const uint16_t* K = (const uint16_t*)dh;
  const uint16_t* V = (const uint16_t*)((char*)dh + bytes);
  for (int R : {3200, 12800, 102400}) {
    std::vector<int> ids(R);
    srand(R);
    for (int i = 0; i < R; ++i) ids[i] = (int)(((uint64_t)rand() * 2654435761ull) % (uint64_t)nrows);
    int* dids;
    CK(cudaMalloc(&dids, R * sizeof(int)));
    CK(cudaMemcpy(dids, ids.data(), R * sizeof(int), cudaMemcpyHostToDevice));
    float best = 1e30f;
    for (int it = 0; it < 10; ++it) {
      CK(cudaEventRecord(a));
      gather_rows<<<(R * 32 + 255) / 256, 256>>>(K, V, dids, R, dout);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    printf("uva_gather rows=%d bytes=%d us=%.2f GBs=%.1f\n", R, R * 512, best * 1e3, R * 512.0 / (best * 1e-3) / 1e9);
    best = 1e30f;
    for (int it = 0; it < 10; ++it) {
      CK(cudaEventRecord(a));
      gather_rows_v4<<<(R * 32 + 255) / 256, 256>>>(K, V, dids, R, dout);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    printf("uva_gather_v4 rows=%d bytes=%d us=%.2f GBs=%.1f\n", R, R * 512, best * 1e3, R * 512.0 / (best * 1e-3) / 1e9);
    CK(cudaFree(dids));
  }
  return 0;
}
