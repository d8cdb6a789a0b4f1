// Calibration microbenchmarks for B200 (not part of the product): launch cost, dependent-load latency
// (L2 / HBM), one-round streaming kernels, smem atomics throughput. nvcc -arch=sm_100a -O3 -o mb microbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e = (x);                                                    \
    if (e != cudaSuccess) {                                                 \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                              \
    }                                                                       \
  } while (0)

__global__ void k_empty() {}

__global__ void k_chase(const unsigned* __restrict__ next, int hops, unsigned* out) {
  unsigned p = 0;
  for (int i = 0; i < hops; ++i) p = next[p];
  if (threadIdx.x == 0) out[blockIdx.x] = p;
}

__global__ void k_stream1(const uint4* __restrict__ in, uint4* out, size_t n) {  // one 16 B load per thread
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint4 v = in[i];
    if (v.x == 0xdeadbeef) out[i] = v;
  }
}

__global__ void k_stream_loop(const uint4* __restrict__ in, unsigned* out, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = in[i];
    acc += v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0xdeadbeef) out[0] = acc;
}

__global__ void k_atoms(unsigned* out, int iters, int spread) {
  __shared__ unsigned h[32 * 128];
  for (int i = threadIdx.x; i < 32 * 128; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned* hw = h + (threadIdx.x >> 5) * 128;
  unsigned x = threadIdx.x * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    unsigned bin = spread ? (x >> 25) : ((x >> 29) & 7);  // 128 bins vs 8 hot bins
    atomicAdd(&hw[bin], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[0];
}

float time_ms(void (*f)(cudaStream_t), cudaStream_t s, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f(s);
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) f(s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

static unsigned* g_next;
static unsigned* g_out;
static uint4* g_big;
static int g_hops;
static size_t g_n;

int main() {
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  const size_t N = (size_t)1 << 28;  // 1 GiB of u32 for the chase
  std::vector<unsigned> h(N / 64);
  // random cycle over 16M entries spaced 256 B apart (defeats caches and prefetch)
  const size_t M = N / 64;
  std::vector<unsigned> perm(M);
  for (size_t i = 0; i < M; ++i) perm[i] = (unsigned)i;
  srand(1);
  for (size_t i = M - 1; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
  std::vector<unsigned> nxt(N, 0);
  for (size_t i = 0; i < M; ++i) nxt[(size_t)perm[i] * 64] = perm[(i + 1) % M] * 64;
  CK(cudaMalloc(&g_next, N * 4));
  CK(cudaMemcpy(g_next, nxt.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&g_out, 1 << 20));
  g_n = (size_t)1 << 26;  // 1 GiB of uint4
  CK(cudaMalloc(&g_big, g_n * 16));
  CK(cudaMemset(g_big, 1, g_n * 16));

  printf("empty kernel 1x1           : %.2f us/launch (back-to-back)\n",
         1000 * time_ms([](cudaStream_t s) { k_empty<<<1, 1, 0, s>>>(); }, s, 1000));
  printf("empty kernel 148x1024      : %.2f us/launch\n",
         1000 * time_ms([](cudaStream_t s) { k_empty<<<148, 1024, 0, s>>>(); }, s, 1000));
  for (int hops : {1, 10, 100}) {
    g_hops = hops;
    float ms = time_ms([](cudaStream_t s) { k_chase<<<1, 1, 0, s>>>(g_next, g_hops, g_out); }, s, 20);
    printf("dependent HBM chase %4d hops: %.2f us total, %.0f ns/hop (incl. launch)\n", hops, ms * 1000,
           ms * 1e6 / hops);
  }
  for (size_t mb : {1, 4, 16, 64, 1024}) {
    g_n = mb * (1 << 20) / 16;
    float ms = time_ms([](cudaStream_t s) {
      k_stream1<<<(unsigned)((g_n + 255) / 256), 256, 0, s>>>(g_big, g_big, g_n);
    }, s, 50);
    printf("stream one load/thread %5zu MB: %.2f us  %.0f GB/s\n", mb, ms * 1000, mb * 1.048576e6 / (ms * 1e-3) / 1e9);
  }
  for (size_t mb : {16, 64, 1024}) {
    g_n = mb * (1 << 20) / 16;
    float ms = time_ms([](cudaStream_t s) { k_stream_loop<<<148 * 4, 512, 0, s>>>(g_big, g_out, g_n); }, s, 50);
    printf("stream grid-stride 592x512 %5zu MB: %.2f us  %.0f GB/s\n", mb, ms * 1000,
           mb * 1.048576e6 / (ms * 1e-3) / 1e9);
  }
  for (int spread : {1, 0}) {
    g_hops = spread;
    float ms = time_ms([](cudaStream_t s) { k_atoms<<<148, 1024, 0, s>>>(g_out, 1000, g_hops); }, s, 10);
    printf("smem atomicAdd per-warp hist (%s): %.3f ns per warp-instr per SM\n", spread ? "128 bins" : "8 hot bins",
           ms * 1e6 / (1000.0 * 32));
  }
  return 0;
}
