// Kernel-boundary cost in a CUDA graph (plain / PDL) vs an in-kernel grid barrier (cooperative launch).
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_empty(int* p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0]++;
}
__global__ void k_gridsync(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}
__device__ unsigned g_bar[2];
__global__ void k_mybar(int iters) {  // sense-free counter barrier: target = (i+1)*gridDim
  unsigned* cnt = &g_bar[0];
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(cnt, 1u);
      const unsigned target = (unsigned)(i + 1) * gridDim.x;
      while (true) {
        unsigned v;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(cnt));
        if (v >= target) break;
      }
    }
    __syncthreads();
  }
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  int* d;
  cudaMalloc(&d, 4);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int grid : {148, 592}) {
      cudaGraph_t gr;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < 100; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid; cfg.blockDim = 1024 / (grid / 148); cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = pdl;
        cudaLaunchKernelEx(&cfg, k_empty, d);
      }
      cudaStreamEndCapture(s, &gr);
      cudaGraphExec_t ge;
      cudaGraphInstantiate(&ge, gr, 0);
      cudaGraphLaunch(ge, s);
      cudaStreamSynchronize(s);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a, s);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("graph of 100 empty kernels grid=%d pdl=%d: %.2f us per kernel\n", grid, pdl, ms * 1000 / 1000);
    }
  }
  {
    int iters = 1000;
    void* args[] = {&iters};
    cudaLaunchCooperativeKernel((void*)k_gridsync, 148, 1024, args, 0, s);
    cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaLaunchCooperativeKernel((void*)k_gridsync, 148, 1024, args, 0, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cg grid.sync 148x1024: %.3f us per barrier (%s)\n", ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  {
    int iters = 1000;
    cudaMemset(g_bar, 0, 0);
    void* p; cudaGetSymbolAddress(&p, g_bar); cudaMemset(p, 0, 8);
    void* args[] = {&iters};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaLaunchCooperativeKernel((void*)k_mybar, 148, 1024, args, 0, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("counter grid barrier 148x1024: %.3f us per barrier (%s)\n", ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
