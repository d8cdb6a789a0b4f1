// Device helpers shared by the kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "internal.h"

namespace pkv {

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Plain (coherent) 16-byte load: used for UVA host memory and data written by earlier kernels.
// Same load as an ordered (volatile) asm statement: stays where it is written, e.g. ahead of a barrier, so a
// batch of independent loads is really in flight together (the compiler otherwise sinks them to their use).
__device__ __forceinline__ uint4 ldg_nc_v4_early(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 32-byte load (sm_100 LDG.256), ordered like ldg_nc_v4_early: one request covers a whole 32-byte sector, where
// two 16-byte loads from different instructions each request the same sector from L2 again.
struct u32x8 {
  uint32_t w[8];
};
__device__ __forceinline__ u32x8 ldg_nc_v8_early(const void* p) {
  u32x8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
                 "=r"(r.w[7])
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ldg_v4(const void* p) {
  uint4 r;
  asm("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ uint2 ldg_v2(const void* p) {
  uint2 r;
  asm("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Order-preserving map of an fp64 value to uint64 (ascending). -0.0 is canonicalised to +0.0.
__device__ __forceinline__ unsigned long long ord_f64(double x) {
  x = __dadd_rn(x, 0.0);  // -0.0 + 0.0 = +0.0
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// Order-preserving map of an fp32 value to uint32 (ascending). -0.0 canonicalised to +0.0.
__device__ __forceinline__ uint32_t ord_f32(float x) {
  x = __fadd_rn(x, 0.0f);
  uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}

__device__ __forceinline__ double shfl_xor_d(double v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

__device__ __forceinline__ int sign_bit(const DevCfg& c, int d) { return (c.sign_mask[d >> 5] >> (d & 31)) & 1; }

}  // namespace pkv

namespace pkv {

// Optional phase timestamps (clock64 of CTA (0,0,0), thread 0) for kernel anatomy studies; enabled through
// pkv_phase_profile(). Slot layout: g_phase[kind * 16 + phase].
static __device__ unsigned long long* g_phase = nullptr;  // one copy per translation unit
static inline cudaError_t set_phase_ptr_tu(unsigned long long* p) {
  return cudaMemcpyToSymbol(g_phase, &p, sizeof(p));
}
#ifdef PKV_PHASE_PROFILE
__device__ __forceinline__ void phase_mark(int kind, int ph) {
  if (g_phase && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_phase[kind * 16 + ph] = t;
  }
}

// Per-CTA end timestamps of one kernel kind (slots 256.. of the phase buffer) for imbalance studies.
__device__ __forceinline__ void cta_mark(int kind, int which) {
  if (g_phase && threadIdx.x == 0) {
    const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (cta < 2048) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_phase[256 + 4096 * which + 2 * cta + (kind == K_RERANK ? 1 : 0)] = t;
    }
  }
}
#else  // marks compile away in the product build (build with PKV_PHASE_PROFILE=1 for scripts/phase_profile.py)
__device__ __forceinline__ void phase_mark(int, int) {}
__device__ __forceinline__ void cta_mark(int, int) {}
#endif

// Programmatic dependent launch: a kernel launched with pdl_launch may start while the previous kernel on the
// stream drains; it must call pdl_wait() before touching that kernel's outputs. Disable with PKV_NO_PDL=1.
bool pdl_enabled();

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// pdl_launch for a kernel whose grid is tiled by thread-block clusters of cluster_x CTAs along x.
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                               int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace pkv
