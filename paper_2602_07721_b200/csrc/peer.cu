// One-shot all-gather over peer memory: the "peer" exchange transport of the sequence-sharded
// path (comm.cpp, pkv_comm_init_peer). Every rank owns a symmetric exchange arena that all ranks map (CUDA IPC
// across processes, plain pointers within one). One kernel per exchange: CTA j stores chunk j of this rank's
// slot straight into every peer's arena (NVLink stores on an NVSwitch system), fences at system scope, raises
// its flag in every peer's arena, waits until every rank's chunk j has landed in its own arena, and copies those
// chunks into the caller's exchange buffer — no NCCL call, no host involvement, CUDA-graph capturable.
//
// Arena layout (bytes): [0, 4096) flags u32 [MAX_RANKS src][PX_CTAS]; [4096, 8192) epochs u32 [PX_CTAS] (local
// use only); then two parity halves of `half` bytes, each [world][slot bytes]. CTA j counts its exchanges in
// epochs[j]; exchange e of CTA j writes parity e & 1 and flag value e. All ranks run the same exchange sequence
// with the same grid, so the counters agree; a rank can be at most one exchange ahead of a peer (it cannot
// finish exchange e + 1 before that peer has sent e + 1, which follows the peer's exchange e in stream order),
// so two parities suffice and a flag never runs ahead of the value its receiver waits for.
#include "common.cuh"

namespace pkv {

constexpr int PX_CTAS = 8;
constexpr int PX_THREADS = 256;
constexpr size_t PX_HDR = 8192;

struct PeerTable {
  char* arena[MAX_RANKS];
};

namespace {

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// copy words [w0, w1) (u32 units) of src to dst, 16-byte vectors where both are aligned
__device__ __forceinline__ void copy_words(uint32_t* dst, const uint32_t* src, size_t w0, size_t w1) {
  const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0 && (w0 & 3) == 0;
  size_t w = w0 + threadIdx.x * (vec ? 4 : 1);
  if (vec) {
    for (; w + 4 <= w1; w += PX_THREADS * 4)
      *reinterpret_cast<uint4*>(dst + w) = *reinterpret_cast<const uint4*>(src + w);
    // tail (< 4 words) by the thread that would own it
    if (w < w1)
      for (size_t x = w; x < w1; ++x) dst[x] = src[x];
  } else {
    for (; w < w1; w += PX_THREADS) dst[w] = src[w];
  }
}

__global__ void __launch_bounds__(PX_THREADS) peer_allgather_kernel(PeerTable t, int rank, int world, uint32_t* buf,
                                                                     size_t words, size_t half) {
  const int j = blockIdx.x;
  char* mine = t.arena[rank];
  unsigned* epochs = reinterpret_cast<unsigned*>(mine + 4096);
  __shared__ unsigned s_e;
  if (threadIdx.x == 0) s_e = epochs[j] + 1u;
  __syncthreads();
  const unsigned e = s_e;
  const size_t par = PX_HDR + (size_t)(e & 1u) * half;
  // this CTA's chunk of a slot, in words (a multiple of 4 so chunks stay 16-byte aligned)
  const size_t per = ((words + PX_CTAS - 1) / PX_CTAS + 3) & ~(size_t)3;
  const size_t w0 = min(words, (size_t)j * per), w1 = min(words, w0 + per);
  const uint32_t* src = buf + (size_t)rank * words;
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    uint32_t* dst = reinterpret_cast<uint32_t*>(t.arena[p] + par) + (size_t)rank * words;
    copy_words(dst, src, w0, w1);
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < world && threadIdx.x != rank)
    st_release_sys(reinterpret_cast<unsigned*>(t.arena[threadIdx.x]) + rank * PX_CTAS + j, e);
  if (threadIdx.x < world && threadIdx.x != rank) {
    const unsigned* f = reinterpret_cast<const unsigned*>(mine) + threadIdx.x * PX_CTAS + j;
    while ((int)(ld_acquire_sys(f) - e) < 0) {
    }
    __threadfence();
  }
  __syncthreads();
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    copy_words(buf + (size_t)r * words, reinterpret_cast<const uint32_t*>(mine + par) + (size_t)r * words, w0, w1);
  }
  if (threadIdx.x == 0) epochs[j] = e;
}

}  // namespace

cudaError_t launch_peer_allgather(char* const* arenas, int rank, int world, uint32_t* buf, size_t words, size_t half,
                                  cudaStream_t stream) {
  PeerTable t{};
  for (int r = 0; r < world && r < MAX_RANKS; ++r) t.arena[r] = arenas[r];
  ProfScope p_(K_MERGE, stream);
  peer_allgather_kernel<<<PX_CTAS, PX_THREADS, 0, stream>>>(t, rank, world, buf, words, half);
  return cudaGetLastError();
}

size_t peer_header_bytes() { return PX_HDR; }

}  // namespace pkv
