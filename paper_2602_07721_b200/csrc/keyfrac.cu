// Per-subspace centroid occupancy of the retrieval zone (the key-fraction reading of rho, DESIGN
// AMB-8b): occ[b][g][s][c] = number of indexed keys of (sequence b, KV head g) whose subspace-s centroid id is c.
// Query prep then probes each subspace's centroids in rank order until the probed ones hold >= rho_keys keys
// ("only let the top-rho fraction contribute a non-zero bonus", "collision processing scales with
// rho n"). Maintained by encode_keys / append_decode_keys while enabled (pkv_index_set_occupancy).
#include "common.cuh"

namespace pkv {
namespace {

constexpr int OC_THREADS = 256;
constexpr int OC_KEYS = 4096;  // keys per CTA

// keys [t0, t1) of every (sequence, KV head): a shared-memory histogram of the CTA's keys, then one global atomic
// per non-empty (subspace, centroid) bin. Key t's id row is rotated left by t mod 16 bytes (byte i = subspace
// (i + t) mod 16, scan.cu).
__global__ void __launch_bounds__(OC_THREADS) occupancy_kernel(const uint8_t* __restrict__ ids, int64_t cap,
                                                                int64_t t0, int64_t t1, uint32_t* occ) {
  __shared__ uint32_t h[NB * NC];
  const int bh = blockIdx.y;
  for (int i = threadIdx.x; i < NB * NC; i += OC_THREADS) h[i] = 0u;
  __syncthreads();
  const int64_t k0 = t0 + (int64_t)blockIdx.x * OC_KEYS;
  const int64_t k1 = min(t1, k0 + OC_KEYS);
  const uint8_t* ib = ids + (int64_t)bh * cap * NB;
  for (int64_t t = k0 + threadIdx.x; t < k1; t += OC_THREADS) {
    const uint4 r = ldg_v4(ib + t * NB);
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    const int rot = (int)(t & 15);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const uint32_t c = (w[i >> 2] >> (8 * (i & 3))) & 0xffu;
      atomicAdd(&h[((i + rot) & 15) * NC + c], 1u);
    }
  }
  __syncthreads();
  uint32_t* o = occ + (int64_t)bh * NB * NC;
  for (int i = threadIdx.x; i < NB * NC; i += OC_THREADS)
    if (h[i]) atomicAdd(o + i, h[i]);
}

}  // namespace

cudaError_t launch_occupancy(const pkv_index* ix, int64_t t0, int64_t t1, cudaStream_t stream) {
  if (t1 <= t0) return cudaSuccess;
  dim3 grid((unsigned)((t1 - t0 + OC_KEYS - 1) / OC_KEYS), ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_ENCODE, stream);
  occupancy_kernel<<<grid, OC_THREADS, 0, stream>>>(ix->ids, ix->cap, t0, t1, ix->occ);
  return cudaGetLastError();
}

}  // namespace pkv
