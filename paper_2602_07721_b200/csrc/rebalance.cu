// Append rebalancing across sequence shards. Decode appends land on the last rank, so
// its shard grows by update_size keys per flush; a boundary shift moves the oldest keys of shard r+1
// to the end of shard r. Shards stay contiguous and ordered by position, so the sharded select's newest-rank-first
// tie rule (AMB-12) and every other invariant of the sharded path are unchanged.
//
// Exchange entry of one (sequence, KV head, key): the key's canonical centroid-id row (subspace b in byte b, 16 B)
// followed by its record (rec_bytes), laid out [batch][n_kv][count] x entry. The index stores key t's id row rotated
// left by (t mod 16) bytes (scan.cu), so a key that changes position is re-rotated on the way.
#include "common.cuh"

namespace pkv {
namespace {

constexpr int RB_THREADS = 256;

// rotate a 16-byte row left by r bytes: byte i of the result = byte (i + r) mod 16 of the input
__device__ __forceinline__ uint4 rotl_row(uint4 v, int r) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  const int wr = (r >> 2) & 3, br = 8 * (r & 3);
  uint32_t o[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t lo = w[(k + wr) & 3], hi = w[(k + wr + 1) & 3];
    o[k] = br ? __funnelshift_r(lo, hi, br) : lo;
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// one thread per (unit, key): copy key `src0 + i` of `ids/rec` into entry i of the buffer (canonical row)
__global__ void export_entries_kernel(const uint8_t* __restrict__ ids, const uint8_t* __restrict__ rec, int64_t cap,
                                      int rb, int64_t src0, int64_t count, uint8_t* __restrict__ buf) {
  const int64_t i = (int64_t)blockIdx.x * RB_THREADS + threadIdx.x;
  if (i >= count) return;
  const int64_t u = blockIdx.y, t = src0 + i;
  const int64_t eb = 16 + rb;
  uint8_t* e = buf + (u * count + i) * eb;
  const uint4 row = *reinterpret_cast<const uint4*>(ids + (u * cap + t) * NB);
  *reinterpret_cast<uint4*>(e) = rotl_row(row, (int)((16 - (t & 15)) & 15));
  const uint4* r = reinterpret_cast<const uint4*>(rec + (u * cap + t) * rb);
  for (int c = 0; c < rb / 16; ++c) reinterpret_cast<uint4*>(e + 16)[c] = r[c];
}

// one thread per (unit, key): entry i of the buffer becomes key `dst0 + i` (row rotated for its new position)
__global__ void import_entries_kernel(uint8_t* __restrict__ ids, uint8_t* __restrict__ rec, int64_t cap, int rb,
                                      int64_t dst0, int64_t count, const uint8_t* __restrict__ buf) {
  const int64_t i = (int64_t)blockIdx.x * RB_THREADS + threadIdx.x;
  if (i >= count) return;
  const int64_t u = blockIdx.y, t = dst0 + i;
  const int64_t eb = 16 + rb;
  const uint8_t* e = buf + (u * count + i) * eb;
  *reinterpret_cast<uint4*>(ids + (u * cap + t) * NB) = rotl_row(*reinterpret_cast<const uint4*>(e), (int)(t & 15));
  uint4* r = reinterpret_cast<uint4*>(rec + (u * cap + t) * rb);
  for (int c = 0; c < rb / 16; ++c) r[c] = reinterpret_cast<const uint4*>(e + 16)[c];
}

}  // namespace

cudaError_t launch_export_entries(const pkv_index* ix, int64_t src0, int64_t count, void* buf, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((count + RB_THREADS - 1) / RB_THREADS), ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_EXPORT, stream);
  export_entries_kernel<<<grid, RB_THREADS, 0, stream>>>(ix->ids, ix->rec, ix->cap, ix->dcfg.rec_bytes, src0, count,
                                                         static_cast<uint8_t*>(buf));
  return cudaGetLastError();
}

cudaError_t launch_import_entries(pkv_index* ix, int64_t dst0, int64_t count, const void* buf, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((count + RB_THREADS - 1) / RB_THREADS), ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_EXPORT, stream);
  import_entries_kernel<<<grid, RB_THREADS, 0, stream>>>(ix->ids, ix->rec, ix->cap, ix->dcfg.rec_bytes, dst0, count,
                                                         static_cast<const uint8_t*>(buf));
  return cudaGetLastError();
}

}  // namespace pkv
