// Key encoder: prefill summarisation and decode-flush append (PAPER §4.1).
//
// One half-warp per key, lane b = subspace b (coordinates 8b..8b+7). Per key:
//   y' = H (s (.) k)  — the SRHT rotation as radix-2 Walsh-Hadamard butterflies, computed EXACTLY:
//       fast path: block-floating-point int32 butterflies (exact when every nonzero element of the key is
//       within 16 binades of the largest; 255*2^16*128 < 2^31), else fp64 butterflies in the oracle's order
//       (bit-identical to the oracle in every case).
//   S_b = fp64 left-to-right sum of y_j^2; centroid id = sign pattern (Eq. 6); 3-bit magnitude by the
//   midpoint rule y_j^2 >= M_t S_b on the Prop. 1 levels (AMB-5) — the fp64 op sequence of the oracle.
//   w'_b = w_b / ||sign*L[idx]|| = S_b / (sqrt(128) <sign*L[idx], y_b>)  (Eq. 7, 9 with AMB-6; alpha clamp 1e-3)
// Bytes per key: 256 in (bf16 K), 144 out (16 ids + 64 nibbles + 64 w'). HBM-bound.
#include <cuda_fp16.h>

#include "common.cuh"

namespace pkv {
namespace {

constexpr int KEYS_PER_BLOCK = 16;  // 256 threads

template <typename T>
__device__ __forceinline__ T shfl_x(T v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m, 16);
}

// Walsh-Hadamard butterflies over the 128 coordinates held 8-per-lane by a half-warp.
// Stage order h = 1, 2, 4 (in-lane), 8, 16, 32, 64 (across lanes), pair (i, i+h) -> (a+b, a-b).
template <typename T>
__device__ __forceinline__ void fwht128(T v[8], int lane16) {
#pragma unroll
  for (int h = 1; h < 8; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if ((i & h) == 0) {
        T a = v[i], b = v[i + h];
        v[i] = a + b;
        v[i + h] = a - b;
      }
    }
  }
#pragma unroll
  for (int x = 1; x < 16; x <<= 1) {
    const bool upper = (lane16 & x) != 0;
    const T sgn = upper ? T(-1) : T(1);  // upper: o - v, lower: v + o — one multiply-add either way
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      T o = shfl_x(v[i], x);
      v[i] = v[i] * sgn + o;
    }
  }
}

// One key (sequence/KV head bh, key tt of the call) per half-warp; lane16 = subspace.
__device__ __forceinline__ void encode_one(const uint16_t* __restrict__ K, int64_t sb, int64_t sh, int64_t st,
                                           int64_t t0, int n_kv, int64_t cap, const DevCfg& cfg,
                                           uint8_t* __restrict__ ids, uint8_t* __restrict__ rec, float* sL,
                                           unsigned long long* stats, int bh, int64_t tt, bool live, bool stage) {
  const int lane16 = threadIdx.x & 15;
  const int b = bh / n_kv, h = bh - b * n_kv;
  const int64_t t = t0 + tt;

  const uint4 raw = ldg_nc_v4(K + b * sb + h * sh + tt * st + 8 * lane16);
  if (stage) {  // the levels go to shared memory while the key is in flight (block-uniform)
    if (threadIdx.x < 8) sL[threadIdx.x] = cfg.levels[threadIdx.x];
    __syncthreads();
  }
  const uint32_t w4[4] = {raw.x, raw.y, raw.z, raw.w};
  uint32_t e[8], mant[8], sgn[8];
  int emax = 0;
  bool sub = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t bits = (i & 1) ? (w4[i >> 1] >> 16) : (w4[i >> 1] & 0xffffu);
    e[i] = (bits >> 7) & 0xffu;
    mant[i] = bits & 0x7fu;
    sgn[i] = ((bits >> 15) & 1u) ^ (uint32_t)sign_bit(cfg, 8 * lane16 + i);
    emax = max(emax, (int)e[i]);
    sub |= (e[i] == 0u && mant[i] != 0u) || e[i] == 0xffu;
  }
#pragma unroll
  for (int x = 1; x < 16; x <<= 1) emax = max(emax, shfl_x(emax, x));
  bool ok = !sub;
#pragma unroll
  for (int i = 0; i < 8; ++i) ok &= (e[i] == 0u) || ((int)e[i] >= emax - 16);
  const bool warp_ok = __all_sync(0xffffffffu, ok);

  double y[8];
  if (warp_ok) {
    int v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int nabs = (e[i] == 0u) ? 0 : (int)((128u | mant[i]) << (e[i] - (uint32_t)emax + 16u));
      v[i] = sgn[i] ? -nabs : nabs;
    }
    fwht128<int>(v, lane16);
    const double pscale = __longlong_as_double((long long)(1023 + emax - 150) << 52);  // 2^(emax-150), emax >= 1
#pragma unroll
    for (int i = 0; i < 8; ++i) y[i] = emax ? (double)v[i] * pscale : 0.0;  // exact: |v| < 2^31
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t bits = (i & 1) ? (w4[i >> 1] >> 16) : (w4[i >> 1] & 0xffffu);
      const double x = (double)__uint_as_float(bits << 16);
      y[i] = sign_bit(cfg, 8 * lane16 + i) ? -x : x;
    }
    fwht128<double>(y, lane16);
  }

  // ---- per-subspace decisions, fp64, fixed op order (no FMA contraction) ----
  double sq[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) sq[i] = __dmul_rn(y[i], y[i]);
  double S = sq[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) S = __dadd_rn(S, sq[i]);
  double th[7];
#pragma unroll
  for (int i = 0; i < 7; ++i) th[i] = __dmul_rn(cfg.mid_sq[i], S);

  uint32_t id = 0, code = 0;
  float dot = 0.f, vn2 = 0.f;
  const bool degenerate = (S == 0.0);
  // AMB-7 / SURVEY §8(b): zero subspaces and zero keys are encoded deterministically and counted, not rejected.
  // stats[0] zero keys, [1] keys with at least one zero subspace, [2] zero subspaces (rare: one atomic per key).
  const unsigned zmask = __ballot_sync(0xffffffffu, degenerate && live) >> (threadIdx.x & 16);
  if (lane16 == 0 && (zmask & 0xffffu)) {
    const unsigned z = zmask & 0xffffu;
    if (z == 0xffffu) atomicAdd(stats + 0, 1ull);
    atomicAdd(stats + 1, 1ull);
    atomicAdd(stats + 2, (unsigned long long)__popc(z));
  }
  // weights in fp32 on y scaled by 2^(119 - emax): |y| < 128 * 2^(emax - 126) so |y * scale| < 1 (ratios only)
  const double scale = __longlong_as_double((long long)(1023 + 119 - emax) << 52);
  const double unscale = __longlong_as_double((long long)(1023 - 119 + emax) << 52);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool pos = y[i] >= 0.0;
#ifdef PKV_ENC_LINEAR
    uint32_t idx = 0;
#pragma unroll
    for (int t2 = 0; t2 < 7; ++t2) idx += (uint32_t)(sq[i] >= th[t2]);
#else
    const bool b2 = sq[i] >= th[3];
    const double t1 = b2 ? th[5] : th[1];
    const bool b1 = sq[i] >= t1;
    const double t0v = b2 ? (b1 ? th[6] : th[4]) : (b1 ? th[2] : th[0]);
    const bool b0 = sq[i] >= t0v;
    uint32_t idx = 4u * b2 + 2u * b1 + (uint32_t)b0;
#endif
    uint32_t sbit = pos ? 1u : 0u;
    if (degenerate) {  // AMB-7: encode(e_1)
      idx = (i == 0) ? 7u : 0u;
      sbit = 1u;
    }
    id |= (pos ? 1u : 0u) << i;
    code |= ((sbit << 3) | idx) << (4 * i);
    const float L = sL[idx];
    const float yf = (float)(y[i] * scale);
    dot = fmaf(sbit ? L : -L, yf, dot);
    vn2 = fmaf(L, L, vn2);
  }
  const float Sf = (float)(S * scale * scale);
  float wprime = 0.f;
  if (!degenerate) {
    // alpha = dot / (||v~|| sqrt(S)); clamp at 1e-3 (AMB-6)
    const bool clamped = (dot <= 0.f) || (dot * dot < 1e-6f * vn2 * Sf);
    const float w_rel = clamped ? sqrtf(Sf * (1.0f / 128.0f)) / (1e-3f * sqrtf(vn2)) : Sf / (11.313708498984761f * dot);
    wprime = (float)((double)w_rel * unscale);
  }

  // ---- stores ----
  uint32_t idw = 0;
  const int q = lane16 & 3;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t o = __shfl_sync(0xffffffffu, id, (int)((4 * q + j + t) & 15), 16);
    idw |= (o & 0xffu) << (8 * j);
  }
  // fp16 weights (AMB-20 variant): w'_b = h_b * 2^E with one exponent per key, E = floor(log2 max_b w'_b) - 14
  // so that every h_b < 2^15 is a normal fp16 down to max * 2^-28; bit (b mod 8) of E (8-bit two's
  // complement) rides in the otherwise-zero sign bit of h_b, so each half of the record decodes E alone.
  uint32_t hbits = 0;
  if (cfg.w16) {
    float m = wprime;
#pragma unroll
    for (int x = 1; x < 16; x <<= 1) m = fmaxf(m, shfl_x(m, x));
    int E = (m > 0.f) ? ((__float_as_int(m) >> 23) & 0xff) - 127 - 14 : 0;
    E = max(-126, min(126, E));
    const float down = __int_as_float((127 - E) << 23);  // 2^-E, exact scaling
    hbits = (uint32_t)__half_as_ushort(__float2half_rn(wprime * down)) | ((((uint32_t)E >> (lane16 & 7)) & 1u) << 15);
  }
  if (live) {
    const int64_t row = (b * n_kv + h) * cap + t;
    if (lane16 < 4) reinterpret_cast<uint32_t*>(ids + row * NB)[lane16] = idw;
    uint8_t* r = rec + row * cfg.rec_bytes;
    reinterpret_cast<uint32_t*>(r)[lane16] = code;
    if (cfg.w16) reinterpret_cast<uint16_t*>(r + 64)[lane16] = (uint16_t)hbits;
    else reinterpret_cast<float*>(r + 64)[lane16] = wprime;
  }
}

// Grid (ceil(count / 16), batch * n_kv), keys [t0, t0 + count): 64 registers, 4 CTAs per SM (the list variant
// below is a separate kernel: its grid-stride loop and index division in this one cost 95 registers and 27%).
__global__ void __launch_bounds__(256, 4) encode_kernel(const uint16_t* __restrict__ K, int64_t sb, int64_t sh,
                                                        int64_t st, int64_t t0, int64_t count, int n_kv,
                                                        int64_t cap, DevCfg cfg, uint8_t* __restrict__ ids,
                                                        uint8_t* __restrict__ rec, unsigned long long* stats) {
  __shared__ float sL[8];  // magnitude levels: per-lane indexed (a divergent constant-bank read would serialise)
  int64_t tt = (int64_t)blockIdx.x * KEYS_PER_BLOCK + (threadIdx.x >> 4);
  const bool live = tt < count;
  if (!live) tt = count - 1;  // keep the half-warp shuffles full; results discarded
  encode_one(K, sb, sh, st, t0, n_kv, cap, cfg, ids, rec, sL, stats, blockIdx.y, tt, live, true);
}

// The keys list[0 .. *list_n) (entry = bh * count + tt, written by the tensor-core encoder for keys outside its
// exact range), grid-stride over the list.
__global__ void __launch_bounds__(256) encode_list_kernel(const uint16_t* __restrict__ K, int64_t sb, int64_t sh,
                                                          int64_t st, int64_t t0, int64_t count, int n_kv,
                                                          int64_t cap, DevCfg cfg, uint8_t* __restrict__ ids,
                                                          uint8_t* __restrict__ rec, unsigned long long* stats,
                                                          const int32_t* list, const int32_t* list_n) {
  __shared__ float sL[8];
  if (threadIdx.x < 8) sL[threadIdx.x] = cfg.levels[threadIdx.x];
  __syncthreads();
  const int n = *list_n;
  // both half-warps of a warp run the same number of rounds (encode_one shuffles over the full warp): the round
  // count is taken over the warp's pair of entries, and a half whose entry is past the list encodes a dummy key
  // (the list's first entry) without storing it
  for (int k0 = blockIdx.x * KEYS_PER_BLOCK + ((threadIdx.x >> 5) << 1); k0 < n; k0 += gridDim.x * KEYS_PER_BLOCK) {
    const int kk = k0 + ((threadIdx.x >> 4) & 1);
    const bool live = kk < n;
    const int e = list[live ? kk : 0];
    encode_one(K, sb, sh, st, t0, n_kv, cap, cfg, ids, rec, sL, stats, (int)(e / count), e % count, live, false);
  }
}

__global__ void export_kernel(const uint8_t* __restrict__ ids_in, const uint8_t* __restrict__ rec_in, int64_t start,
                              int64_t count, int n_kv, int64_t cap, int64_t total, int w16, int rec_bytes,
                              uint8_t* ids, uint8_t* codes, float* w) {
  const int64_t kk = (int64_t)blockIdx.x * 16 + (threadIdx.x >> 4);
  const int s = threadIdx.x & 15;
  if (kk >= total) return;
  const int64_t i = kk % count, bh = kk / count;
  const int64_t t = start + i;
  const int64_t row = bh * cap + t;
  if (ids) ids[kk * NB + s] = ids_in[row * NB + ((s - t) & 15)];
  const uint8_t* r = rec_in + row * rec_bytes;
  if (codes) reinterpret_cast<uint32_t*>(codes + kk * 64)[s] = reinterpret_cast<const uint32_t*>(r)[s];
  if (w) {
    if (w16) {  // h_b * 2^E, E from the sign bits of the 8 halves of this half of the record
      const uint16_t* hw = reinterpret_cast<const uint16_t*>(r + 64) + (s & 8);
      uint32_t e8 = 0;
      for (int i = 0; i < 8; ++i) e8 |= (uint32_t)(hw[i] >> 15) << i;
      const int E = (int)(int8_t)e8;
      const float hv = __half2float(__ushort_as_half((unsigned short)(hw[s & 7] & 0x7fffu)));
      w[kk * NB + s] = hv * __int_as_float((127 + E) << 23);
    } else {
      w[kk * NB + s] = reinterpret_cast<const float*>(r + 64)[s];
    }
  }
}

}  // namespace

cudaError_t launch_encode_list(const pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t0,
                               int64_t count, const int32_t* list, const int32_t* list_n, cudaStream_t stream) {
  ProfScope p_(K_ENCODE, stream);
  encode_list_kernel<<<ix->num_sms * 2, 256, 0, stream>>>(static_cast<const uint16_t*>(K), sb, sh, st, t0, count,
                                                     ix->cfg.n_kv_heads, ix->cap, ix->dcfg, ix->ids, ix->rec,
                                                     ix->stats, list, list_n);
  return cudaGetLastError();
}

cudaError_t launch_encode(const pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t0,
                          int64_t count, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((count + KEYS_PER_BLOCK - 1) / KEYS_PER_BLOCK), ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_ENCODE, stream);
  encode_kernel<<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(K), sb, sh, st, t0, count,
                                          ix->cfg.n_kv_heads, ix->cap, ix->dcfg, ix->ids, ix->rec, ix->stats);
  return cudaGetLastError();
}

cudaError_t launch_export(const pkv_index* ix, int64_t start, int64_t count, uint8_t* ids, uint8_t* codes,
                          float* w, cudaStream_t stream) {
  const int64_t total = (int64_t)ix->batch * ix->cfg.n_kv_heads * count;
  if (total == 0) return cudaSuccess;
  ProfScope p_(K_EXPORT, stream);
  export_kernel<<<(unsigned)((total + 15) / 16), 256, 0, stream>>>(ix->ids, ix->rec, start, count,
                                                                   ix->cfg.n_kv_heads, ix->cap, total,
                                                                   ix->dcfg.w16, ix->dcfg.rec_bytes, ids, codes, w);
  return cudaGetLastError();
}

cudaError_t set_phase_encode(unsigned long long* p) { return set_phase_ptr_tu(p); }

}  // namespace pkv
