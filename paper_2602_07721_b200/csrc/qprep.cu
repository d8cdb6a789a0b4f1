// Query preparation (a1): normalise & rotate q, rank the 256 analytic centroids of every
// subspace by the query-centroid dot product ("cheap dot product q^T c") and turn ranks into the
// multi-tier collision bonuses, packed 4 query heads per u32 for the scan's lookup table; also
// the rerank tables sign*L[idx]*q~_j used by the RSQ-IP estimate (Eq. 10).
//
// Grid (16 subspaces, n_kv, batch), 4 warps; warp w handles query head g*G + w. Exact contract shared with
// the oracle (AMB-9): y' = fp64 butterflies of s (.) q; score_c = fp64 left-to-right sum of +-y'_j from 0.0;
// order (score desc, id asc) — here a warp-wide bitonic sort of 256 (key, id) pairs, 8 per lane.
#include "common.cuh"

namespace pkv {
namespace {

__device__ __forceinline__ bool less_kv(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// Ascending bitonic sort of 256 (key, id) pairs; lane L holds positions 8L..8L+7.
__device__ __forceinline__ void bitonic256(unsigned long long key[8], uint32_t id[8], int lane) {
#pragma unroll
  for (int k = 2; k <= 256; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 8) {
        const int lm = j >> 3;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key[e], lm);
          const uint32_t oi = __shfl_xor_sync(0xffffffffu, id[e], lm);
          const bool asc = (((8 * lane + e) & k) == 0);
          const bool mine_less = less_kv(key[e], id[e], ok, oi);
          const bool keep_min = (asc == lower);
          if (keep_min != mine_less) {
            key[e] = ok;
            id[e] = oi;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if ((e & j) == 0) {
            const int p = e | j;
            const bool asc = (((8 * lane + e) & k) == 0);
            const bool a_less = less_kv(key[e], id[e], key[p], id[p]);
            if (asc != a_less) {
              const unsigned long long tk = key[e];
              key[e] = key[p];
              key[p] = tk;
              const uint32_t ti = id[e];
              id[e] = id[p];
              id[p] = ti;
            }
          }
        }
      }
    }
  }
}

__global__ void __launch_bounds__(128) qprep_kernel(const uint16_t* __restrict__ q, int T, DevCfg cfg,
                                                    uint32_t* __restrict__ lut, float* __restrict__ rtab,
                                                    float* __restrict__ qnorm, float* __restrict__ qrot,
                                                    float* __restrict__ dbg_q_rot) {
  __shared__ uint8_t bonus_s[GMAX][NC];
  const int sb = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = cfg.G;
  if (warp < G) {
    const int h = g * G + warp;
    const uint16_t* qh = q + ((int64_t)b * cfg.n_q + h) * D;
    const uint2 raw = ldg_v2(qh + 4 * lane);
    const float qf[4] = {bf16_lo(raw.x), bf16_hi(raw.x), bf16_lo(raw.y), bf16_hi(raw.y)};
    double v[4];
    float qn2 = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      qn2 = fmaf(qf[i], qf[i], qn2);
      v[i] = sign_bit(cfg, 4 * lane + i) ? -(double)qf[i] : (double)qf[i];
    }
    // butterflies h = 1, 2 in-lane; 4..64 across lanes (oracle order)
#pragma unroll
    for (int hh = 1; hh < 4; hh <<= 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if ((i & hh) == 0) {
          const double a = v[i], c = v[i + hh];
          v[i] = __dadd_rn(a, c);
          v[i + hh] = __dsub_rn(a, c);
        }
      }
    }
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) {
      const bool upper = (lane & x) != 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double o = shfl_xor_d(v[i], x);
        v[i] = upper ? __dsub_rn(o, v[i]) : __dadd_rn(v[i], o);
      }
    }
    double yn2 = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) yn2 = fma(v[i], v[i], yn2);
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) {
      yn2 += shfl_xor_d(yn2, x);
      qn2 += __shfl_xor_sync(0xffffffffu, qn2, x);
    }
    const double inv_yn = yn2 > 0.0 ? 1.0 / sqrt(yn2) : 0.0;
    // subspace sb coordinates 8sb..8sb+7 live in lanes 2sb, 2sb+1
    double yb[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) yb[j] = __shfl_sync(0xffffffffu, v[j & 3], 2 * sb + (j >> 2));
    // centroid scores for ids 8*lane + e
    unsigned long long key[8];
    uint32_t id[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t c = 8u * lane + e;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, ((c >> j) & 1u) ? yb[j] : -yb[j]);
      key[e] = ~ord_f64(acc);  // ascending key == descending score
      id[e] = c;
    }
    bitonic256(key, id, lane);
    const int chunk = max(1, T / cfg.n_tiers);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int rank = 8 * lane + e;
      int bonus = 0;
      if (rank < T) bonus = cfg.tier_bonus[min(rank / chunk, cfg.n_tiers - 1)];
      bonus_s[warp][id[e]] = (uint8_t)bonus;
    }
    // rerank table rows for coordinates 8sb..8sb+7 of head h: entry (j, n) = sign(n) L[n&7] q~_{8sb+j}
    float* rt = rtab + (((int64_t)b * cfg.n_q + h) * D + 8 * sb) * 16;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e2 = 4 * lane + r;
      const int j = e2 >> 4, n = e2 & 15;
      double yj = yb[0];
#pragma unroll
      for (int jj = 1; jj < 8; ++jj) yj = (j == jj) ? yb[jj] : yj;
      const float qt = (float)(yj * inv_yn);
      const float L = cfg.levels[n & 7];
      rt[e2] = (n & 8) ? L * qt : -L * qt;
    }
    if (lane == 2 * sb || lane == 2 * sb + 1) {
      float* qr = qrot + ((int64_t)b * cfg.n_q + h) * D;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        qr[4 * lane + i] = (float)(v[i] * inv_yn);
        if (dbg_q_rot) dbg_q_rot[((int64_t)b * cfg.n_q + h) * D + 4 * lane + i] = (float)(v[i] * inv_yn);
      }
    }
    if (sb == 0 && lane == 0) qnorm[(int64_t)b * cfg.n_q + h] = sqrtf(qn2);
  }
  __syncthreads();
  uint32_t* lg = lut + ((int64_t)b * cfg.n_kv + g) * NC * NB;
  for (int c = threadIdx.x; c < NC; c += blockDim.x) {
    uint32_t wv = 0;
    for (int w = 0; w < G; ++w) wv |= (uint32_t)bonus_s[w][c] << (8 * w);
    lg[c * NB + sb] = wv;
  }
}

}  // namespace

cudaError_t launch_qprep(const pkv_index* ix, const void* q, int T, float* dbg_q_rot, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(NB, ix->cfg.n_kv_heads, ix->batch);
  ProfScope p_(K_QPREP, stream);
  qprep_kernel<<<grid, 128, 0, stream>>>(static_cast<const uint16_t*>(q), T, ix->dcfg, ws->lut, ws->rtab,
                                          ws->qnorm, ws->qrot, dbg_q_rot);
  return cudaGetLastError();
}

}  // namespace pkv
