// Query preparation (a1): normalise & rotate q, rank the 256 analytic centroids of every
// subspace by the query-centroid dot product ("cheap dot product q^T c") and turn ranks into the
// multi-tier collision bonuses, written as one byte per query head into the packed u32 lookup table
// of the scan; also the rerank tables sign*L[idx]*q~_j used by the RSQ-IP estimate (Eq. 10).
//
// Grid (16 subspaces, n_q heads, batch), 128 threads. Exact contract shared with the oracle (AMB-9):
// y' = fp64 butterflies of s (.) q; score_c = fp64 left-to-right sum of +-y'_j from 0.0; order (score desc,
// id asc). The complement symmetry score(255-c) = -score(c) halves the sort to 128 "leaders", one per thread;
// the bitonic network runs in registers and warp shuffles, only its 3 stages with distance >= 32 in smem.
#include "common.cuh"

namespace pkv {
namespace {

constexpr int QP_THREADS = 128;

struct KV {
  unsigned long long k;
  uint32_t id;
};

__device__ __forceinline__ KV shfl_kv(const KV& v, int m) {
  KV o;
  o.k = __shfl_xor_sync(0xffffffffu, v.k, m);
  o.id = __shfl_xor_sync(0xffffffffu, v.id, m);
  return o;
}

// One stage (k, j) for the element at position p held by this thread, partner value `o` at position p ^ j.
// Branch-free: (key, id) pairs are distinct, so "mine < o" == !(o < mine).
__device__ __forceinline__ void ce(KV& mine, const KV& o, int p, int k, int j) {
  const bool keep_min = (((p & j) == 0) == ((p & k) == 0));
  const bool o_less = (o.k < mine.k) | ((o.k == mine.k) & (o.id < mine.id));
  const bool take = keep_min == o_less;
  mine.k = take ? o.k : mine.k;
  mine.id = take ? o.id : mine.id;
}

__global__ void __launch_bounds__(QP_THREADS) qprep_kernel(const uint16_t* q, int T, DevCfg cfg,
                                                          uint32_t* lut, float* rtab,
                                                          float* qnorm, float* qrot,
                                                          float* dbg_q_rot, unsigned int* ucount) {
  __shared__ unsigned long long sk[NC / 2];
  __shared__ uint32_t si[NC / 2];
  phase_mark(K_QPREP, 0);
  const int sb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = h / cfg.G, hh = h % cfg.G;
  pdl_wait();  // the query of this layer follows the previous layer's work
  pdl_trigger();
  if (sb == 0 && hh == 0 && t == 0) ucount[b * cfg.n_kv + g] = 0u;  // the select of this step counts from 0
  phase_mark(K_QPREP, 1);
  // warp 0 rotates the query (fp64 butterflies) and publishes this subspace's 8 coordinates and 1/||y'||
  __shared__ double s_yb[8];
  __shared__ double s_inv;
  if (warp == 0) {
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
#pragma unroll
    for (int x = 1; x < 4; x <<= 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if ((i & x) == 0) {
          const double a2 = v[i], c = v[i + x];
          v[i] = __dadd_rn(a2, c);
          v[i + x] = __dsub_rn(a2, c);
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
    if (lane == 2 * sb || lane == 2 * sb + 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) s_yb[4 * (lane - 2 * sb) + i] = v[i];
      float* qr = qrot + ((int64_t)b * cfg.n_q + h) * D;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        qr[4 * lane + i] = (float)(v[i] * inv_yn);
        if (dbg_q_rot) dbg_q_rot[((int64_t)b * cfg.n_q + h) * D + 4 * lane + i] = (float)(v[i] * inv_yn);
      }
    }
    if (lane == 0) s_inv = inv_yn;
    if (sb == 0 && lane == 0) qnorm[(int64_t)b * cfg.n_q + h] = sqrtf(qn2);
  }
  __syncthreads();
  double yb[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) yb[j] = s_yb[j];
  const double inv_yn = s_inv;
  // rerank table rows for coordinates 8sb..8sb+7 (one entry per thread): sign(n) L[n&7] q~_{8sb+j}
  {
    const int j = t >> 4, nb = t & 15;
    double yj = yb[0];
#pragma unroll
    for (int jj = 1; jj < 8; ++jj) yj = (j == jj) ? yb[jj] : yj;
    const float qt = (float)(yj * inv_yn);
    const float L = cfg.levels[nb & 7];
    rtab[(((int64_t)b * cfg.n_q + h) * D + 8 * sb) * 16 + t] = (nb & 8) ? L * qt : -L * qt;
  }
  phase_mark(K_QPREP, 2);
  // Complement symmetry: score(255 - c) == -score(c) exactly (every partial sum of the left-to-right fp64 sum
  // is negated, round-to-nearest is odd-symmetric and an exact zero is +0.0 either way). So the (score desc,
  // id asc) order of all 256 is: the 128 "leaders" (of each pair {c, 255-c} the one that comes first) in
  // order, then their complements in reverse order -> rank(255 - c) = 255 - rank(c). Only the leaders are
  // sorted, one per thread. Thread t owns the pair {t, 255 - t}; t < 128 <= 255 - t breaks a zero tie.
  KV e;
  {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, ((t >> j) & 1) ? yb[j] : -yb[j]);
    const bool neg = acc < 0.0;
    e.k = ~ord_f64(neg ? -acc : acc);  // ascending key == descending score; ties by ascending id
    e.id = neg ? (uint32_t)(NC - 1 - t) : (uint32_t)t;
  }
  // Fast path: when the fp64 scores have 8 trailing zero mantissa bits (always, unless the query spans more than
  // ~27 binades: each y' is an exact sum of bf16 values and the 8-term score sums are exact too), the leader id
  // fits in those bits and the sort moves one 64-bit composite (2 shuffles per stage instead of 3): ordering by
  // composite == ordering by (key, id). Otherwise the (key, id) pair network below.
  if (__syncthreads_and((e.k & 0xffull) == 0xffull)) {
    unsigned long long c = (e.k & ~0xffull) | e.id;
#pragma unroll
    for (int k = 2; k <= NC / 2; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        unsigned long long o;
        if (j < 32) {
          o = __shfl_xor_sync(0xffffffffu, c, j);
        } else {
          sk[t] = c;
          __syncthreads();
          o = sk[t ^ j];
          __syncthreads();
        }
        const bool keep_min = (((t & j) == 0) == ((t & k) == 0));
        c = (keep_min == (o < c)) ? o : c;
      }
    }
    e.id = (uint32_t)(c & 0xffull);
  } else {
#pragma unroll
    for (int k = 2; k <= NC / 2; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        KV o;
        if (j < 32) {
          o = shfl_kv(e, j);
        } else {
          sk[t] = e.k;
          si[t] = e.id;
          __syncthreads();
          o = KV{sk[t ^ j], si[t ^ j]};
          __syncthreads();
        }
        ce(e, o, t, k, j);
      }
    }
  }
  phase_mark(K_QPREP, 3);
  // position t == rank of leader e.id, 255 - t == rank of its complement; write this head's bonus byte of the
  // packed LUT entry of both
  const int chunk = max(1, T / cfg.n_tiers);
  uint8_t* lb = reinterpret_cast<uint8_t*>(lut + ((int64_t)b * cfg.n_kv + g) * NC * NB);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int rank = u ? NC - 1 - t : t;
    const uint32_t id = u ? NC - 1 - e.id : e.id;
    int bonus = 0;
    if (rank < T) bonus = cfg.tier_bonus[min(rank / chunk, cfg.n_tiers - 1)];
    lb[((int64_t)id * NB + sb) * 4 + hh] = (uint8_t)bonus;
  }
  phase_mark(K_QPREP, 4);
}

}  // namespace

cudaError_t launch_qprep(const pkv_index* ix, const void* q, int T, float* dbg_q_rot, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(NB, ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_QPREP, stream);
  return pdl_launch(qprep_kernel, grid, dim3(QP_THREADS), 0, stream, static_cast<const uint16_t*>(q), T, ix->dcfg,
                    ws->lut, ws->rtab, ws->qnorm, ws->qrot, dbg_q_rot, ws->ucount);
}

cudaError_t set_phase_qprep(unsigned long long* p) { return set_phase_ptr_tu(p); }

}  // namespace pkv
