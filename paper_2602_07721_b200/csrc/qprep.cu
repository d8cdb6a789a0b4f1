// Query preparation (a1): normalise & rotate q, rank the 256 analytic centroids of every
// subspace by the query-centroid dot product ("cheap dot product q^T c") and turn ranks into the
// multi-tier collision bonuses, written as one byte per query head into the packed u32 lookup table
// of the scan; also the rerank tables sign*L[idx]*q~_j used by the RSQ-IP estimate (Eq. 10).
//
// Grid (8 subspace pairs, n_q heads, batch), 128 threads. Exact contract shared with the oracle (AMB-9):
// y' = fp64 butterflies of s (.) q; score_c = fp64 left-to-right sum of +-y'_j from 0.0; order (score desc,
// id asc). The complement symmetry score(255-c) = -score(c) halves the sort to 128 "leaders", two per thread;
// the bitonic network runs in registers and warp shuffles, only its stage with distance 64 in smem.
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

// CTA = two subspaces (sb0 = 2*blockIdx.x, sb0 + 1) of one query head, 64 threads each, 2 leaders per thread
// (position p = 2*tl + i): distance 1 inside a thread, 2..32 by shuffles, 64 through shared memory. 128-thread
// CTAs, half the CTAs of one subspace per CTA: a batch of 8 x 32 heads fits one wave.
__global__ void __launch_bounds__(QP_THREADS) qprep_kernel(const uint16_t* q, int T, DevCfg cfg,
                                                          uint32_t* lut, float* rtab,
                                                          float* qnorm, float* qrot,
                                                          float* dbg_q_rot, unsigned int* ucount,
                                                          const uint32_t* occ, int64_t rho_keys) {
  __shared__ unsigned long long sk[2][NC / 2];
  __shared__ uint32_t si[2][NC / 2];
  phase_mark(K_QPREP, 0);
  const int h = blockIdx.y, b = blockIdx.z;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int half = t >> 6, tl = t & 63;  // this thread's subspace (of the pair) and its index in that sort
  const int sb = 2 * blockIdx.x + half;
  const int g = h / cfg.G, hh = h % cfg.G;
  pdl_wait();  // the query of this layer follows the previous layer's work
  pdl_trigger();
  if (blockIdx.x == 0 && hh == 0 && t == 0) ucount[b * cfg.n_kv + g] = 0u;  // the select counts from 0
  phase_mark(K_QPREP, 1);
  // warp 0 rotates the query (fp64 butterflies) and publishes the pair's 16 coordinates and 1/||y'||
  __shared__ double s_yb[16];
  __shared__ double s_inv;
  const int sp = 2 * blockIdx.x;  // first subspace of the pair: coordinates 8sp .. 8sp+15 = lanes 2sp .. 2sp+3
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
    if (lane >= 2 * sp && lane < 2 * sp + 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) s_yb[4 * (lane - 2 * sp) + i] = v[i];
      float* qr = qrot + ((int64_t)b * cfg.n_q + h) * D;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        qr[4 * lane + i] = (float)(v[i] * inv_yn);
        if (dbg_q_rot) dbg_q_rot[((int64_t)b * cfg.n_q + h) * D + 4 * lane + i] = (float)(v[i] * inv_yn);
      }
    }
    if (lane == 0) s_inv = inv_yn;
    if (blockIdx.x == 0 && lane == 0) qnorm[(int64_t)b * cfg.n_q + h] = sqrtf(qn2);
  }
  __syncthreads();
  double yb[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) yb[j] = s_yb[8 * half + j];
  const double inv_yn = s_inv;
  // rerank table rows for coordinates 8sb..8sb+7 (two entries per thread): sign(n) L[n&7] q~_{8sb+j}
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int te = 2 * tl + i;
    const int j = te >> 4, nb = te & 15;
    double yj = yb[0];
#pragma unroll
    for (int jj = 1; jj < 8; ++jj) yj = (j == jj) ? yb[jj] : yj;
    const float qt = (float)(yj * inv_yn);
    const float L = cfg.levels[nb & 7];
    rtab[(((int64_t)b * cfg.n_q + h) * D + 8 * sb) * 16 + te] = (nb & 8) ? L * qt : -L * qt;
  }
  phase_mark(K_QPREP, 2);
  // Complement symmetry: score(255 - c) == -score(c) exactly (every partial sum of the left-to-right fp64 sum
  // is negated, round-to-nearest is odd-symmetric and an exact zero is +0.0 either way). So the (score desc,
  // id asc) order of all 256 is: the 128 "leaders" (of each pair {c, 255-c} the one that comes first) in
  // order, then their complements in reverse order -> rank(255 - c) = 255 - rank(c). Only the leaders are
  // sorted. Element i of thread tl is the pair {c, 255 - c}, c = 2*tl + i (c < 128 <= 255 - c breaks a zero tie).
  KV e[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int c = 2 * tl + i;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, ((c >> j) & 1) ? yb[j] : -yb[j]);
    const bool neg = acc < 0.0;
    e[i].k = ~ord_f64(neg ? -acc : acc);  // ascending key == descending score; ties by ascending id
    e[i].id = neg ? (uint32_t)(NC - 1 - c) : (uint32_t)c;
  }
  // Fast path: when the fp64 scores have 8 trailing zero mantissa bits (always, unless the query spans more than
  // ~27 binades: each y' is an exact sum of bf16 values and the 8-term score sums are exact too), the leader id
  // fits in those bits and the sort moves one 64-bit composite (2 shuffles per element and stage instead of 3):
  // ordering by composite == ordering by (key, id). Otherwise the (key, id) pair network below.
  if (__syncthreads_and(((e[0].k & 0xffull) == 0xffull) && ((e[1].k & 0xffull) == 0xffull))) {
    unsigned long long c[2] = {(e[0].k & ~0xffull) | e[0].id, (e[1].k & ~0xffull) | e[1].id};
#pragma unroll
    for (int k = 2; k <= NC / 2; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        if (j == 1) {  // positions 2tl, 2tl + 1: inside the thread
          const bool asc = ((2 * tl) & k) == 0;
          const unsigned long long lo = c[0] < c[1] ? c[0] : c[1], hi = c[0] < c[1] ? c[1] : c[0];
          c[0] = asc ? lo : hi;
          c[1] = asc ? hi : lo;
        } else {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int p = 2 * tl + i;
            unsigned long long o;
            if (j < 64) {
              o = __shfl_xor_sync(0xffffffffu, c[i], j >> 1);
            } else {
              sk[half][p] = c[i];
              __syncthreads();
              o = sk[half][p ^ j];
              __syncthreads();
            }
            const bool keep_min = (((p & j) == 0) == ((p & k) == 0));
            c[i] = (keep_min == (o < c[i])) ? o : c[i];
          }
        }
      }
    }
    e[0].id = (uint32_t)(c[0] & 0xffull);
    e[1].id = (uint32_t)(c[1] & 0xffull);
  } else {
#pragma unroll
    for (int k = 2; k <= NC / 2; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        if (j == 1) {
          const KV lo = e[0], hi = e[1];
          KV a2 = lo, b2 = hi;
          ce(a2, hi, 2 * tl, k, 1);
          ce(b2, lo, 2 * tl + 1, k, 1);
          e[0] = a2;
          e[1] = b2;
        } else {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int p = 2 * tl + i;
            KV o;
            if (j < 64) {
              o = shfl_kv(e[i], j >> 1);
            } else {
              sk[half][p] = e[i].k;
              si[half][p] = e[i].id;
              __syncthreads();
              o = KV{sk[half][p ^ j], si[half][p ^ j]};
              __syncthreads();
            }
            ce(e[i], o, p, k, j);
          }
        }
      }
    }
  }
  phase_mark(K_QPREP, 3);
  // Key-fraction reading of rho (AMB-8b): this subspace probes its centroids in rank order until the
  // probed ones hold >= rho_keys indexed keys: T_b = 1 + the first rank whose inclusive occupancy prefix reaches
  // rho_keys. Ranks 0..127 are the sorted leaders (rank p at thread p/2), ranks 128..255 their complements in
  // reverse (rank 255 - p), so the prefix before complement rank 255 - p is (all leaders) + (complements of the
  // leaders after p). Two block scans over the 64 threads of each subspace (the pair's halves are independent).
  if (occ != nullptr) {
    __shared__ uint32_t s_wsum[4][2];  // per warp: leader total, complement total
    __shared__ int s_T[2];
    const uint32_t* ob = occ + (((int64_t)b * cfg.n_kv + g) * NB + sb) * NC;
    uint32_t oL[2], oC[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      oL[i] = ob[e[i].id];
      oC[i] = ob[NC - 1 - e[i].id];
    }
    const uint32_t sL = oL[0] + oL[1], sC = oC[0] + oC[1];
    uint32_t iL = sL, iC = sC;  // inclusive scans over this warp's lanes
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, iL, x), c = __shfl_up_sync(0xffffffffu, iC, x);
      if (lane >= x) {
        iL += a;
        iC += c;
      }
    }
    if (lane == 31) {
      s_wsum[warp][0] = iL;
      s_wsum[warp][1] = iC;
    }
    if (tl == 0) s_T[half] = 0;  // rho_keys == 0 would probe nothing (never reached: rho_keys >= 1 here)
    __syncthreads();
    const int w0 = 2 * half;  // the two warps of this subspace: w0 (threads 0..31 of the half), w0 + 1
    const bool upper = (warp & 1) != 0;
    const uint32_t TL = s_wsum[w0][0] + s_wsum[w0 + 1][0], TC = s_wsum[w0][1] + s_wsum[w0 + 1][1];
    const uint32_t exL = (upper ? s_wsum[w0][0] : 0u) + iL - sL;  // leaders before rank 2tl
    const uint32_t exC = (upper ? s_wsum[w0][1] : 0u) + iC - sC;  // complements of leaders before 2tl
    const uint64_t tgt = (uint64_t)rho_keys;
    // (rank, keys before it, keys through it)
    const uint32_t rk[4] = {(uint32_t)(2 * tl), (uint32_t)(2 * tl + 1), (uint32_t)(NC - 1 - 2 * tl),
                            (uint32_t)(NC - 2 - 2 * tl)};
    const uint32_t bef[4] = {exL, exL + oL[0], TL + TC - exC - oC[0], TL + TC - exC - oC[0] - oC[1]};
    const uint32_t thr[4] = {oL[0], oL[1], oC[0], oC[1]};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if ((uint64_t)bef[i] < tgt && (uint64_t)bef[i] + thr[i] >= tgt) s_T[half] = (int)rk[i] + 1;
    __syncthreads();
    T = s_T[half];
  }
  // position p = 2*tl + i == rank of leader e[i].id, 255 - p == rank of its complement; write both bonus bytes
  // into this (head, subspace)'s own 256-byte row (the scan packs the 4 heads' bytes per centroid; rows of
  // different CTAs share no sector — bytes of one packed word written by 4 CTAs measured 1.2 us of stores)
  const int chunk = max(1, T / cfg.n_tiers);
  uint8_t* lb = reinterpret_cast<uint8_t*>(lut + ((int64_t)b * cfg.n_kv + g) * NC * NB);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int p = 2 * tl + i;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int rank = u ? NC - 1 - p : p;
      const uint32_t id = u ? NC - 1 - e[i].id : e[i].id;
      int bonus = 0;
      if (rank < T) bonus = cfg.tier_bonus[min(rank / chunk, cfg.n_tiers - 1)];
      lb[(hh * NB + sb) * NC + id] = (uint8_t)bonus;
    }
  }
  phase_mark(K_QPREP, 4);
}

}  // namespace

cudaError_t launch_qprep(const pkv_index* ix, const void* q, int T, int64_t rho_keys, float* dbg_q_rot,
                         cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(NB / 2, ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_QPREP, stream);
  return pdl_launch(qprep_kernel, grid, dim3(QP_THREADS), 0, stream, static_cast<const uint16_t*>(q), T, ix->dcfg,
                    ws->lut, ws->rtab, ws->qnorm, ws->qrot, dbg_q_rot, ws->ucount,
                    rho_keys > 0 ? (const uint32_t*)ix->occ : (const uint32_t*)nullptr, rho_keys);
}

cudaError_t set_phase_qprep(unsigned long long* p) { return set_phase_ptr_tu(p); }

}  // namespace pkv
