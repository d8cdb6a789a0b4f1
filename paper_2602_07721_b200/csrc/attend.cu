// Gather + sparse attention (a7): Eq. 2-3 over hot rows U retrieved rows, with the full-precision
// K/V rows read either from HBM or, for the million-token offload case, directly from pinned host memory
// through UVA ("(iv) a UVA-based kernel") — no staging copy.
//
// attend_partial_kernel  grid (splits, n_kv, batch), 4 warps. Work items of one (sequence, KV head): the n_hot hot
//                        rows (each scored against the G query heads of the group: read once, used G times) and
//                        the G*k retrieved rows (each for its own query head). A warp keeps an online-softmax
//                        state (m, l, o) per query head in the log2 domain; lane L owns dims 4L..4L+3; rows are
//                        fetched 4 items at a time (8 x 8-byte loads in flight per lane) to cover UVA latency.
//                        Emits one partial (m, l, o[128]) per (query head, split).
// attend_combine_kernel  LSE merge of the partials (all splits, all ranks when sharded) -> bf16 out, natural lse.
#include <algorithm>

#include "common.cuh"

namespace pkv {
namespace {

constexpr int AT_WARPS = 4;
constexpr int AT_BATCH = 8;
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ float4 bf16x4(uint2 w) {
  return make_float4(bf16_lo(w.x), bf16_hi(w.x), bf16_lo(w.y), bf16_hi(w.y));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int x = 16; x > 0; x >>= 1) v += __shfl_xor_sync(0xffffffffu, v, x);
  return v;
}

struct SoftState {
  float m, l, o[4];
};
static_assert(AT_BATCH * GMAX == 32, "transpose-reduction maps one (row, head) pair per lane");

__global__ void __launch_bounds__(AT_WARPS * 32) attend_partial_kernel(AttendArgs a, int n_q, int n_kv, int G,
                                                                       int items_per_split, float* part,
                                                                       unsigned int* ticket, void* out,
                                                                       float* lse, float* out_f32) {
  phase_mark(K_ATTEND, 0);
  __shared__ __align__(16) float sm_x[AT_WARPS][AT_BATCH * GMAX];
  __shared__ float sm_m[AT_WARPS][GMAX], sm_l[AT_WARPS][GMAX];
  __shared__ float sm_o[AT_WARPS][GMAX][D];
  __shared__ float sm_w[GMAX][MAX_SPLITS];
  __shared__ float sm_M[GMAX], sm_L[GMAX];
  __shared__ int sm_last;
  pdl_trigger();
  const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float qscale = a.scale * LOG2E;
  float4 qv[GMAX];
#pragma unroll
  for (int hh = 0; hh < GMAX; ++hh) {
    if (hh < G) {
      const uint16_t* qp = static_cast<const uint16_t*>(a.q) + ((int64_t)b * n_q + g * G + hh) * D + 4 * lane;
      const float4 f = bf16x4(ldg_v2(qp));
      qv[hh] = make_float4(f.x * qscale, f.y * qscale, f.z * qscale, f.w * qscale);
    } else {
      qv[hh] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  SoftState st[GMAX];
#pragma unroll
  for (int hh = 0; hh < GMAX; ++hh) {
    st[hh].m = -INFINITY;
    st[hh].l = 0.f;
    st[hh].o[0] = st[hh].o[1] = st[hh].o[2] = st[hh].o[3] = 0.f;
  }
  const int n_items = a.n_hot + G * a.k;
  const int i0 = split * items_per_split;
  const int i1 = min(n_items, i0 + items_per_split);
  const uint16_t* Kb = static_cast<const uint16_t*>(a.K);
  const uint16_t* Vb = static_cast<const uint16_t*>(a.V);
  const uint16_t* Kh = static_cast<const uint16_t*>(a.K_hot) + ((int64_t)b * n_kv + g) * a.hot_rows * D;
  const uint16_t* Vh = static_cast<const uint16_t*>(a.V_hot) + ((int64_t)b * n_kv + g) * a.hot_rows * D;
  bool waited = false;
  for (int base = i0 + warp * AT_BATCH; base < i1; base += AT_WARPS * AT_BATCH) {
    uint2 kr[AT_BATCH], vr[AT_BATCH];
    int head[AT_BATCH];  // -1: hot row (all heads), -2: skip, else query head within the group
    // hot rows do not depend on the retrieval: issue them before waiting on the previous kernel
#pragma unroll
    for (int u = 0; u < AT_BATCH; ++u) {
      const int it = base + u;
      head[u] = -2;
      kr[u] = make_uint2(0, 0);
      vr[u] = make_uint2(0, 0);
      if (it < i1 && it < a.n_hot) {
        head[u] = -1;
        kr[u] = ldg_v2(Kh + (int64_t)it * D + 4 * lane);
        vr[u] = ldg_v2(Vh + (int64_t)it * D + 4 * lane);
      }
    }
    if (!waited) {
      pdl_wait();  // top-k ids come from the retrieval kernels
      phase_mark(K_ATTEND, 1);
      waited = true;
    }
    int id[AT_BATCH];
#pragma unroll
    for (int u = 0; u < AT_BATCH; ++u) {
      const int it = base + u;
      id[u] = -1;
      if (it < i1 && it >= a.n_hot) {
        const int r = it - a.n_hot;
        id[u] = a.idx[((int64_t)b * n_q + g * G + r / a.k) * a.k + r % a.k];
      }
    }
#pragma unroll
    for (int u = 0; u < AT_BATCH; ++u) {
      const int it = base + u;
      if (it < i1 && it >= a.n_hot && id[u] >= 0 && id[u] >= a.own_lo && id[u] < a.own_hi) {
        head[u] = (it - a.n_hot) / a.k;
        const int64_t off = (int64_t)b * a.sb + (int64_t)g * a.sh + ((int64_t)id[u] - a.id_offset) * a.st + 4 * lane;
        kr[u] = ldg_v2(Kb + off);
        vr[u] = ldg_v2(Vb + off);
      }
    }
    // all (row, head) partial dots of the batch, then one transpose-reduction: 31 shuffles leave the full dot
    // of pair L = (row L/4, head L%4) in lane L (instead of a serial 5-shuffle chain per row and head)
    float v[AT_BATCH * GMAX];
#pragma unroll
    for (int u = 0; u < AT_BATCH; ++u) {
      const float4 kf = bf16x4(kr[u]);
#pragma unroll
      for (int hh = 0; hh < GMAX; ++hh)
        v[u * GMAX + hh] = kf.x * qv[hh].x + kf.y * qv[hh].y + kf.z * qv[hh].z + kf.w * qv[hh].w;
    }
#pragma unroll
    for (int m = 16, V = 32; m >= 1; m >>= 1, V >>= 1) {
      const bool upper = (lane & m) != 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < V / 2) {
          const float send = upper ? v[i] : v[i + V / 2];
          const float keep = upper ? v[i + V / 2] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
      }
    }
    sm_x[warp][lane] = v[0];
    __syncwarp();
    float x[AT_BATCH * GMAX];
#pragma unroll
    for (int i = 0; i < AT_BATCH * GMAX / 4; ++i) {
      const float4 t4 = reinterpret_cast<const float4*>(sm_x[warp])[i];
      x[4 * i] = t4.x;
      x[4 * i + 1] = t4.y;
      x[4 * i + 2] = t4.z;
      x[4 * i + 3] = t4.w;
    }
    __syncwarp();
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) {
      if (hh >= G) break;
      float mx = st[hh].m;
#pragma unroll
      for (int u = 0; u < AT_BATCH; ++u)
        if (head[u] == -1 || head[u] == hh) mx = fmaxf(mx, x[u * GMAX + hh]);
      if (mx == -INFINITY) continue;  // no row of this head in the batch
      const float c = exp2f(st[hh].m - mx);
      float l = st[hh].l * c;
      float o0 = st[hh].o[0] * c, o1 = st[hh].o[1] * c, o2 = st[hh].o[2] * c, o3 = st[hh].o[3] * c;
#pragma unroll
      for (int u = 0; u < AT_BATCH; ++u) {
        if (head[u] == -1 || head[u] == hh) {
          const float pu = exp2f(x[u * GMAX + hh] - mx);
          const float4 vf = bf16x4(vr[u]);
          l += pu;
          o0 = fmaf(pu, vf.x, o0);
          o1 = fmaf(pu, vf.y, o1);
          o2 = fmaf(pu, vf.z, o2);
          o3 = fmaf(pu, vf.w, o3);
        }
      }
      st[hh].m = mx;
      st[hh].l = l;
      st[hh].o[0] = o0;
      st[hh].o[1] = o1;
      st[hh].o[2] = o2;
      st[hh].o[3] = o3;
    }
  }
  if (!waited) pdl_wait();
  // merge the 4 warps' states
#pragma unroll
  for (int hh = 0; hh < GMAX; ++hh) {
    if (lane == 0) {
      sm_m[warp][hh] = st[hh].m;
      sm_l[warp][hh] = st[hh].l;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) sm_o[warp][hh][4 * lane + i] = st[hh].o[i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * D; e += AT_WARPS * 32) {
    const int hh = e / D, d = e % D;
    float M = -INFINITY;
    for (int w = 0; w < AT_WARPS; ++w) M = fmaxf(M, sm_m[w][hh]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < AT_WARPS; ++w) {
        const float c = exp2f(sm_m[w][hh] - M);
        L += sm_l[w][hh] * c;
        O += sm_o[w][hh][d] * c;
      }
    }
    float* p = part + (((int64_t)b * n_q + g * G + hh) * MAX_SPLITS + split) * PART;
    if (d == 0) {
      p[0] = M;
      p[1] = L;
    }
    p[2 + d] = O;
  }
  phase_mark(K_ATTEND, 2);
  if (ticket == nullptr) return;  // sharded: the LSE merge runs after the all-gather
  // fused LSE merge: the last CTA of this (sequence, KV head) to finish combines all splits
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(&ticket[b * n_kv + g], 1u);
    sm_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!sm_last) return;
  __threadfence();
  const int nsplits = gridDim.x;
  if (warp < G) {
    const int hh = warp;
    const float* base = part + ((int64_t)b * n_q + g * G + hh) * MAX_SPLITS * PART;
    float M = -INFINITY;
    for (int s = lane; s < nsplits; s += 32) M = fmaxf(M, __ldcg(base + (int64_t)s * PART));
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, x));
    float L = 0.f;
    for (int s = lane; s < nsplits; s += 32) {
      const float m = __ldcg(base + (int64_t)s * PART);
      const float c = (m == -INFINITY) ? 0.f : exp2f(m - M);  // partial o is unnormalised: rescale only
      sm_w[hh][s] = c;
      L += c * __ldcg(base + (int64_t)s * PART + 1);
    }
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) L += __shfl_xor_sync(0xffffffffu, L, x);
    if (lane == 0) {
      sm_M[hh] = M;
      sm_L[hh] = L;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * D; e += AT_WARPS * 32) {
    const int hh = e / D, d = e % D;
    const float* base = part + ((int64_t)b * n_q + g * G + hh) * MAX_SPLITS * PART;
    float O = 0.f;
    for (int s = 0; s < nsplits; ++s) O += sm_w[hh][s] * __ldcg(base + (int64_t)s * PART + 2 + d);
    const float L = sm_L[hh];
    const int64_t bhq = (int64_t)b * n_q + g * G + hh;
    const float o = L > 0.f ? O / L : 0.f;
    static_cast<__nv_bfloat16*>(out)[bhq * D + d] = __float2bfloat16_rn(o);
    if (out_f32) out_f32[bhq * D + d] = o;
    if (lse && d == 0) lse[bhq] = L > 0.f ? (sm_M[hh] + log2f(L)) * 0.6931471805599453f : -INFINITY;
  }
  if (threadIdx.x == 0) ticket[b * n_kv + g] = 0u;  // re-arm for the next launch / graph replay
}

__global__ void __launch_bounds__(D) attend_combine_kernel(const float* parts, int nsplits, int P,
                                                            int64_t rank_stride, int n_q, void* out, float* lse,
                                                            float* out_f32) {
  const int h = blockIdx.x, b = blockIdx.y, d = threadIdx.x;
  const int64_t bhq = (int64_t)b * n_q + h;
  float M = -INFINITY;
  for (int r = 0; r < P; ++r)
    for (int s = 0; s < nsplits; ++s) M = fmaxf(M, parts[r * rank_stride + (bhq * MAX_SPLITS + s) * PART]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int r = 0; r < P; ++r) {
      for (int s = 0; s < nsplits; ++s) {
        const float* p = parts + r * rank_stride + (bhq * MAX_SPLITS + s) * PART;
        const float m = p[0];
        if (m == -INFINITY) continue;
        const float c = exp2f(m - M);
        L += p[1] * c;
        O += p[2 + d] * c;
      }
    }
  }
  const float o = L > 0.f ? O / L : 0.f;
  static_cast<__nv_bfloat16*>(out)[bhq * D + d] = __float2bfloat16_rn(o);
  if (out_f32) out_f32[bhq * D + d] = o;
  if (lse && d == 0) lse[bhq] = L > 0.f ? (M + log2f(L)) * 0.6931471805599453f : -INFINITY;
}

__global__ void fill_empty_topk_kernel(int32_t* idx, float* est, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    idx[i] = -1;
    est[i] = -INFINITY;
  }
}

}  // namespace

cudaError_t launch_fill_empty_topk(int32_t* out_idx, float* out_est, int64_t count, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  ProfScope p_(K_DEBUG, stream);
  fill_empty_topk_kernel<<<(unsigned)std::min<int64_t>(64, (count + 255) / 256), 256, 0, stream>>>(out_idx, out_est,
                                                                                                  count);
  return cudaGetLastError();
}

int plan_attend_splits(const pkv_index* ix, int total_items) {
  // one round of AT_BATCH rows per warp: every row load of a CTA is in flight at once
  (void)ix;
  int splits = (total_items + AT_WARPS * AT_BATCH - 1) / (AT_WARPS * AT_BATCH);
  if (splits > MAX_SPLITS) splits = MAX_SPLITS;
  if (splits < 1) splits = 1;
  return splits;
}

cudaError_t launch_attend_partial(const pkv_index* ix, const AttendArgs& a, int splits, float* part_out,
                                  unsigned int* ticket, void* out, float* lse, cudaStream_t stream) {
  const int G = ix->dcfg.G;
  const int n_items = a.n_hot + G * a.k;
  const int per = (n_items + splits - 1) / splits;
  dim3 grid(splits, ix->cfg.n_kv_heads, ix->batch);
  ProfScope p_(K_ATTEND, stream);
  return pdl_launch(attend_partial_kernel, grid, dim3(AT_WARPS * 32), 0, stream, a, ix->cfg.n_q_heads,
                    ix->cfg.n_kv_heads, G, per > 0 ? per : 1, part_out, ticket, out, lse, ix->dbg_out_f32);
}

cudaError_t launch_attend_combine(const pkv_index* ix, const float* parts, int nsplits, int P, void* out, float* lse,
                                  cudaStream_t stream) {
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  const int64_t rank_stride = (int64_t)ix->batch * ix->cfg.n_q_heads * MAX_SPLITS * PART;
  ProfScope p_(K_COMBINE, stream);
  attend_combine_kernel<<<grid, D, 0, stream>>>(parts, nsplits, P, rank_stride, ix->cfg.n_q_heads, out, lse,
                                                ix->dbg_out_f32);
  return cudaGetLastError();
}

cudaError_t set_phase_attend(unsigned long long* p) { return set_phase_ptr_tu(p); }

}  // namespace pkv
