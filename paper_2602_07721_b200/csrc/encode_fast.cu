// Key encoder, two threads per key (default; PAPER §4.1). The half-warp encoder (encode.cu)
// spends most of its instructions on what a 16-lane layout costs: 4 of the 7 butterfly stages through shuffles,
// per-lane redundant range checks, and fp64 decision sequences with fp64 selects. Here a CTA stages 64 key rows in
// shared memory with coalesced 16-byte loads, and each thread holds 64 coordinates of a key in registers:
//   * exact integers: with emax the largest exponent of the key and every nonzero element within 16 binades of it,
//     x_i = s_i k_i 2^(150 - emax) is an integer below 2^24 (exact truncating convert); the 7 Walsh-Hadamard
//     stages (6 in the thread, the last with the partner thread through one shuffle per value) run in int32
//     without overflow (|y| < 2^31) — y is EXACT;
//   * decisions certified in fp32: id bits are the signs of the exact y; the 3-bit magnitude (AMB-5) comes from
//     r = y_j^2 / S_b in fp32 (relative error <= ~16u, u = 2^-24) through a 72-bucket table of r (8 buckets per
//     binade, at most one threshold M_t per bucket, none within 1e-4 of a bucket edge: ef_buckets_ok); a decision
//     with r farther than 64u from its bucket's threshold is the decision of the oracle's fp64 sequence (AMB-2),
//     whose own rounding is ~2^-50 relative;
//   * weights (Eq. 7, 9, AMB-6) in fp32 from the same fp32 coordinates as encode.cu (identical formulas).
// A key outside the exact range (elements more than 16 binades apart, subnormal, inf/nan, tiny), with a zero
// subspace (AMB-7, counted in the stats by the exact kernel), or with an uncertified decision (~1% of keys) is
// appended to a list that the exact half-warp kernel encodes right after (encode_list_kernel), overwriting it.
#include "common.cuh"

namespace pkv {
namespace {

constexpr int EF_THREADS = 128;
constexpr int EF_KEYS = EF_THREADS / 2;            // keys per CTA, two threads per key
constexpr int EF_ROW = 272;                        // shared row stride: 256 B + 16 B padding (conflict-free reads)
constexpr int EF_SMEM = EF_KEYS * EF_ROW;          // the bf16 rows; then each warp stages its 16 records there
constexpr float EF_MARGIN = 96.f * 5.9604645e-8f;  // 96 u, relative to a threshold of r (64u + the 3 packed bits)
constexpr int EF_BUCKETS = 72;                     // r in [2^-9, 1): 9 binades x 8

// One subspace's decisions and weight (8 exact coordinates y): id bits, magnitude codes, certification slack, w'.
// Not inlined: the eight call sites share one copy of the code (the fully unrolled loop was 8 copies and the
// kernel stalled on instruction fetch 19% of the time).
__device__ __forceinline__ uint32_t umad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

struct EfSub {
  uint32_t idb, cw;
  float wp, dmin;
  int sok;
};
__device__ __noinline__ EfSub ef_subspace(int4 ya, int4 yb, const float4* sB, double unscale) {
  const int v[8] = {ya.x, ya.y, ya.z, ya.w, yb.x, yb.y, yb.z, yb.w};
  EfSub o;
  float f[8], q[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    f[j] = (float)v[j];
    q[j] = f[j] * f[j];
  }
  const float S = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
  o.sok = S > 0.f;  // a zero subspace takes the exact path (AMB-7 encoding + stats)
  // r = q / S: relative error <= ~16u (q 3u, S 7u, reciprocal 2u)
  const float invS = 1.0f / S;
  uint32_t idb = 0u, cw = 0u;
  float dot = 0.f, vn2 = 0.f, dmin = 3.0e38f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t pos = (uint32_t)(~v[j]) >> 31;  // y >= 0 (an int has no -0)
    const float r = q[j] * invS;
    const int k = min(EF_BUCKETS - 1, max(0, (int)(__float_as_uint(r) >> 20) - (118 << 3)));
    const float4 bt = sB[k];
    const float thr = bt.x;
    const bool up = r >= thr;
    const uint32_t idx = __float_as_uint(bt.w) + (up ? 1u : 0u);  // = (thr bits & 7) + up
    dmin = fminf(dmin, fabsf(r - thr) - EF_MARGIN * thr);
    // disjoint bit fields packed by multiply-adds (FMA pipe; the ALU pipe is this kernel's bound)
    const uint32_t nib = umad(pos, 8u, idx);
    idb = umad(pos, 1u << j, idb);
    cw = umad(nib, 1u << (4 * j), cw);
    const float Lm = up ? bt.z : bt.y;
    const float Ls = __uint_as_float(__float_as_uint(Lm) | (__float_as_uint(f[j]) & 0x80000000u));  // sign * L[idx]
    dot = fmaf(Ls, f[j], dot);
    vn2 = fmaf(Ls, Ls, vn2);
  }
  dot *= 4.656612873077393e-10f;  // y' 2^(119 - emax) = v 2^-31: encode.cu's scaled coordinates, |.| < 1
  // w' = w / ||sign L[idx]|| (encode.cu): alpha = dot / (||v~|| sqrt(S)), floor 1e-3 (AMB-6)
  const float Sf = S * 2.168404344971009e-19f;  // (2^-31)^2
  const bool clamped = (dot <= 0.f) || (dot * dot < 1e-6f * vn2 * Sf);
  const float w_rel =
      clamped ? sqrtf(Sf * (1.0f / 128.0f)) / (1e-3f * sqrtf(vn2)) : Sf / (11.313708498984761f * dot);
  o.wp = (float)((double)w_rel * unscale);
  o.idb = idb;
  o.cw = cw;
  o.dmin = dmin;
  return o;
}

#ifndef PKV_EF_MINB
#define PKV_EF_MINB 5  // 96 registers, 5 CTAs per SM: 301.4 vs 307.5 us (4 CTAs), 302.4 (6 CTAs) per 1M keys
#endif
__global__ void __launch_bounds__(EF_THREADS, PKV_EF_MINB) encode_fast_kernel(const uint16_t* __restrict__ K, int64_t sb,
                                                                     int64_t sh, int64_t st, int64_t count, int n_kv,
                                                                     int64_t cap, int64_t t0, DevCfg cfg,
                                                                     uint8_t* __restrict__ ids,
                                                                     uint8_t* __restrict__ rec, int32_t* fb_list,
                                                                     int32_t* fb_n) {
  extern __shared__ __align__(16) uint8_t rows[];  // EF_SMEM bytes
  // magnitude buckets of r = y^2 / S: (threshold with the idx below it in its 3 low bits, L[idx below],
  // L[idx above]) — the decision and its level come from one load
  __shared__ float4 sB[EF_BUCKETS];
  __shared__ __align__(16) uint4 sS[16];           // per 32-bit word of a key row: the rotation signs of its two bf16
  const int tid = threadIdx.x, bh = blockIdx.y, half = tid & 1;
  const int b = bh / n_kv, h = bh - b * n_kv;
  const int64_t tile0 = (int64_t)blockIdx.x * EF_KEYS;
  if (tid < EF_BUCKETS) {
    // bucket k: r in [2^-9 (1 + (k&7)/8) 2^(k>>3), next edge); bucket 0 also takes everything below
    const float lo = ldexpf(1.f + (float)(tid & 7) * 0.125f, (tid >> 3) - 9);
    const float hi = (tid & 7) == 7 ? ldexpf(1.f, (tid >> 3) - 8)
                                    : ldexpf(1.f + (float)((tid & 7) + 1) * 0.125f, (tid >> 3) - 9);
    int below = 0;
    float thr = 3.0e38f;
    for (int t = 0; t < 7; ++t) {
      const float m = (float)cfg.mid_sq[t];
      below += m < lo;
      if (m >= lo && m < hi) thr = m;
    }
    sB[tid] = make_float4(__uint_as_float((__float_as_uint(thr) & ~7u) | (uint32_t)below), cfg.levels[below],
                          cfg.levels[below < 7 ? below + 1 : 7], __uint_as_float((uint32_t)below));
  }
  if (tid < 64) {  // word i holds coordinates 2i (low half) and 2i + 1 (high half)
    const uint32_t w = cfg.sign_mask[tid >> 4];
    reinterpret_cast<uint32_t*>(sS)[tid] =
        (((w >> ((2 * tid) & 31)) & 1u) << 15) | (((w >> ((2 * tid + 1) & 31)) & 1u) << 31);
  }
  // ---- rows of the tile: 16 threads per 256-byte row, all 8 loads of a thread in flight at once
  {
    const uint16_t* Kb = K + b * sb + h * sh;
    uint4 ld[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = i * EF_THREADS + tid, r = c >> 4, part = c & 15;
      ld[i] = (tile0 + r < count) ? ldg_nc_v4(Kb + (tile0 + r) * st + 8 * part) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = i * EF_THREADS + tid, r = c >> 4, part = c & 15;
      *reinterpret_cast<uint4*>(rows + r * EF_ROW + 16 * part) = ld[i];
    }
  }
  __syncthreads();
  const int kk = tid >> 1;  // this thread's key in the tile; it holds coordinates 64*half .. 64*half + 63
  const int64_t tt = tile0 + kk;
  const bool live = tt < count;
  const uint8_t* my = rows + kk * EF_ROW + 128 * half;
  // ---- exponent range of the key (zeros excluded from the minimum), combined with the partner thread
  uint32_t mx = 0u, mn = 0x7fff7fffu;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint4 x4 = *reinterpret_cast<const uint4*>(my + 16 * i);
    const uint32_t xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t a = xs[e] & 0x7fff7fffu;
      mx = __vmaxu2(mx, a);
      // zero halves -> 0x7fff (never the minimum): bit 15 of a + 0x7fff is set iff the half is nonzero (no carry
      // crosses the halves), z marks the zero halves, z - (z >> 15) fills them with 0x7fff
      const uint32_t z = ~(a + 0x7fff7fffu) & 0x80008000u;
      mn = __vminu2(mn, a | (z - (z >> 15)));
    }
  }
  mx = __vmaxu2(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  mn = __vminu2(mn, __shfl_xor_sync(0xffffffffu, mn, 1));
  const int emax = (int)(max(mx >> 16, mx & 0xffffu) >> 7);
  const int emin = (int)(min(mn >> 16, mn & 0xffffu) >> 7);
  bool ok = live && emax >= 23 && emax <= 254 && emin + 16 >= emax;
  // ---- exact integers x_i = s_i k_i 2^(150 - emax): |x| < 2^24, an exact truncating convert
  const float scale = __int_as_float((277 - (ok ? emax : 150)) << 23);
  int v[64];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint4 x4 = *reinterpret_cast<const uint4*>(my + 16 * i);
    const uint4 s4 = sS[8 * half + i];  // broadcast within each half
    const uint32_t xs[4] = {x4.x ^ s4.x, x4.y ^ s4.y, x4.z ^ s4.z, x4.w ^ s4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[8 * i + 2 * e] = __float2int_rz(__uint_as_float(xs[e] << 16) * scale);
      v[8 * i + 2 * e + 1] = __float2int_rz(__uint_as_float(xs[e] & 0xffff0000u) * scale);
    }
  }
  // ---- y = H x (exact in int32): stages h = 1 .. 32 inside the thread, h = 64 with the partner
#pragma unroll
  for (int hh = 1; hh < 64; hh <<= 1) {
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if ((i & hh) == 0) {
        const int a = v[i], c = v[i + hh];
        v[i] = a + c;
        v[i + hh] = a - c;
      }
    }
  }
  {
    const int sg = half ? -1 : 1;  // lower half: v + o; upper half: o - v
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = v[i] * sg + __shfl_xor_sync(0xffffffffu, v[i], 1);
  }
  // ---- this thread's 8 subspaces 8*half .. 8*half + 7 (y still in registers): id bits, certified magnitude codes,
  // weights. The codes and weights of the warp's 16 keys are staged in the warp's (consumed) row buffer and written
  // as one contiguous 2 KB block (a key that fails certification is re-encoded by the exact list kernel after
  // this one, overwriting it).
  const double unscale = __longlong_as_double((long long)(1023 - 119 + (ok ? emax : 150)) << 52);
  unsigned long long id8 = 0ull;  // id bytes of this thread's 8 subspaces
  uint32_t code[8];
  float wp[8];
  float dmin = 3.0e38f;  // smallest |r - threshold| / threshold margin slack over the thread's coordinates
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const EfSub o = ef_subspace(make_int4(v[8 * s], v[8 * s + 1], v[8 * s + 2], v[8 * s + 3]),
                                make_int4(v[8 * s + 4], v[8 * s + 5], v[8 * s + 6], v[8 * s + 7]), sB, unscale);
    ok &= o.sok != 0;
    dmin = fminf(dmin, o.dmin);
    id8 |= (unsigned long long)o.idb << (8 * s);
    code[s] = o.cw;
    wp[s] = o.wp;
  }
  ok &= dmin > 0.f;
  {
    __syncwarp();  // the warp's rows are consumed: its 16 records go there
    uint8_t* stage = rows + (tid >> 5) * 16 * EF_ROW;
    uint4* me = reinterpret_cast<uint4*>(stage + (kk & 15) * REC + 32 * half);
    me[0] = make_uint4(code[0], code[1], code[2], code[3]);
    me[1] = make_uint4(code[4], code[5], code[6], code[7]);
    me[4] = make_uint4(__float_as_uint(wp[0]), __float_as_uint(wp[1]), __float_as_uint(wp[2]), __float_as_uint(wp[3]));
    me[5] = make_uint4(__float_as_uint(wp[4]), __float_as_uint(wp[5]), __float_as_uint(wp[6]), __float_as_uint(wp[7]));
    __syncwarp();
    const int64_t k0 = tile0 + (kk & ~15);  // the warp's first key
    uint8_t* grec = rec + ((int64_t)bh * cap + t0 + k0) * REC;
    const int lane = tid & 31;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = lane + 32 * i;  // 16-byte chunk of the warp's 2 KB: key c >> 3
      if (k0 + (c >> 3) < count)
        reinterpret_cast<uint4*>(grec)[c] = reinterpret_cast<const uint4*>(stage)[c];
    }
  }
  const int64_t row = (int64_t)bh * cap + t0 + (live ? tt : 0);
  // ---- the key's id row (both halves), or the exact kernel's list
  const uint32_t idw[2] = {(uint32_t)id8, (uint32_t)(id8 >> 32)};
  const uint32_t p0 = __shfl_xor_sync(0xffffffffu, idw[0], 1), p1 = __shfl_xor_sync(0xffffffffu, idw[1], 1);
  const int pok = __shfl_xor_sync(0xffffffffu, (int)ok, 1);  // unconditionally: every lane takes part
  ok = ok && pok != 0;
  if (live && ok && half == 0) {
    const uint32_t w4[4] = {idw[0], idw[1], p0, p1};  // canonical order: subspace b in byte b
    // id row rotated left by (t mod 16) bytes: byte i = subspace (i + t) mod 16 (scan.cu)
    const int rot = (int)((t0 + tt) & 15);
    const int wr = rot >> 2, br = 8 * (rot & 3);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t lo = w4[(k + wr) & 3], hi = w4[(k + wr + 1) & 3];
      o[k] = br ? __funnelshift_r(lo, hi, br) : lo;
    }
    *reinterpret_cast<uint4*>(ids + row * NB) = make_uint4(o[0], o[1], o[2], o[3]);
  }
  const bool to_list = live && !ok && half == 0;
  const unsigned m = __ballot_sync(0xffffffffu, to_list);
  if (m) {
    int base = 0;
    if ((tid & 31) == 0) base = atomicAdd(fb_n, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (to_list) fb_list[base + __popc(m & ((1u << (tid & 31)) - 1u))] = (int32_t)(bh * count + tt);
  }
}

}  // namespace

// The bucket table's preconditions for a configuration's thresholds M_t (as fp32): M_0 >= 2^-9 * 1.125 (bucket 0
// also takes every r below it), M_6 < 1, at most one threshold per bucket, and none within 1e-4 (relative) of a
// bucket edge. The default Prop. 1 levels satisfy them (closest: M_5 = 2^-3 * 1.5013, 9e-4 from an edge); a
// configuration that does not takes the half-warp encoder.
bool ef_buckets_ok(const DevCfg& c) {
  int prev_bucket = -1;
  for (int t = 0; t < 7; ++t) {
    const float m = (float)c.mid_sq[t];
    if (!(m >= ldexpf(1.125f, -9)) || !(m < 1.f)) return false;
    int e;
    const float fr = frexpf(m, &e);  // m = fr * 2^e, fr in [0.5, 1)
    const float mant = 2.f * fr;     // [1, 2)
    const int k = (e - 1 + 9) * 8 + (int)((mant - 1.f) * 8.f);
    if (k <= prev_bucket) return false;
    prev_bucket = k;
    for (int j = 0; j <= 8; ++j) {  // edges of this binade (and the next binade's first)
      const float edge = ldexpf(1.f + 0.125f * (float)j, e - 1);
      if (fabsf(m - edge) <= 1e-4f * edge) return false;
    }
  }
  return true;
}

cudaError_t launch_encode_fast(const pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t0,
                               int64_t count, int32_t* list, int32_t* list_n, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((count + EF_KEYS - 1) / EF_KEYS), ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_ENCODE, stream);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(encode_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, EF_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  encode_fast_kernel<<<grid, EF_THREADS, EF_SMEM, stream>>>(static_cast<const uint16_t*>(K), sb, sh, st, count,
                                                             ix->cfg.n_kv_heads, ix->cap, t0, ix->dcfg, ix->ids,
                                                             ix->rec, list, list_n);
  return cudaGetLastError();
}

}  // namespace pkv
