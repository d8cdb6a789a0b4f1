// Key encoder on the 5th-generation tensor cores (tcgen05): the SRHT rotation y' = H (s (.) k) as a
// 128 x 128 x 128 GEMM per tile of 128 keys, EXACT, then the per-subspace decisions of PAPER §4.1.
//
// Exactness (AMB-2 requires codes that are functions of the exact y'): a key whose non-zero elements lie within
// 16 binades of its largest is, in units of 2^(emax-150), a vector of integers v_j with |v_j| < 2^24 (the
// integer path of encode.cu). Each v_j is split into three 8-bit digits v = a 2^16 + b 2^8 + c; digits are
// exact in bf16, R = H diag(s) is +-1, and a digit GEMM accumulates at most 128 x 255 < 2^15 in magnitude, so
// every partial sum is an integer representable in fp32 — the tensor-core result is exact whatever its internal
// order. y = A 2^16 + B 2^8 + C is then assembled exactly in 64-bit integers. Keys outside that range (wide
// spans, subnormals, inf/nan) are listed for the half-warp encoder of encode.cu, which handles every key.
//
// Decisions: the sign bit is exact (integer y). The 3-bit magnitude index idx_j = #{t: fl(y_j^2) >= fl(M_t S)}
// (fp64 op sequence of the oracle) is taken in fp32 and certified: when y_j^2 is at least 2^-17 (relative) away
// from the two thresholds bracketing it, the fp64 decisions are the same (fp32 rounding here ~2^-22, fp64
// rounding in the oracle ~2^-50); otherwise that subspace is decided again with the exact fp64 sequence.
// Weights w' in fp32 as in encode.cu (ratios are scale-free).
//
// Kernel: persistent, 128 threads (thread t = key t of the tile, = TMEM lane t), one CTA per SM. Shared memory:
// R (32 KB, built once) and the three digit tiles (3 x 32 KB) in the UMMA K-major, no-swizzle canonical layout
// (8 x 16-byte core matrices, LBO = 128 B along K, SBO = 2 KB along M/N). One elected thread issues 3 x 8
// tcgen05.mma (M = N = 128, K = 16, bf16 -> fp32) into 3 x 128 TMEM columns and commits to an mbarrier; the
// epilogue reads its lane with tcgen05.ld.32x32b.x32.
#include "common.cuh"

#include <cuda_fp16.h>

namespace pkv {
namespace {

constexpr int TC_KEYS = 128;
constexpr int TC_TILE_BYTES = TC_KEYS * D * 2;            // one 128 x 128 bf16 operand
constexpr int TC_SMEM = 4 * TC_TILE_BYTES + 1024;         // R + 3 digit tiles + alignment slack
constexpr uint32_t TC_TMEM_COLS = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (row, k) in the K-major no-swizzle canonical layout of a 128 x 128 bf16 tile
__device__ __forceinline__ uint32_t umma_off(int row, int kchunk) {  // kchunk: 8-element (16-byte) chunk of k
  return (uint32_t)((row >> 3) * 2048 + kchunk * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);         // start address
  d |= (uint64_t)(128u >> 4) << 16;                 // leading byte offset: next core matrix along K
  d |= (uint64_t)(2048u >> 4) << 32;                // stride byte offset: next 8-row group along M/N
  d |= (uint64_t)1 << 46;                           // descriptor version (sm_100)
  return d;                                         // base offset 0, legacy LBO mode, SWIZZLE_NONE
}

// instruction descriptor: kind::f16, A = B = bf16, D = f32, K-major A and B, M = 128, N = 128
constexpr uint32_t TC_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(TC_IDESC), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__global__ void __launch_bounds__(TC_KEYS, 1) encode_tc_kernel(const uint16_t* __restrict__ K, int64_t sb, int64_t sh,
                                                               int64_t st, int64_t t0, int64_t count, int n_kv,
                                                               int64_t cap, int64_t total_tiles, int tiles_per_head,
                                                               DevCfg cfg, uint8_t* __restrict__ ids,
                                                               uint8_t* __restrict__ rec, int32_t* fb_list,
                                                               int32_t* fb_count) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sR = sm;                         // R[n][k] = H[n][k] s_k
  uint8_t* sA = sm + TC_TILE_BYTES;         // digit tiles A0 (2^16), A1 (2^8), A2 (1)
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base_s;
  __shared__ float sL[8];
  const int t = threadIdx.x, warp = t >> 5;

  // R, once per CTA: row n, chunk c holds k = 8c .. 8c+7
  for (int i = t; i < D * 16; i += TC_KEYS) {
    const int n = i >> 4, c = i & 15;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t lohi = 0;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int k = 8 * c + 2 * e + h2;
        const int neg = (__popc(n & k) & 1) ^ sign_bit(cfg, k);
        lohi |= (uint32_t)(neg ? 0xBF80u : 0x3F80u) << (16 * h2);  // bf16 -1 / +1
      }
      w[e] = lohi;
    }
    *reinterpret_cast<uint4*>(sR + umma_off(n, c)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (t < 8) sL[t] = cfg.levels[t];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_s)),
                 "n"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base_s;
  uint32_t phase = 0;

  for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    const int64_t bh = tile / tiles_per_head;
    const int64_t tt = (tile - bh * tiles_per_head) * TC_KEYS + t;  // key of this thread (relative to t0)
    const bool live = tt < count;
    const int64_t b = bh / n_kv, h = bh - b * n_kv;
    // ---- 1. load the key, split into exact 8-bit digits, stage the three digit tiles
    uint32_t w[64];
    {
      const uint16_t* src = K + b * sb + h * sh + (live ? tt : 0) * st;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const uint4 v = live ? ldg_nc_v4(src + 8 * c) : make_uint4(0, 0, 0, 0);
        w[4 * c] = v.x;
        w[4 * c + 1] = v.y;
        w[4 * c + 2] = v.z;
        w[4 * c + 3] = v.w;
      }
    }
    int emax = 0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const uint32_t bits = (w[i] >> (16 * h2)) & 0xffffu;
        const int e = (int)((bits >> 7) & 0xffu);
        emax = max(emax, e);
        bad |= (e == 0 && (bits & 0x7fu) != 0) || e == 0xff;
      }
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) {
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int e = (int)((w[i] >> (16 * h2 + 7)) & 0xffu);
        bad |= e != 0 && e < emax - 16;
      }
    }
    bool fast = live && !bad;  // cleared below for keys with a zero subspace (counted by the half-warp encoder)
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      uint32_t dg[3][4];
#pragma unroll
      for (int e4 = 0; e4 < 4; ++e4) {
        uint32_t out[3] = {0, 0, 0};
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const uint32_t bits = (w[4 * c + e4] >> (16 * h2)) & 0xffffu;
          const uint32_t e = (bits >> 7) & 0xffu;
          const uint32_t v = (fast && e != 0u) ? ((128u | (bits & 0x7fu)) << (e - (uint32_t)emax + 16u)) : 0u;
          const uint32_t sgn = (bits & 0x8000u);
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            const uint32_t dig = (v >> (16 - 8 * p)) & 0xffu;
            const uint32_t bf = dig ? ((__float_as_uint((float)dig) >> 16) | sgn) : 0u;  // exact in bf16
            out[p] |= bf << (16 * h2);
          }
        }
#pragma unroll
        for (int p = 0; p < 3; ++p) dg[p][e4] = out[p];
      }
#pragma unroll
      for (int p = 0; p < 3; ++p)
        *reinterpret_cast<uint4*>(sA + p * TC_TILE_BYTES + umma_off(t, c)) =
            make_uint4(dg[p][0], dg[p][1], dg[p][2], dg[p][3]);
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic-proxy stores -> tensor-core reads
    __syncthreads();
    // ---- 2. three exact digit GEMMs into TMEM columns [0,128), [128,256), [256,384)
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t rb = smem_u32(sR);
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const uint32_t ab = smem_u32(sA + p * TC_TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16(tmem + 128u * p, umma_desc(ab + 256u * kk), umma_desc(rb + 256u * kk), kk > 0 ? 1u : 0u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&mbar)));
    }
    {  // wait for the MMAs (mbarrier phase flips once per tile)
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(&mbar)), "r"(phase));
      }
      phase ^= 1u;
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // ---- 3. epilogue: exact y, decisions, weights, stores (4 subspaces per 32-column load)
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    uint32_t idw[16], code[16];
    float wp[16];
    const double pscale = __longlong_as_double((long long)(1023 + emax - 150) << 52);  // unit of the integers
#pragma unroll 1
    for (int g = 0; g < 4; ++g) {
      uint32_t ra[32], rb2[32], rc[32];
      tmem_ld32(lane_addr + 32u * g, ra);
      tmem_ld32(lane_addr + 128u + 32u * g, rb2);
      tmem_ld32(lane_addr + 256u + 32u * g, rc);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        long long yi[8];
        float yf[8], sq[8];
        float S = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = 8 * s4 + j;
          yi[j] = ((long long)(int)__uint_as_float(ra[col]) << 16) + ((long long)(int)__uint_as_float(rb2[col]) << 8) +
                  (long long)(int)__uint_as_float(rc[col]);
          yf[j] = (float)yi[j];
          sq[j] = yf[j] * yf[j];
          S += sq[j];
        }
        const int sbi = 4 * g + s4;
        uint32_t id = 0, cw = 0;
        bool certain = true;
        float thf[7];
#pragma unroll
        for (int k2 = 0; k2 < 7; ++k2) thf[k2] = (float)cfg.mid_sq[k2] * S;
        uint32_t nib[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool pos = yi[j] >= 0;
          const float x = sq[j];
          const bool b2 = x >= thf[3];
          const bool b1 = x >= (b2 ? thf[5] : thf[1]);
          const bool b0 = x >= (b2 ? (b1 ? thf[6] : thf[4]) : (b1 ? thf[2] : thf[0]));
          const int idx = 4 * b2 + 2 * b1 + (int)b0;
          // certify against the bracketing thresholds (relative margin 2^-17)
          const float lo = idx > 0 ? thf[idx - 1] : -1.f, hi = idx < 7 ? thf[idx] : 3.4e38f;
          certain &= (idx == 0 || x - lo > 7.62939453125e-06f * lo) && (idx == 7 || hi - x > 7.62939453125e-06f * hi);
          id |= (pos ? 1u : 0u) << j;
          nib[j] = ((pos ? 1u : 0u) << 3) | (uint32_t)idx;
        }
        const bool degenerate = (S == 0.f);  // all eight y are exactly zero (integers)
        fast &= !degenerate;                 // AMB-7 keys go to the half-warp encoder, which counts them
        if (!certain && !degenerate) {        // exact fp64 sequence of the oracle for this subspace
          double yd[8], sqd[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            yd[j] = (double)yi[j] * pscale;
            sqd[j] = __dmul_rn(yd[j], yd[j]);
          }
          double Sd = sqd[0];
#pragma unroll
          for (int j = 1; j < 8; ++j) Sd = __dadd_rn(Sd, sqd[j]);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t idx = 0;
#pragma unroll
            for (int k2 = 0; k2 < 7; ++k2) idx += (uint32_t)(sqd[j] >= __dmul_rn(cfg.mid_sq[k2], Sd));
            nib[j] = (nib[j] & 8u) | idx;
          }
        }
        float dot = 0.f, vn2 = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t nb = nib[j];
          if (degenerate) nb = (j == 0) ? 15u : 8u;  // AMB-7: encode(e_1): sign +, idx 7 on coordinate 0
          cw |= nb << (4 * j);
          const float L = sL[nb & 7u];
          dot = fmaf((nb & 8u) ? L : -L, yf[j], dot);
          vn2 = fmaf(L, L, vn2);
        }
        idw[sbi] = id;
        code[sbi] = cw;
        float wrel = 0.f;
        if (!degenerate) {
          const bool clamped = (dot <= 0.f) || (dot * dot < 1e-6f * vn2 * S);
          wrel = clamped ? sqrtf(S * (1.0f / 128.0f)) / (1e-3f * sqrtf(vn2)) : S / (11.313708498984761f * dot);
        }
        wp[sbi] = (float)((double)wrel * pscale);
      }
    }
    // ---- 4. stores (or hand the key to the exact half-warp encoder)
    if (live && !fast) {
      const int slot = atomicAdd(fb_count, 1);
      fb_list[slot] = (int32_t)(bh * count + tt);
    }
    if (fast) {
      const int64_t tg = t0 + tt;
      const int64_t row = bh * cap + tg;
      uint32_t rot[4];
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {  // byte i of the stored row = id of subspace (i + t) mod 16
        uint32_t v = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) v |= (idw[(4 * j4 + e + (int)(tg & 15)) & 15] & 0xffu) << (8 * e);
        rot[j4] = v;
      }
      *reinterpret_cast<uint4*>(ids + row * NB) = make_uint4(rot[0], rot[1], rot[2], rot[3]);
      uint8_t* r = rec + row * cfg.rec_bytes;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4)
        reinterpret_cast<uint4*>(r)[q4] = make_uint4(code[4 * q4], code[4 * q4 + 1], code[4 * q4 + 2], code[4 * q4 + 3]);
      if (cfg.w16) {  // fp16 weights with the per-key exponent in the sign bits (encode.cu)
        float m = 0.f;
#pragma unroll
        for (int s2 = 0; s2 < 16; ++s2) m = fmaxf(m, wp[s2]);
        int E = (m > 0.f) ? ((__float_as_int(m) >> 23) & 0xff) - 127 - 14 : 0;
        E = max(-126, min(126, E));
        const float down = __int_as_float((127 - E) << 23);
        uint32_t hw[8];
#pragma unroll
        for (int s2 = 0; s2 < 16; s2 += 2) {
          const uint32_t h0 = (uint32_t)__half_as_ushort(__float2half_rn(wp[s2] * down)) | ((((uint32_t)E >> (s2 & 7)) & 1u) << 15);
          const uint32_t h1 = (uint32_t)__half_as_ushort(__float2half_rn(wp[s2 + 1] * down)) |
                              ((((uint32_t)E >> ((s2 + 1) & 7)) & 1u) << 15);
          hw[s2 >> 1] = h0 | (h1 << 16);
        }
        reinterpret_cast<uint4*>(r + 64)[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        reinterpret_cast<uint4*>(r + 64)[1] = make_uint4(hw[4], hw[5], hw[6], hw[7]);
      } else {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          reinterpret_cast<float4*>(r + 64)[q4] = make_float4(wp[4 * q4], wp[4 * q4 + 1], wp[4 * q4 + 2], wp[4 * q4 + 3]);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();  // TMEM and the digit tiles are rewritten by the next tile
    asm volatile("tcgen05.fence::after_thread_sync;\n");
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TC_TMEM_COLS));
}

}  // namespace

cudaError_t init_encode_tc_attrs() {
  return cudaFuncSetAttribute(encode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
}

cudaError_t launch_encode_tc(const pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t0,
                             int64_t count, int32_t* fb_list, int32_t* fb_count, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const int tiles_per_head = (int)((count + TC_KEYS - 1) / TC_KEYS);
  const int64_t total = (int64_t)tiles_per_head * ix->batch * ix->cfg.n_kv_heads;
  const int grid = (int)std::min<int64_t>(total, ix->num_sms);
  ProfScope p_(K_ENCODE, stream);
  encode_tc_kernel<<<grid, TC_KEYS, TC_SMEM, stream>>>(static_cast<const uint16_t*>(K), sb, sh, st, t0, count,
                                                       ix->cfg.n_kv_heads, ix->cap, total, tiles_per_head, ix->dcfg,
                                                       ix->ids, ix->rec, fb_list, fb_count);
  return cudaGetLastError();
}

}  // namespace pkv
