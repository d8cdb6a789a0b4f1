// Stage I on the GPU: collision scan (a3) and bucket_topk (a4) — PAPER §4.2.2 (1).
//
// scan_kernel      every key of every KV head: score = sum_b LUT_b[id_b], 4 query heads per KV head packed as
//                  bytes of one u32 (max score 96 < 128, no carries). Reads 16 B of centroid ids per key.
//                  Lookup table in shared memory, 64 tables interleaved (word = c*64 + t, table t serves
//                  subspace t mod 16): lane L at step i reads subspace (L+i) mod 16 from table L+i, so the 32
//                  lanes of a warp hit 32 distinct banks for ANY ids (conflict-free). The encoder stores key t's
//                  id row rotated by t mod 16 bytes, so byte i of the row is that subspace; one PRMT builds the
//                  smem address (id byte -> bits 8..15, table offset -> bits 0..7). Per-warp score histograms
//                  in shared memory; per-chunk totals to global (deterministic, no global atomics).
// select_kernel    threshold s* = max{s : #(score >= s) >= C} per query head from cumulative chunk histograms,
//                  ties in the s* bucket handed out newest first (AMB-12), then the chunk's candidate ids.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace pkv {
namespace {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_WARPS = SCAN_THREADS / 32;
constexpr int LUT_WORDS = NC * 64;                 // 64 KB
constexpr int LUT_STG_STRIDE = 66;  // words per staged (query head, subspace) row: 64 + 2 (conflict-free transposes)
constexpr int SCAN_SMEM = LUT_WORDS * 4 + SCAN_WARPS * GMAX * HB * 4 + GMAX * NB * LUT_STG_STRIDE * 4;
constexpr int SCAN_UNROLL = 4;

template <int RES, bool FAST>
__device__ __forceinline__ uint32_t lut_load(uint32_t addr, uint32_t lut_base) {
  uint32_t v;
  if (FAST) {
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(RES));
  } else {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr + lut_base));
  }
  return v;
}

// Warp w of a chunk's CTA owns the contiguous key segment [t_begin + w*seg, +seg), seg a multiple of 128 keys; the
// select kernel uses the same segments, so the per-warp histograms of the scan give it every warp's output offsets.
__host__ __device__ __forceinline__ uint32_t warp_seg(uint32_t len) { return ((len + 32 * 128 - 1) / (32 * 128)) * 128; }

template <bool CHECK>
__device__ __forceinline__ void load_rows(uint4 (&row)[SCAN_UNROLL], const uint8_t* __restrict__ ids_bh, uint32_t base,
                                          uint32_t t_end) {
#pragma unroll
  for (int u = 0; u < SCAN_UNROLL; ++u) {
    const uint32_t t = base + (uint32_t)u * 32;
    row[u] = (!CHECK || t < t_end) ? ldg_nc_v4(ids_bh + (size_t)t * NB) : make_uint4(0, 0, 0, 0);
  }
}

// Score one key (16 conflict-free LUT reads) and record it; G query heads packed in the bytes of acc.
template <int RES, bool FAST, int G>
__device__ __forceinline__ void score_key(const uint4& r, const uint32_t (&p)[16], uint32_t lut_base,
                                          uint32_t* __restrict__ scores_bh, uint32_t* hist_w, uint32_t t) {
  const uint32_t wds[4] = {r.x, r.y, r.z, r.w};
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t a = prmt(wds[i >> 2], p[i], 0x5504u | ((uint32_t)(i & 3) << 4));
    acc += lut_load<RES, FAST>(a, lut_base);
  }
  scores_bh[t] = acc;
#pragma unroll
  for (int hh = 0; hh < G; ++hh) atomicAdd(&hist_w[hh * HB + prmt(acc, 0u, 0x4440u | (uint32_t)hh)], 1u);
}

// Main loop over this warp's segment [seg0, seg1), software-pipelined: rows of the next round are in flight while
// this round is scored. Full rounds run without per-key bounds checks; only the last round checks.
template <int RES, bool FAST, int G>
__device__ __forceinline__ void scan_loop(uint4 (&row)[SCAN_UNROLL], const uint8_t* __restrict__ ids_bh,
                                          uint32_t* __restrict__ scores_bh, uint32_t* hist_w, uint32_t seg0,
                                          uint32_t seg1, uint32_t lut_base) {
  const int lane = threadIdx.x & 31;
  uint32_t p[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) p[i] = (uint32_t)(lane + i) * 4u;
  constexpr uint32_t STEP = 32 * SCAN_UNROLL;
  uint32_t wbase = seg0;  // warp-uniform
  for (; wbase + STEP <= seg1; wbase += STEP) {  // all rows of this round in range
    uint4 nxt[SCAN_UNROLL];
    load_rows<true>(nxt, ids_bh, wbase + STEP + lane, seg1);
#pragma unroll
    for (int u = 0; u < SCAN_UNROLL; ++u)
      score_key<RES, FAST, G>(row[u], p, lut_base, scores_bh, hist_w, wbase + lane + u * 32);
#pragma unroll
    for (int u = 0; u < SCAN_UNROLL; ++u) row[u] = nxt[u];
  }
  if (wbase < seg1) {  // last, partial round (no further rows to prefetch)
#pragma unroll
    for (int u = 0; u < SCAN_UNROLL; ++u) {
      const uint32_t t = wbase + lane + u * 32;
      if (t < seg1) score_key<RES, FAST, G>(row[u], p, lut_base, scores_bh, hist_w, t);
    }
  }
}

template <int RES>
__global__ void __launch_bounds__(SCAN_THREADS, 1)
    scan_kernel(const uint8_t* __restrict__ ids, const uint32_t* lut_g, uint32_t* scores, uint32_t* chunk_hist,
                uint16_t* warp_hist, int64_t cap, int64_t sstride, int64_t n, int64_t chunk, int G) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* lut = smem;
  uint32_t* hist = smem + LUT_WORDS;
  const int bh = blockIdx.y, j = blockIdx.x;
  const int64_t t_begin = (int64_t)j * chunk;
  const int64_t t_end = min(n, t_begin + chunk);
  const uint8_t* ids_bh = ids + (int64_t)bh * cap * NB;
  pdl_trigger();
  phase_mark(K_SCAN, 0);
  // the centroid ids do not depend on the query: start streaming them before qprep has finished
  const uint32_t seg = warp_seg((uint32_t)(t_end - t_begin));
  const uint32_t seg0 = (uint32_t)t_begin + (threadIdx.x >> 5) * seg;
  const uint32_t seg1 = min((uint32_t)t_end, seg0 + seg);
  uint4 row[SCAN_UNROLL];
  load_rows<true>(row, ids_bh, seg0 + (threadIdx.x & 31), seg1);
  for (int i = threadIdx.x; i < SCAN_WARPS * GMAX * HB; i += SCAN_THREADS) hist[i] = 0u;
  pdl_wait();  // lookup table comes from qprep
  phase_mark(K_SCAN, 1);
  // qprep writes one 256-byte row of bonuses per (query head, subspace): lutb[hh][s][c] (no two CTAs share a
  // sector). (1) a coalesced copy of the 4 x 16 rows into a staging area, (2) thread (s, 4 centroids) packs the 4
  // heads' bytes of each centroid into one word (byte hh = head hh) and writes the 4 interleaved replicas
  // c*64 + s + 16 r, the two half-warps starting one replica apart (conflict-free stores)
  uint32_t* stg = hist + SCAN_WARPS * GMAX * HB;
  {
    const uint32_t* lw = lut_g + (int64_t)bh * NC * NB;  // 4 heads x 16 rows x 64 words
    uint32_t v[GMAX];
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) v[hh] = lw[hh * NB * (NC / 4) + threadIdx.x];
    const int s = threadIdx.x >> 6, c4 = threadIdx.x & 63;
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) stg[(hh * NB + s) * LUT_STG_STRIDE + c4] = v[hh];
  }
  __syncthreads();
  {
    const int s = threadIdx.x & 15, c4 = threadIdx.x >> 4, rot = c4 & 1;
    uint32_t h[GMAX];
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) h[hh] = stg[(hh * NB + s) * LUT_STG_STRIDE + c4];
    const uint32_t a0 = prmt(h[0], h[1], 0x5140u), a1 = prmt(h[0], h[1], 0x7362u);  // h0.0 h1.0 h0.1 h1.1 | .2 .3
    const uint32_t b0 = prmt(h[2], h[3], 0x5140u), b1 = prmt(h[2], h[3], 0x7362u);
    const uint32_t w[4] = {prmt(a0, b0, 0x5410u), prmt(a0, b0, 0x7632u), prmt(a1, b1, 0x5410u),
                           prmt(a1, b1, 0x7632u)};  // centroid 4 c4 + k: its 4 heads' bonus bytes
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = 4 * c4 + k;
#pragma unroll
      for (int r = 0; r < 4; ++r) lut[c * 64 + s + 16 * ((r + rot) & 3)] = w[k];
    }
  }
  __syncthreads();
  const uint32_t lut_base = (uint32_t)__cvta_generic_to_shared(lut);
  phase_mark(K_SCAN, 2);
  uint32_t* scores_bh = scores + (int64_t)bh * sstride;
  uint32_t* hist_w = hist + (threadIdx.x >> 5) * GMAX * HB;
  if (lut_base == (uint32_t)RES) {
    if (G == 4) scan_loop<RES, true, 4>(row, ids_bh, scores_bh, hist_w, seg0, seg1, lut_base);
    else if (G == 2) scan_loop<RES, true, 2>(row, ids_bh, scores_bh, hist_w, seg0, seg1, lut_base);
    else if (G == 3) scan_loop<RES, true, 3>(row, ids_bh, scores_bh, hist_w, seg0, seg1, lut_base);
    else scan_loop<RES, true, 1>(row, ids_bh, scores_bh, hist_w, seg0, seg1, lut_base);
  } else {
    scan_loop<RES, false, 4>(row, ids_bh, scores_bh, hist_w, seg0, seg1, lut_base);  // G <= 4: unused bytes are 0
  }
  if (warp_hist != nullptr) {
    // this warp's cumulative counts cum_w[h][s] = #(score_h >= s) in its segment (u16: a segment holds < 2^16 keys),
    // read by the select kernel instead of a counting pass over the scores
    __syncwarp();
    const int lane = threadIdx.x & 31;
    uint16_t* wo = warp_hist + (((int64_t)bh * gridDim.x + j) * SCAN_WARPS + (threadIdx.x >> 5)) * GMAX * HB;
    for (int hh = 0; hh < G; ++hh) {
      uint32_t v[4], tot = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[e] = hist_w[hh * HB + 4 * lane + e];
        tot += v[e];
      }
      uint32_t inc = tot;
#pragma unroll
      for (int x = 1; x < 32; x <<= 1) {
        const uint32_t o = __shfl_down_sync(0xffffffffu, inc, x);
        if (lane + x < 32) inc += o;
      }
      uint32_t run = inc - tot;
      uint32_t c[4];
#pragma unroll
      for (int e = 3; e >= 0; --e) {
        run += v[e];
        c[e] = run;
      }
      reinterpret_cast<uint2*>(wo + hh * HB)[lane] = make_uint2(c[0] | (c[1] << 16), c[2] | (c[3] << 16));
    }
  }
  __syncthreads();
  phase_mark(K_SCAN, 3);
  // per-CTA totals, then cumulative (suffix) counts cum[s] = #(score >= s), one warp per query head
  for (int i = threadIdx.x; i < GMAX * HB; i += SCAN_THREADS) {
    uint32_t s = 0;
    for (int w = 0; w < SCAN_WARPS; ++w) s += hist[w * GMAX * HB + i];
    hist[i] = s;  // warp 0's slot reused: every warp's reads of slot i precede this write (same thread)
  }
  __syncthreads();
  uint32_t* out = chunk_hist + ((int64_t)bh * MAX_CHUNKS + j) * GMAX * HB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < GMAX) {
    // lane l owns bins 4l..4l+3; suffix sums across lanes from the top
    uint32_t v[4], tot = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[e] = hist[warp * HB + 4 * lane + e];
      tot += v[e];
    }
    uint32_t inc = tot;  // inclusive suffix over lanes >= lane
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) {
      const uint32_t o = __shfl_down_sync(0xffffffffu, inc, x);
      if (lane + x < 32) inc += o;
    }
    uint32_t run = inc - tot;  // counts of bins above this lane's range
#pragma unroll
    for (int e = 3; e >= 0; --e) {
      run += v[e];
      out[warp * HB + 4 * lane + e] = run;
    }
  }
  phase_mark(K_SCAN, 4);
}

// sel layout per (b, q head): [0] s*, [1] gt_local, [2] C_local, [3] take_local (written by chunk 0's CTA)
constexpr int SEL_STRIDE = 4 + 4 * MAX_CHUNKS;
constexpr int SEL_THREADS = 1024;
constexpr int SEL_SMEM = 32 * 4 * 128 * 8;  // per-warp compaction lists: up to 4 groups of 128 keys x uint2

// Fused threshold + compaction (bucket_topk). Chunk histograms are CUMULATIVE:
// cum_j[h][s] = #(score >= s) in chunk j. Every CTA of a (sequence, KV head) recomputes, for its query heads,
//   s*      = max{s : sum_j cum_j[s] >= C}            (global over ranks when sharded: all_hist)
//   ties    : C - #(> s*) taken newest first — newest rank, then newest chunk, then newest key (AMB-12)
//   offsets : gt_off = sum_{j' < j} #(> s*) in j',  tie quota/offset from the suffix of newer chunks
// and then writes its chunk's candidates: two passes over the packed scores (L2), warp-level ballots,
// one block scan of the per-warp counts (no per-tile block synchronisation).
template <int VB>  // 128-key groups per lane batch (VB * 4 keys per lane in flight)
__global__ void __launch_bounds__(SEL_THREADS) select_kernel(
    const uint32_t* chunk_hist, const uint32_t* all_hist, int P, int rank, int batch, const uint32_t* scores,
    int64_t cap, int64_t n, int64_t chunk, int nchunks, int n_q, int n_kv, int G, int64_t C, int64_t id_offset,
    int64_t cand_stride, int32_t* cand, int32_t* sel, const uint8_t* rec, int64_t rec_head_bytes, int rec_bytes,
    unsigned int* ucount, int32_t* uid, int32_t* upos, const uint16_t* warp_hist) {
  phase_mark(K_SELECT, 0);
  cta_mark(K_SELECT, 1);
  __shared__ uint32_t Hg[GMAX][HB];   // global cumulative counts
  __shared__ uint32_t Hl[GMAX][HB];   // this rank's cumulative counts
  __shared__ int s_star[GMAX], gt_local[GMAX], take_local[GMAX];
  __shared__ int p_base[GMAX], p_take[GMAX], p_eq[GMAX];
  __shared__ uint32_t wcnt[32][2 * GMAX];
  extern __shared__ uint2 sel_list[];  // per-warp compaction lists (VB * 128 entries each), SEL_SMEM bytes
  pdl_trigger();
  pdl_wait();
  phase_mark(K_SELECT, 1);
  const int bh = blockIdx.y, j = blockIdx.x;
  const int b = bh / n_kv, g = bh % n_kv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t* chb = chunk_hist + (int64_t)bh * MAX_CHUNKS * GMAX * HB;
  // B's input does not depend on the threshold: the first VB groups of this warp's segment are loaded now, so
  // their L2 latency overlaps A1-A3. Warp segments are whole multiples of 128 keys: a lane reads 4 consecutive
  // keys as one 16-byte vector.
  const uint32_t t_begin = (uint32_t)j * (uint32_t)chunk;
  const uint32_t t_end = (uint32_t)min(n, (int64_t)t_begin + chunk);
  const uint32_t len = t_end - t_begin;
  const uint32_t seg = warp_seg(len);
  const uint32_t seg0 = t_begin + warp * seg;
  const uint32_t seg1 = min(t_end, seg0 + seg);
  const uint32_t* sc = scores + (int64_t)bh * cap;
  uint4 vreg[VB];
  const uint32_t ngrp = (seg1 > seg0) ? (seg1 - seg0 + 127) / 128 : 0;  // 128-key groups of this warp
#pragma unroll
  for (int k2 = 0; k2 < VB; ++k2) {
    const uint32_t t = seg0 + 128u * k2 + 4u * lane;
    vreg[k2] = (t < seg1) ? *reinterpret_cast<const uint4*>(sc + t) : make_uint4(0, 0, 0, 0);
  }
  // A1: local and global cumulative totals. Thread (half, hh, s): half of the chunks, loads batched 16 at a time
  // so that many L2 requests are in flight (a load->add chain per chunk would serialise their latency).
  __shared__ uint32_t Hpart[GMAX][HB];
  {
    const int e = threadIdx.x & (GMAX * HB - 1), half = threadIdx.x / (GMAX * HB);
    const int hh = e / HB, s = e % HB;
    const int c_lo = half ? nchunks / 2 : 0, c_hi = half ? nchunks : nchunks / 2;
    uint32_t l = 0;
    for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
      uint32_t v[16];
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2)
        v[k2] = (hh < G && c0 + k2 < c_hi) ? chb[((int64_t)(c0 + k2) * GMAX + hh) * HB + s] : 0u;
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) l += v[k2];
    }
    if (half) Hpart[hh][s] = l;
    __syncthreads();
    if (!half && hh < G) {
      l += Hpart[hh][s];
      Hl[hh][s] = l;
      uint32_t t = l;
      if (P > 1) {
        uint32_t v[MAX_RANKS];
#pragma unroll
        for (int r = 0; r < MAX_RANKS; ++r)
          v[r] = r < P ? all_hist[(((int64_t)r * batch + b) * n_q + g * G + hh) * HB + s] : 0u;
        t = 0;
#pragma unroll
        for (int r = 0; r < MAX_RANKS; ++r) t += v[r];
      }
      Hg[hh][s] = t;
    }
  }
  __syncthreads();
  phase_mark(K_SELECT, 2);
  // A2: threshold per query head (warp hh)
  if (warp < G) {
    const int hh = warp;
    int ss = -1;
    if (C > 0) {
#pragma unroll
      for (int e = 0; e < HB / 32; ++e) {
        const int s = lane + 32 * e;
        const unsigned m = __ballot_sync(0xffffffffu, Hg[hh][s] >= (uint32_t)C);
        if (m) ss = 32 * e + 31 - __clz(m);
      }
    }
    if (lane == 0) {
      int take = 0, gtl = 0, st = HB;
      if (ss >= 0) {
        st = ss;
        const int64_t gt_g = (ss + 1 < HB) ? Hg[hh][ss + 1] : 0;
        int64_t need = C - gt_g;
        for (int r = P - 1; r > rank && P > 1; --r) {
          const uint32_t* hr = all_hist + (((int64_t)r * batch + b) * n_q + g * G + hh) * HB;
          need -= (int64_t)hr[ss] - (ss + 1 < HB ? hr[ss + 1] : 0);
          if (need < 0) need = 0;
        }
        gtl = (ss + 1 < HB) ? (int)Hl[hh][ss + 1] : 0;
        const int64_t eql = (int64_t)Hl[hh][ss] - gtl;
        take = (int)(need < eql ? need : eql);
      }
      s_star[hh] = st;
      gt_local[hh] = gtl;
      take_local[hh] = take;
    }
    __syncwarp();
    // A3: this chunk's offsets. A head's candidate list holds its selected keys (score > s*, and the taken s*
    // ties) in key order, chunk after chunk. Ties are handed out newest first, so the chunks after this one take
    // min(tl, eq_after) of them, this chunk min(eq, rest), the older chunks what remains:
    //   base = #(> s*) in older chunks + max(0, tl - eq_after - eq)
    const int st = s_star[hh];
    uint32_t gt_before = 0, eq_after = 0;
    int my_gt = 0, my_eq = 0;
    for (int jj = lane; jj < nchunks; jj += 32) {
      const uint32_t* cj = chb + ((int64_t)jj * GMAX + hh) * HB;
      const uint32_t gtv = (st + 1 < HB) ? cj[st + 1] : 0;
      const uint32_t eqv = (st < HB) ? cj[st] - gtv : 0;
      if (jj < j) gt_before += gtv;
      if (jj > j) eq_after += eqv;
      if (jj == j) {
        my_gt = (int)gtv;
        my_eq = (int)eqv;
      }
    }
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) {
      gt_before += __shfl_xor_sync(0xffffffffu, gt_before, x);
      eq_after += __shfl_xor_sync(0xffffffffu, eq_after, x);
      my_gt += __shfl_xor_sync(0xffffffffu, my_gt, x);
      my_eq += __shfl_xor_sync(0xffffffffu, my_eq, x);
    }
    if (lane == 0) {
      const int tl = take_local[hh];
      const int taken_after = (int)eq_after < tl ? (int)eq_after : tl;
      const int rem = tl - taken_after;
      p_take[hh] = rem < my_eq ? rem : my_eq;
      p_eq[hh] = my_eq;
      p_base[hh] = (int)gt_before + max(0, tl - (int)eq_after - my_eq);
      (void)my_gt;
      if (j == 0) {
        int32_t* o = sel + ((int64_t)b * n_q + g * G + hh) * SEL_STRIDE;
        o[0] = st;
        o[1] = gt_local[hh];
        o[2] = gt_local[hh] + tl;
        o[3] = tl;
      }
    }
  }
  __syncthreads();
  phase_mark(K_SELECT, 3);
  // B: compaction of this chunk. Warp w owns the contiguous segment [seg0, seg1).
  // Packed comparisons (scores <= 127, 4 query heads per u32): with K_gt = 0x7f - s*, K_ge = 0x80 - s* per byte,
  // bit 7 of byte h of (score + K_gt) is [score_h > s*_h] and of (score + K_ge) is [score_h >= s*_h] — no carries
  // cross bytes. Unused heads get s* = 127, which no score reaches.
  uint32_t kgt = 0, kge = 0;
#pragma unroll
  for (int hh = 0; hh < GMAX; ++hh) {
    const uint32_t st = (hh < G && s_star[hh] < HB) ? (uint32_t)s_star[hh] : 127u;
    kgt |= (0x7fu - st) << (8 * hh);
    kge |= (0x80u - st) << (8 * hh);
  }
  // pass 1: per-head counts of this warp's segment; lane l reads keys 4l..4l+3 of each 128-key group, VB groups
  // (16 keys per lane) in flight, kept in registers for pass 2 when the segment is short enough (the 128K case)
  uint32_t tot_gt[GMAX] = {0, 0, 0, 0}, tot_eq[GMAX] = {0, 0, 0, 0};
  if (warp_hist != nullptr) {
    // the dense scan recorded this warp segment's cumulative counts: #(> s*) = cum[s*+1], #(== s*) = cum[s*] - cum[s*+1]
    const uint16_t* wh = warp_hist + (((int64_t)bh * nchunks + j) * 32 + warp) * GMAX * HB;
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) {
      const int st = (hh < G) ? s_star[hh] : HB;
      const uint32_t ge = st < HB ? wh[hh * HB + st] : 0u;
      const uint32_t gt = st + 1 < HB ? wh[hh * HB + st + 1] : 0u;
      tot_gt[hh] = lane == 0 ? gt : 0u;  // summed over the warp's lanes below
      tot_eq[hh] = lane == 0 ? ge - gt : 0u;
    }
  }
  for (uint32_t g0 = 0; warp_hist == nullptr && g0 < ngrp; g0 += VB) {
    if (g0 > 0) {
#pragma unroll
      for (int k2 = 0; k2 < VB; ++k2) {
        const uint32_t t = seg0 + 128u * (g0 + k2) + 4u * lane;
        vreg[k2] = (t < seg1) ? *reinterpret_cast<const uint4*>(sc + t) : make_uint4(0, 0, 0, 0);
      }
    }
    uint32_t cgt = 0, ceq = 0;  // per-byte counts (<= 16 per batch: no carries)
#pragma unroll
    for (int k2 = 0; k2 < VB; ++k2) {
      const uint32_t t = seg0 + 128u * (g0 + k2) + 4u * lane;
      const uint32_t vv[4] = {vreg[k2].x, vreg[k2].y, vreg[k2].z, vreg[k2].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t gtb = (vv[e] + kgt) & 0x80808080u;
        const uint32_t geb = (vv[e] + kge) & 0x80808080u;
        if (t + e < seg1) {
          cgt += gtb >> 7;
          ceq += (geb & ~gtb) >> 7;
        }
      }
    }
#pragma unroll
    for (int hh = 0; hh < GMAX; ++hh) {
      tot_gt[hh] += (cgt >> (8 * hh)) & 0xffu;
      tot_eq[hh] += (ceq >> (8 * hh)) & 0xffu;
    }
  }
#pragma unroll
  for (int hh = 0; hh < GMAX; ++hh) {
    const uint32_t a1 = __reduce_add_sync(0xffffffffu, tot_gt[hh]);
    const uint32_t a2 = __reduce_add_sync(0xffffffffu, tot_eq[hh]);
    if (lane == 0) {
      wcnt[warp][2 * hh] = a1;
      wcnt[warp][2 * hh + 1] = a2;
    }
  }
  __syncthreads();
  if (warp < 2 * GMAX) {  // warp k scans column k over the 32 warps
    const int k = warp;
    const uint32_t v = wcnt[lane][k];
    uint32_t inc = v;
#pragma unroll
    for (int x = 1; x < 32; x <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, inc, x);
      if (lane >= x) inc += o;
    }
    wcnt[lane][k] = inc - v;  // exclusive base of warp `lane`
  }
  __syncthreads();
  // per-head running state in registers (the entry loop below is the select's hot loop; 1024-thread CTAs leave
  // 64 registers per thread, so nothing in it is re-read from shared memory or the parameter bank):
  //   base: list position of this warp's next selected key; the chunk's tie quota goes to its newest warps
  //   first, so this warp takes tw of its ew ties: all of them, none, or (one warp per chunk and head) the
  //   newest tw, for which es counts the ties already passed
  int base[GMAX], ew[GMAX], tw[GMAX], es[GMAX];
#pragma unroll
  for (int hh = 0; hh < GMAX; ++hh) {
    const int pre_gt = (int)wcnt[warp][2 * hh], pre_eq = (int)wcnt[warp][2 * hh + 1];
    ew[hh] = (warp < 31 ? (int)wcnt[warp + 1][2 * hh + 1] : p_eq[hh]) - pre_eq;
    const int suf = p_eq[hh] - pre_eq;  // ties in this warp and the newer ones
    base[hh] = p_base[hh] + pre_gt + max(0, p_take[hh] - suf);
    tw[hh] = min(ew[hh], max(0, p_take[hh] - (suf - ew[hh])));
    es[hh] = 0;
  }
  int32_t* const cd0 = cand + ((int64_t)b * n_q + g * G) * cand_stride;
  const int cs = (int)cand_stride;  // the group's lists span < 4 * capacity < 2^31 entries: 32-bit offsets
  const int32_t idoff = (int32_t)id_offset;
  const uint32_t lt = (1u << lane) - 1u;
  const bool do_prefetch = rec != nullptr, do_union = uid != nullptr;
  // Fast entry loop: every head of this warp takes all of its s* ties or none of them (true for all warps but at
  // most one per chunk and head) and no union list is built. A key is then picked for head h iff its flag byte h
  // has bit 7 (>) or, when the warp takes its ties, bit 6 (==): one mask, no per-head branches (1M: the entry
  // loop was ~185 instructions per 32 entries with the per-head branches).
#ifdef PKV_NO_FAST_ENTRY
  bool fast = false;  // A/B build: the per-head-branch loop for every warp
#else
  bool fast = !do_union;
#endif
  uint32_t pmask = 0;
#pragma unroll
  for (int hh = 0; hh < GMAX; ++hh) {
    if (hh < G && tw[hh] != 0 && tw[hh] != ew[hh]) fast = false;
    pmask |= (tw[hh] == 0 ? 0x80u : 0xc0u) << (8 * hh);  // heads >= G never have a flag set
  }
  phase_mark(K_SELECT, 4);
  // pass 2: keys with score >= s* for at least one head (~4 x beta of them) are first compacted, in key
  // order, into a per-warp list; the per-head ballots then run over that list only. Key (lane l, element e)
  // of a group precedes (l', e') iff l < l' or (l == l' and e < e'): its list slot is the number of kept keys
  // of lower lanes (one ballot per element position) plus its own earlier kept elements.
  uint2* wl = sel_list + warp * (VB * 128);
  for (uint32_t g0 = 0; g0 < ngrp; g0 += VB) {
    // vreg holds groups 0..VB-1 from the prologue unless pass 1 streamed the segment (no per-warp histograms)
    if (ngrp > VB && (g0 > 0 || warp_hist == nullptr)) {
#pragma unroll
      for (int k2 = 0; k2 < VB; ++k2) {
        const uint32_t t = seg0 + 128u * (g0 + k2) + 4u * lane;
        vreg[k2] = (t < seg1) ? *reinterpret_cast<const uint4*>(sc + t) : make_uint4(0, 0, 0, 0);
      }
    }
    if (g0 + VB < ngrp) {  // the next batch towards L1 while this one is compacted (no registers held)
#pragma unroll
      for (int k2 = 0; k2 < VB; ++k2) {
        const uint32_t t = seg0 + 128u * (g0 + VB + k2) + 4u * lane;
        if (t < seg1) asm volatile("prefetch.global.L1 [%0];" ::"l"(sc + t));
      }
    }
    uint32_t nl = 0;
#pragma unroll
    for (int k2 = 0; k2 < VB; ++k2) {
      const uint32_t t = seg0 + 128u * (g0 + k2) + 4u * lane;
      const uint32_t vv[4] = {vreg[k2].x, vreg[k2].y, vreg[k2].z, vreg[k2].w};
      uint32_t fl[4];
      bool keep[4];
      uint32_t below = 0, total = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t gtb = (vv[e] + kgt) & 0x80808080u;
        const uint32_t geb = (vv[e] + kge) & 0x80808080u;
        keep[e] = (t + e < seg1) && geb != 0u;
        fl[e] = gtb | ((geb & ~gtb) >> 1);  // bit 7: >, bit 6: ==
        const uint32_t m = __ballot_sync(0xffffffffu, keep[e]);
        below += __popc(m & lt);
        total += __popc(m);
      }
      uint32_t slot = nl + below;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (keep[e]) wl[slot++] = make_uint2(t + e, fl[e]);
      }
      nl += total;
    }
    __syncwarp();
    for (uint32_t l0 = 0; fast && l0 < nl; l0 += 32) {
      const bool valid = l0 + lane < nl;
      const uint2 ent = valid ? wl[l0 + lane] : make_uint2(0u, 0u);  // invalid lanes: no flags
      if (valid && do_prefetch) {  // warm L2 with the record the rerank kernel will gather for this key
        const uint8_t* r = rec + (int64_t)bh * rec_head_bytes + (int64_t)ent.x * rec_bytes;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(r));
        if (rec_bytes != 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(r + rec_bytes - 1));
      }
      const uint32_t pk = ent.y & pmask;
      const int32_t gid = (int32_t)ent.x + idoff;
#pragma unroll
      for (int hh = 0; hh < GMAX; ++hh) {
        const bool pick = (pk & (0xc0u << (8 * hh))) != 0u;
        const uint32_t m = __ballot_sync(0xffffffffu, pick);
        if (pick) cd0[hh * cs + base[hh] + __popc(m & lt)] = gid;
        base[hh] += __popc(m);
      }
    }
    for (uint32_t l0 = 0; !fast && l0 < nl; l0 += 32) {
      const bool valid = l0 + lane < nl;
      const uint2 ent = valid ? wl[l0 + lane] : make_uint2(0u, 0u);
      if (valid && do_prefetch) {  // warm L2 with the record the rerank kernel will gather for this key
        const uint8_t* r = rec + (int64_t)bh * rec_head_bytes + (int64_t)ent.x * rec_bytes;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(r));
        if (rec_bytes != 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(r + rec_bytes - 1));
      }
      int pos[GMAX];
      const int32_t gid = (int32_t)ent.x + idoff;
#pragma unroll
      for (int hh = 0; hh < GMAX; ++hh) {
        const bool fg = (ent.y & (0x80u << (8 * hh))) != 0u;
        const bool fe = (ent.y & (0x40u << (8 * hh))) != 0u;
        bool pick;
        if (tw[hh] == 0) {  // warp-uniform: none of this warp's ties is taken
          pick = fg;
        } else if (tw[hh] == ew[hh]) {  // all of them
          pick = fg | fe;
        } else {  // the chunk's tie boundary: a tie is taken iff fewer than tw ties of this warp are newer
          const uint32_t me = __ballot_sync(0xffffffffu, fe);
          pick = fg | (fe && ew[hh] - 1 - (es[hh] + __popc(me & lt)) < tw[hh]);
          es[hh] += __popc(me);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, pick);
        pos[hh] = pick ? base[hh] + __popc(m & lt) : -1;
        if (pick) cd0[hh * cs + pos[hh]] = gid;
        base[hh] += __popc(m);
      }
      if (do_union) {  // union entry: the key once, with its position in every head's candidate list
        const bool any = (pos[0] & pos[1] & pos[2] & pos[3]) != -1;  // positions >= 0, or -1
        const uint32_t ma = __ballot_sync(0xffffffffu, any);
        uint32_t ub = 0;
        if (lane == 0 && ma) ub = atomicAdd(&ucount[bh], (uint32_t)__popc(ma));
        ub = __shfl_sync(0xffffffffu, ub, 0);
        if (any) {
          const int64_t u = (int64_t)bh * cand_stride + ub + __popc(ma & lt);
          uid[u] = (int32_t)ent.x;
          reinterpret_cast<int4*>(upos)[u] = make_int4(pos[0], pos[1], pos[2], pos[3]);
        }
      }
    }
    __syncwarp();
  }
  phase_mark(K_SELECT, 5);
  cta_mark(K_SELECT, 0);
}

__global__ void dbg_scores_kernel(const uint32_t* __restrict__ scores, int64_t cap, int64_t n, int n_q, int n_kv,
                                  int G, uint8_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int bh = blockIdx.y;
  if (t >= n) return;
  const int b = bh / n_kv, g = bh % n_kv;
  const uint32_t s = scores[(int64_t)bh * cap + t];
  for (int hh = 0; hh < G; ++hh) out[((int64_t)b * n_q + g * G + hh) * n + t] = (uint8_t)(s >> (8 * hh));
}

}  // namespace

cudaError_t init_scan_attrs() {
  cudaError_t e = cudaFuncSetAttribute(scan_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAN_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(select_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SEL_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(select_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SEL_SMEM / 2);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(scan_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAN_SMEM);
}

// packed-score row stride: the capacity rounded to 4 keys, so every row is 16-byte aligned for the select's
// vector loads
int64_t score_stride(const pkv_index* ix) { return (ix->cap + 3) & ~(int64_t)3; }

// PKV_NO_WARP_HIST=1: the select counts its warps' keys itself (A/B switch; results are identical)
static bool warp_hist_on() {
  static const bool on = [] {
    const char* e = getenv("PKV_NO_WARP_HIST");
    return !(e && e[0] == '1');
  }();
  return on;
}

ScanPlan plan_scan(const pkv_index* ix, int64_t n) {
  if (ix->postings) {  // the inverted-list scan works on fixed chunks
    ScanPlan p;
    p.chunk = POST_CHUNK;
    p.nchunks = (int)std::max<int64_t>(1, (n + POST_CHUNK - 1) / POST_CHUNK);
    return p;
  }
  // One 1024-thread CTA per SM (~114 KB smem): never more CTAs than SMs, so there is no second wave.
  ScanPlan p;
  const int units = ix->batch * ix->cfg.n_kv_heads;
  int target = ix->num_sms / units;
  if (target < 1) target = 1;
  int64_t chunk = (n + target - 1) / target;
  if (chunk < 2048) chunk = 2048;
  chunk = (chunk + 31) / 32 * 32;
  int nch = (int)((n + chunk - 1) / chunk);
  if (nch > MAX_CHUNKS) {
    chunk = ((n + MAX_CHUNKS - 1) / MAX_CHUNKS + 31) / 32 * 32;
    nch = (int)((n + chunk - 1) / chunk);
  }
  if (nch < 1) nch = 1;
  p.nchunks = nch;
  p.chunk = chunk;
  // per-warp histograms (u16 counts): segments below 2^16 keys and the workspace's CTA slots
  // used only when a select warp's segment spans several register batches (> 512 keys: the 1M case), where
  // the select's counting pass would read the scores twice; below that the counting pass runs on registers and
  // measured faster than the scan's extra epilogue (128K: 48.0 vs 48.9 us/layer; 1M: 192.6 vs 194.7)
  const uint32_t wseg = warp_seg((uint32_t)std::min<int64_t>(chunk, 1 << 30));
  p.warp_hist = wseg > 4 * 128 && wseg < 65536 &&
                (int64_t)nch * units <= ix->ws->warp_hist_ctas && warp_hist_on();
  return p;
}

cudaError_t launch_scan(const pkv_index* ix, int64_t n, const ScanPlan& plan, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(plan.nchunks, ix->batch * ix->cfg.n_kv_heads);
  cudaError_t e;
  if (ix->smem_reserved == 1024) {
    ProfScope p_(K_SCAN, stream);
    e = pdl_launch(scan_kernel<1024>, grid, dim3(SCAN_THREADS), SCAN_SMEM, stream, (const uint8_t*)ix->ids,
                   (const uint32_t*)ws->lut, ws->scores, ws->chunk_hist, plan.warp_hist ? ws->warp_hist : nullptr,
                   ix->cap, score_stride(ix), n, plan.chunk, ix->dcfg.G);
  } else {
    ProfScope p_(K_SCAN, stream);
    e = pdl_launch(scan_kernel<0>, grid, dim3(SCAN_THREADS), SCAN_SMEM, stream, (const uint8_t*)ix->ids,
                   (const uint32_t*)ws->lut, ws->scores, ws->chunk_hist, plan.warp_hist ? ws->warp_hist : nullptr,
                   ix->cap, score_stride(ix), n, plan.chunk, ix->dcfg.G);
  }
  return e;
}

// L2 prefetch of the rerank records by the select kernel (PKV_SELECT_PREFETCH=0 disables it, for A/B)
static bool prefetch_rec() {
  static const bool on = [] {
    const char* e = getenv("PKV_SELECT_PREFETCH");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t launch_select(const pkv_index* ix, int64_t n, const ScanPlan& plan, const uint32_t* all_hist, int P,
                          int rank, int64_t C, int64_t id_offset, cudaStream_t stream) {
  const Workspace* ws = ix->ws;
  dim3 grid(plan.nchunks, ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_SELECT, stream);
  // 128-key groups per warp: ceil(chunk / (32 * 128)); two of them fit one batch (the 128K case), longer chunks
  // stream four groups per batch
  const bool small = (plan.chunk + 32 * 128 - 1) / (32 * 128) <= 2;
  return pdl_launch(small ? select_kernel<2> : select_kernel<4>, grid, dim3(SEL_THREADS),
                    small ? SEL_SMEM / 2 : SEL_SMEM, stream, (const uint32_t*)ws->chunk_hist, all_hist, P,
                    rank, ix->batch, (const uint32_t*)ws->scores, score_stride(ix), n, plan.chunk, plan.nchunks,
                    ix->cfg.n_q_heads, ix->cfg.n_kv_heads, ix->dcfg.G, C, id_offset, ws->cap, ws->cand, ws->sel,
                    // only when the candidates' records fit the L2 comfortably (128K: 32 MB); at 1M (214 MB) the
                    // prefetches evict each other and measured slower
                    prefetch_rec() && (int64_t)ix->batch * ix->cfg.n_q_heads * C * ix->dcfg.rec_bytes <= (48ll << 20)
                        ? (const uint8_t*)ix->rec
                        : (const uint8_t*)nullptr,
                    ix->cap * ix->dcfg.rec_bytes, ix->dcfg.rec_bytes, ws->ucount,
                    union_rerank() ? ws->uid : (int32_t*)nullptr, ws->upos,
                    plan.warp_hist ? (const uint16_t*)ws->warp_hist : (const uint16_t*)nullptr);
}

cudaError_t launch_dbg_scores(const pkv_index* ix, int64_t n, uint8_t* out, cudaStream_t stream) {
  dim3 grid((unsigned)((n + 255) / 256), ix->batch * ix->cfg.n_kv_heads);
  ProfScope p_(K_DEBUG, stream);
  dbg_scores_kernel<<<grid, 256, 0, stream>>>(ix->ws->scores, score_stride(ix), n, ix->cfg.n_q_heads, ix->cfg.n_kv_heads,
                                              ix->dcfg.G, out);
  return cudaGetLastError();
}

__global__ void head_hist_kernel(const uint32_t* chunk_hist, int nchunks, int n_q, int n_kv, int G,
                                 uint32_t* out) {
  const int h = blockIdx.x, b = blockIdx.y, bin = threadIdx.x;
  const int g = h / G, hh = h % G;
  const uint32_t* ch = chunk_hist + ((int64_t)(b * n_kv + g) * MAX_CHUNKS) * GMAX * HB + hh * HB;
  uint32_t s = 0;
  for (int j = 0; j < nchunks; ++j) s += ch[(int64_t)j * GMAX * HB + bin];
  out[((int64_t)b * n_q + h) * HB + bin] = s;
}

cudaError_t launch_head_hist(const pkv_index* ix, const ScanPlan& plan, uint32_t* head_hist_out,
                             cudaStream_t stream) {
  dim3 grid(ix->cfg.n_q_heads, ix->batch);
  ProfScope p_(K_HEADHIST, stream);
  head_hist_kernel<<<grid, HB, 0, stream>>>(ix->ws->chunk_hist, plan.nchunks, ix->cfg.n_q_heads,
                                            ix->cfg.n_kv_heads, ix->dcfg.G, head_hist_out);
  return cudaGetLastError();
}

cudaError_t set_phase_scan(unsigned long long* p) { return set_phase_ptr_tu(p); }

}  // namespace pkv
