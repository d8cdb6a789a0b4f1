// C ABI entry points: validation, index lifetime, and the stream-ordered orchestration of the kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "comm.h"
#include "internal.h"

namespace pkv {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string g_err;

pkv_status set_error(pkv_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

pkv_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PKV_OK;
  return set_error(PKV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

constexpr int SEL_STRIDE = 4 + 4 * MAX_CHUNKS;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

#define PKV_CUDA(expr, what)                                    \
  do {                                                          \
    cudaError_t e_ = (expr);                                    \
    if (e_ != cudaSuccess) return cuda_status(e_, what);        \
  } while (0)

pkv_status validate_config(const pkv_config* c) {
  if (!c) return set_error(PKV_ERR_INVALID_ARG, "null config");
  if (c->head_dim != PKV_HEAD_DIM || c->n_subspaces != PKV_SUBSPACES || c->subspace_dim != PKV_SUBSPACE_DIM)
    return set_error(PKV_ERR_UNSUPPORTED, "only D=128, B=16, m=8 are supported");
  if (c->rot_rounds != 1) return set_error(PKV_ERR_UNSUPPORTED, "only rot_rounds=1 is supported");
  if (c->n_q_heads <= 0 || c->n_kv_heads <= 0 || c->n_q_heads % c->n_kv_heads)
    return set_error(PKV_ERR_INVALID_ARG, "n_q_heads must be a positive multiple of n_kv_heads");
  if (c->n_q_heads / c->n_kv_heads > GMAX) return set_error(PKV_ERR_UNSUPPORTED, "GQA group size must be <= 4");
  if (c->n_tiers < 1 || c->n_tiers > PKV_MAX_TIERS) return set_error(PKV_ERR_INVALID_ARG, "n_tiers out of range");
  for (int i = 0; i < c->n_tiers; ++i) {
    if (c->tier_bonus[i] < 1) return set_error(PKV_ERR_INVALID_ARG, "tier bonuses must be >= 1");
    if (i && c->tier_bonus[i] >= c->tier_bonus[i - 1])
      return set_error(PKV_ERR_INVALID_ARG, "tier bonuses must be strictly decreasing");
  }
  if (c->tier_bonus[0] * PKV_SUBSPACES > HB - 1)
    return set_error(PKV_ERR_UNSUPPORTED, "max collision score must be <= 127 (tier_bonus[0] <= 7)");
  for (int i = 0; i < 8; ++i)
    if (!(c->mag_levels[i] > 0.f) || (i && !(c->mag_levels[i] > c->mag_levels[i - 1])) || !(c->mag_levels[i] < 1.f))
      return set_error(PKV_ERR_INVALID_ARG, "magnitude levels must be increasing in (0,1)");
  if (c->w_fp16 != 0 && c->w_fp16 != 1) return set_error(PKV_ERR_INVALID_ARG, "w_fp16 must be 0 or 1");
  return PKV_OK;
}

DevCfg make_devcfg(const pkv_config& c) {
  DevCfg d;
  std::memset(&d, 0, sizeof(d));
  d.n_q = c.n_q_heads;
  d.n_kv = c.n_kv_heads;
  d.G = c.n_q_heads / c.n_kv_heads;
  d.n_tiers = c.n_tiers;
  for (int i = 0; i < PKV_MAX_TIERS; ++i) d.tier_bonus[i] = c.tier_bonus[i];
  for (int i = 0; i < 8; ++i) d.levels[i] = c.mag_levels[i];
  for (int i = 0; i < 7; ++i) d.mid_sq[i] = c.mag_mid_sq[i];
  for (int j = 0; j < PKV_HEAD_DIM; ++j)
    if (c.rot_sign[j]) d.sign_mask[j >> 5] |= 1u << (j & 31);
  d.w16 = c.w_fp16;
  d.rec_bytes = c.w_fp16 ? 96 : REC;
  return d;
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

pkv_status alloc_workspace(Workspace* ws, int batch, int n_q, int n_kv, int64_t cap) {
  ws->batch = batch;
  ws->n_q = n_q;
  ws->n_kv = n_kv;
  ws->cap = cap;
  const size_t bq = (size_t)batch * n_q, bk = (size_t)batch * n_kv;
  size_t sizes[19] = {
      bk * NC * NB * 4,                                  // lut
      bq * D * 16 * 4,                                   // rtab
      bq * 4,                                            // qnorm
      bq * D * 4,                                        // qrot
      bk * (size_t)((cap + 3) & ~3LL) * 4 + 16,          // scores (rows 16-byte aligned for vector loads)
      bk * MAX_CHUNKS * GMAX * HB * 4,                   // chunk_hist
      (size_t)MAX_RANKS * bq * HB * 4,                   // head_hist
      bq * SEL_STRIDE * 4,                               // sel
      bq * (size_t)cap * 4,                              // cand
      bq * (size_t)cap * 4,                              // est
      (size_t)MAX_RANKS * bq * MAX_TOPK * 8,             // topk exchange: per rank [idx | est] (one all-gather)
      (size_t)std::max<size_t>(bk, 256) * 32 * GMAX * HB * 2,  // warp_hist (scan CTAs <= max(units, SMs))
      (size_t)MAX_RANKS * bq * MAX_SPLITS * PART * 4,    // part
      bk * 4,                                            // ticket
      (size_t)topk_segments(cap) * bq * MAX_TOPK * 4,    // seg_est
      (size_t)topk_segments(cap) * bq * MAX_TOPK * 4,    // seg_idx
      bk * 4,                                            // ucount
      bk * (size_t)cap * 4,                              // uid
      bk * (size_t)cap * 16};                            // upos
  size_t total = 0;
  for (size_t s : sizes) total += align_up(s);
  void* base = nullptr;
  cudaError_t e = cudaMalloc(&base, total);
  if (e != cudaSuccess) return cuda_status(e, "workspace cudaMalloc");
  char* p = static_cast<char*>(base);
  auto take = [&](int i) {
    char* r = p;
    p += align_up(sizes[i]);
    return r;
  };
  ws->lut = reinterpret_cast<uint32_t*>(take(0));
  ws->rtab = reinterpret_cast<float*>(take(1));
  ws->qnorm = reinterpret_cast<float*>(take(2));
  ws->qrot = reinterpret_cast<float*>(take(3));
  ws->scores = reinterpret_cast<uint32_t*>(take(4));
  ws->chunk_hist = reinterpret_cast<uint32_t*>(take(5));
  ws->head_hist = reinterpret_cast<uint32_t*>(take(6));
  ws->sel = reinterpret_cast<int32_t*>(take(7));
  ws->cand = reinterpret_cast<int32_t*>(take(8));
  ws->est = reinterpret_cast<float*>(take(9));
  ws->topk_idx = reinterpret_cast<int32_t*>(take(10));
  ws->topk_est = reinterpret_cast<float*>(ws->topk_idx + bq * MAX_TOPK);  // rank r: idx at 2r*slot, est after
  ws->warp_hist = reinterpret_cast<uint16_t*>(take(11));
  ws->warp_hist_ctas = (int64_t)std::max<size_t>(bk, 256);
  ws->part = reinterpret_cast<float*>(take(12));
  ws->ticket = reinterpret_cast<unsigned int*>(take(13));
  ws->seg_est = reinterpret_cast<float*>(take(14));
  ws->seg_idx = reinterpret_cast<int32_t*>(take(15));
  ws->seg_slots = topk_segments(cap);
  ws->ucount = reinterpret_cast<unsigned int*>(take(16));
  ws->uid = reinterpret_cast<int32_t*>(take(17));
  ws->upos = reinterpret_cast<int32_t*>(take(18));
  ws->base = base;
  ws->bytes = total;
  e = cudaMemset(base, 0, total);
  if (e != cudaSuccess) return cuda_status(e, "workspace memset");
  return PKV_OK;
}

void release_workspace(Workspace* ws) {
  if (!ws) return;
  if (--ws->refs == 0) {
    if (ws->base) cudaFree(ws->base);
    if (ws->ta_msg) cudaFree(ws->ta_msg);
    delete ws;
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Fused T+A exchange buffer, allocated on first use (an eager call precedes any graph capture).
pkv_status ensure_ta_msg(Workspace* ws) {
  if (ws->ta_msg) return PKV_OK;
  const size_t words = (size_t)MAX_RANKS * ws->batch * ws->n_q * ta_slot(TA_MAXK);
  cudaError_t e = cudaMalloc(&ws->ta_msg, words * 4);
  if (e != cudaSuccess) {
    ws->ta_msg = nullptr;
    return cuda_status(e, "exchange buffer cudaMalloc");
  }
  return PKV_OK;
}

pkv_status check_kv_layout(const void* K, int64_t sb, int64_t sh, int64_t st, const char* who) {
  if (!K) return set_error(PKV_ERR_INVALID_ARG, std::string(who) + ": null K/V pointer");
  if (!aligned16(K)) return set_error(PKV_ERR_INVALID_ARG, std::string(who) + ": K/V must be 16-byte aligned");
  if (sb < 0 || sh < 0 || st < 0 || (sb % 8) || (sh % 8) || (st % 8))
    return set_error(PKV_ERR_INVALID_ARG, std::string(who) + ": strides must be non-negative multiples of 8");
  return PKV_OK;
}

// -------------------------------------------------------------- retrieval phases (shared by all modes)
pkv_status phase_scan(pkv_index* ix, const void* q, const pkv_retrieve_params* p, ScanPlan& plan, cudaStream_t s) {
  const int64_t n = ix->n;
  PKV_CUDA(launch_qprep(ix, q, p->probes_T, p->rho_keys, p->dbg_q_rot, s), "qprep");
  plan = plan_scan(ix, n > 0 ? n : 1);
  if (n > 0 && ix->postings) {
    PKV_CUDA(launch_postings_scan(ix, n, score_stride(ix), s), "postings scan");
  } else if (n > 0) {
    PKV_CUDA(launch_scan(ix, n, plan, s), "scan");
  } else {
    PKV_CUDA(cudaMemsetAsync(ix->ws->chunk_hist, 0,
                             (size_t)ix->batch * ix->cfg.n_kv_heads * MAX_CHUNKS * GMAX * HB * 4, s),
             "hist clear");
  }
  if (p->dbg_scores && n > 0) PKV_CUDA(launch_dbg_scores(ix, n, p->dbg_scores, s), "dbg scores");
  return PKV_OK;
}

pkv_status phase_select_rerank(pkv_index* ix, const pkv_retrieve_params* p, const ScanPlan& plan,
                               const uint32_t* all_hist, int P, int rank, cudaStream_t s) {
  const int64_t n = ix->n;
  PKV_CUDA(launch_select(ix, n > 0 ? n : 0, plan, all_hist, P, rank, p->n_cand, ix->shard_offset, s), "select");
  if (n > 0) {
    const int64_t cmax = std::min<int64_t>(p->n_cand, n);
    if (cmax > 0) PKV_CUDA(launch_rerank(ix, cmax, ix->shard_offset, s), "rerank");
  }
  return PKV_OK;
}

// Key encoder. Default: the thread-per-key kernel (encode_fast.cu: exact int32 butterflies, fp32 decisions
// certified against the oracle's fp64 sequence) with the exact half-warp kernel (encode.cu) for the keys it hands
// back. PKV_ENCODER=half: the half-warp kernel alone (round 1's default); PKV_ENCODER=tc: the tensor-core kernel
// (encode_tc.cu, exact 8-bit-digit GEMMs) + the same fallback. fp16 weights always take the half-warp kernel.
// Read at every call (tests switch it).
static std::string encoder_kind() {
  const char* e = getenv("PKV_ENCODER");
  return e ? std::string(e) : std::string("fast");
}
bool use_tc_encoder() { return encoder_kind() == "tc"; }

pkv_status run_encoder(pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t0, int64_t count,
                       cudaStream_t stream) {
  if (count <= 0) return PKV_OK;
  const std::string kind = encoder_kind();
  if (kind == "half" || ix->dcfg.w16 || (kind != "tc" && kind != "fast") || (kind == "fast" && !ef_buckets_ok(ix->dcfg))) {
    PKV_CUDA(launch_encode(ix, K, sb, sh, st, t0, count, stream), "encode");
    return PKV_OK;
  }
  const int64_t units = (int64_t)ix->batch * ix->cfg.n_kv_heads;
  if (!ix->enc_fb) PKV_CUDA(cudaMalloc(&ix->enc_fb, (size_t)(units * ix->cap + 1) * 4), "encoder list");
  int32_t* fb_n = ix->enc_fb + units * ix->cap;
  PKV_CUDA(cudaMemsetAsync(fb_n, 0, 4, stream), "encoder list reset");
  if (kind == "tc")
    PKV_CUDA(launch_encode_tc(ix, K, sb, sh, st, t0, count, ix->enc_fb, fb_n, stream), "encode (tensor cores)");
  else
    PKV_CUDA(launch_encode_fast(ix, K, sb, sh, st, t0, count, ix->enc_fb, fb_n, stream), "encode (thread per key)");
  PKV_CUDA(launch_encode_list(ix, K, sb, sh, st, t0, count, ix->enc_fb, fb_n, stream), "encode (fallback)");
  return PKV_OK;
}

// Sequence-sharded retrieve_and_attend with the fused T+A exchange: H all-gather, local
// candidates and top-k, then ONE all-gather of (est, id, logit, v row) + hot partial per head, and a replicated
// merge + attention. Two collectives per layer instead of three.
pkv_status retrieve_and_attend_sharded(pkv_index* ix, const void* q, const pkv_retrieve_params* p, const void* K,
                                       const void* V, int64_t sb, int64_t sh, int64_t st, const void* K_hot,
                                       const void* V_hot, int32_t n_hot, float scale, int32_t* out_idx,
                                       float* out_est, void* out, float* lse, cudaStream_t stream) {
  if (!p) return set_error(PKV_ERR_INVALID_ARG, "retrieve_and_attend: null params");
  const int64_t n_global = comm_global_n(ix, p);
  if (n_global < 0) return set_error(PKV_ERR_INVALID_ARG, "retrieve_and_attend: global retrieval length unknown");
  pkv_status st0 = check_retrieve(ix, q, p, n_global, out_idx, out_est);
  if (st0 != PKV_OK) return st0;
  if (n_hot < 0 || (n_hot > 0 && (!K_hot || !V_hot || !aligned16(K_hot) || !aligned16(V_hot))))
    return set_error(PKV_ERR_INVALID_ARG, "retrieve_and_attend: bad hot rows");
  st0 = check_kv_layout(K, sb, sh, st, "retrieve_and_attend(K)");
  if (st0 == PKV_OK) st0 = check_kv_layout(V, sb, sh, st, "retrieve_and_attend(V)");
  if (st0 != PKV_OK) return st0;
  DeviceGuard g(ix->device);
  Workspace* ws = ix->ws;
  st0 = ensure_ta_msg(ws);
  if (st0 != PKV_OK) return st0;
  ScanPlan plan;
  st0 = phase_scan(ix, q, p, plan, stream);
  if (st0 != PKV_OK) return st0;
  const size_t hist_slot = (size_t)ix->batch * ix->cfg.n_q_heads * HB;
  PKV_CUDA(launch_head_hist(ix, plan, ws->head_hist + ix->rank * hist_slot, stream), "head hist");
  st0 = comm_allgather_u32(ix, ws->head_hist, hist_slot, stream);
  if (st0 != PKV_OK) return st0;
  st0 = phase_select_rerank(ix, p, plan, ws->head_hist, ix->world, ix->rank, stream);
  if (st0 != PKV_OK) return st0;
  PKV_CUDA(launch_topk(ix, p->n_cand, p->top_k, ws->topk_idx, ws->topk_est, MAX_TOPK, stream), "topk");
  const size_t rank_words = (size_t)ix->batch * ix->cfg.n_q_heads * ta_slot(p->top_k);
  const bool last = ix->rank == ix->world - 1;
  PKV_CUDA(launch_ta_pack(ix, ws->topk_idx, ws->topk_est, p->top_k, q, K, V, sb, sh, st, scale, ix->shard_offset,
                          K_hot, V_hot, last ? n_hot : 0, ws->ta_msg + ix->rank * rank_words, stream),
           "exchange pack");
  st0 = comm_allgather_u32(ix, ws->ta_msg, rank_words, stream);
  if (st0 != PKV_OK) return st0;
  PKV_CUDA(launch_ta_merge(ix, ws->ta_msg, ix->world, p->top_k, out_idx, out_est, out, lse, stream), "exchange merge");
  return PKV_OK;
}

}  // namespace

pkv_status check_retrieve(const pkv_index* ix, const void* q, const pkv_retrieve_params* p, int64_t n_global,
                          const int32_t* out_idx, const float* out_est) {
  if (!ix || !q || !p || !out_idx || !out_est) return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: null pointer");
  if (!aligned16(q)) return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: q must be 16-byte aligned");
  if (p->probes_T < 1 || p->probes_T > PKV_CENTROIDS)
    return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: probes_T out of [1,256]");
  if (p->top_k < 1 || p->top_k > MAX_TOPK) return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: top_k out of [1,1024]");
  if (n_global < 1) return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: empty retrieval zone");
  if (p->n_cand < std::min<int64_t>(p->top_k, n_global) || p->n_cand > n_global)
    return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: n_cand must be in [min(top_k, n), n]");
  if (p->rho_keys < 0 || p->rho_keys > n_global)
    return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: rho_keys must be in [0, n]");
  if (p->rho_keys > 0 && !ix->occ)
    return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: rho_keys needs pkv_index_set_occupancy(index, 1)");
  if (p->rho_keys > 0 && ix->world > 1)
    return set_error(PKV_ERR_UNSUPPORTED, "retrieve_topk: the key-fraction reading is not sequence-sharded");
  return PKV_OK;
}

pkv_status attend_hot_only(pkv_index* ix, const void* q, const void* K_hot, const void* V_hot, int n_hot,
                           int hot_rows, int top_k, float scale, int32_t* out_idx, float* out_est, void* out,
                           float* lse, cudaStream_t stream) {
  if (n_hot < 1 || hot_rows < n_hot || !K_hot || !V_hot || !aligned16(K_hot) || !aligned16(V_hot) || !aligned16(q))
    return set_error(PKV_ERR_INVALID_ARG, "attend_hot_only: bad hot rows");
  const int64_t bq = (int64_t)ix->batch * ix->cfg.n_q_heads;
  PKV_CUDA(launch_fill_empty_topk(out_idx, out_est, bq * top_k, stream), "fill");
  AttendArgs a{q, nullptr, nullptr, 0, 0, 0, nullptr, 0, K_hot, V_hot, n_hot, scale, 0, 0, 0, hot_rows};
  PKV_CUDA(launch_attend_partial(ix, a, plan_attend_splits(ix, n_hot), ix->ws->part, ix->ws->ticket, out, lse, stream),
           "attend");
  return PKV_OK;
}

}  // namespace pkv

using namespace pkv;

extern "C" {

const char* pkv_last_error(void) { return g_err.c_str(); }
const char* pkv_version(void) { return "pariskv-b200 0.1 (sm_100a)"; }

pkv_status pkv_launch_count(uint64_t* total) {
  if (!total) return set_error(PKV_ERR_INVALID_ARG, "null");
  *total = g_launches.load();
  return PKV_OK;
}

pkv_status pkv_index_create(const pkv_config* cfg, int32_t batch, int64_t capacity, int32_t device, pkv_index** out) {
  if (!out) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_create: null out");
  *out = nullptr;
  pkv_status st = validate_config(cfg);
  if (st != PKV_OK) return st;
  if (batch < 1 || capacity < 1 || capacity > (int64_t)INT32_MAX - 1)
    return set_error(PKV_ERR_INVALID_ARG, "pkv_index_create: batch >= 1 and 1 <= capacity < 2^31 required");
  int ndev = 0;
  PKV_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_create: bad device");
  DeviceGuard g(device);
  pkv_index* ix = new (std::nothrow) pkv_index();
  if (!ix) return set_error(PKV_ERR_CUDA, "host allocation failed");
  ix->cfg = *cfg;
  ix->dcfg = make_devcfg(*cfg);
  ix->device = device;
  ix->batch = batch;
  ix->cap = capacity;
  cudaDeviceGetAttribute(&ix->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&ix->smem_reserved, cudaDevAttrReservedSharedMemoryPerBlock, device);
  const size_t units = (size_t)batch * cfg->n_kv_heads;
  cudaError_t e = cudaMalloc(&ix->ids, units * capacity * NB);
  if (e == cudaSuccess) e = cudaMalloc(&ix->rec, units * capacity * ix->dcfg.rec_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&ix->stats, 4 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(ix->stats, 0, 4 * sizeof(unsigned long long));
  // the encoders' hand-back list (4 B per key + count): allocated here, not inside a (timed, capturable) encode
  if (e == cudaSuccess) e = cudaMalloc(&ix->enc_fb, (units * capacity + 1) * 4);
  if (e != cudaSuccess) {
    cudaFree(ix->enc_fb);
    cudaFree(ix->stats);
    cudaFree(ix->rec);
    cudaFree(ix->ids);
    delete ix;
    return cuda_status(e, "index cudaMalloc");
  }
  ix->ws = new Workspace();
  ix->ws->device = device;
  st = alloc_workspace(ix->ws, batch, cfg->n_q_heads, cfg->n_kv_heads, capacity);
  if (st == PKV_OK) {
    e = init_scan_attrs();
    if (e == cudaSuccess) e = init_rerank_attrs();
    if (e == cudaSuccess) e = init_postings_attrs();
    if (e == cudaSuccess) e = init_encode_tc_attrs();
    if (e != cudaSuccess) st = cuda_status(e, "cudaFuncSetAttribute");
  }
  if (st != PKV_OK) {
    release_workspace(ix->ws);
    cudaFree(ix->ids);
    cudaFree(ix->rec);
    cudaFree(ix->stats);
    delete ix;
    return st;
  }
  *out = ix;
  return PKV_OK;
}

pkv_status pkv_index_destroy(pkv_index* ix) {
  if (!ix) return PKV_OK;
  DeviceGuard g(ix->device);
  comm_destroy(ix->comm);
  release_workspace(ix->ws);
  cudaFree(ix->ids);
  cudaFree(ix->rec);
  cudaFree(ix->occ);
  cudaFree(ix->post_off);
  cudaFree(ix->post_key);
  cudaFree(ix->enc_fb);
  cudaFree(ix->stats);
  delete ix;
  return PKV_OK;
}

pkv_status pkv_index_get_stats(const pkv_index* ix, pkv_index_stats* out, cudaStream_t stream) {
  if (!ix || !out) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_get_stats: null pointer");
  DeviceGuard g(ix->device);
  unsigned long long h[4] = {0, 0, 0, 0};
  PKV_CUDA(cudaMemcpyAsync(h, ix->stats, sizeof(h), cudaMemcpyDeviceToHost, stream), "stats copy");
  PKV_CUDA(cudaStreamSynchronize(stream), "stats sync");
  out->n_keys = ix->n;
  out->zero_keys = (int64_t)h[0];
  out->keys_with_zero_subspace = (int64_t)h[1];
  out->zero_subspaces = (int64_t)h[2];
  return PKV_OK;
}

pkv_status pkv_index_set_debug_output(pkv_index* ix, float* out_f32) {
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_set_debug_output: null index");
  ix->dbg_out_f32 = out_f32;
  return PKV_OK;
}

pkv_status pkv_index_set_postings(pkv_index* ix, int32_t enable, cudaStream_t stream) {
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_set_postings: null index");
  DeviceGuard g(ix->device);
  if (!enable) {
    ix->postings = false;
    return PKV_OK;
  }
  if (!ix->post_off) {
    const int64_t units = (int64_t)ix->batch * ix->cfg.n_kv_heads;
    const int64_t nch = (ix->cap + POST_CHUNK - 1) / POST_CHUNK;
    if (nch > MAX_CHUNKS) return set_error(PKV_ERR_UNSUPPORTED, "pkv_index_set_postings: capacity > 256 chunks of 8192");
    cudaError_t e = cudaMalloc(&ix->post_off, (size_t)units * nch * NB * (NC + 1) * 2);
    if (e == cudaSuccess) e = cudaMalloc(&ix->post_key, (size_t)units * nch * NB * POST_CHUNK * 2);
    if (e != cudaSuccess) {
      cudaFree(ix->post_off);
      cudaFree(ix->post_key);
      ix->post_off = nullptr;
      ix->post_key = nullptr;
      return cuda_status(e, "pkv_index_set_postings");
    }
  }
  ix->postings = true;
  PKV_CUDA(launch_postings_build(ix, 0, (ix->n + POST_CHUNK - 1) / POST_CHUNK, stream), "postings");
  return PKV_OK;
}

pkv_status pkv_index_set_occupancy(pkv_index* ix, int32_t enable, cudaStream_t stream) {
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_set_occupancy: null index");
  DeviceGuard g(ix->device);
  if (!enable) {
    cudaFree(ix->occ);
    ix->occ = nullptr;
    return PKV_OK;
  }
  const size_t bytes = (size_t)ix->batch * ix->cfg.n_kv_heads * NB * NC * 4;
  if (!ix->occ) {
    cudaError_t e = cudaMalloc(&ix->occ, bytes);
    if (e != cudaSuccess) {
      ix->occ = nullptr;
      return cuda_status(e, "pkv_index_set_occupancy");
    }
  }
  PKV_CUDA(cudaMemsetAsync(ix->occ, 0, bytes, stream), "occupancy clear");
  PKV_CUDA(launch_occupancy(ix, 0, ix->n, stream), "occupancy");
  return PKV_OK;
}

pkv_status pkv_index_len(const pkv_index* ix, int64_t* n_out) {
  if (!ix || !n_out) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_len: null pointer");
  *n_out = ix->n;
  return PKV_OK;
}

pkv_status pkv_index_share_workspace(pkv_index* ix, pkv_index* donor) {
  if (!ix || !donor) return set_error(PKV_ERR_INVALID_ARG, "share_workspace: null");
  if (ix == donor || ix->ws == donor->ws) return PKV_OK;
  if (ix->device != donor->device || ix->batch != donor->batch || ix->cfg.n_q_heads != donor->cfg.n_q_heads ||
      ix->cfg.n_kv_heads != donor->cfg.n_kv_heads || donor->ws->cap < ix->cap)
    return set_error(PKV_ERR_INVALID_ARG, "share_workspace: incompatible donor");
  DeviceGuard g(ix->device);
  release_workspace(ix->ws);
  ix->ws = donor->ws;
  ix->ws->refs++;
  return PKV_OK;
}

pkv_status encode_keys(pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t n,
                       cudaStream_t stream) {
  NvtxRange nvtx_("pkv:encode_keys");
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "encode_keys: null index");
  if (n < 0) return set_error(PKV_ERR_INVALID_ARG, "encode_keys: n < 0");
  if (n > ix->cap) return set_error(PKV_ERR_CAPACITY, "encode_keys: n exceeds capacity");
  if (n > 0) {
    pkv_status s = check_kv_layout(K, sb, sh, st, "encode_keys");
    if (s != PKV_OK) return s;
  }
  DeviceGuard g(ix->device);
  PKV_CUDA(cudaMemsetAsync(ix->stats, 0, 4 * sizeof(unsigned long long), stream), "stats reset");
  if (n > 0) {
    pkv_status se = run_encoder(ix, K, sb, sh, st, 0, n, stream);
    if (se != PKV_OK) return se;
  }
  ix->n = n;
  if (ix->postings) PKV_CUDA(launch_postings_build(ix, 0, (n + POST_CHUNK - 1) / POST_CHUNK, stream), "postings");
  if (ix->occ) {
    PKV_CUDA(cudaMemsetAsync(ix->occ, 0, (size_t)ix->batch * ix->cfg.n_kv_heads * NB * NC * 4, stream),
             "occupancy clear");
    PKV_CUDA(launch_occupancy(ix, 0, n, stream), "occupancy");
  }
  return PKV_OK;
}

pkv_status append_decode_keys(pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t,
                              cudaStream_t stream) {
  NvtxRange nvtx_("pkv:append_decode_keys");
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "append_decode_keys: null index");
  if (t < 0) return set_error(PKV_ERR_INVALID_ARG, "append_decode_keys: t < 0");
  if (ix->n + t > ix->cap) return set_error(PKV_ERR_CAPACITY, "append_decode_keys: capacity exceeded");
  if (t > 0) {
    pkv_status s = check_kv_layout(K, sb, sh, st, "append_decode_keys");
    if (s != PKV_OK) return s;
  }
  DeviceGuard g(ix->device);
  if (t > 0) {
    pkv_status se = run_encoder(ix, K, sb, sh, st, ix->n, t, stream);
    if (se != PKV_OK) return se;
  }
  const int64_t first = ix->n / POST_CHUNK;  // the partial chunk and the new ones are rebuilt
  if (ix->occ && t > 0) PKV_CUDA(launch_occupancy(ix, ix->n, ix->n + t, stream), "occupancy(append)");
  ix->n += t;
  if (ix->postings && t > 0)
    PKV_CUDA(launch_postings_build(ix, first, (ix->n + POST_CHUNK - 1) / POST_CHUNK, stream), "postings(append)");
  return PKV_OK;
}

pkv_status pkv_index_export(const pkv_index* ix, int64_t start, int64_t count, uint8_t* ids, uint8_t* codes, float* w,
                            cudaStream_t stream) {
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "export: null index");
  if (start < 0 || count < 0 || start + count > ix->n)
    return set_error(PKV_ERR_INVALID_ARG, "export: range outside [0, n)");
  DeviceGuard g(ix->device);
  PKV_CUDA(launch_export(ix, start, count, ids, codes, w, stream), "export");
  return PKV_OK;
}

pkv_status retrieve_topk(pkv_index* ix, const void* q, const pkv_retrieve_params* p, int32_t* out_idx, float* out_est,
                         cudaStream_t stream) {
  NvtxRange nvtx_("pkv:retrieve_topk");
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: null index");
  if (!p) return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: null params");
  const int64_t n_global = ix->comm ? comm_global_n(ix, p) : ix->n;
  if (n_global < 0) return set_error(PKV_ERR_INVALID_ARG, "retrieve_topk: global retrieval length unknown");
  pkv_status st = check_retrieve(ix, q, p, n_global, out_idx, out_est);
  if (st != PKV_OK) return st;
  DeviceGuard g(ix->device);
  ScanPlan plan;
  st = phase_scan(ix, q, p, plan, stream);
  if (st != PKV_OK) return st;
  Workspace* ws = ix->ws;
  const size_t hist_slot = (size_t)ix->batch * ix->cfg.n_q_heads * HB;
  const size_t topk_slot = (size_t)ix->batch * ix->cfg.n_q_heads * MAX_TOPK;
  if (ix->comm) {
    PKV_CUDA(launch_head_hist(ix, plan, ws->head_hist + ix->rank * hist_slot, stream), "head hist");
    st = comm_allgather_u32(ix, ws->head_hist, hist_slot, stream);
    if (st != PKV_OK) return st;
    st = phase_select_rerank(ix, p, plan, ws->head_hist, ix->world, ix->rank, stream);
    if (st != PKV_OK) return st;
    // (T) local top-k lists, ids and estimates of a rank adjacent: one all-gather of 2*slot words per rank
    PKV_CUDA(launch_topk(ix, p->n_cand, p->top_k, ws->topk_idx + ix->rank * 2 * topk_slot,
                         ws->topk_est + ix->rank * 2 * topk_slot, MAX_TOPK, stream),
             "topk");
    st = comm_allgather_u32(ix, reinterpret_cast<uint32_t*>(ws->topk_idx), 2 * topk_slot, stream);
    if (st != PKV_OK) return st;
    PKV_CUDA(launch_topk_merge(ix, ix->world, p->top_k, ws->topk_est, ws->topk_idx, 2 * topk_slot, out_idx, out_est,
                               stream),
             "topk merge");
  } else {
    st = phase_select_rerank(ix, p, plan, nullptr, 1, 0, stream);
    if (st != PKV_OK) return st;
    PKV_CUDA(launch_topk(ix, p->n_cand, p->top_k, out_idx, out_est, p->top_k, stream), "topk");
  }
  if (p->dbg_cand || p->dbg_est) PKV_CUDA(launch_dbg_cand(ix, p->n_cand, p->dbg_cand, p->dbg_est, stream), "dbg cand");
  return PKV_OK;
}

pkv_status sparse_attend(pkv_index* ix, const void* q, const void* K, const void* V, int64_t sb, int64_t sh, int64_t st,
                         const int32_t* idx, int32_t k, const void* K_hot, const void* V_hot, int32_t n_hot,
                         float scale, void* out, float* lse, cudaStream_t stream) {
  NvtxRange nvtx_("pkv:sparse_attend");
  if (!ix || !q || !out) return set_error(PKV_ERR_INVALID_ARG, "sparse_attend: null pointer");
  if (k < 0 || n_hot < 0 || k > MAX_TOPK) return set_error(PKV_ERR_INVALID_ARG, "sparse_attend: bad k / n_hot");
  if (k > 0) {
    if (!idx) return set_error(PKV_ERR_INVALID_ARG, "sparse_attend: null idx");
    pkv_status s1 = check_kv_layout(K, sb, sh, st, "sparse_attend(K)");
    if (s1 != PKV_OK) return s1;
    s1 = check_kv_layout(V, sb, sh, st, "sparse_attend(V)");
    if (s1 != PKV_OK) return s1;
  }
  if (n_hot > 0 && (!K_hot || !V_hot || !aligned16(K_hot) || !aligned16(V_hot)))
    return set_error(PKV_ERR_INVALID_ARG, "sparse_attend: bad hot rows");
  if (k == 0 && n_hot == 0) return set_error(PKV_ERR_INVALID_ARG, "sparse_attend: empty attention set");
  if (!aligned16(q)) return set_error(PKV_ERR_INVALID_ARG, "sparse_attend: q must be 16-byte aligned");
  DeviceGuard g(ix->device);
  const int G = ix->dcfg.G;
  const int splits = plan_attend_splits(ix, n_hot + G * k);
  const bool last = !ix->comm || ix->rank == ix->world - 1;
  AttendArgs a{q, K, V, sb, sh, st, idx, k, K_hot, V_hot, last ? n_hot : 0, scale,
               ix->comm ? ix->shard_offset : 0, ix->comm ? ix->shard_offset + ix->n : INT64_MAX,
               ix->comm ? ix->shard_offset : 0, n_hot};
  Workspace* ws = ix->ws;
  const size_t part_slot = (size_t)ix->batch * ix->cfg.n_q_heads * MAX_SPLITS * PART;
  const int slot = ix->comm ? ix->rank : 0;
  if (!ix->comm) {
    PKV_CUDA(launch_attend_partial(ix, a, splits, ws->part, ws->ticket, out, lse, stream), "attend");
    return PKV_OK;
  }
  PKV_CUDA(launch_attend_partial(ix, a, splits, ws->part + slot * part_slot, nullptr, nullptr, nullptr, stream),
           "attend");
  pkv_status s2 = comm_allgather_u32(ix, reinterpret_cast<uint32_t*>(ws->part), part_slot, stream);
  if (s2 != PKV_OK) return s2;
  PKV_CUDA(launch_attend_combine(ix, ws->part, splits, ix->world, out, lse, stream), "combine");
  return PKV_OK;
}

pkv_status retrieve_and_attend(pkv_index* ix, const void* q, const pkv_retrieve_params* p, const void* K, const void* V,
                               int64_t sb, int64_t sh, int64_t st, const void* K_hot, const void* V_hot, int32_t n_hot,
                               float scale, int32_t* out_idx, float* out_est, void* out, float* lse,
                               cudaStream_t stream) {
  return retrieve_and_attend_rows(ix, q, p, K, V, sb, sh, st, K_hot, V_hot, n_hot, n_hot, scale, out_idx, out_est, out,
                                  lse, stream);
}

pkv_status retrieve_and_attend_rows(pkv_index* ix, const void* q, const pkv_retrieve_params* p, const void* K,
                                    const void* V, int64_t sb, int64_t sh, int64_t st, const void* K_hot,
                                    const void* V_hot, int32_t n_hot, int32_t hot_rows, float scale, int32_t* out_idx,
                                    float* out_est, void* out, float* lse, cudaStream_t stream) {
  return pkv::retrieve_and_attend_rows_after(ix, q, p, K, V, sb, sh, st, K_hot, V_hot, n_hot, hot_rows, scale,
                                             out_idx, out_est, out, lse, nullptr, stream);
}

}  // extern "C"

namespace pkv {

// retrieve_and_attend_rows whose row gather (the last kernel) also waits for `attend_after` (may be null): the
// streaming manager's asynchronous offload of evicted K/V rows must land in the store before those rows can be
// gathered, while query prep, scan, select and rerank of the same step run alongside it.
pkv_status retrieve_and_attend_rows_after(pkv_index* ix, const void* q, const pkv_retrieve_params* p, const void* K,
                                          const void* V, int64_t sb, int64_t sh, int64_t st, const void* K_hot,
                                          const void* V_hot, int32_t n_hot, int32_t hot_rows, float scale,
                                          int32_t* out_idx, float* out_est, void* out, float* lse,
                                          cudaEvent_t attend_after, cudaStream_t stream) {
  NvtxRange nvtx_("pkv:retrieve_and_attend");
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "retrieve_and_attend: null index");
  if (attend_after && ix->comm) return set_error(PKV_ERR_UNSUPPORTED, "retrieve_and_attend: ordered gather when sharded");
  if (ix->comm) {  // sequence-sharded: one fused T+A exchange when k fits its slots, else the two calls
    if (hot_rows != n_hot) return set_error(PKV_ERR_UNSUPPORTED, "retrieve_and_attend: strided hot rows when sharded");
    if (p && p->top_k <= TA_MAXK && out)
      return retrieve_and_attend_sharded(ix, q, p, K, V, sb, sh, st, K_hot, V_hot, n_hot, scale, out_idx, out_est, out,
                                         lse, stream);
    pkv_status st1 = retrieve_topk(ix, q, p, out_idx, out_est, stream);
    if (st1 != PKV_OK) return st1;
    return sparse_attend(ix, q, K, V, sb, sh, st, out_idx, p->top_k, K_hot, V_hot, n_hot, scale, out, lse, stream);
  }
  pkv_status st0 = check_retrieve(ix, q, p, ix->n, out_idx, out_est);
  if (st0 != PKV_OK) return st0;
  if (!out) return set_error(PKV_ERR_INVALID_ARG, "retrieve_and_attend: null out");
  st0 = check_kv_layout(K, sb, sh, st, "retrieve_and_attend(K)");
  if (st0 == PKV_OK) st0 = check_kv_layout(V, sb, sh, st, "retrieve_and_attend(V)");
  if (st0 != PKV_OK) return st0;
  if (n_hot < 0 || (n_hot > 0 && (!K_hot || !V_hot || !aligned16(K_hot) || !aligned16(V_hot))))
    return set_error(PKV_ERR_INVALID_ARG, "retrieve_and_attend: bad hot rows");
  if (n_hot > 0 && hot_rows < n_hot)
    return set_error(PKV_ERR_INVALID_ARG, "retrieve_and_attend_rows: hot_rows must be >= n_hot");
  if (n_hot > 16 * 64) return set_error(PKV_ERR_UNSUPPORTED, "retrieve_and_attend: n_hot must be <= 1024");
  DeviceGuard g(ix->device);
  ScanPlan plan;
  const int64_t C_cap = std::min<int64_t>(p->n_cand, ix->n);
  const bool clustered = topk_segments(C_cap) == 1;
  st0 = phase_scan(ix, q, p, plan, stream);
  if (st0 != PKV_OK) return st0;
  st0 = phase_select_rerank(ix, p, plan, nullptr, 1, 0, stream);
  if (st0 != PKV_OK) return st0;
  // The hot rows (sink + local + buffer) are attended by the last kernel: in the cluster top-k kernel ahead of
  // its dependency wait (overlapping the rerank kernel's drain); after the segmented top-k for very long lists.
  if (attend_after) PKV_CUDA(cudaStreamWaitEvent(stream, attend_after, 0), "wait for the offload");
  if (!clustered) {
    PKV_CUDA(launch_topk(ix, p->n_cand, p->top_k, out_idx, out_est, p->top_k, stream), "topk");
    PKV_CUDA(launch_topk_attend_rows(ix, p->top_k, out_idx, q, K, V, sb, sh, st, scale, K_hot, V_hot, n_hot, hot_rows,
                                     out, lse, stream),
             "attend rows");
  } else {
    PKV_CUDA(launch_topk_attend(ix, C_cap, p->top_k, out_idx, out_est, q, K, V, sb, sh, st, scale, K_hot, V_hot, n_hot,
                                hot_rows, out, lse, stream),
             "topk+attend");
  }
  if (p->dbg_cand || p->dbg_est) PKV_CUDA(launch_dbg_cand(ix, p->n_cand, p->dbg_cand, p->dbg_est, stream), "dbg cand");
  return PKV_OK;
}

}  // namespace pkv

extern "C" {

// ---------------------------------------------------------------- single-process sharded emulation
namespace {
// The emulation sets each shard's offset for the duration of one call; restored on every return path so a
// later unsharded call on the same index returns local ids again.
struct OffsetScope {
  pkv_index* const* shards;
  int P;
  int64_t saved[MAX_RANKS];
  OffsetScope(pkv_index* const* s, const int64_t* offsets, int p) : shards(s), P(p) {
    for (int r = 0; r < P; ++r) {
      saved[r] = shards[r]->shard_offset;
      shards[r]->shard_offset = offsets[r];
    }
  }
  ~OffsetScope() {
    for (int r = 0; r < P; ++r) shards[r]->shard_offset = saved[r];
  }
};
}  // namespace

pkv_status pkv_retrieve_topk_sharded_local(pkv_index* const* shards, const int64_t* offsets, int32_t P, const void* q,
                                           const pkv_retrieve_params* p, int32_t* out_idx, float* out_est,
                                           cudaStream_t stream) {
  if (!shards || !offsets || P < 1 || P > MAX_RANKS)
    return set_error(PKV_ERR_INVALID_ARG, "sharded_local: need 1 <= P <= 8 shards");
  int64_t n_global = 0;
  for (int r = 0; r < P; ++r) {
    if (!shards[r] || shards[r]->device != shards[0]->device || shards[r]->batch != shards[0]->batch ||
        shards[r]->comm || (r && shards[r]->ws == shards[0]->ws))
      return set_error(PKV_ERR_INVALID_ARG, "sharded_local: shards must be distinct, same device/batch, own workspace");
    if (offsets[r] != n_global) return set_error(PKV_ERR_INVALID_ARG, "sharded_local: offsets must be contiguous");
    n_global += shards[r]->n;
  }
  pkv_status st = check_retrieve(shards[0], q, p, n_global, out_idx, out_est);
  if (st != PKV_OK) return st;
  DeviceGuard g(shards[0]->device);
  Workspace* w0 = shards[0]->ws;
  const size_t hist_slot = (size_t)shards[0]->batch * shards[0]->cfg.n_q_heads * HB;
  const size_t topk_slot = (size_t)shards[0]->batch * shards[0]->cfg.n_q_heads * MAX_TOPK;
  ScanPlan plans[MAX_RANKS];
  OffsetScope scope(shards, offsets, P);
  for (int r = 0; r < P; ++r) {
    pkv_retrieve_params pr = *p;
    pr.dbg_scores = nullptr;
    pr.dbg_cand = nullptr;
    pr.dbg_est = nullptr;
    if (r) pr.dbg_q_rot = nullptr;
    st = phase_scan(shards[r], q, &pr, plans[r], stream);
    if (st != PKV_OK) return st;
    PKV_CUDA(launch_head_hist(shards[r], plans[r], w0->head_hist + r * hist_slot, stream), "head hist");
  }
  for (int r = 0; r < P; ++r) {
    st = phase_select_rerank(shards[r], p, plans[r], w0->head_hist, P, r, stream);
    if (st != PKV_OK) return st;
    PKV_CUDA(launch_topk(shards[r], p->n_cand, p->top_k, w0->topk_idx + r * 2 * topk_slot,
                         w0->topk_est + r * 2 * topk_slot, MAX_TOPK, stream),
             "topk");
  }
  PKV_CUDA(launch_topk_merge(shards[0], P, p->top_k, w0->topk_est, w0->topk_idx, 2 * topk_slot, out_idx, out_est,
                             stream),
           "merge");
  return PKV_OK;
}

pkv_status pkv_sparse_attend_sharded_local(pkv_index* const* shards, const int64_t* offsets, int32_t P, const void* q,
                                           const void* const* Ks, const void* const* Vs, int64_t sb, int64_t sh,
                                           int64_t st, const int32_t* idx, int32_t k, const void* K_hot,
                                           const void* V_hot, int32_t n_hot, float scale, void* out, float* lse,
                                           cudaStream_t stream) {
  if (!shards || !offsets || !Ks || !Vs || P < 1 || P > MAX_RANKS || !q || !out)
    return set_error(PKV_ERR_INVALID_ARG, "attend_sharded_local: bad arguments");
  if (k < 0 || n_hot < 0 || k > MAX_TOPK || (k == 0 && n_hot == 0))
    return set_error(PKV_ERR_INVALID_ARG, "attend_sharded_local: bad k / n_hot");
  if (n_hot > 0 && (!K_hot || !V_hot || !aligned16(K_hot) || !aligned16(V_hot)))
    return set_error(PKV_ERR_INVALID_ARG, "attend_sharded_local: bad hot rows");
  if (k > 0 && !idx) return set_error(PKV_ERR_INVALID_ARG, "attend_sharded_local: null idx");
  if (!aligned16(q)) return set_error(PKV_ERR_INVALID_ARG, "attend_sharded_local: q must be 16-byte aligned");
  for (int r = 1; r < P; ++r)
    if (!shards[r] || shards[r]->ws == shards[0]->ws || shards[r]->device != shards[0]->device)
      return set_error(PKV_ERR_INVALID_ARG, "attend_sharded_local: shards need their own workspace");
  DeviceGuard g(shards[0]->device);
  const int G = shards[0]->dcfg.G;
  const int splits = plan_attend_splits(shards[0], n_hot + G * k);
  Workspace* w0 = shards[0]->ws;
  const size_t part_slot = (size_t)shards[0]->batch * shards[0]->cfg.n_q_heads * MAX_SPLITS * PART;
  for (int r = 0; r < P; ++r) {
    if (k > 0) {
      pkv_status s1 = check_kv_layout(Ks[r], sb, sh, st, "attend_sharded_local(K)");
      if (s1 == PKV_OK) s1 = check_kv_layout(Vs[r], sb, sh, st, "attend_sharded_local(V)");
      if (s1 != PKV_OK) return s1;
    }
    AttendArgs a{q, Ks[r], Vs[r], sb, sh, st, idx, k, K_hot, V_hot, r == P - 1 ? n_hot : 0, scale, offsets[r],
                 offsets[r] + shards[r]->n, offsets[r], n_hot};
    PKV_CUDA(launch_attend_partial(shards[r], a, splits, w0->part + r * part_slot, nullptr, nullptr, nullptr, stream),
             "attend");
  }
  PKV_CUDA(launch_attend_combine(shards[0], w0->part, splits, P, out, lse, stream), "combine");
  return PKV_OK;
}

pkv_status pkv_retrieve_and_attend_sharded_local(pkv_index* const* shards, const int64_t* offsets, int32_t P,
                                                const void* q, const void* const* Ks, const void* const* Vs,
                                                int64_t sb, int64_t sh, int64_t st, const pkv_retrieve_params* p,
                                                const void* K_hot, const void* V_hot, int32_t n_hot, float scale,
                                                int32_t* out_idx, float* out_est, void* out, float* lse,
                                                cudaStream_t stream) {
  if (!shards || !offsets || !Ks || !Vs || P < 1 || P > MAX_RANKS || !q || !p || !out)
    return set_error(PKV_ERR_INVALID_ARG, "retrieve_and_attend_sharded_local: bad arguments");
  if (p->top_k > TA_MAXK) return set_error(PKV_ERR_UNSUPPORTED, "retrieve_and_attend_sharded_local: top_k > 256");
  if (n_hot < 0 || (n_hot > 0 && (!K_hot || !V_hot || !aligned16(K_hot) || !aligned16(V_hot))))
    return set_error(PKV_ERR_INVALID_ARG, "retrieve_and_attend_sharded_local: bad hot rows");
  int64_t n_global = 0;
  for (int r = 0; r < P; ++r) {
    if (!shards[r] || shards[r]->device != shards[0]->device || shards[r]->batch != shards[0]->batch ||
        shards[r]->comm || (r && shards[r]->ws == shards[0]->ws))
      return set_error(PKV_ERR_INVALID_ARG, "sharded_local: shards must be distinct, same device/batch, own workspace");
    if (offsets[r] != n_global) return set_error(PKV_ERR_INVALID_ARG, "sharded_local: offsets must be contiguous");
    pkv_status s1 = check_kv_layout(Ks[r], sb, sh, st, "sharded_local(K)");
    if (s1 == PKV_OK) s1 = check_kv_layout(Vs[r], sb, sh, st, "sharded_local(V)");
    if (s1 != PKV_OK) return s1;
    n_global += shards[r]->n;
  }
  pkv_status st0 = check_retrieve(shards[0], q, p, n_global, out_idx, out_est);
  if (st0 != PKV_OK) return st0;
  DeviceGuard g(shards[0]->device);
  Workspace* w0 = shards[0]->ws;
  st0 = ensure_ta_msg(w0);
  if (st0 != PKV_OK) return st0;
  const size_t hist_slot = (size_t)shards[0]->batch * shards[0]->cfg.n_q_heads * HB;
  const size_t rank_words = (size_t)shards[0]->batch * shards[0]->cfg.n_q_heads * ta_slot(p->top_k);
  ScanPlan plans[MAX_RANKS];
  pkv_retrieve_params pr = *p;
  pr.dbg_scores = nullptr;
  pr.dbg_cand = nullptr;
  pr.dbg_est = nullptr;
  pr.dbg_q_rot = nullptr;
  OffsetScope scope(shards, offsets, P);
  for (int r = 0; r < P; ++r) {
    st0 = phase_scan(shards[r], q, &pr, plans[r], stream);
    if (st0 != PKV_OK) return st0;
    PKV_CUDA(launch_head_hist(shards[r], plans[r], w0->head_hist + r * hist_slot, stream), "head hist");
  }
  for (int r = 0; r < P; ++r) {  // each shard's local top-k in its own workspace, packed into slot r
    st0 = phase_select_rerank(shards[r], &pr, plans[r], w0->head_hist, P, r, stream);
    if (st0 != PKV_OK) return st0;
    Workspace* wr = shards[r]->ws;
    PKV_CUDA(launch_topk(shards[r], pr.n_cand, pr.top_k, wr->topk_idx, wr->topk_est, MAX_TOPK, stream), "topk");
    PKV_CUDA(launch_ta_pack(shards[r], wr->topk_idx, wr->topk_est, pr.top_k, q, Ks[r], Vs[r], sb, sh, st, scale,
                            offsets[r], K_hot, V_hot, r == P - 1 ? n_hot : 0, w0->ta_msg + r * rank_words, stream),
             "exchange pack");
  }
  PKV_CUDA(launch_ta_merge(shards[0], w0->ta_msg, P, pr.top_k, out_idx, out_est, out, lse, stream), "exchange merge");
  return PKV_OK;
}

pkv_status pkv_nccl_unique_id(uint8_t out[128]) { return comm_unique_id(out); }

pkv_status pkv_comm_init(pkv_index* ix, const uint8_t id[128], int32_t rank, int32_t world, int64_t shard_offset) {
  if (!ix || !id || world < 1 || world > MAX_RANKS || rank < 0 || rank >= world || shard_offset < 0)
    return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_init: bad arguments (world must be in [1, 8])");
  DeviceGuard g(ix->device);
  return comm_init(ix, id, rank, world, shard_offset);
}

pkv_status pkv_comm_init_peer(pkv_index* ix, int32_t rank, int32_t world, int64_t shard_offset, size_t arena_bytes,
                              uint8_t ipc_handle[64], void** arena) {
  if (!ix || world < 1 || world > MAX_RANKS || rank < 0 || rank >= world || shard_offset < 0)
    return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_init_peer: bad arguments (world must be in [1, 8])");
  DeviceGuard g(ix->device);
  return comm_init_peer(ix, rank, world, shard_offset, arena_bytes, ipc_handle, arena);
}

pkv_status pkv_comm_peer_connect(pkv_index* ix, const uint8_t* ipc_handles) {
  if (!ix || !ipc_handles) return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_peer_connect: null pointer");
  DeviceGuard g(ix->device);
  return comm_peer_connect(ix, ipc_handles, nullptr);
}

pkv_status pkv_comm_peer_connect_local(pkv_index* ix, void* const* arenas) {
  if (!ix || !arenas) return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_peer_connect_local: null pointer");
  DeviceGuard g(ix->device);
  return comm_peer_connect(ix, nullptr, arenas);
}

pkv_status pkv_comm_init_host(pkv_index* ix, pkv_host_allgather_fn fn, void* ctx, int32_t rank, int32_t world,
                              int64_t shard_offset) {
  if (!ix || !fn || world < 1 || world > MAX_RANKS || rank < 0 || rank >= world || shard_offset < 0)
    return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_init_host: bad arguments (world must be in [1, 8])");
  DeviceGuard g(ix->device);
  return comm_init_host(ix, fn, ctx, rank, world, shard_offset);
}

pkv_status pkv_comm_set_global_len(pkv_index* ix, int64_t n_global) {
  if (!ix || n_global < 0) return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_set_global_len: bad arguments");
  return comm_set_global_len(ix, n_global);
}

pkv_status pkv_comm_share(pkv_index* ix, pkv_index* donor, int64_t shard_offset) {
  if (!ix || !donor || shard_offset < 0) return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_share: bad arguments");
  if (ix->device != donor->device) return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_share: different devices");
  return comm_share(ix, donor, shard_offset);
}


// ------------------------------------------------------------------ append rebalancing
pkv_status pkv_index_entry_bytes(const pkv_index* ix, int64_t* bytes_per_key) {
  if (!ix || !bytes_per_key) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_entry_bytes: null pointer");
  *bytes_per_key = (int64_t)ix->batch * ix->cfg.n_kv_heads * (NB + ix->dcfg.rec_bytes);
  return PKV_OK;
}

pkv_status pkv_index_export_front(const pkv_index* ix, int64_t count, void* buf, cudaStream_t stream) {
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_export_front: null index");
  if (count < 0 || count > ix->n) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_export_front: count outside [0, n]");
  if (count > 0 && !buf) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_export_front: null buffer");
  DeviceGuard g(ix->device);
  PKV_CUDA(launch_export_entries(ix, 0, count, buf, stream), "export front");
  return PKV_OK;
}

// postings and occupancy of an index whose contents changed in [t0, n): rebuilt from the first affected chunk
static pkv_status refresh_derived(pkv_index* ix, int64_t t0, bool full, cudaStream_t stream) {
  if (ix->postings)
    PKV_CUDA(launch_postings_build(ix, full ? 0 : t0 / POST_CHUNK, (ix->n + POST_CHUNK - 1) / POST_CHUNK, stream),
             "postings (rebalance)");
  if (ix->occ) {
    if (full)
      PKV_CUDA(cudaMemsetAsync(ix->occ, 0, (size_t)ix->batch * ix->cfg.n_kv_heads * NB * NC * 4, stream),
               "occupancy clear");
    PKV_CUDA(launch_occupancy(ix, full ? 0 : t0, ix->n, stream), "occupancy (rebalance)");
  }
  return PKV_OK;
}

pkv_status pkv_index_import_back(pkv_index* ix, const void* buf, int64_t count, cudaStream_t stream) {
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_import_back: null index");
  if (count < 0) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_import_back: count < 0");
  if (count > 0 && !buf) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_import_back: null buffer");
  if (ix->n + count > ix->cap) return set_error(PKV_ERR_CAPACITY, "pkv_index_import_back: capacity exceeded");
  if (count == 0) return PKV_OK;
  DeviceGuard g(ix->device);
  const int64_t t0 = ix->n;
  PKV_CUDA(launch_import_entries(ix, t0, count, buf, stream), "import back");
  ix->n += count;
  return refresh_derived(ix, t0, false, stream);
}

pkv_status pkv_index_drop_front(pkv_index* ix, int64_t count, cudaStream_t stream) {
  if (!ix) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_drop_front: null index");
  if (count < 0 || count > ix->n) return set_error(PKV_ERR_INVALID_ARG, "pkv_index_drop_front: count outside [0, n]");
  if (count == 0) return PKV_OK;
  DeviceGuard g(ix->device);
  const int64_t keep = ix->n - count;
  if (keep > 0) {  // the kept keys move down by `count` through a stream-ordered scratch copy (the ranges overlap)
    int64_t eb = 0;
    pkv_index_entry_bytes(ix, &eb);
    void* tmp = nullptr;
    PKV_CUDA(cudaMallocAsync(&tmp, (size_t)(keep * eb), stream), "drop_front scratch");
    cudaError_t e = launch_export_entries(ix, count, keep, tmp, stream);
    if (e == cudaSuccess) e = launch_import_entries(ix, 0, keep, tmp, stream);
    cudaFreeAsync(tmp, stream);
    PKV_CUDA(e, "drop front");
  }
  ix->n = keep;
  ix->shard_offset += count;
  return refresh_derived(ix, 0, true, stream);
}

pkv_status pkv_index_shift_boundary(pkv_index* older, pkv_index* newer, int64_t count, cudaStream_t stream) {
  if (!older || !newer || older == newer) return set_error(PKV_ERR_INVALID_ARG, "shift_boundary: two indices needed");
  if (older->device != newer->device || older->batch != newer->batch ||
      older->cfg.n_kv_heads != newer->cfg.n_kv_heads || older->dcfg.rec_bytes != newer->dcfg.rec_bytes ||
      std::memcmp(older->dcfg.sign_mask, newer->dcfg.sign_mask, sizeof(older->dcfg.sign_mask)) != 0)
    return set_error(PKV_ERR_INVALID_ARG, "shift_boundary: indices of different devices / shapes / rotations");
  if (count < 0 || count > newer->n) return set_error(PKV_ERR_INVALID_ARG, "shift_boundary: count outside [0, n]");
  if (older->n + count > older->cap) return set_error(PKV_ERR_CAPACITY, "shift_boundary: capacity exceeded");
  if (count == 0) return PKV_OK;
  DeviceGuard g(older->device);
  int64_t eb = 0;
  pkv_index_entry_bytes(newer, &eb);
  void* buf = nullptr;
  PKV_CUDA(cudaMallocAsync(&buf, (size_t)(count * eb), stream), "shift_boundary buffer");
  pkv_status st = pkv_index_export_front(newer, count, buf, stream);
  if (st == PKV_OK) st = pkv_index_import_back(older, buf, count, stream);
  if (st == PKV_OK) st = pkv_index_drop_front(newer, count, stream);
  cudaFreeAsync(buf, stream);
  return st;
}

pkv_status pkv_rebalance_plan(const int64_t* lengths, int32_t P, int64_t granule, int64_t* shift) {
  if (!lengths || !shift || P < 1 || P > 64 || granule < 1)
    return set_error(PKV_ERR_INVALID_ARG, "pkv_rebalance_plan: bad arguments");
  int64_t N = 0;
  for (int r = 0; r < P; ++r) {
    if (lengths[r] < 0) return set_error(PKV_ERR_INVALID_ARG, "pkv_rebalance_plan: negative length");
    N += lengths[r];
  }
  // boundary r (start of shard r, now at b_r) moves right towards the balanced position r*N/P by whole granules,
  // never left; then min(., next boundary) keeps the boundaries ordered (shard r+1 can always give what r needs
  // once it has received its own share from r+2: apply shift[P-2] first, shift[0] last)
  int64_t b[65], nb[65];
  b[0] = 0;
  for (int r = 1; r <= P; ++r) b[r] = b[r - 1] + lengths[r - 1];
  nb[P] = N;
  for (int r = 1; r < P; ++r) {
    const int64_t target = (int64_t)((__int128)r * N / P);
    nb[r] = target > b[r] ? b[r] + (target - b[r]) / granule * granule : b[r];
  }
  for (int r = P - 1; r >= 1; --r) nb[r] = std::min(nb[r], nb[r + 1]);
  for (int r = 1; r < P; ++r) shift[r - 1] = nb[r] - b[r];
  return PKV_OK;
}

}  // extern "C"
