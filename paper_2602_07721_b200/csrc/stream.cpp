// Streaming decode: the four-region KV cache of PAPER §4.2.3 "Buffer Update" on top of the
// retrieval index. Host-side bookkeeping plus stream-ordered copies; the GPU work is append_decode_keys
// (encoder) and retrieve_and_attend_rows (the decode hot path). See include/pariskv.h for the contract.
//
// Hot buffer layout, per (sequence, KV head), row capacity R = sink + local_size + update_size:
//   rows [0, n_sink)                          Sink
//   rows [sink, sink + n_local)               Local (oldest first)
//   rows [sink + n_local, ... + n_buf)        Update buffer (oldest first)
// so the attended hot rows are always the contiguous prefix... except for an unfilled sink, which prefill
// forbids (n_tokens >= sink). A flush evicts the oldest e = n_local + n_buf - local_size rows of Local U Update
// (rows [sink, sink + e)) to the retrieval zone and moves the remaining local_size rows down to row sink.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "internal.h"

using namespace pkv;

struct pkv_stream {
  pkv_index* ix = nullptr;
  pkv_stream_config cfg{};
  int rows = 0;             // hot row capacity per (sequence, KV head)
  int n_local = 0, n_buf = 0;
  bool prefilled = false;
  uint16_t* Kh = nullptr;   // hot K [batch][n_kv][rows][128]
  uint16_t* Vh = nullptr;
  uint16_t* scratch = nullptr;  // [batch][n_kv][local_size][128] for overlapping Local shifts
  uint16_t* Ks = nullptr;   // retrieval store K [batch][n_kv][cap][128] (device pointer; host-mapped if offloaded)
  uint16_t* Vs = nullptr;
  void* Ks_host = nullptr;  // host allocation when offloaded
  void* Vs_host = nullptr;
  // asynchronous offload of evicted rows ("offloading the corresponding full-precision KV pairs
  // asynchronously"): a flush copies the evicted rows to device staging buffers on the caller's stream, a side
  // stream moves them to the store (over the host link when offloaded) while the step's retrieval kernels run,
  // and only the step's row gather waits for it (ev_join)
  uint16_t* Kst = nullptr;  // staging [batch][n_kv][update_size][128]
  uint16_t* Vst = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

namespace {

constexpr size_t ROWB = (size_t)D * 2;  // bytes per bf16 row

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// copy `nrows` rows of every (sequence, KV head): dst row r0 of a head block with `dst_rows` capacity, from a
// source whose row t of (b, h) lives at src + b*sb + h*sh + t*st (elements)
cudaError_t copy_rows(uint16_t* dst, int64_t dst_rows, int64_t r0, const uint16_t* src, int64_t sb, int64_t sh,
                      int64_t st, int64_t nrows, int batch, int n_kv, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  for (int b = 0; b < batch; ++b) {
    // one 2-D copy per sequence: heads are the "height", rows of a head the "width" when rows are contiguous
    if (st == D) {
      cudaError_t e = cudaMemcpy2DAsync(dst + ((int64_t)b * n_kv * dst_rows + r0) * D, dst_rows * ROWB,
                                        src + b * sb, sh * 2, nrows * ROWB, n_kv, cudaMemcpyDefault, s);
      if (e != cudaSuccess) return e;
    } else {
      for (int h = 0; h < n_kv; ++h) {
        cudaError_t e = cudaMemcpy2DAsync(dst + (((int64_t)b * n_kv + h) * dst_rows + r0) * D, ROWB,
                                          src + b * sb + h * sh, st * 2, ROWB, nrows, cudaMemcpyDefault, s);
        if (e != cudaSuccess) return e;
      }
    }
  }
  return cudaSuccess;
}

}  // namespace

extern "C" {

pkv_status pkv_stream_create(pkv_index* ix, const pkv_stream_config* c, pkv_stream** out) {
  if (!ix || !c || !out) return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_create: null pointer");
  if (c->sink < 0 || c->local_size < 0 || c->update_size < 1 ||
      (int64_t)c->sink + c->local_size + c->update_size > 1024)
    return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_create: need sink, local_size >= 0, update_size >= 1, "
                                          "sink + local_size + update_size <= 1024");
  if (ix->comm) return set_error(PKV_ERR_UNSUPPORTED, "pkv_stream_create: sequence-sharded index");
  Guard g(ix->device);
  pkv_stream* s = new (std::nothrow) pkv_stream();
  if (!s) return set_error(PKV_ERR_CUDA, "host allocation failed");
  s->ix = ix;
  s->cfg = *c;
  s->rows = c->sink + c->local_size + c->update_size;
  const int64_t heads = (int64_t)ix->batch * ix->cfg.n_kv_heads;
  const size_t hot = (size_t)heads * s->rows * ROWB, store = (size_t)heads * ix->cap * ROWB;
  cudaError_t e = cudaMalloc(&s->Kh, hot);
  if (e == cudaSuccess) e = cudaMalloc(&s->Vh, hot);
  if (e == cudaSuccess && c->local_size > 0)
    e = cudaMalloc(&s->scratch, (size_t)heads * c->local_size * ROWB);
  if (e == cudaSuccess) e = cudaMalloc(&s->Kst, (size_t)heads * c->update_size * ROWB);
  if (e == cudaSuccess) e = cudaMalloc(&s->Vst, (size_t)heads * c->update_size * ROWB);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) {
    if (c->offload_host) {
      e = cudaHostAlloc(&s->Ks_host, store, cudaHostAllocMapped);
      if (e == cudaSuccess) e = cudaHostAlloc(&s->Vs_host, store, cudaHostAllocMapped);
      if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&s->Ks, s->Ks_host, 0);
      if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&s->Vs, s->Vs_host, 0);
    } else {
      e = cudaMalloc(&s->Ks, store);
      if (e == cudaSuccess) e = cudaMalloc(&s->Vs, store);
    }
  }
  if (e != cudaSuccess) {
    pkv_stream_destroy(s);
    return cuda_status(e, "pkv_stream_create");
  }
  *out = s;
  return PKV_OK;
}

pkv_status pkv_stream_destroy(pkv_stream* s) {
  if (!s) return PKV_OK;
  Guard g(s->ix->device);
  cudaFree(s->Kh);
  cudaFree(s->Vh);
  cudaFree(s->scratch);
  if (s->side) cudaStreamSynchronize(s->side);  // an offload still in flight finishes before its buffers go
  cudaFree(s->Kst);
  cudaFree(s->Vst);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  if (s->side) cudaStreamDestroy(s->side);
  if (s->cfg.offload_host) {
    cudaFreeHost(s->Ks_host);
    cudaFreeHost(s->Vs_host);
  } else {
    cudaFree(s->Ks);
    cudaFree(s->Vs);
  }
  delete s;
  return PKV_OK;
}

pkv_status pkv_stream_prefill(pkv_stream* s, const void* K, const void* V, int64_t sb, int64_t sh, int64_t st,
                              int64_t n_tokens, cudaStream_t stream) {
  NvtxRange nvtx_("pkv:stream_prefill");
  if (!s || !K || !V) return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_prefill: null pointer");
  pkv_index* ix = s->ix;
  const int sink = s->cfg.sink;
  if (n_tokens < sink) return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_prefill: n_tokens < sink");
  if (sb < 0 || sh < 0 || st < D) return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_prefill: bad strides");
  const int64_t rest = n_tokens - sink;
  const int n_local = (int)std::min<int64_t>(s->cfg.local_size, rest);
  const int64_t n_ret = rest - n_local;
  if (n_ret > ix->cap) return set_error(PKV_ERR_CAPACITY, "pkv_stream_prefill: retrieval zone exceeds capacity");
  Guard g(ix->device);
  const uint16_t* k = static_cast<const uint16_t*>(K);
  const uint16_t* v = static_cast<const uint16_t*>(V);
  const int batch = ix->batch, n_kv = ix->cfg.n_kv_heads;
  // the encoder reads the retrieval keys in place; an empty retrieval zone still resets the index
  pkv_status r = encode_keys(ix, k + sink * st, sb, sh, st, n_ret, stream);
  if (r != PKV_OK) return r;
  cudaError_t e = copy_rows(s->Kh, s->rows, 0, k, sb, sh, st, sink, batch, n_kv, stream);
  if (e == cudaSuccess) e = copy_rows(s->Vh, s->rows, 0, v, sb, sh, st, sink, batch, n_kv, stream);
  if (e == cudaSuccess) e = copy_rows(s->Ks, ix->cap, 0, k + sink * st, sb, sh, st, n_ret, batch, n_kv, stream);
  if (e == cudaSuccess) e = copy_rows(s->Vs, ix->cap, 0, v + sink * st, sb, sh, st, n_ret, batch, n_kv, stream);
  if (e == cudaSuccess)
    e = copy_rows(s->Kh, s->rows, sink, k + (sink + n_ret) * st, sb, sh, st, n_local, batch, n_kv, stream);
  if (e == cudaSuccess)
    e = copy_rows(s->Vh, s->rows, sink, v + (sink + n_ret) * st, sb, sh, st, n_local, batch, n_kv, stream);
  if (e != cudaSuccess) return cuda_status(e, "pkv_stream_prefill");
  s->n_local = n_local;
  s->n_buf = 0;
  s->prefilled = true;
  return PKV_OK;
}

pkv_status pkv_stream_decode(pkv_stream* s, const void* q, const void* k_new, const void* v_new,
                             const pkv_retrieve_params* params, float scale, int32_t* out_idx, float* out_est,
                             void* out, float* lse, cudaStream_t stream) {
  NvtxRange nvtx_("pkv:stream_decode");
  // Every argument is validated, for the state this step will produce, before anything is enqueued or changed:
  // a failing call leaves the regions and the index as they were (header contract).
  if (!s || !q || !k_new || !v_new || !params || !out_idx || !out_est || !out)
    return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_decode: null pointer");
  if (!s->prefilled) return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_decode: prefill first");
  if (params->top_k < 1 || params->top_k > MAX_TOPK)
    return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_decode: top_k out of [1,1024]");
  pkv_index* ix = s->ix;
  const int sink = s->cfg.sink, L = s->cfg.local_size, U = s->cfg.update_size;
  const int batch = ix->batch, n_kv = ix->cfg.n_kv_heads;
  const bool flush = s->n_buf + 1 == U;
  const int evict = flush ? std::max(0, s->n_local + U - L) : 0;
  if (flush && ix->n + evict > ix->cap)
    return set_error(PKV_ERR_CAPACITY, "pkv_stream_decode: flush would exceed the index capacity");
  const int64_t n_after = ix->n + evict;                                   // retrieval zone after this step
  const int keep = flush ? s->n_local + s->n_buf + 1 - evict : s->n_local;  // Local after this step
  const int buf_after = flush ? 0 : s->n_buf + 1;
  const int n_hot = sink + keep + buf_after;
  pkv_retrieve_params p = *params;
  if (n_after > 0 && (p.probes_T <= 0 || p.n_cand <= 0)) {  // schedule for the post-flush retrieval length
    int32_t T = 0;
    int64_t C = 0;
    pkv_status r = pkv_schedule(n_after, p.top_k, &T, &C);
    if (r != PKV_OK) return r;
    if (p.probes_T <= 0) p.probes_T = T;
    if (p.n_cand <= 0) p.n_cand = C;
  }
  if (n_after > 0) {
    pkv_status r = check_retrieve(ix, q, &p, n_after, out_idx, out_est);
    if (r != PKV_OK) return r;
  } else if (n_hot < 1 || (reinterpret_cast<uintptr_t>(q) & 15u)) {
    return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_decode: nothing to attend / misaligned q");
  }
  Guard g(ix->device);
  const int64_t hb = (int64_t)n_kv * s->rows * D;  // elements per sequence in the hot buffer
  const int64_t row = sink + s->n_local + s->n_buf;
  // (1) the new token joins the Update buffer
  cudaError_t e = copy_rows(s->Kh, s->rows, row, static_cast<const uint16_t*>(k_new), (int64_t)n_kv * D, D, D, 1,
                            batch, n_kv, stream);
  if (e == cudaSuccess)
    e = copy_rows(s->Vh, s->rows, row, static_cast<const uint16_t*>(v_new), (int64_t)n_kv * D, D, D, 1, batch,
                  n_kv, stream);
  if (e != cudaSuccess) return cuda_status(e, "pkv_stream_decode(append)");
  s->n_buf += 1;
  if (flush) {
    // (2) evict the oldest rows of Local U Update into Retrieval: encode + append (iii), K/V to the store (i)
    const int64_t n0 = ix->n;
    if (evict > 0) {
      // (i) evicted rows -> staging (device, this stream), then -> the store on the side stream, asynchronously
      const int64_t sh_st = (int64_t)U * D, sb_st = (int64_t)n_kv * U * D;
      e = copy_rows(s->Kst, U, 0, s->Kh + (int64_t)sink * D, hb, (int64_t)s->rows * D, D, evict, batch, n_kv,
                    stream);
      if (e == cudaSuccess)
        e = copy_rows(s->Vst, U, 0, s->Vh + (int64_t)sink * D, hb, (int64_t)s->rows * D, D, evict, batch, n_kv,
                      stream);
      if (e == cudaSuccess) e = cudaEventRecord(s->ev_fork, stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s->side, s->ev_fork, 0);
      if (e == cudaSuccess) e = copy_rows(s->Ks, ix->cap, n0, s->Kst, sb_st, sh_st, D, evict, batch, n_kv, s->side);
      if (e == cudaSuccess) e = copy_rows(s->Vs, ix->cap, n0, s->Vst, sb_st, sh_st, D, evict, batch, n_kv, s->side);
      if (e == cudaSuccess) e = cudaEventRecord(s->ev_join, s->side);
      if (e != cudaSuccess) return cuda_status(e, "pkv_stream_decode(offload)");
      // (iii) encode and index the evicted keys (read in place, before the Local shift below)
      pkv_status r = append_decode_keys(ix, s->Kh + (int64_t)sink * D, hb, (int64_t)s->rows * D, D, evict, stream);
      if (r != PKV_OK) {
        cudaStreamWaitEvent(stream, s->ev_join, 0);  // join the side stream (capture-safe) before reporting
        return r;
      }
    }
    // (3) the newest local_size rows become Local (ii)
    if (e == cudaSuccess && evict > 0 && keep > 0) {
      for (uint16_t* H : {s->Kh, s->Vh}) {
        const uint16_t* src = H + (int64_t)(sink + evict) * D;
        if (evict >= keep) {  // disjoint ranges
          e = copy_rows(H, s->rows, sink, src, hb, (int64_t)s->rows * D, D, keep, batch, n_kv, stream);
        } else {              // overlapping: through the scratch buffer
          e = copy_rows(s->scratch, L, 0, src, hb, (int64_t)s->rows * D, D, keep, batch, n_kv, stream);
          if (e == cudaSuccess)
            e = copy_rows(H, s->rows, sink, s->scratch, (int64_t)n_kv * L * D, (int64_t)L * D, D, keep, batch, n_kv,
                          stream);
        }
        if (e != cudaSuccess) break;
      }
    }
    if (e != cudaSuccess) return cuda_status(e, "pkv_stream_decode(flush)");
    s->n_local = keep;
    s->n_buf = 0;
  }
  // (4) retrieval over the updated index + attention over Sink U Local U Update and the retrieved rows; a still
  // empty retrieval zone (prompt <= sink + local_size, no eviction yet) attends the hot rows alone
  if (n_after == 0)
    return attend_hot_only(ix, q, s->Kh, s->Vh, n_hot, s->rows, p.top_k, scale, out_idx, out_est, out, lse, stream);
  const bool offloading = flush && evict > 0;
  pkv_status r = retrieve_and_attend_rows_after(ix, q, &p, s->Ks, s->Vs, (int64_t)n_kv * ix->cap * D, ix->cap * D, D,
                                                s->Kh, s->Vh, n_hot, s->rows, scale, out_idx, out_est, out, lse,
                                                offloading ? s->ev_join : nullptr, stream);
  if (r != PKV_OK && offloading) cudaStreamWaitEvent(stream, s->ev_join, 0);
  return r;
}

pkv_status pkv_stream_state(const pkv_stream* s, int64_t* n_retrieval, int32_t* n_local, int32_t* n_buffer,
                            const void** K_store, const void** V_store, const void** K_hot, const void** V_hot) {
  if (!s) return set_error(PKV_ERR_INVALID_ARG, "pkv_stream_state: null stream");
  if (n_retrieval) *n_retrieval = s->ix->n;
  if (n_local) *n_local = s->n_local;
  if (n_buffer) *n_buffer = s->n_buf;
  if (K_store) *K_store = s->Ks;
  if (V_store) *V_store = s->Vs;
  if (K_hot) *K_hot = s->Kh;
  if (V_hot) *V_hot = s->Vh;
  return PKV_OK;
}

}  // extern "C"
