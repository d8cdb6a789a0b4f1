// Optional per-kernel CUDA-event timing (eager mode only; bench.py uses it for the live roofline numbers).
// When enabled, every kernel launch is bracketed by two events recorded on the launch stream.
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <vector>

#include "internal.h"

namespace pkv {
namespace {

struct Rec {
  int kind;
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
int64_t g_count[K_NUM_KINDS] = {};
double g_ms[K_NUM_KINDS] = {};

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void drain() {  // caller holds g_mu
  for (auto& r : g_recs) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      g_count[r.kind]++;
      g_ms[r.kind] += ms;
    }
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
}

const char* kNames[K_NUM_KINDS] = {"encode", "qprep", "scan", "select", "unused", "rerank", "topk",
                                   "topk_merge", "attend", "combine", "head_hist", "export", "debug"};

}  // namespace

thread_local int t_kind = -1;  // kind of the launch being bracketed (pdl_enabled's per-kernel mask)

ProfScope::ProfScope(int kind, cudaStream_t s) : kind_(kind), s_(s) {
  t_kind = kind;
  if (g_on) {
    std::lock_guard<std::mutex> l(g_mu);
    a_ = get_event();
    cudaEventRecord(a_, s_);
  }
}

ProfScope::~ProfScope() {
  g_launches++;
  if (a_) {
    std::lock_guard<std::mutex> l(g_mu);
    cudaEvent_t b = get_event();
    cudaEventRecord(b, s_);
    g_recs.push_back(Rec{kind_, a_, b});
    if (g_recs.size() > 4096) drain();
  }
}

}  // namespace pkv

extern "C" pkv_status pkv_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> l(pkv::g_mu);
  pkv::drain();
  for (int i = 0; i < pkv::K_NUM_KINDS; ++i) {
    pkv::g_count[i] = 0;
    pkv::g_ms[i] = 0.0;
  }
  pkv::g_on = on != 0;
  return PKV_OK;
}

extern "C" pkv_status pkv_profile_read(int32_t kind, int64_t* launches, double* total_ms) {
  if (kind < 0 || kind >= pkv::K_NUM_KINDS || !launches || !total_ms)
    return pkv::set_error(PKV_ERR_INVALID_ARG, "pkv_profile_read: bad kind");
  std::lock_guard<std::mutex> l(pkv::g_mu);
  pkv::drain();
  *launches = pkv::g_count[kind];
  *total_ms = pkv::g_ms[kind];
  return PKV_OK;
}

extern "C" const char* pkv_kernel_name(int32_t kind) {
  return (kind >= 0 && kind < pkv::K_NUM_KINDS) ? pkv::kNames[kind] : "";
}

namespace pkv {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PKV_NO_PDL");
    return !(e && e[0] == '1');
  }();
  // Bit k: kernel kind k (KernelKind) is launched WITHOUT programmatic serialisation. Default: the query-prep
  // and rerank kernels — their early-resident CTAs (waiting in griddepcontrol.wait on SMs still running the
  // predecessor) measured 4-5 us/layer slower at 128K; scan, select and the fused top-k keep their pre-wait
  // work (centroid-id prefetch, hot-row attention). PKV_NO_PDL_MASK overrides (diagnostics).
  static const unsigned mask = [] {
    const char* e = std::getenv("PKV_NO_PDL_MASK");
    return e ? (unsigned)std::strtoul(e, nullptr, 0) : ((1u << K_QPREP) | (1u << K_RERANK));
  }();
  return on && !(t_kind >= 0 && ((mask >> t_kind) & 1u));
}
}  // namespace pkv

extern "C" pkv_status pkv_phase_profile(unsigned long long* device_buf) {
  cudaError_t e = pkv::set_phase_scan(device_buf);
  if (e == cudaSuccess) e = pkv::set_phase_rerank(device_buf);
  if (e == cudaSuccess) e = pkv::set_phase_qprep(device_buf);
  if (e == cudaSuccess) e = pkv::set_phase_attend(device_buf);
  if (e == cudaSuccess) e = pkv::set_phase_encode(device_buf);
  return pkv::cuda_status(e, "pkv_phase_profile");
}
