// Internal declarations shared by the host side (api.cpp, comm.cpp, levels.cpp) and the kernel
// launchers (*.cu). Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "../../include/pariskv.h"

namespace pkv {

constexpr int D = PKV_HEAD_DIM;        // 128
constexpr int NB = PKV_SUBSPACES;      // 16 subspaces
constexpr int M = PKV_SUBSPACE_DIM;    // 8
constexpr int NC = PKV_CENTROIDS;      // 256 analytic centroids per subspace (Eq. 5)
constexpr int HB = 128;                // histogram bins (max collision score <= 127)
constexpr int GMAX = 4;                // query heads per KV head packed in one u32 (bytes)
constexpr int REC = 128;               // bytes per rerank record: 64 B nibbles + 16 x fp32 w'
constexpr int MAX_TOPK = 1024;
constexpr int MAX_CHUNKS = 256;        // scan chunks per (sequence, KV head)
constexpr int MAX_SPLITS = 64;         // attention split-k partials per (sequence, q head)
constexpr int PART = D + 2;            // floats per attention partial: m, l, o[128]

// Device-side copy of the offline constants, passed to kernels by value.
struct DevCfg {
  int n_q, n_kv, G;
  int n_tiers;
  int tier_bonus[PKV_MAX_TIERS];
  float levels[8];
  double mid_sq[7];
  unsigned int sign_mask[4];  // bit d of word d/32 = rot_sign[d]
  int w16;                    // 1: fp16 weights + per-key exponent (96-byte records), 0: fp32 (128-byte)
  int rec_bytes;              // record stride: 96 or 128
};

struct Workspace {
  int device = -1;
  int batch = 0, n_q = 0, n_kv = 0;
  int64_t cap = 0;
  uint32_t* lut = nullptr;        // [batch][n_kv][4 heads][16 s][256 c] bonus bytes (head j = query head g*G+j)
  float* rtab = nullptr;          // [batch][n_q][128 coord][16 nibble] rerank tables sign*L[idx]*q~
  float* qnorm = nullptr;         // [batch][n_q]
  float* qrot = nullptr;          // [batch][n_q][128]
  uint32_t* scores = nullptr;     // [batch][n_kv][cap] packed collision scores
  uint32_t* chunk_hist = nullptr; // [batch][n_kv][MAX_CHUNKS][GMAX][HB]
  uint32_t* head_hist = nullptr;  // [MAX_RANKS][batch][n_q][HB] (per-rank totals; sharded exchange H)
  int32_t* sel = nullptr;         // [batch][n_q][4 + 4*MAX_CHUNKS] threshold + per-chunk offsets
  int32_t* cand = nullptr;        // [batch][n_q][cap]
  float* est = nullptr;           // [batch][n_q][cap]
  uint32_t* ta_msg = nullptr;     // fused T+A exchange: [MAX_RANKS][batch][n_q][ta_slot(TA_MAXK)] words
  int32_t* topk_idx = nullptr;    // sharded exchange T: rank r's ids at topk_idx + 2r*slot,
  float* topk_est = nullptr;      //   its estimates at topk_est + 2r*slot (= ids + slot); slot = batch*n_q*MAX_TOPK
  float* part = nullptr;          // [MAX_RANKS][batch][n_q][MAX_SPLITS][PART] (exchange A)
  unsigned int* ticket = nullptr; // [batch][n_kv] split-completion counters of the fused attention merge
  float* seg_est = nullptr;       // [seg_slots][batch][n_q][MAX_TOPK] segmented top-k of long candidate lists
  int32_t* seg_idx = nullptr;
  int seg_slots = 1;              // = topk_segments(cap): segment lists a head's candidate list can need
  // GQA-union rerank: per (sequence, KV head) the keys that are a candidate of at least one of
  // its query heads, each with its candidate position in every head's list (-1: not a candidate of that head)
  unsigned int* ucount = nullptr; // [batch][n_kv] union sizes (zeroed by qprep, counted by select)
  int32_t* uid = nullptr;         // [batch][n_kv][cap] local key index
  int32_t* upos = nullptr;        // [batch][n_kv][cap][4] candidate positions per query head of the group
  uint16_t* warp_hist = nullptr;  // [warp_hist_ctas][32 warps][GMAX][HB] per-warp cumulative score counts (scan)
  int64_t warp_hist_ctas = 0;
  void* base = nullptr;
  size_t bytes = 0;
  int refs = 1;
};

constexpr int MAX_RANKS = 8;
constexpr int SEG_SLOTS = 64;  // most segments of one candidate list in the segmented top-k (rerank.cu)

struct Comm;  // comm.cpp

}  // namespace pkv

struct pkv_index {
  pkv_config cfg;
  pkv::DevCfg dcfg;
  int device = 0;
  int batch = 0;
  int64_t cap = 0;
  int64_t n = 0;
  uint8_t* ids = nullptr;   // [batch][n_kv][cap][16]; row of key t rotated left by (t mod 16) bytes
  uint8_t* rec = nullptr;   // [batch][n_kv][cap][rec_bytes]: 64 B nibbles + 16 x fp32 w' (or 16 x fp16 w')
  // inverted lists (pkv_index_set_postings): per (b, kv, chunk of POST_CHUNK keys, subspace)
  // bucket offsets u16 [257] and the chunk's key offsets u16 [POST_CHUNK] sorted by centroid id
  float* dbg_out_f32 = nullptr;         // optional fp32 copy of every attention output (pkv_index_set_debug_output)
  unsigned long long* stats = nullptr;  // device [4]: zero keys, keys with a zero subspace, zero subspaces, spare
  int32_t* enc_fb = nullptr;  // [batch*n_kv*cap + 1]: keys handed back by the fast / tensor-core encoder, count at the end
  bool postings = false;
  uint32_t* occ = nullptr;  // [batch][n_kv][16][256] centroid occupancy (pkv_index_set_occupancy); null = off
  uint16_t* post_off = nullptr;
  uint16_t* post_key = nullptr;
  pkv::Workspace* ws = nullptr;
  pkv::Comm* comm = nullptr;
  int rank = 0, world = 1;
  int64_t shard_offset = 0;
  int num_sms = 148;
  int smem_reserved = 1024;
};

namespace pkv {

// NVTX range around one public call (nsys / ncu timelines: "pkv:retrieve_and_attend" etc.); header-only NVTX 3,
// a no-op unless a tool is attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Kernel kinds for launch accounting / optional event timing (profile.cpp)
enum KernelKind { K_ENCODE, K_QPREP, K_SCAN, K_SELECT, K_UNUSED4, K_RERANK, K_TOPK, K_MERGE, K_ATTEND,
                  K_COMBINE, K_HEADHIST, K_EXPORT, K_DEBUG, K_NUM_KINDS };
class ProfScope {  // bracket one kernel launch: counts it, and records events when profiling is on
 public:
  ProfScope(int kind, cudaStream_t s);
  ~ProfScope();

 private:
  int kind_;
  cudaStream_t s_;
  cudaEvent_t a_ = nullptr;
};

cudaError_t set_phase_scan(unsigned long long* p);
cudaError_t set_phase_rerank(unsigned long long* p);
cudaError_t set_phase_qprep(unsigned long long* p);
cudaError_t set_phase_attend(unsigned long long* p);
cudaError_t set_phase_encode(unsigned long long* p);

// Shared validation / hot-row-only attention (api.cpp), used by the streaming manager (stream.cpp)
pkv_status retrieve_and_attend_rows_after(pkv_index* ix, const void* q, const pkv_retrieve_params* p, const void* K,
                                          const void* V, int64_t sb, int64_t sh, int64_t st, const void* K_hot,
                                          const void* V_hot, int32_t n_hot, int32_t hot_rows, float scale,
                                          int32_t* out_idx, float* out_est, void* out, float* lse,
                                          cudaEvent_t attend_after, cudaStream_t stream);
pkv_status check_retrieve(const pkv_index* ix, const void* q, const pkv_retrieve_params* p, int64_t n_global,
                          const int32_t* out_idx, const float* out_est);
// Attention over the hot rows alone (empty retrieval zone): out_idx/out_est [batch][n_q][top_k] get -1 / -inf.
pkv_status attend_hot_only(pkv_index* ix, const void* q, const void* K_hot, const void* V_hot, int n_hot,
                           int hot_rows, int top_k, float scale, int32_t* out_idx, float* out_est, void* out,
                           float* lse, cudaStream_t stream);

// Error plumbing (api.cpp)
pkv_status set_error(pkv_status s, const std::string& msg);
pkv_status cuda_status(cudaError_t e, const char* what);
extern std::atomic<uint64_t> g_launches;

// Host-side constants (levels.cpp)
void prop1_levels(int m, double out_levels[8]);

// Launchers (*.cu). All enqueue on `stream` and return the launch error.
// tensor-core encoder (encode_tc.cu): keys outside its exact range are appended to fb_list (count fb_count)
cudaError_t init_encode_tc_attrs();
cudaError_t launch_encode_tc(const pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t0,
                             int64_t count, int32_t* fb_list, int32_t* fb_count, cudaStream_t stream);
// half-warp encoder over a device list (entries bh * count + tt)
bool ef_buckets_ok(const DevCfg& c);
cudaError_t launch_encode_fast(const pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t0,
                               int64_t count, int32_t* list, int32_t* list_n, cudaStream_t stream);
cudaError_t launch_encode_list(const pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t0,
                               int64_t count, const int32_t* list, const int32_t* list_n, cudaStream_t stream);
cudaError_t launch_encode(const pkv_index* ix, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t0,
                          int64_t count, cudaStream_t stream);
cudaError_t launch_export(const pkv_index* ix, int64_t start, int64_t count, uint8_t* ids, uint8_t* codes,
                          float* w, cudaStream_t stream);
cudaError_t launch_qprep(const pkv_index* ix, const void* q, int T, int64_t rho_keys, float* dbg_q_rot,
                         cudaStream_t stream);
cudaError_t launch_occupancy(const pkv_index* ix, int64_t t0, int64_t t1, cudaStream_t stream);
cudaError_t launch_export_entries(const pkv_index* ix, int64_t src0, int64_t count, void* buf, cudaStream_t stream);
cudaError_t launch_import_entries(pkv_index* ix, int64_t dst0, int64_t count, const void* buf, cudaStream_t stream);

constexpr int POST_CHUNK = 8192;  // keys per inverted-list chunk (u16 offsets)

struct ScanPlan {
  int nchunks;
  int64_t chunk;           // keys per chunk (multiple of 32)
  bool warp_hist = false;  // the scan records per-warp cumulative histograms for the select (dense scan only)
};
ScanPlan plan_scan(const pkv_index* ix, int64_t n);
int64_t score_stride(const pkv_index* ix);
cudaError_t init_postings_attrs();
cudaError_t launch_postings_build(const pkv_index* ix, int64_t chunk0, int64_t chunk1, cudaStream_t stream);
// inverted-list variant of the scan: same scores / per-chunk histograms, chunks of POST_CHUNK keys
cudaError_t launch_postings_scan(const pkv_index* ix, int64_t n, int64_t sstride, cudaStream_t stream);
cudaError_t init_scan_attrs();
cudaError_t init_rerank_attrs();
cudaError_t launch_scan(const pkv_index* ix, int64_t n, const ScanPlan& plan, cudaStream_t stream);
// Per-head totals of the chunk histograms -> head_hist[slot].
cudaError_t launch_head_hist(const pkv_index* ix, const ScanPlan& plan, uint32_t* head_hist_out,
                             cudaStream_t stream);
// Fused threshold + compaction. all_hist: [P][batch][n_q][HB] gathered cumulative per-rank totals (P > 1).
cudaError_t launch_select(const pkv_index* ix, int64_t n, const ScanPlan& plan, const uint32_t* all_hist, int P,
                          int rank, int64_t C, int64_t id_offset, cudaStream_t stream);
cudaError_t launch_rerank(const pkv_index* ix, int64_t C_cap, int64_t id_offset, cudaStream_t stream);
// GQA-union rerank (PKV_RERANK=union; measured slower than the per-query-head kernel, which stays the default):
// select emits the union lists, the rerank reads every record once per KV head and scores it for all the
// group's query heads
bool union_rerank();
cudaError_t launch_dbg_scores(const pkv_index* ix, int64_t n, uint8_t* out, cudaStream_t stream);
cudaError_t launch_topk(const pkv_index* ix, int64_t C_cap, int k, int32_t* out_idx, float* out_est,
                        int out_stride, cudaStream_t stream);
// Final top-k fused with the gather + attention of the selected rows and of the hot rows (row t of (b, h) at
// K_hot + ((b*n_kv + h)*hot_rows + t)*D), one thread-block cluster per query head.
cudaError_t launch_topk_attend(const pkv_index* ix, int64_t C_cap, int k, int32_t* out_idx, float* out_est,
                               const void* q, const void* K, const void* V, int64_t sb, int64_t sh, int64_t st,
                               float scale, const void* K_hot,
                               const void* V_hot, int n_hot, int hot_rows, void* out, float* lse,
                               cudaStream_t stream);
int topk_segments(int64_t C_cap);
// Attention over the given top-k rows (no selection) and the hot rows (segmented top-k path).
cudaError_t launch_topk_attend_rows(const pkv_index* ix, int k, const int32_t* idx, const void* q, const void* K,
                                    const void* V, int64_t sb, int64_t sh, int64_t st, float scale,
                                    const void* K_hot, const void* V_hot, int n_hot, int hot_rows, void* out,
                                    float* lse, cudaStream_t stream);  // > 1: long lists take the segmented top-k + merge (no fused attend)
cudaError_t launch_topk_merge_strided(const pkv_index* ix, int P, int k, const float* all_est, const int32_t* all_idx,
                                      int32_t* out_idx, float* out_est, int out_stride, cudaStream_t stream);
// Sharded fused exchange (T+A): per (rank, sequence, head) a slot of ta_slot(k) words holding the rank's local
// top-k entries (est, id, logit), their value rows and the rank's hot-row partial; one all-gather, then a
// replicated merge + attention.
constexpr int TA_MAXK = 256;
int64_t ta_slot(int k);
cudaError_t launch_ta_pack(const pkv_index* ix, const int32_t* lidx, const float* lest, int k, const void* q,
                           const void* K, const void* V, int64_t sb, int64_t sh, int64_t st, float scale, int64_t off,
                           const void* K_hot, const void* V_hot, int n_hot, uint32_t* msg, cudaStream_t stream);
cudaError_t launch_ta_merge(const pkv_index* ix, const uint32_t* msg, int P, int k, int32_t* out_idx, float* out_est,
                            void* out, float* lse, cudaStream_t stream);
cudaError_t launch_topk_merge(const pkv_index* ix, int P, int k, const float* all_est, const int32_t* all_idx,
                              int64_t rank_stride, int32_t* out_idx, float* out_est, cudaStream_t stream);
cudaError_t launch_dbg_cand(const pkv_index* ix, int64_t C, int32_t* dbg_cand, float* dbg_est,
                            cudaStream_t stream);

struct AttendArgs {
  const void* q;
  const void* K;
  const void* V;
  int64_t sb, sh, st;
  const int32_t* idx;
  int k;
  const void* K_hot;
  const void* V_hot;
  int n_hot;
  float scale;
  int64_t own_lo, own_hi;  // global ids owned by this shard
  int64_t id_offset;       // local row = id - id_offset
  int hot_rows;            // row capacity of a (sequence, KV head) block of the hot rows (>= n_hot)
};
int plan_attend_splits(const pkv_index* ix, int total_rows);
// ticket != nullptr: the last CTA of each (sequence, KV head) also does the LSE merge into out/lse.
cudaError_t launch_attend_partial(const pkv_index* ix, const AttendArgs& a, int splits, float* part_out,
                                  unsigned int* ticket, void* out, float* lse, cudaStream_t stream);
// out_idx = -1, out_est = -inf for `count` entries (retrieval over an empty zone)
cudaError_t launch_fill_empty_topk(int32_t* out_idx, float* out_est, int64_t count, cudaStream_t stream);
cudaError_t launch_attend_combine(const pkv_index* ix, const float* parts, int nsplits, int P, void* out,
                                  float* lse, cudaStream_t stream);

}  // namespace pkv
