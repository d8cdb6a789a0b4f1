/*
 * pariskv.h — C ABI of the B200 (sm_100a) ParisKV decode-time KV-cache retrieval hot path.
 *
 * ParisKV: "Fast and Drift-Robust KV-Cache Retrieval for Long-Context LLMs" (arXiv 2602.07721).
 * Citations: P:n = PAPER.md line n (section / equation), S:n = SPEC.md line n, AMB-x = a reading of
 * the paper listed in DESIGN.md.
 *
 * The four calls of the hot path:
 *   encode_keys          prefill key summarisation (§4.1)
 *   append_decode_keys   sliding-window flush: encode evicted keys and append them
 *   retrieve_topk        per decode step: query prep, collision voting, bucket_topk, RSQ-IP rerank,
 *                        final top-k (Eq. 10)
 *   sparse_attend        attention over hot rows U retrieved rows, K/V in HBM or pinned host memory
 *                        read through UVA (Eq. 2-3)
 *
 * Conventions shared by every entry point
 *   - Every function returns pkv_status (0 = PKV_OK). No C++ exception crosses the ABI.
 *     pkv_last_error() returns a thread-local message for the last non-OK status.
 *   - Argument errors (PKV_ERR_INVALID_ARG, PKV_ERR_CAPACITY) are detected on the host before any work
 *     is enqueued: a failing call has no side effect.
 *   - Ownership: the caller owns every input and output buffer (q, K, V, hot rows, idx, est, out, lse) and
 *     keeps it alive until the stream work completes. The library owns the index metadata (centroid ids,
 *     4-bit codes, weights), the per-index workspace and the NCCL communicator.
 *   - Streams: all device work is enqueued on the caller's stream. retrieve_topk and sparse_attend perform
 *     no host synchronisation and no allocation, so they can be captured in a CUDA graph.
 *     Asynchronous device faults surface at the caller's next synchronisation (PKV_ERR_CUDA is returned
 *     only for launch-time errors).
 *   - Dtypes: K, V, q and hot rows are bf16 (reading AMB-21). Head dim D = 128, B = 16 subspaces of
 *     m = 8 dimensions, 256 centroids per subspace (the paper's default).
 *   - Strided K/V layout: element (b, h, t, d) of a [batch][n_kv][tokens][D] tensor is at
 *     base + b*sb + h*sh + t*st + d (strides in ELEMENTS; d is contiguous). sb, sh, st must be multiples
 *     of 8 and base 16-byte aligned (16-byte vector loads).
 *   - GQA: query head h reads KV head h / (n_q_heads / n_kv_heads); retrieval is per query head (AMB-13).
 */
#ifndef PARISKV_H
#define PARISKV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* cudaStream_t;

typedef enum {
  PKV_OK = 0,
  PKV_ERR_INVALID_ARG = -1, /* bad pointer, shape, stride, alignment or parameter                 */
  PKV_ERR_CAPACITY = -2,    /* append would exceed the index capacity (no partial append)          */
  PKV_ERR_CUDA = -3,        /* CUDA runtime / launch error                                         */
  PKV_ERR_UNSUPPORTED = -4, /* configuration this build does not implement (e.g. D != 128)         */
  PKV_ERR_NCCL = -5         /* NCCL error in a sequence-sharded call                                */
} pkv_status;

#define PKV_HEAD_DIM 128
#define PKV_SUBSPACES 16
#define PKV_SUBSPACE_DIM 8
#define PKV_CENTROIDS 256
#define PKV_MAX_TIERS 8

/* Offline constants ("an analytic centroid codebook and a quantization configuration").
 * Fill with pkv_config_init; fields may then be edited (tiers) before pkv_index_create copies it. */
typedef struct {
  int32_t head_dim;                  /* D = 128 (only value supported)                                   */
  int32_t n_subspaces;               /* B = 16                                            */
  int32_t subspace_dim;              /* m = D/B = 8                                                      */
  int32_t n_q_heads;                 /* query heads per sequence (e.g. 32)                               */
  int32_t n_kv_heads;                /* KV heads per sequence (e.g. 8); n_q_heads % n_kv_heads == 0, the  */
                                     /* GQA group G = n_q/n_kv must be <= 4 (4 heads share a packed u32) */
  int32_t n_tiers;                   /* multi-tier collision bonus: 6                             */
  int32_t tier_bonus[PKV_MAX_TIERS]; /* bonus per tier, strictly decreasing, e.g. {6,5,4,3,2,1} (AMB-10) */
  float mag_levels[8];               /* Prop. 1 magnitude levels L0<...<L7 (AMB-5), fp32       */
  double mag_mid_sq[7];              /* M_t = ((L_{t-1}+L_t)/2)^2 in fp64, exact from the fp32 levels     */
  uint8_t rot_sign[PKV_HEAD_DIM];    /* SRHT sign diagonal s_j: 0 -> +1, 1 -> -1 (AMB-1)          */
  int32_t rot_rounds;                /* 1 (only value supported)                                         */
  int32_t w_fp16;                    /* rerank weight precision (AMB-20): 0 = fp32 w' in a */
                                     /* 128-byte record (default); 1 = fp16 w' with a per-key power-of-two */
                                     /* scale 2^E (E in [-126,126], kept in the 16 free sign bits) in a    */
                                     /* 96-byte record. Estimates then carry an extra relative error of at */
                                     /* most 2^-11 per subspace term (AMB-20)                */
} pkv_config;

/* Fill cfg with the paper defaults: D=128, B=16, m=8, 6 tiers {6..1}, Prop. 1 levels for m=8 computed on
 * the host (conditional means of |u_j| over 8 equal-probability bins of u_j^2 ~ Beta(1/2,(m-1)/2)),
 * the given head counts and the caller's 128 rotation sign bits (the harness draws them from a seed).
 * Host-only; no device is touched. */
pkv_status pkv_config_init(pkv_config* cfg, int32_t n_q_heads, int32_t n_kv_heads, const uint8_t* rot_sign);

/* Adaptive (rho, beta) schedule vs retrieval-zone length n (reading AMB-11 = S:329 in basis points):
 * T = ceil(rho*256) probes per subspace, C = min(n, max(min(top_k, n), ceil(beta*n))). Host-only. */
pkv_status pkv_schedule(int64_t n, int32_t top_k, int32_t* probes_T, int64_t* n_cand);

/* ---------------------------------------------------------------------------------------------------
 * Index: GPU-resident key summaries of the retrieval zone of `batch` sequences x n_kv_heads KV heads
 * (centroid ids, 4-bit codes, w). Per key and KV head: 16 B of centroid ids + a 128 B rerank
 * record (64 B packed nibbles + 16 fp32 weights). Device memory is allocated on `device` at creation for
 * `capacity` keys per (sequence, KV head), together with the retrieval workspace.
 * ------------------------------------------------------------------------------------------------- */
typedef struct pkv_index pkv_index;

pkv_status pkv_index_create(const pkv_config* cfg, int32_t batch, int64_t capacity, int32_t device,
                            pkv_index** out);
pkv_status pkv_index_destroy(pkv_index* index);
/* Number of keys per (sequence, KV head) currently in the retrieval zone. */
pkv_status pkv_index_len(const pkv_index* index, int64_t* n_out);
/* Let `index` use `donor`'s retrieval workspace instead of its own (frees its own). Both indices must
 * have the same config head counts and batch, and donor capacity >= index capacity. Work on the two
 * indices must then be serialised (e.g. one stream for all layers). */
pkv_status pkv_index_share_workspace(pkv_index* index, pkv_index* donor);

/* (1) encode_keys — prefill (§4.1): encode tokens [0, n) of K (device bf16, layout above,
 * tokens = retrieval-zone positions) and make them the index content (replaces previous content).
 * Per key: y' = H (s (.) k) exactly (integer / fp64 Walsh-Hadamard butterflies), centroid id per subspace
 * = sign pattern (Eq. 6), 3-bit magnitude by the midpoint rule on the Prop. 1 levels (AMB-5), sign bit,
 * and w_b = ||k|| r_b / alpha_b (Eq. 7, 9) stored pre-divided by ||sign*L[idx]|| (AMB-6).
 * Errors: INVALID_ARG (null/misaligned K, n < 0), CAPACITY (n > capacity). */
pkv_status encode_keys(pkv_index* index, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t n,
                       cudaStream_t stream);

/* (2) append_decode_keys — decode flush: encode t more keys (same layout, token 0 of K is
 * the new key at retrieval position n) and append them at positions [n, n+t). CAPACITY if n+t > capacity
 * (nothing appended). */
pkv_status append_decode_keys(pkv_index* index, const void* K, int64_t sb, int64_t sh, int64_t st, int64_t t,
                              cudaStream_t stream);

/* Parameters of one retrieval. probes_T and n_cand come from pkv_schedule(n_global, top_k, ...) on the
 * host (the GLOBAL retrieval length when sequence-sharded). Optional debug outputs (device pointers,
 * NULL = not written) expose intermediate results for parity tests. */
typedef struct {
  int32_t probes_T;     /* T in [1, 256]                                                             */
  int64_t n_cand;       /* C in [0, n] (global n when sharded)                                      */
  int32_t top_k;        /* k >= 1                                                                     */
  uint8_t* dbg_scores;  /* [batch][n_q][n_local] collision scores                              */
  int32_t* dbg_cand;    /* [batch][n_q][n_cand] candidate ids (global), set semantics, -1 padded      */
  float* dbg_est;       /* [batch][n_q][n_cand] RSQ-IP estimate aligned with dbg_cand                  */
  float* dbg_q_rot;     /* [batch][n_q][D] rotated unit query q~ = R q/||q||               */
  int64_t n_global;     /* sequence-sharded calls: the global retrieval length n_cand is checked against; */
                        /* <= 0 takes the communicator's record (pkv_comm_init / pkv_comm_set_global_len). */
                        /* Ignored by unsharded calls (the index length is used).                        */
  int64_t rho_keys;     /* 0: rho read as a fraction of CENTROIDS, T = probes_T probes per subspace      */
                        /* (AMB-8). > 0: the KEY-fraction reading (AMB-8b, "only let the     */
                        /* top-rho fraction contribute a non-zero bonus", "scales with rho n"): per */
                        /* (query head, subspace) the centroids are probed in rank order until they hold */
                        /* >= rho_keys indexed keys (pkv_schedule_key_fraction gives ceil(rho n)); the 6 */
                        /* tiers split that subspace's probe count T_b as AMB-10 splits T. Needs         */
                        /* pkv_index_set_occupancy(index, 1); in [0, n]; UNSUPPORTED when sharded.       */
} pkv_retrieve_params;

/* (3) retrieve_topk — per decode step. q: device bf16 [batch][n_q][D] contiguous.
 * Outputs (device): out_idx int32 [batch][n_q][top_k] retrieval-zone token ids (global ids when sharded),
 * ordered by estimate descending, ties -> larger id, padded with -1 when n < top_k;
 * out_est fp32 [batch][n_q][top_k] the RSQ-IP estimate of <k, q> (Eq. 10, includes ||q||, AMB-14),
 * -inf where padded. Requires n >= 1 and n_cand >= min(top_k, n). */
pkv_status retrieve_topk(pkv_index* index, const void* q, const pkv_retrieve_params* params, int32_t* out_idx,
                         float* out_est, cudaStream_t stream);

/* (4) sparse_attend — Eq. 2-3 over C(q) = hot rows U {retrieval rows idx[0..k), idx >= 0}:
 * logits = <k_i, q> * scale in fp32 from the full-precision bf16 rows, softmax, o = sum p_i v_i.
 * q: device bf16 [batch][n_q][D]. K, V: retrieval-zone rows in the strided layout above; they may be
 * device pointers or pointers into cudaHostAllocMapped / cudaHostRegister'ed pinned host memory, read by
 * the kernel through UVA — no copy is made. idx: device int32 [batch][n_q][k] (from
 * retrieve_topk; -1 entries skipped; ids must be distinct per row). K_hot, V_hot: device bf16
 * [batch][n_kv][n_hot][D] contiguous (sink + local + update buffer), may be NULL when
 * n_hot == 0. out: device bf16 [batch][n_q][D]; lse: device fp32 [batch][n_q] = log sum exp(logits)
 * (natural log), may be NULL. When sequence-sharded, idx holds global ids, K/V are this rank's rows
 * (local row = id - shard_offset), hot rows are attended by the LAST rank only, and every rank receives
 * the merged output. INVALID_ARG if k < 0, n_hot < 0, both sets empty, or misaligned pointers. */
pkv_status sparse_attend(pkv_index* index, const void* q, const void* K, const void* V, int64_t sb, int64_t sh,
                         int64_t st, const int32_t* idx, int32_t k, const void* K_hot, const void* V_hot,
                         int32_t n_hot, float scale, void* out, float* lse, cudaStream_t stream);

/* (3)+(4) retrieve_and_attend — one decode step of one layer: exactly retrieve_topk followed by sparse_attend
 * with the same arguments (K/V rows strided as above, HBM or UVA), scheduled as one unit on the caller's
 * stream (CUDA-graph capturable, no host sync): the final top-k selection is fused with the gather and
 * attention of the selected rows and of the hot rows (sink + local + buffer), one thread-block
 * cluster per query head; the hot rows are attended before that kernel waits on the rerank kernel. out_idx/out_est are identical to retrieve_topk's; out/lse equal
 * sparse_attend's up to fp32 summation order. n_hot <= 1024. When sequence-sharded it calls the two entry
 * points. Ordering: K_hot/V_hot are read before the kernels wait on their stream predecessor's completion
 * (programmatic dependent launch), so a producer kernel that itself triggers early must not write them. */
pkv_status retrieve_and_attend(pkv_index* index, const void* q, const pkv_retrieve_params* params, const void* K,
                               const void* V, int64_t sb, int64_t sh, int64_t st, const void* K_hot,
                               const void* V_hot, int32_t n_hot, float scale, int32_t* out_idx, float* out_est,
                               void* out, float* lse, cudaStream_t stream);

/* retrieve_and_attend with hot rows stored with a row capacity hot_rows >= n_hot per (sequence, KV head):
 * hot row t of (b, h) at K_hot + ((b*n_kv + h)*hot_rows + t)*128 (the region manager's layout). Not
 * supported on a sequence-sharded index unless hot_rows == n_hot. */
pkv_status retrieve_and_attend_rows(pkv_index* index, const void* q, const pkv_retrieve_params* params,
                                    const void* K, const void* V, int64_t sb, int64_t sh, int64_t st,
                                    const void* K_hot, const void* V_hot, int32_t n_hot, int32_t hot_rows,
                                    float scale, int32_t* out_idx, float* out_est, void* out, float* lse,
                                    cudaStream_t stream);

/* Same for retrieve_and_attend (top_k <= 256): the fused exchange of SURVEY §8(f3) — per query head every
 * shard contributes its local top-k entries with their attention logits and value rows (and shard P-1 its
 * hot-row partial) to ONE exchange buffer; a replicated merge selects the global top-k exactly as
 * retrieve_topk does and attends the selected entries. A communicator-attached index takes the same path in
 * retrieve_and_attend (two collectives per layer: score histograms, then this exchange). */
pkv_status pkv_retrieve_and_attend_sharded_local(pkv_index* const* shards, const int64_t* offsets, int32_t P,
                                                const void* q, const void* const* Ks, const void* const* Vs,
                                                int64_t sb, int64_t sh, int64_t st,
                                                const pkv_retrieve_params* params, const void* K_hot,
                                                const void* V_hot, int32_t n_hot, float scale, int32_t* out_idx,
                                                float* out_est, void* out, float* lse, cudaStream_t stream);

/* ---------------------------------------------------------------------------------------------------
 * Streaming decode: the four-region KV cache of PAPER §4.2.3 "Buffer Update".
 *   Sink      the first `sink` tokens, kept on the GPU (full precision, always attended)
 *   Retrieval every older token: indexed (centroid ids, 4-bit codes, w) in `index`, full-precision K/V in a
 *             store owned by the stream — HBM, or pinned host memory read through UVA (offload setting)
 *   Local     the newest `local_size` tokens before the buffer, on the GPU, always attended
 *   Update    up to `update_size` newly generated tokens, on the GPU, always attended
 * Each decode token is appended to the Update buffer; when it holds update_size tokens the oldest tokens of
 * Local U Update beyond local_size are evicted into Retrieval: their keys are encoded and appended to the
 * index (append_decode_keys, on the GPU) and their K/V rows copied to the store, and the rest is shifted to
 * become the new Local. Retrieval ids returned by pkv_stream_decode are store positions:
 * retrieval id i is token sink + i of the sequence. All copies and kernels run on the caller's stream
 * (asynchronous to the host); decode steps without a flush are CUDA-graph capturable.
 * ------------------------------------------------------------------------------------------------- */
typedef struct pkv_stream pkv_stream; /* opaque */
typedef struct {
  int32_t sink;         /* 16 */
  int32_t local_size;   /* 256 (Table 1) */
  int32_t update_size;  /* 512 (Table 1 "Update"; the flush size m of P:458) */
  int32_t offload_host; /* 0: retrieval K/V in HBM; 1: in pinned host memory (UVA reads) */
} pkv_stream_config;
/* Create a stream over `index` (which it uses but does not own; its capacity bounds the retrieval zone).
 * Allocates the hot buffer [batch][n_kv][sink + local_size + update_size][128] bf16 (K and V) and the
 * retrieval store [batch][n_kv][capacity][128] bf16 (K and V). Errors: INVALID_ARG (sizes < 0, sink +
 * local_size + update_size > 1024 or update_size < 1), CUDA (allocation). */
pkv_status pkv_stream_create(pkv_index* index, const pkv_stream_config* config, pkv_stream** out);
pkv_status pkv_stream_destroy(pkv_stream* s);
/* Prefill with n_tokens >= sink tokens (K, V device bf16, element (b,h,t,d) at base + b*sb + h*sh + t*st + d):
 * tokens [0, sink) -> Sink, the newest min(local_size, n_tokens - sink) -> Local, the rest -> Retrieval
 * (encode_keys + store copy). Replaces any previous content. Errors: INVALID_ARG, CAPACITY. */
pkv_status pkv_stream_prefill(pkv_stream* s, const void* K, const void* V, int64_t sb, int64_t sh, int64_t st,
                              int64_t n_tokens, cudaStream_t stream);
/* One decode step of this layer: append (k_new, v_new) (device bf16 [batch][n_kv][128]) to the Update buffer,
 * flush when it is full, then retrieve_and_attend with q over Sink U Local U Update (hot rows) and the
 * retrieved rows of the store. params: probes_T/n_cand <= 0 take the schedule for the current retrieval
 * length (pkv_schedule). Outputs as retrieve_and_attend. CAPACITY if a flush would overflow the index (no
 * side effect). */
pkv_status pkv_stream_decode(pkv_stream* s, const void* q, const void* k_new, const void* v_new,
                             const pkv_retrieve_params* params, float scale, int32_t* out_idx, float* out_est,
                             void* out, float* lse, cudaStream_t stream);
/* Region sizes: retrieval tokens, local tokens, buffered tokens, and the retrieval store's device-visible
 * K/V base pointers ([batch][n_kv][capacity][128] bf16) and hot buffer pointers. Any output may be NULL. */
pkv_status pkv_stream_state(const pkv_stream* s, int64_t* n_retrieval, int32_t* n_local, int32_t* n_buffer,
                            const void** K_store, const void** V_store, const void** K_hot, const void** V_hot);

/* Inverted-list collision variant ("collision processing scales with rho*n"): with
 * enable = 1 the index also keeps, per chunk of 8192 keys and per subspace, its keys bucketed by centroid id
 * (32 B per key and KV head, built now and maintained by encode_keys / append_decode_keys), and retrievals
 * visit only the buckets of probed centroids instead of scanning every key's 16 ids. Scores, candidates and
 * results are identical to the dense scan's. enable = 0 returns to the dense scan (buffers are kept).
 * Errors: UNSUPPORTED if the capacity exceeds 256 chunks (2,097,152 keys), CUDA on allocation failure. */
pkv_status pkv_index_set_postings(pkv_index* index, int32_t enable, cudaStream_t stream);

/* Key-fraction reading of rho: enable = 1 allocates the per-(sequence, KV head,
 * subspace) centroid occupancy histogram (16 x 256 u32 counts: how many indexed keys carry each centroid id),
 * counts the current retrieval zone on `stream`, and keeps it current on every later encode_keys /
 * append_decode_keys; enable = 0 frees it. Required by retrieve calls with rho_keys > 0. */
pkv_status pkv_index_set_occupancy(pkv_index* index, int32_t enable, cudaStream_t stream);

/* rho_keys = ceil(rho * n) with rho from the same (rho, beta) schedule as pkv_schedule (AMB-11). */
pkv_status pkv_schedule_key_fraction(int64_t n, int64_t* rho_keys);

/* Degenerate-key accounting (AMB-7; replaces the per-key API error of S:89): keys whose rotated
 * subspace b has S_b = 0 get the deterministic encoding of e_1 in that subspace (id 0xFF, w_b = 0) and are
 * counted on the device by the encoder. Counts cover the current index content (encode_keys resets them,
 * append_decode_keys adds). pkv_index_get_stats enqueues a copy on `stream` and synchronises that stream. */
typedef struct {
  int64_t n_keys;                  /* keys per (sequence, KV head) in the retrieval zone (= pkv_index_len)   */
  int64_t zero_keys;               /* keys (over all sequences and KV heads) that are entirely zero         */
  int64_t keys_with_zero_subspace; /* keys with at least one subspace of S_b = 0 (includes zero_keys)       */
  int64_t zero_subspaces;          /* total (key, subspace) pairs with S_b = 0                              */
} pkv_index_stats;
pkv_status pkv_index_get_stats(const pkv_index* index, pkv_index_stats* out, cudaStream_t stream);

/* Test hook: when out_f32 != NULL every later attention call on this index (sparse_attend,
 * retrieve_and_attend[_rows], the sharded paths — shard 0's pointer in the *_sharded_local emulation) also
 * writes the fp32 attention output, before its bf16 rounding, to out_f32 (device [batch][n_q][D]). The
 * caller keeps the buffer alive; NULL disables. Lets parity tests check the fp32 accumulation against the
 * 2e-3 bar apart from the bf16 rounding of `out` (AMB-17). Host-only. */
pkv_status pkv_index_set_debug_output(pkv_index* index, float* out_f32);

/* Diagnostics: copy metadata of positions [start, start+count) into caller device buffers in the
 * canonical layout: ids uint8 [batch][n_kv][count][16] (subspace order), codes uint8
 * [batch][n_kv][count][64] (coordinate c -> byte c>>1, low nibble for even c; nibble = sign<<3 | idx),
 * w fp32 [batch][n_kv][count][16] = w_b / ||sign*L[idx]||_b (the stored weight, AMB-6). Any pointer may
 * be NULL. */
pkv_status pkv_index_export(const pkv_index* index, int64_t start, int64_t count, uint8_t* ids, uint8_t* codes,
                            float* w, cudaStream_t stream);

/* ---------------------------------------------------------------------------------------------------
 * Sequence sharding across GPUs (not in the paper, which is single-GPU).
 * Rank r owns retrieval positions [shard_offset, shard_offset + n_local) of every sequence/KV head in its
 * own index. After pkv_comm_init, retrieve_topk and sparse_attend exchange three small messages per call
 * over NCCL on the caller's stream: per-head score histograms, local top-k lists and partial softmax
 * states, and return the same results as an unsharded index over the concatenated shards.
 * ------------------------------------------------------------------------------------------------- */
/* 128-byte NCCL unique id, to be broadcast from rank 0 to all ranks by the caller. */
pkv_status pkv_nccl_unique_id(uint8_t out[128]);
/* Attach an NCCL communicator to `index` (collective over `world` ranks; call on every rank; also sums the
 * ranks' current index lengths into the global length, one synchronous exchange). */
pkv_status pkv_comm_init(pkv_index* index, const uint8_t id[128], int32_t rank, int32_t world,
                         int64_t shard_offset);
/* Host-staged transport (for CPU process groups such as gloo, tests, and several ranks sharing one GPU, where
 * NCCL cannot run): fn performs an all-gather in HOST memory — buf holds `world` slots of bytes_per_rank
 * bytes, slot `rank` holds this rank's contribution on entry, and on return every slot must hold its rank's
 * contribution; fn returns 0 on success (any other value -> PKV_ERR_NCCL). Each exchange then copies the
 * rank's slot to pinned host memory, synchronises the stream, calls fn and copies all slots back: results
 * are identical to the NCCL transport, but calls synchronise and are not graph-capturable. Collective over
 * `world` ranks (every rank calls it); it also sums the ranks' current index lengths into the global length. */
typedef int32_t (*pkv_host_allgather_fn)(void* ctx, void* buf, size_t bytes_per_rank, int32_t rank, int32_t world);
pkv_status pkv_comm_init_host(pkv_index* index, pkv_host_allgather_fn fn, void* ctx, int32_t rank, int32_t world,
                              int64_t shard_offset);
/* Peer transport: the exchanges become one-shot all-gather kernels over peer memory — each rank
 * stores its slot straight into every peer's symmetric "arena" (NVLink stores on an NVSwitch system), raises
 * per-CTA flags there and waits for the peers' flags in its own arena: no NCCL call and no host involvement per
 * exchange, stream-ordered and CUDA-graph capturable (peer.cu). Two steps, both on every rank:
 *   pkv_comm_init_peer: allocates this rank's arena (arena_bytes >= 8192 + 2 * world * the largest exchange
 *     message; 64 MB covers batch 8 x 32 query heads) and attaches the communicator; returns the arena's
 *     CUDA IPC handle (ipc_handle, 64 bytes, may be NULL) and its device pointer (arena, may be NULL);
 *   pkv_comm_peer_connect: opens the peers' IPC handles (ipc_handles = world x 64 bytes, this rank's ignored),
 *     for ranks in different processes; or pkv_comm_peer_connect_local with the world arena pointers, for
 *     ranks in one process.
 * The global retrieval length is not exchanged at attach: set it with pkv_comm_set_global_len or pass
 * pkv_retrieve_params.n_global. Every rank must issue the same sequence of sharded calls (the exchanges
 * pair up by order); ranks that share one GPU must run their streams concurrently and keep grids small enough
 * to co-reside (the exchange kernel of one rank spins until the others arrive). */
pkv_status pkv_comm_init_peer(pkv_index* index, int32_t rank, int32_t world, int64_t shard_offset,
                              size_t arena_bytes, uint8_t ipc_handle[64], void** arena);
pkv_status pkv_comm_peer_connect(pkv_index* index, const uint8_t* ipc_handles);
pkv_status pkv_comm_peer_connect_local(pkv_index* index, void* const* arenas);
/* Global retrieval length recorded by the communicator (validation of n_cand in sharded calls). pkv_comm_init
 * and pkv_comm_init_host set it to the sum of the ranks' lengths at attach time; after appends on any rank the
 * caller updates it here on every rank, or passes pkv_retrieve_params.n_global per call. */
pkv_status pkv_comm_set_global_len(pkv_index* index, int64_t n_global);
/* Attach `donor`'s communicator to `index` as well (e.g. one communicator for all layers of a model). The
 * two indices must then be used from the same stream order on every rank. */
pkv_status pkv_comm_share(pkv_index* index, pkv_index* donor, int64_t shard_offset);
/* Single-process emulation for tests: treat `shards[0..P)` (indices on the SAME device, shard p owning
 * positions [offsets[p], offsets[p]+n_p)) as one sharded index and run the sharded algorithm with the
 * exchanges done by device copies. Inputs and outputs as retrieve_topk (out_idx/out_est written once). */
pkv_status pkv_retrieve_topk_sharded_local(pkv_index* const* shards, const int64_t* offsets, int32_t P,
                                           const void* q, const pkv_retrieve_params* params, int32_t* out_idx,
                                           float* out_est, cudaStream_t stream);
/* Same for sparse_attend: Ks[p], Vs[p] are shard p's rows (local row = id - offsets[p]); hot rows belong
 * to shard P-1. */
pkv_status pkv_sparse_attend_sharded_local(pkv_index* const* shards, const int64_t* offsets, int32_t P,
                                           const void* q, const void* const* Ks, const void* const* Vs,
                                           int64_t sb, int64_t sh, int64_t st, const int32_t* idx, int32_t k,
                                           const void* K_hot, const void* V_hot, int32_t n_hot, float scale,
                                           void* out, float* lse, cudaStream_t stream);

/* ---------------------------------------------------------------------------------------------------
 * Append rebalancing across sequence shards (not in the paper). Decode appends (one
 * update_size flush per 512 steps) land on the last rank, whose shard grows. A boundary shift moves the `count`
 * OLDEST keys of shard r+1 to the END of shard r: both shards stay contiguous and ordered by position, so the
 * sharded select's newest-rank-first tie rule (AMB-12) and all sharded results are unchanged (bit-identical to
 * the unsharded index). The caller moves the matching K/V rows the same way (local row = id - shard_offset).
 * The index's degenerate-key statistics (pkv_index_get_stats) count the keys encoded INTO that index and are
 * not moved. Postings / occupancy tables, when enabled, are rebuilt.
 * ------------------------------------------------------------------------------------------------- */
/* Bytes of one key's exchange entry over all sequences and KV heads: batch * n_kv * (16 + record bytes). An
 * entry buffer of `count` keys is laid out [batch][n_kv][count] x (canonical 16-byte centroid-id row — subspace
 * b in byte b — followed by the key's record). */
pkv_status pkv_index_entry_bytes(const pkv_index* index, int64_t* bytes_per_key);
/* Write the entries of keys [0, count) of `index` (its oldest) into the device buffer `buf` (count *
 * pkv_index_entry_bytes bytes, caller-owned, on the index's device). Stream-ordered; the index is unchanged.
 * INVALID_ARG: count outside [0, n] or null buffer. */
pkv_status pkv_index_export_front(const pkv_index* index, int64_t count, void* buf, cudaStream_t stream);
/* Append `count` entries from the device buffer `buf` after the index's newest key (they become keys
 * [n, n + count)). CAPACITY if n + count exceeds the capacity (nothing changes). */
pkv_status pkv_index_import_back(pkv_index* index, const void* buf, int64_t count, cudaStream_t stream);
/* Remove keys [0, count): the rest move down by count (stream-ordered scratch copy) and shard_offset grows by
 * count. INVALID_ARG: count outside [0, n]. */
pkv_status pkv_index_drop_front(pkv_index* index, int64_t count, cudaStream_t stream);
/* Both indices on one device (same batch, KV heads, record format and rotation): export_front(newer) +
 * import_back(older) + drop_front(newer) through a stream-ordered buffer. Across GPUs the caller runs the three
 * steps on the two ranks and moves the buffer between them (NCCL send/recv, a peer copy). */
pkv_status pkv_index_shift_boundary(pkv_index* older, pkv_index* newer, int64_t count, cudaStream_t stream);
/* Host-only policy: for P contiguous shards of lengths[0..P), shift[r] (r < P-1) = keys to move from shard r+1 to
 * shard r so that every boundary moves right, by whole `granule`s, towards the balanced position r*N/P (never
 * left; boundaries stay ordered). Apply shift[P-2] first and shift[0] last. Touches no device. */
pkv_status pkv_rebalance_plan(const int64_t* lengths, int32_t P, int64_t granule, int64_t* shift);

/* Total number of kernels this library has launched in the process (host-side counter, for launch
 * accounting in bench.py; graph replays are not counted). */
pkv_status pkv_launch_count(uint64_t* total);
/* Optional per-kernel timing for benchmarks: when enabled, every kernel launch is bracketed by two CUDA
 * events on its stream (eager launches only; do not enable while capturing a graph). pkv_profile_read
 * synchronises and returns the launch count and summed device time of one kernel kind; kinds are numbered
 * 0..12 = encode, qprep, scan, select, (unused), rerank, topk, topk_merge, attend, combine, head_hist,
 * export, debug (pkv_kernel_name). Enabling or disabling resets the counters. */
pkv_status pkv_profile_enable(int32_t on);
pkv_status pkv_profile_read(int32_t kind, int64_t* launches, double* total_ms);
const char* pkv_kernel_name(int32_t kind);
/* Library build/version string. */
const char* pkv_version(void);
const char* pkv_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PARISKV_H */
