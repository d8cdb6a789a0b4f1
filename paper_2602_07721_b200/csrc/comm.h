// Sequence-sharded exchange: NCCL, or a caller-supplied host all-gather. Host side only.
#pragma once

#include "internal.h"

namespace pkv {

pkv_status comm_unique_id(uint8_t out[128]);
pkv_status comm_init(pkv_index* ix, const uint8_t id[128], int rank, int world, int64_t shard_offset);
pkv_status comm_init_host(pkv_index* ix, pkv_host_allgather_fn fn, void* ctx, int rank, int world,
                          int64_t shard_offset);
pkv_status comm_init_peer(pkv_index* ix, int rank, int world, int64_t shard_offset, size_t arena_bytes,
                          uint8_t ipc_handle[64], void** arena_out);
pkv_status comm_peer_connect(pkv_index* ix, const uint8_t* handles, void* const* arenas);
void comm_destroy(Comm* c);
pkv_status comm_share(pkv_index* ix, pkv_index* donor, int64_t shard_offset);
// In-place all-gather of `slot` u32 words per rank: buf[r*slot .. (r+1)*slot) is rank r's contribution.
pkv_status comm_allgather_u32(pkv_index* ix, uint32_t* buf, size_t slot, cudaStream_t stream);
// Global retrieval length of a sharded call: params->n_global when > 0, else the length recorded by the
// communicator (summed over the ranks at init, or set with pkv_comm_set_global_len); -1 if unknown.
int64_t comm_global_n(const pkv_index* ix, const pkv_retrieve_params* p);
pkv_status comm_set_global_len(pkv_index* ix, int64_t n_global);

}  // namespace pkv
