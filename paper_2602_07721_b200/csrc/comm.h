// Sequence-sharded exchange over NCCL. Host side only.
#pragma once

#include "internal.h"

namespace pkv {

pkv_status comm_unique_id(uint8_t out[128]);
pkv_status comm_init(pkv_index* ix, const uint8_t id[128], int rank, int world, int64_t shard_offset);
void comm_destroy(Comm* c);
pkv_status comm_share(pkv_index* ix, pkv_index* donor, int64_t shard_offset);
// In-place all-gather of `slot` u32 words per rank: buf[r*slot .. (r+1)*slot) is rank r's contribution.
pkv_status comm_allgather_u32(pkv_index* ix, uint32_t* buf, size_t slot, cudaStream_t stream);
// Global retrieval length is the caller's business when sharded (T and C come from the host schedule on
// the global length); validation then only bounds-checks against INT64_MAX.
int64_t comm_global_n(const pkv_index* ix);

}  // namespace pkv
