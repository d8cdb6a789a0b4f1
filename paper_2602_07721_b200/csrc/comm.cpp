// NCCL plumbing for the sequence-sharded retrieval. Three in-place all-gathers per
// layer and decode step, all on the caller's stream: (H) per-head score histograms, (T) local top-k lists,
// (A) partial softmax states. The unique id is produced here and broadcast by the caller (torch.distributed).
#include <nccl.h>

#include <cstring>

#include <string>

#include "comm.h"

namespace pkv {

struct Comm {
  ncclComm_t comm = nullptr;
  int refs = 1;
};

static pkv_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return PKV_OK;
  return set_error(PKV_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

pkv_status comm_unique_id(uint8_t out[128]) {
  if (!out) return set_error(PKV_ERR_INVALID_ARG, "pkv_nccl_unique_id: null");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  pkv_status s = nccl_status(ncclGetUniqueId(&id), "ncclGetUniqueId");
  if (s != PKV_OK) return s;
  std::memcpy(out, &id, 128);
  return PKV_OK;
}

pkv_status comm_init(pkv_index* ix, const uint8_t id_bytes[128], int rank, int world, int64_t shard_offset) {
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, 128);
  Comm* c = new Comm();
  pkv_status s = nccl_status(ncclCommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  if (s != PKV_OK) {
    delete c;
    return s;
  }
  comm_destroy(ix->comm);
  ix->comm = c;
  ix->rank = rank;
  ix->world = world;
  ix->shard_offset = shard_offset;
  return PKV_OK;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (--c->refs > 0) return;
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
}

pkv_status comm_share(pkv_index* ix, pkv_index* donor, int64_t shard_offset) {
  if (!donor->comm) return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_share: donor has no communicator");
  if (ix->comm == donor->comm) {
    ix->shard_offset = shard_offset;
    return PKV_OK;
  }
  comm_destroy(ix->comm);
  ix->comm = donor->comm;
  ix->comm->refs++;
  ix->rank = donor->rank;
  ix->world = donor->world;
  ix->shard_offset = shard_offset;
  return PKV_OK;
}

pkv_status comm_allgather_u32(pkv_index* ix, uint32_t* buf, size_t slot, cudaStream_t stream) {
  return nccl_status(ncclAllGather(buf + ix->rank * slot, buf, slot, ncclUint32, ix->comm->comm, stream),
                     "ncclAllGather");
}

int64_t comm_global_n(const pkv_index* ix) {
  (void)ix;
  return INT64_MAX;
}

}  // namespace pkv
