// Exchange plumbing for the sequence-sharded retrieval. Per layer and decode step the library
// all-gathers (H) per-head score histograms and then either (T) local top-k lists and (A) partial softmax
// states, or the fused T+A message — all in place in one device buffer on the caller's stream.
// Two transports:
//   NCCL  (pkv_comm_init): ncclAllGather over NVLink; stream-ordered and CUDA-graph capturable. The unique id
//         is produced here and broadcast by the caller (torch.distributed).
//   host  (pkv_comm_init_host): the caller's host all-gather (e.g. a gloo process group): the rank's slot is
//         copied to pinned host memory, the stream synchronised, the callback run, and all slots copied back.
//         Synchronous, not capturable — for CPU process groups, tests, and ranks that share one GPU.
//   peer  (pkv_comm_init_peer + pkv_comm_peer_connect[_local]): a one-shot all-gather kernel that stores the
//         rank's slot straight into every peer's symmetric arena over NVLink (peer.cu).
#include <nccl.h>

#include <cstring>

#include <string>

#include "comm.h"

namespace pkv {

struct Comm {
  ncclComm_t comm = nullptr;
  pkv_host_allgather_fn host_fn = nullptr;
  void* host_ctx = nullptr;
  void* stage = nullptr;  // pinned host staging buffer of the host transport
  size_t stage_bytes = 0;
  int rank = 0, world = 1;
  int64_t global_n = -1;
  int refs = 1;
  // peer transport
  char* arena = nullptr;            // this rank's symmetric arena (cudaMalloc)
  size_t arena_bytes = 0;
  char* peers[MAX_RANKS] = {};      // every rank's arena as seen from this process (peers[rank] == arena)
  bool opened[MAX_RANKS] = {};      // peers[r] came from cudaIpcOpenMemHandle
  bool connected = false;
};

cudaError_t launch_peer_allgather(char* const* arenas, int rank, int world, uint32_t* buf, size_t words, size_t half,
                                  cudaStream_t stream);
size_t peer_header_bytes();

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

static pkv_status raw_allgather(Comm* c, void* buf, size_t bytes, cudaStream_t stream) {
  if (c->arena) {
    if (!c->connected) return set_error(PKV_ERR_INVALID_ARG, "peer exchange: pkv_comm_peer_connect first");
    const size_t half = (c->arena_bytes - peer_header_bytes()) / 2;
    if ((bytes & 3) || bytes * c->world > half)
      return set_error(PKV_ERR_CAPACITY, "peer exchange: message larger than the arena (pkv_comm_init_peer)");
    return cuda_status(launch_peer_allgather(c->peers, c->rank, c->world, static_cast<uint32_t*>(buf), bytes / 4, half,
                                             stream),
                       "peer all-gather");
  }
  if (c->comm)
    return nccl_status(ncclAllGather(static_cast<char*>(buf) + c->rank * bytes, buf, bytes, ncclChar, c->comm, stream),
                       "ncclAllGather");
  const size_t total = bytes * c->world;
  if (c->stage_bytes < total) {
    if (c->stage) cudaFreeHost(c->stage);
    c->stage = nullptr;
    c->stage_bytes = 0;
    if (cudaMallocHost(&c->stage, total) != cudaSuccess) return set_error(PKV_ERR_CUDA, "host exchange staging");
    c->stage_bytes = total;
  }
  char* h = static_cast<char*>(c->stage);
  cudaError_t e = cudaMemcpyAsync(h + c->rank * bytes, static_cast<char*>(buf) + c->rank * bytes, bytes,
                                  cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_status(e, "host exchange (device to host)");
  if (c->host_fn(c->host_ctx, h, bytes, c->rank, c->world) != 0)
    return set_error(PKV_ERR_NCCL, "host all-gather callback failed");
  e = cudaMemcpyAsync(buf, h, total, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // the staging buffer is reused by the next exchange
  return cuda_status(e, "host exchange (host to device)");
}

// Global length at attach time: all-gather of every rank's local length (one synchronous exchange).
static pkv_status reduce_global_n(Comm* c, int64_t local_n) {
  int64_t* d = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(int64_t) * c->world);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d + c->rank, &local_n, sizeof(int64_t), cudaMemcpyHostToDevice, s);
  pkv_status st = cuda_status(e, "global length exchange");
  if (st == PKV_OK) st = raw_allgather(c, d, sizeof(int64_t), s);
  int64_t h[MAX_RANKS] = {};
  if (st == PKV_OK) {
    e = cudaMemcpyAsync(h, d, sizeof(int64_t) * c->world, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    st = cuda_status(e, "global length exchange");
  }
  if (st == PKV_OK) {
    c->global_n = 0;
    for (int r = 0; r < c->world; ++r) c->global_n += h[r];
  }
  if (s) cudaStreamDestroy(s);
  cudaFree(d);
  return st;
}

static void attach(pkv_index* ix, Comm* c, int64_t shard_offset) {
  comm_destroy(ix->comm);
  ix->comm = c;
  ix->rank = c->rank;
  ix->world = c->world;
  ix->shard_offset = shard_offset;
}

pkv_status comm_init(pkv_index* ix, const uint8_t id_bytes[128], int rank, int world, int64_t shard_offset) {
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, 128);
  Comm* c = new Comm();
  c->rank = rank;
  c->world = world;
  pkv_status s = nccl_status(ncclCommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  if (s == PKV_OK) s = reduce_global_n(c, ix->n);
  if (s != PKV_OK) {
    comm_destroy(c);
    return s;
  }
  attach(ix, c, shard_offset);
  return PKV_OK;
}

pkv_status comm_init_host(pkv_index* ix, pkv_host_allgather_fn fn, void* ctx, int rank, int world,
                          int64_t shard_offset) {
  Comm* c = new Comm();
  c->host_fn = fn;
  c->host_ctx = ctx;
  c->rank = rank;
  c->world = world;
  pkv_status s = reduce_global_n(c, ix->n);
  if (s != PKV_OK) {
    comm_destroy(c);
    return s;
  }
  attach(ix, c, shard_offset);
  return PKV_OK;
}

pkv_status comm_init_peer(pkv_index* ix, int rank, int world, int64_t shard_offset, size_t arena_bytes,
                          uint8_t ipc_handle[64], void** arena_out) {
  if (arena_bytes < peer_header_bytes() + 2 * 4096)
    return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_init_peer: arena too small");
  Comm* c = new Comm();
  c->rank = rank;
  c->world = world;
  c->arena_bytes = arena_bytes;
  cudaError_t e = cudaMalloc(&c->arena, arena_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->arena, 0, peer_header_bytes());  // flags and epochs start at 0
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h{};
  if (e == cudaSuccess && ipc_handle) e = cudaIpcGetMemHandle(&h, c->arena);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    comm_destroy(c);
    return cuda_status(e, "pkv_comm_init_peer");
  }
  if (ipc_handle) std::memcpy(ipc_handle, &h, 64);
  if (arena_out) *arena_out = c->arena;
  c->peers[rank] = c->arena;
  attach(ix, c, shard_offset);
  return PKV_OK;
}

pkv_status comm_peer_connect(pkv_index* ix, const uint8_t* handles, void* const* arenas) {
  Comm* c = ix->comm;
  if (!c || !c->arena) return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_peer_connect: pkv_comm_init_peer first");
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    if (arenas) {
      c->peers[r] = static_cast<char*>(arenas[r]);
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + 64 * r, 64);
      void* p = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return cuda_status(e, "pkv_comm_peer_connect: cudaIpcOpenMemHandle");
      c->peers[r] = static_cast<char*>(p);
      c->opened[r] = true;
    }
    if (!c->peers[r]) return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_peer_connect: null peer arena");
  }
  c->connected = true;
  return PKV_OK;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (--c->refs > 0) return;
  for (int r = 0; r < MAX_RANKS; ++r)
    if (c->opened[r]) cudaIpcCloseMemHandle(c->peers[r]);
  if (c->arena) cudaFree(c->arena);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->stage) cudaFreeHost(c->stage);
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
  return raw_allgather(ix->comm, buf, slot * sizeof(uint32_t), stream);
}

int64_t comm_global_n(const pkv_index* ix, const pkv_retrieve_params* p) {
  if (p && p->n_global > 0) return p->n_global;
  return ix->comm ? ix->comm->global_n : ix->n;
}

pkv_status comm_set_global_len(pkv_index* ix, int64_t n_global) {
  if (!ix->comm) return set_error(PKV_ERR_INVALID_ARG, "pkv_comm_set_global_len: index has no communicator");
  ix->comm->global_n = n_global;
  return PKV_OK;
}

}  // namespace pkv
