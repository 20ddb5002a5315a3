// NCCL plumbing for the sequence-sharded full cache.
//
// One communicator per process/GPU, created from a unique id that rank 0
// makes and the host ships to the other ranks (torch.distributed store).
// The forward's per-layer exchange (forward.cu) and the rebuild's score /
// retrieval-buffer exchanges (caches.py) go through these calls, on the
// caller's stream, so they order with the kernels around them.
#include <nccl.h>

#include "hs_common.cuh"

namespace hs {

static int nccl_error(const char *what, ncclResult_t r) {
  return set_error(HS_ERR_CUDA, "%s: %s", what, ncclGetErrorString(r));
}

int shard_all_gather(const HsShard *sh, const void *send, void *recv, size_t bytes, cudaStream_t st) {
  ncclResult_t r = ncclAllGather(send, recv, bytes, ncclChar, reinterpret_cast<ncclComm_t>(sh->comm), st);
  if (r != ncclSuccess) return nccl_error("all_gather", r);
  return HS_OK;
}

}  // namespace hs

extern "C" size_t hs_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

extern "C" int hs_comm_unique_id(void *id) {
  ncclResult_t r = ncclGetUniqueId(reinterpret_cast<ncclUniqueId *>(id));
  return r == ncclSuccess ? HS_OK : hs::nccl_error("ncclGetUniqueId", r);
}

extern "C" int hs_comm_init(void **comm, const void *id, int world, int rank) {
  HS_REQUIRE(world >= 1 && rank >= 0 && rank < world, HS_ERR_VALUE, "comm_init: rank %d of %d", rank, world);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, world, uid, rank);
  if (r != ncclSuccess) return hs::nccl_error("ncclCommInitRank", r);
  *comm = c;
  return HS_OK;
}

extern "C" int hs_comm_destroy(void *comm) {
  if (!comm) return HS_OK;
  ncclResult_t r = ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? HS_OK : hs::nccl_error("ncclCommDestroy", r);
}

extern "C" int hs_all_gather(void *comm, const void *send, void *recv, size_t bytes, void *stream) {
  HS_REQUIRE(comm != nullptr, HS_ERR_VALUE, "all_gather: no communicator");
  HsShard sh{comm, 0, 0};
  return hs::shard_all_gather(&sh, send, recv, bytes, hs::as_stream(stream));
}

extern "C" int hs_all_reduce_sum(void *comm, void *buf, size_t count, int dtype, void *stream) {
  HS_REQUIRE(comm != nullptr, HS_ERR_VALUE, "all_reduce: no communicator");
  ncclDataType_t t;
  switch (dtype) {
    case 0: t = ncclBfloat16; break;
    case 1: t = ncclFloat32; break;
    case 2: t = ncclFloat64; break;
    case 3: t = ncclInt32; break;
    default: return hs::set_error(HS_ERR_VALUE, "all_reduce: dtype %d", dtype);
  }
  ncclResult_t r = ncclAllReduce(buf, buf, count, t, ncclSum, reinterpret_cast<ncclComm_t>(comm),
                                 hs::as_stream(stream));
  return r == ncclSuccess ? HS_OK : hs::nccl_error("all_reduce", r);
}
