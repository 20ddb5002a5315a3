// Collectives for the sequence-sharded full cache.
//
// Two communicator kinds sit behind HsShard.comm:
//
// * NCCL (hs_comm_init): one communicator per process/GPU, created
//   non-blocking from a unique id that rank 0 makes and the host ships to
//   the other ranks (torch.distributed).  Every call polls
//   ncclCommGetAsyncError until the operation is enqueued, under a deadline
//   (HS_NCCL_TIMEOUT_S, default 300 s); a peer that never arrives aborts the
//   communicator and surfaces as HS_ERR_CUDA instead of a hang.
// * loopback (hs_loopback_create): G ranks inside ONE process, each driven
//   by its own host thread and CUDA stream, exchanging through device-to-
//   device copies.  Same semantics as the NCCL calls (rank-ordered all-gather,
//   all-gather-v, sum all-reduce), so a G-shard session runs on one GPU and
//   is checked bit for bit against the unsharded one.
//
// The forward's per-layer exchange (forward.cu, prefill.cu), the rebuild's
// score all-gather and its chunk exchange (hs_retrieval_exchange, caches.py)
// go through these calls on the caller's stream.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <set>
#include <stdlib.h>
#include <string.h>
#include <vector>

#include "hs_common.cuh"

namespace hs {

// ---------------------------------------------------------------- loopback group
struct LbGroup;
struct LbComm {
  LbGroup *g;
  int rank;
};

struct LbSlot {
  const void *send;
  void *recv;
  size_t bytes;                     // all-gather: bytes per rank; all-reduce: element count
  const size_t *counts;             // all-gather-v: bytes per rank (recv is rank-ordered)
  cudaStream_t st;
};

struct LbGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;
  std::vector<LbSlot> slot;
  std::vector<cudaEvent_t> ready, done;
  std::vector<LbComm> comms;

  // all ranks' host threads meet here; false on timeout (the group is then
  // broken: every later collective fails fast)
  bool barrier(double timeout_s) {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

static std::mutex g_lb_mu;
static std::set<const void *> g_lb_comms;   // loopback communicator handles

static bool is_loopback(const void *comm) {
  std::lock_guard<std::mutex> lk(g_lb_mu);
  return g_lb_comms.count(comm) != 0;
}

static double timeout_s() {
  static double t = -1.0;
  if (t < 0) {
    const char *e = getenv("HS_NCCL_TIMEOUT_S");
    t = e ? atof(e) : 300.0;
    if (t <= 0) t = 300.0;
  }
  return t;
}

static int lb_fail(const char *what) {
  return set_error(HS_ERR_CUDA, "%s: loopback peer did not arrive within %.0f s", what, timeout_s());
}

// Rank `c->rank` contributes `me`; `issue` enqueues this rank's copies on its
// stream once every rank's inputs are ready.  Protocol: record ready ->
// barrier -> wait peers' ready, copy -> record done -> barrier -> wait peers'
// done (no rank reuses its send buffer before the peers' reads finished).
template <typename Issue>
static int lb_collective(LbComm *c, const LbSlot &me, const char *what, Issue issue) {
  LbGroup *g = c->g;
  const int r = c->rank;
  g->slot[r] = me;
  if (cudaEventRecord(g->ready[r], me.st) != cudaSuccess) return set_error(HS_ERR_CUDA, "%s: event record", what);
  if (!g->barrier(timeout_s())) return lb_fail(what);
  for (int p = 0; p < g->world; ++p)
    if (p != r && cudaStreamWaitEvent(me.st, g->ready[p], 0) != cudaSuccess)
      return set_error(HS_ERR_CUDA, "%s: stream wait", what);
  int rc = issue(g, r);
  if (rc != HS_OK) return rc;
  if (cudaEventRecord(g->done[r], me.st) != cudaSuccess) return set_error(HS_ERR_CUDA, "%s: event record", what);
  if (!g->barrier(timeout_s())) return lb_fail(what);
  for (int p = 0; p < g->world; ++p)
    if (p != r && cudaStreamWaitEvent(me.st, g->done[p], 0) != cudaSuccess)
      return set_error(HS_ERR_CUDA, "%s: stream wait", what);
  return HS_OK;
}

template <typename T>
__global__ void lb_sum_kernel(const T *parts, int world, size_t n, T *out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;   // rank order, one rounding at the end
    for (int r = 0; r < world; ++r) s += (double)parts[(size_t)r * n + i];
    out[i] = (T)s;
  }
}

__global__ void lb_sum_bf16_kernel(const uint16_t *parts, int world, size_t n, uint16_t *out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int r = 0; r < world; ++r) s += bf16_to_f(parts[(size_t)r * n + i]);
    out[i] = f_to_bf16(s);
  }
}

// ---------------------------------------------------------------- NCCL helpers
static int nccl_error(const char *what, ncclResult_t r) {
  return set_error(HS_ERR_CUDA, "%s: %s", what, ncclGetErrorString(r));
}

// A non-blocking communicator returns ncclInProgress while an operation is
// being set up; poll its async error state until it settles, under the deadline.
static int nccl_settle(ncclComm_t comm, ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return HS_OK;
  if (r != ncclInProgress) return nccl_error(what, r);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    ncclResult_t a = ncclSuccess;
    ncclResult_t q = ncclCommGetAsyncError(comm, &a);
    if (q != ncclSuccess) return nccl_error(what, q);
    if (a == ncclSuccess) return HS_OK;
    if (a != ncclInProgress) return nccl_error(what, a);
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s()) {
      ncclCommAbort(comm);
      return set_error(HS_ERR_CUDA, "%s: timed out after %.0f s (communicator aborted)", what, timeout_s());
    }
  }
}

// ---------------------------------------------------------------- collectives
int shard_all_gather(const HsShard *sh, const void *send, void *recv, size_t bytes, cudaStream_t st) {
  if (is_loopback(sh->comm)) {
    LbComm *c = (LbComm *)sh->comm;
    LbSlot me = {send, recv, bytes, nullptr, st};
    return lb_collective(c, me, "all_gather", [&](LbGroup *g, int r) {
      for (int p = 0; p < g->world; ++p)
        if (cudaMemcpyAsync((char *)recv + (size_t)p * bytes, g->slot[p].send, bytes, cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess)
          return set_error(HS_ERR_CUDA, "all_gather: copy");
      return HS_OK;
    });
  }
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(sh->comm);
  return nccl_settle(comm, ncclAllGather(send, recv, bytes, ncclChar, comm, st), "all_gather");
}

// recv = concat over ranks (rank order) of each rank's `counts[rank]` bytes
int shard_all_gather_v(const HsShard *sh, const void *send, void *recv, const size_t *counts, cudaStream_t st) {
  const int world = sh->world;
  std::vector<size_t> disp(world + 1, 0);
  for (int r = 0; r < world; ++r) disp[r + 1] = disp[r] + counts[r];
  if (is_loopback(sh->comm)) {
    LbComm *c = (LbComm *)sh->comm;
    LbSlot me = {send, recv, counts[c->rank], counts, st};
    return lb_collective(c, me, "all_gather_v", [&](LbGroup *g, int r) {
      for (int p = 0; p < g->world; ++p)
        if (counts[p] && cudaMemcpyAsync((char *)recv + disp[p], g->slot[p].send, counts[p], cudaMemcpyDeviceToDevice,
                                         st) != cudaSuccess)
          return set_error(HS_ERR_CUDA, "all_gather_v: copy");
      return HS_OK;
    });
  }
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(sh->comm);
  ncclResult_t r0 = ncclGroupStart();
  if (r0 != ncclSuccess) return nccl_error("all_gather_v", r0);
  for (int r = 0; r < world; ++r) {
    if (!counts[r]) continue;
    ncclResult_t e = ncclBroadcast(r == sh->rank ? send : nullptr, (char *)recv + disp[r], counts[r], ncclChar, r,
                                   comm, st);
    if (e != ncclSuccess && e != ncclInProgress) {
      ncclGroupEnd();
      return nccl_error("all_gather_v", e);
    }
  }
  return nccl_settle(comm, ncclGroupEnd(), "all_gather_v");
}

// ---------------------------------------------------------------- retrieval exchange
// pack / unpack one layer's slot range [s0, s1) of K and V ([KVH][cap][dh]
// per layer) into / from a contiguous [2][KVH][s1 - s0][dh] block
__global__ void range_pack_kernel(HsCache c, int layer, int s0, int s1, uint4 *buf, int unpack) {
  const int kh = blockIdx.y, which = blockIdx.z, DH = c.head_dim;
  const int n = s1 - s0;
  const size_t vec = (size_t)n * DH / 8;
  uint16_t *base = (which ? c.v : c.k) + (((size_t)layer * c.n_kv_heads + kh) * c.cap + s0) * DH;
  uint4 *blk = buf + ((size_t)which * c.n_kv_heads + kh) * vec;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < vec; e += (size_t)gridDim.x * blockDim.x) {
    if (unpack) reinterpret_cast<uint4 *>(base)[e] = blk[e];
    else blk[e] = reinterpret_cast<const uint4 *>(base)[e];
  }
}

static int range_copy(const HsCache *c, int layer, int s0, int s1, void *buf, int unpack, cudaStream_t st) {
  if (s1 <= s0) return HS_OK;
  dim3 grid(ceil_div((long long)(s1 - s0) * c->head_dim / 8, 256 * 4), c->n_kv_heads, 2);
  range_pack_kernel<<<grid, 256, 0, st>>>(*c, layer, s0, s1, (uint4 *)buf, unpack);
  return check_launch("retrieval_exchange");
}

}  // namespace hs

// ------------------------------------------------------------------ C ABI
extern "C" size_t hs_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

extern "C" int hs_comm_unique_id(void *id) {
  ncclResult_t r = ncclGetUniqueId(reinterpret_cast<ncclUniqueId *>(id));
  return r == ncclSuccess ? HS_OK : hs::nccl_error("ncclGetUniqueId", r);
}

extern "C" int hs_comm_init(void **comm, const void *id, int world, int rank) {
  HS_REQUIRE(world >= 1 && rank >= 0 && rank < world, HS_ERR_VALUE, "comm_init: rank %d of %d", rank, world);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 0;   // returns at once; completion (or a peer that never joins) is polled below
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRankConfig(&c, world, uid, rank, &cfg);
  if (r != ncclSuccess && r != ncclInProgress) return hs::nccl_error("ncclCommInitRank", r);
  int rc = hs::nccl_settle(c, r == ncclSuccess ? ncclInProgress : r, "ncclCommInitRank");
  if (rc != HS_OK) return rc;
  *comm = c;
  return HS_OK;
}

extern "C" int hs_comm_check(void *comm) {
  HS_REQUIRE(comm != nullptr, HS_ERR_VALUE, "comm_check: no communicator");
  if (hs::is_loopback(comm)) {
    hs::LbGroup *g = ((hs::LbComm *)comm)->g;
    std::lock_guard<std::mutex> lk(g->mu);
    return g->broken ? hs::set_error(HS_ERR_CUDA, "loopback group broken (a peer timed out)") : HS_OK;
  }
  ncclResult_t a = ncclSuccess;
  ncclResult_t q = ncclCommGetAsyncError(reinterpret_cast<ncclComm_t>(comm), &a);
  if (q != ncclSuccess) return hs::nccl_error("ncclCommGetAsyncError", q);
  if (a != ncclSuccess && a != ncclInProgress) return hs::nccl_error("communicator", a);
  return HS_OK;
}

extern "C" int hs_comm_abort(void *comm) {
  HS_REQUIRE(comm != nullptr, HS_ERR_VALUE, "comm_abort: no communicator");
  if (hs::is_loopback(comm)) {
    hs::LbGroup *g = ((hs::LbComm *)comm)->g;
    std::lock_guard<std::mutex> lk(g->mu);
    g->broken = true;   // every rank waiting in (or entering) a collective fails at once
    g->cv.notify_all();
    return HS_OK;
  }
  ncclResult_t r = ncclCommAbort(reinterpret_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? HS_OK : hs::nccl_error("ncclCommAbort", r);
}

extern "C" int hs_comm_destroy(void *comm) {
  if (!comm) return HS_OK;
  if (hs::is_loopback(comm)) return HS_OK;   // owned by its group (hs_loopback_destroy)
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
  ncclResult_t r = ncclCommFinalize(c);
  if (r == ncclSuccess || r == ncclInProgress) hs::nccl_settle(c, r == ncclSuccess ? ncclInProgress : r, "finalize");
  r = ncclCommDestroy(c);
  return r == ncclSuccess ? HS_OK : hs::nccl_error("ncclCommDestroy", r);
}

extern "C" int hs_loopback_create(int world, void **comms) {
  HS_REQUIRE(world >= 1 && world <= 64, HS_ERR_VALUE, "loopback: world %d", world);
  hs::LbGroup *g = new hs::LbGroup();
  g->world = world;
  g->slot.resize(world);
  g->ready.resize(world);
  g->done.resize(world);
  g->comms.resize(world);
  for (int r = 0; r < world; ++r) {
    if (cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming) != cudaSuccess)
      return hs::set_error(HS_ERR_CUDA, "loopback: cudaEventCreate");
    g->comms[r] = {g, r};
    comms[r] = &g->comms[r];
  }
  std::lock_guard<std::mutex> lk(hs::g_lb_mu);
  for (int r = 0; r < world; ++r) hs::g_lb_comms.insert(&g->comms[r]);
  return HS_OK;
}

extern "C" int hs_loopback_destroy(void *comm0) {
  if (!comm0 || !hs::is_loopback(comm0)) return hs::set_error(HS_ERR_VALUE, "loopback_destroy: not a loopback comm");
  hs::LbGroup *g = ((hs::LbComm *)comm0)->g;
  {
    std::lock_guard<std::mutex> lk(hs::g_lb_mu);
    for (auto &c : g->comms) hs::g_lb_comms.erase(&c);
  }
  for (int r = 0; r < g->world; ++r) {
    cudaEventDestroy(g->ready[r]);
    cudaEventDestroy(g->done[r]);
  }
  delete g;
  return HS_OK;
}

extern "C" int hs_all_gather(void *comm, const void *send, void *recv, size_t bytes, void *stream) {
  HS_REQUIRE(comm != nullptr, HS_ERR_VALUE, "all_gather: no communicator");
  HsShard sh{comm, 0, 0};
  return hs::shard_all_gather(&sh, send, recv, bytes, hs::as_stream(stream));
}

extern "C" int hs_all_gather_v(void *comm, int rank, int world, const void *send, void *recv,
                               const size_t *bytes_per_rank, void *stream) {
  HS_REQUIRE(comm != nullptr && world >= 1 && rank >= 0 && rank < world, HS_ERR_VALUE, "all_gather_v: bad comm");
  HsShard sh{comm, rank, world};
  return hs::shard_all_gather_v(&sh, send, recv, bytes_per_rank, hs::as_stream(stream));
}

extern "C" int hs_all_reduce_sum(void *comm, void *buf, size_t count, int dtype, void *stream) {
  HS_REQUIRE(comm != nullptr, HS_ERR_VALUE, "all_reduce: no communicator");
  static const size_t esz[4] = {2, 4, 8, 4};
  HS_REQUIRE(dtype >= 0 && dtype <= 3, HS_ERR_VALUE, "all_reduce: dtype %d", dtype);
  cudaStream_t st = hs::as_stream(stream);
  if (hs::is_loopback(comm)) {
    hs::LbComm *c = (hs::LbComm *)comm;
    hs::LbGroup *g = c->g;
    const size_t bytes = count * esz[dtype];
    // every rank reads all send buffers into its own staging row block, then sums in rank order
    std::vector<void *> parts(1);
    if (cudaMallocAsync(&parts[0], bytes * g->world, st) != cudaSuccess)
      return hs::set_error(HS_ERR_CUDA, "all_reduce: staging allocation");
    hs::LbSlot me = {buf, parts[0], bytes, nullptr, st};
    int rc = hs::lb_collective(c, me, "all_reduce", [&](hs::LbGroup *gg, int r) {
      for (int p = 0; p < gg->world; ++p)
        if (cudaMemcpyAsync((char *)parts[0] + p * bytes, gg->slot[p].send, bytes, cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess)
          return hs::set_error(HS_ERR_CUDA, "all_reduce: copy");
      return HS_OK;
    });
    if (rc != HS_OK) return rc;
    const int grid = hs::ceil_div((long long)count, 256 * 8) > 4096 ? 4096 : hs::ceil_div((long long)count, 256 * 8);
    switch (dtype) {
      case 0: hs::lb_sum_bf16_kernel<<<grid, 256, 0, st>>>((const uint16_t *)parts[0], g->world, count, (uint16_t *)buf); break;
      case 1: hs::lb_sum_kernel<float><<<grid, 256, 0, st>>>((const float *)parts[0], g->world, count, (float *)buf); break;
      case 2: hs::lb_sum_kernel<double><<<grid, 256, 0, st>>>((const double *)parts[0], g->world, count, (double *)buf); break;
      default: hs::lb_sum_kernel<int32_t><<<grid, 256, 0, st>>>((const int32_t *)parts[0], g->world, count, (int32_t *)buf); break;
    }
    rc = hs::check_launch("all_reduce");
    cudaFreeAsync(parts[0], st);
    return rc;
  }
  ncclDataType_t t;
  switch (dtype) {
    case 0: t = ncclBfloat16; break;
    case 1: t = ncclFloat32; break;
    case 2: t = ncclFloat64; break;
    default: t = ncclInt32; break;
  }
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
  return hs::nccl_settle(c, ncclAllReduce(buf, buf, count, t, ncclSum, c, st), "all_reduce");
}

extern "C" size_t hs_retrieval_exchange_workspace_bytes(const HsCache *c) {
  // one layer's K and V for the whole view, twice (this rank's block + the gathered blocks)
  return 2 * (size_t)2 * c->n_kv_heads * c->cap * c->head_dim * 2;
}

/* Assemble a replicated retrieval cache after a sharded build: ranges
 * [layer][rank][2] (host int32) are the slot ranges each rank gathered from
 * its own shard (hs_retrieval_gather); per layer every rank packs its range,
 * the blocks are all-gathered (variable sizes, rank order) and unpacked into
 * their slots.  Replaces a sum all-reduce of the whole buffer: each byte
 * crosses the fabric once.                                                   */
extern "C" int hs_retrieval_exchange(const HsShard *sh, const HsCache *c, const int32_t *ranges, void *workspace,
                                     size_t ws_bytes, void *stream) {
  HS_REQUIRE(sh && sh->comm && sh->world >= 1 && sh->rank >= 0 && sh->rank < sh->world, HS_ERR_VALUE,
             "retrieval_exchange: bad shard descriptor");
  HS_REQUIRE(c->kind == HS_KV_SLOTTED && c->head_dim % 8 == 0, HS_ERR_VALUE, "retrieval_exchange: slotted cache");
  HS_REQUIRE(ws_bytes >= hs_retrieval_exchange_workspace_bytes(c), HS_ERR_VALUE, "retrieval_exchange: workspace");
  cudaStream_t st = hs::as_stream(stream);
  const int G = sh->world, me = sh->rank;
  const size_t row = (size_t)2 * c->n_kv_heads * c->head_dim * 2;   // bytes per slot (K and V, all heads)
  char *send = (char *)workspace;
  char *recv = send + hs_retrieval_exchange_workspace_bytes(c) / 2;
  std::vector<size_t> counts(G);
  for (int l = 0; l < c->n_layers; ++l) {
    const int32_t *rg = ranges + (size_t)l * G * 2;
    for (int r = 0; r < G; ++r) {
      HS_REQUIRE(rg[2 * r] >= 0 && rg[2 * r] <= rg[2 * r + 1] && rg[2 * r + 1] <= c->cap, HS_ERR_VALUE,
                 "retrieval_exchange: bad range [%d, %d) of rank %d", rg[2 * r], rg[2 * r + 1], r);
      counts[r] = (size_t)(rg[2 * r + 1] - rg[2 * r]) * row;
    }
    int rc = hs::range_copy(c, l, rg[2 * me], rg[2 * me + 1], send, 0, st);
    if (rc != HS_OK) return rc;
    rc = hs::shard_all_gather_v(sh, send, recv, counts.data(), st);
    if (rc != HS_OK) return rc;
    size_t off = 0;
    for (int r = 0; r < G; ++r) {
      if (r != me) {
        rc = hs::range_copy(c, l, rg[2 * r], rg[2 * r + 1], recv + off, 1, st);
        if (rc != HS_OK) return rc;
      }
      off += counts[r];
    }
  }
  return HS_OK;
}
