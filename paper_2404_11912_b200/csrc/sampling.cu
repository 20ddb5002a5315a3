// Sampling and speculative verification kernels.
//
//   hs_probs         prob_from_logits   (model.py:182-195)
//   hs_sample        sample_from_probs  (model.py:198-202)
//   hs_draft_sample  draft_round body   (speculation.py:221-226)
//   hs_verify_chain  _verify_chain + verify_token/correct_token
//                    (speculation.py:52-72, 187-208)
//
// RNG protocol: the host owns the numpy PCG64 stream of one generate() call
// and uploads its uniforms in order; kernels consume them through a device
// cursor, one per sampling event and one per verification -- exactly the
// reference's consumption order (speculation.py:9-12).
//
// Parallel form: every vocabulary row is processed by one thread-block
// cluster of SMP_CL CTAs (CTA rank r owns the contiguous vocabulary slice r;
// element-wise passes stride over it, the inverse CDF gives each thread a
// contiguous segment staged in shared memory).  Row-wide max /
// argmax / sums / the inverse-CDF prefix are reduced through distributed
// shared memory in a fixed order (thread segment -> warp -> CTA -> CTA rank),
// so every result is deterministic and independent of the launch.  These
// kernels sit on the inner loop's critical path, where one 1024-thread CTA
// walking 32,000 entries was latency-bound (25-47 us); the cluster form
// keeps all of a row's loads in flight at once.
#include <cooperative_groups.h>

#include <cstring>

#include "hs_common.cuh"

namespace cg = cooperative_groups;

namespace hs {

constexpr int SMP_CL = 8;          // CTAs per row (portable cluster size)
constexpr int SMP_THREADS = 512;
constexpr int SMP_WARPS = SMP_THREADS / 32;
constexpr int SEG_REG = 16;        // register-resident entries per thread (V <= 65,536)

struct ArgMax { double v; int i; };

__device__ __forceinline__ ArgMax amax(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

// Cluster-wide reductions.  Each call publishes this CTA's partial in one of
// two shared slots (alternating per call), synchronises the cluster once and
// reads every rank's partial in rank order.  A slot is rewritten two calls
// later, after the intervening cluster barrier: by then every CTA has
// finished reading it.
struct ClRed {
  double d[2];
  int i[2];
};

struct Seg {   // this thread's contiguous slice [j0, j1) of the row
  int j0, j1;
};

__device__ __forceinline__ Seg my_seg(int V) {
  const int per_cta = (V + SMP_CL - 1) / SMP_CL;
  const int rank = (int)cg::this_cluster().block_rank();
  const int c0 = rank * per_cta, c1 = min(V, c0 + per_cta);
  const int per = (per_cta + SMP_THREADS - 1) / SMP_THREADS;
  const int j0 = min(c1, c0 + (int)threadIdx.x * per);
  return Seg{j0, min(c1, j0 + per)};
}

class Cl {
 public:
  __device__ Cl(ClRed *slots, double *wd, int *wi) : s_(slots), wd_(wd), wi_(wi), k_(0) {}

  __device__ ArgMax argmax(ArgMax x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMax y;
      y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
      y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
      x = amax(x, y);
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { wd_[w] = x.v; wi_[w] = x.i; }
    __syncthreads();
    const int b = k_++ & 1;
    if (threadIdx.x == 0) {
      ArgMax r = {wd_[0], wi_[0]};
      for (int k = 1; k < SMP_WARPS; ++k) r = amax(r, ArgMax{wd_[k], wi_[k]});
      s_->d[b] = r.v;
      s_->i[b] = r.i;
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    ArgMax r = {-INFINITY, 0x7fffffff};
    for (int c = 0; c < SMP_CL; ++c) {
      const ClRed *o = cl.map_shared_rank(s_, c);
      r = amax(r, ArgMax{o->d[b], o->i[b]});
    }
    return r;
  }

  // fixed-order sum; `excl` (optional) receives the sum over lower CTA ranks
  __device__ double sum(double x, double *excl = nullptr) {
    x = warp_sum(x);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) wd_[w] = x;
    __syncthreads();
    const int b = k_++ & 1;
    if (threadIdx.x == 0) {
      double r = 0.0;
      for (int k = 0; k < SMP_WARPS; ++k) r += wd_[k];
      s_->d[b] = r;
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int me = (int)cl.block_rank();
    double r = 0.0, e = 0.0;
    for (int c = 0; c < SMP_CL; ++c) {
      const double v = cl.map_shared_rank(s_, c)->d[b];
      if (c == me) e = r;
      r += v;
    }
    if (excl) *excl = e;
    return r;
  }

  __device__ int count(int x) {
    x = warp_sum(x);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) wi_[w] = x;
    __syncthreads();
    const int b = k_++ & 1;
    if (threadIdx.x == 0) {
      int r = 0;
      for (int k = 0; k < SMP_WARPS; ++k) r += wi_[k];
      s_->i[b] = r;
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    int r = 0;
    for (int c = 0; c < SMP_CL; ++c) r += cl.map_shared_rank(s_, c)->i[b];
    return r;
  }

  // exclusive prefix (over the whole row, in entry order) of this thread's
  // segment total: CTA ranks below, then warps below, then lanes below
  __device__ double exclusive_prefix(double local) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();   // wd_ may still be read by a previous reduction
    if (lane == 31) wd_[wid] = incl;
    __syncthreads();
    double wbase = 0.0, cta = 0.0;
    for (int k = 0; k < SMP_WARPS; ++k) {
      if (k == wid) wbase = cta;
      cta += wd_[k];
    }
    __syncthreads();
    double rank_base;
    sum_total_(cta, &rank_base);
    double excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0.0;
    return rank_base + wbase + excl;
  }

  // every CTA must pass this before any exits (its shared memory may still be
  // read by a peer)
  __device__ void finish() { cg::this_cluster().sync(); }

 private:
  __device__ void sum_total_(double cta_total, double *excl) {
    const int b = k_++ & 1;
    if (threadIdx.x == 0) s_->d[b] = cta_total;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int me = (int)cl.block_rank();
    double r = 0.0, e = 0.0;
    for (int c = 0; c < SMP_CL; ++c) {
      const double v = cl.map_shared_rank(s_, c)->d[b];
      if (c == me) e = r;
      r += v;
    }
    *excl = e;
  }

  ClRed *s_;
  double *wd_;
  int *wi_;
  int k_;
};

#define HS_CL_SETUP                      \
  __shared__ ClRed cl_slots_;            \
  __shared__ double cl_wd_[SMP_WARPS];   \
  __shared__ int cl_wi_[SMP_WARPS];      \
  Cl cl(&cl_slots_, cl_wd_, cl_wi_);

// this CTA's contiguous slice [c0, c1) of the row
__device__ __forceinline__ void cta_range(int V, int &c0, int &c1) {
  const int per_cta = (V + SMP_CL - 1) / SMP_CL;
  c0 = (int)cg::this_cluster().block_rank() * per_cta;
  c1 = min(V, c0 + per_cta);
  c0 = min(c0, V);
}

// Element-wise passes walk the CTA slice with a block stride (coalesced):
// entry k of thread t is c0 + t + k * SMP_THREADS.  Argmax (ties to the
// lower index) and the exp / divide passes do not depend on the order; the
// sums are reduced in a fixed order (thread -> warp -> CTA -> rank).
__device__ __forceinline__ ArgMax strided_argmax(const float *logits, int c0, int c1, double inv_t) {
  float x[SEG_REG];
#pragma unroll
  for (int k = 0; k < SEG_REG; ++k) {
    const int j = c0 + (int)threadIdx.x + k * SMP_THREADS;
    x[k] = j < c1 ? logits[j] : -INFINITY;
  }
  ArgMax best = {-INFINITY, 0x7fffffff};
#pragma unroll
  for (int k = 0; k < SEG_REG; ++k) {
    const int j = c0 + (int)threadIdx.x + k * SMP_THREADS;
    if (j < c1) best = amax(best, ArgMax{inv_t == 1.0 ? (double)x[k] : (double)x[k] / inv_t, j});
  }
  return best;
}

__device__ __forceinline__ void one_hot(double *p, int c0, int c1, int hot) {
  for (int j = c0 + (int)threadIdx.x; j < c1; j += SMP_THREADS) p[j] = (j == hot) ? 1.0 : 0.0;
}

// probs of one logits row into p (fp64), whole cluster
__device__ void row_probs(Cl &cl, const float *logits, int V, double T, double *p) {
  int c0, c1;
  cta_range(V, c0, c1);
  if (T == 0.0) {
    one_hot(p, c0, c1, cl.argmax(strided_argmax(logits, c0, c1, 1.0)).i);
    return;
  }
  // max of logits / T (model.py:190-195), then exp(x / T - max) and its sum
  const double mx = cl.argmax(strided_argmax(logits, c0, c1, T)).v;
  double e[SEG_REG];
  double loc = 0.0;
#pragma unroll
  for (int k = 0; k < SEG_REG; ++k) {
    const int j = c0 + (int)threadIdx.x + k * SMP_THREADS;
    e[k] = j < c1 ? exp((double)logits[j] / T - mx) : 0.0;
    loc += e[k];
  }
  const double tot = cl.sum(loc);
#pragma unroll
  for (int k = 0; k < SEG_REG; ++k) {
    const int j = c0 + (int)threadIdx.x + k * SMP_THREADS;
    if (j < c1) p[j] = e[k] / tot;
  }
}

// inverse CDF: min(#{j : cumsum(w/scale)_j <= u}, V-1); w optionally the
// residual max(p - q, 0).  The CTA slice of w is staged in shared memory
// with coalesced loads; the cumulative sum is then segment-sequential per
// thread (contiguous segments) after the fixed-order exclusive prefix of the
// segment totals (deterministic).
__device__ int inv_cdf(Cl &cl, const double *p, const double *q, double scale, int V, double u, double *sw) {
  int c0, c1;
  cta_range(V, c0, c1);
  for (int j = c0 + (int)threadIdx.x; j < c1; j += SMP_THREADS) {
    double x = q ? fmax(p[j] - q[j], 0.0) : p[j];
    if (scale != 1.0) x = x / scale;
    sw[j - c0] = x;
  }
  __syncthreads();
  const Seg s = my_seg(V);
  const int n = s.j1 - s.j0;
  double w[SEG_REG];
  double local = 0.0;
#pragma unroll
  for (int i = 0; i < SEG_REG; ++i) {
    w[i] = i < n ? sw[s.j0 - c0 + i] : 0.0;
    local += w[i];
  }
  double c = cl.exclusive_prefix(local);
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < SEG_REG; ++i) {
    if (i < n) {
      c += w[i];
      cnt += (c <= u) ? 1 : 0;
    }
  }
  cnt = cl.count(cnt);
  __syncthreads();   // sw may be restaged by a later call
  return cnt < V - 1 ? cnt : V - 1;
}

// the residual mass Z = sum max(p - q, 0) (correct_token, speculation.py:65-72)
// and the residual's staging for the inverse CDF in one pass over p, q:
// sw[j - c0] = max(p_j - q_j, 0) for this CTA's slice, Z summed in a fixed
// order (thread's strided entries -> warp -> CTA -> rank)
__device__ double residual_stage(Cl &cl, const double *p, const double *q, int V, double *sw) {
  int c0, c1;
  cta_range(V, c0, c1);
  double z = 0.0;
#pragma unroll
  for (int k = 0; k < SEG_REG; ++k) {
    const int j = c0 + (int)threadIdx.x + k * SMP_THREADS;
    if (j < c1) {
      const double x = fmax(p[j] - q[j], 0.0);
      sw[j - c0] = x;
      z += x;
    }
  }
  return cl.sum(z);   // (its block barrier also orders the staging stores)
}

// inv_cdf over a slice already staged in sw (residual_stage), each entry
// divided by scale in place first: the same values and order as inv_cdf
__device__ int inv_cdf_staged(Cl &cl, double scale, int V, double u, double *sw) {
  int c0, c1;
  cta_range(V, c0, c1);
  if (scale != 1.0)
    for (int j = c0 + (int)threadIdx.x; j < c1; j += SMP_THREADS) sw[j - c0] = sw[j - c0] / scale;
  __syncthreads();
  const Seg s = my_seg(V);
  const int n = s.j1 - s.j0;
  double w[SEG_REG];
  double local = 0.0;
#pragma unroll
  for (int i = 0; i < SEG_REG; ++i) {
    w[i] = i < n ? sw[s.j0 - c0 + i] : 0.0;
    local += w[i];
  }
  double c = cl.exclusive_prefix(local);
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < SEG_REG; ++i) {
    if (i < n) {
      c += w[i];
      cnt += (c <= u) ? 1 : 0;
    }
  }
  cnt = cl.count(cnt);
  __syncthreads();   // sw may be restaged by a later call
  return cnt < V - 1 ? cnt : V - 1;
}

__device__ __forceinline__ bool cl_leader() { return cg::this_cluster().block_rank() == 0 && threadIdx.x == 0; }

// one cluster per row
__global__ void __launch_bounds__(SMP_THREADS) probs_kernel(const float *logits, int V, double T, double *probs) {
  pdl_wait();
  HS_CL_SETUP
  const size_t row = blockIdx.x / SMP_CL;
  row_probs(cl, logits + row * V, V, T, probs + row * V);
  pdl_trigger();
  cl.finish();
}

__global__ void __launch_bounds__(SMP_THREADS) sample_kernel(const double *probs, int V, const double *U,
                                                             int32_t *cursor, int32_t *out) {
  pdl_wait();
  HS_CL_SETUP
  const int cur = *cursor;
  extern __shared__ double sw[];
  const int tok = inv_cdf(cl, probs, nullptr, 1.0, V, U[cur], sw);
  cl.finish();   // every CTA has read the cursor
  if (cl_leader()) { *out = tok; *cursor = cur + 1; }
}

// dyn (optional): a captured step graph's [frontier, window watermark, token]
// slot, written together with the token (the draft lane's next step reads it)
__global__ void __launch_bounds__(SMP_THREADS) draft_sample_kernel(const float *logits, int V, double T,
                                                                   double *probs, const double *U,
                                                                   int32_t *cursor, int32_t *out, int32_t *dyn,
                                                                   int dyn_frontier, int dyn_lo) {
  pdl_wait();
  HS_CL_SETUP
  extern __shared__ double sw[];
  const int cur = *cursor;
  int tok;
  if (T == 0.0) {
    // one-hot argmax row; its inverse CDF at any u in [0, 1) is the argmax
    // itself (model.py:198-202 with a one-hot p), so skip the scan
    int c0, c1;
    cta_range(V, c0, c1);
    const ArgMax best = cl.argmax(strided_argmax(logits, c0, c1, 1.0));
    one_hot(probs, c0, c1, best.i);
    tok = best.i < V ? best.i : V - 1;
  } else {
    row_probs(cl, logits, V, T, probs);
    __syncthreads();   // the CTA's slice of the row is written (it restages only its own slice)
    tok = inv_cdf(cl, probs, nullptr, 1.0, V, U[cur], sw);
  }
  pdl_trigger();
  cl.finish();
  if (cl_leader()) {
    *out = tok;
    *cursor = cur + 1;
    if (dyn) { dyn[0] = dyn_frontier; dyn[1] = dyn_lo; dyn[2] = tok; }
  }
}

// positions (+ token) of a captured step graph; `also` gets the token too
__global__ void graph_step_kernel(int32_t *dyn, int frontier, int lo, int token, int32_t *also) {
  dyn[0] = frontier;
  dyn[1] = lo;
  if (token >= 0) {
    dyn[2] = token;
    if (also) *also = token;
  }
}

// _verify_chain: result[0..n] tokens, [n+1] count, [n+2] accepted, [n+3] status.
// Every CTA of the cluster evaluates the (short) accept chain redundantly:
// thread i checks proposal i with uniform U[cur + i], which is the uniform
// the sequential loop gives it whenever all earlier proposals were accepted;
// the first failing proposal ends the chain.  The row-wide residual sum and
// the correction / bonus draw then run on the whole cluster.
__global__ void __launch_bounds__(SMP_THREADS) verify_chain_kernel(const int32_t *tokens, int n, const double *qd,
                                                                   const double *pd, int V, const double *U,
                                                                   int32_t *cursor, int32_t *result) {
  pdl_wait();
  HS_CL_SETUP
  extern __shared__ double sw[];
  __shared__ int first_s, zero_s;
  const int cur = *cursor;
  if (threadIdx.x == 0) { first_s = n; zero_s = n; }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += SMP_THREADS) {
    const int x = tokens[i];
    const double qx = qd[(size_t)i * V + x];
    const double px = pd[(size_t)i * V + x];
    const bool zero = !(qx > 0.0);
    const bool fail = zero || !(U[cur + i] < fmin(1.0, px / qx));
    if (fail) atomicMin(&first_s, i);
    if (zero) atomicMin(&zero_s, i);
  }
  __syncthreads();
  const int r = first_s;
  // the first failing proposal raises (verify_token's q(x) = 0 check) when its
  // draft probability is 0
  const int status = (r < n && zero_s == r) ? HS_ERR_CONTRACT : 0;
  int tok = 0, used = 0;
  if (!status) {
    if (r < n) {
      // correct_token: residual max(p - q, 0); Z <= 1e-12 -> sample p
      const double *p = pd + (size_t)r * V, *q = qd + (size_t)r * V;
      const double z = residual_stage(cl, p, q, V, sw);
      const double u2 = U[cur + r + 1];
      tok = (z <= 1e-12) ? inv_cdf(cl, p, nullptr, 1.0, V, u2, sw) : inv_cdf_staged(cl, z, V, u2, sw);
      used = r + 2;
    } else {
      tok = inv_cdf(cl, pd + (size_t)n * V, nullptr, 1.0, V, U[cur + n], sw);
      used = n + 1;
    }
  }
  pdl_trigger();
  cl.finish();   // every CTA has read the cursor and its peers' partials
  if (cl_leader()) {
    if (!status) {
      for (int i = 0; i < r; ++i) result[i] = tokens[i];
      result[r] = tok;
      result[n + 1] = r + 1;
      result[n + 2] = r;
      *cursor = cur + used;
    } else {
      *cursor = cur + r;   // the uniforms of the accepted proposals before the failure
    }
    result[n + 3] = status;
  }
}

__global__ void __launch_bounds__(32) verify_token_kernel(int x, const double *q, const double *p, const double *U,
                                                          int32_t *cursor, int32_t *result) {
  if (threadIdx.x != 0) return;
  const int cur = *cursor;
  const double qx = q[x];
  if (!(qx > 0.0)) { result[0] = 0; result[1] = HS_ERR_CONTRACT; return; }
  result[0] = (U[cur] < fmin(1.0, p[x] / qx)) ? 1 : 0;
  result[1] = 0;
  *cursor = cur + 1;
}

__global__ void __launch_bounds__(SMP_THREADS) correct_token_kernel(const double *q, const double *p, int V,
                                                                    const double *U, int32_t *cursor,
                                                                    int32_t *out) {
  pdl_wait();
  HS_CL_SETUP
  const int cur = *cursor;
  extern __shared__ double sw[];
  const double z = residual_stage(cl, p, q, V, sw);
  const int tok = (z <= 1e-12) ? inv_cdf(cl, p, nullptr, 1.0, V, U[cur], sw) : inv_cdf_staged(cl, z, V, U[cur], sw);
  cl.finish();
  if (cl_leader()) { *out = tok; *cursor = cur + 1; }
}

// cluster launch (one SMP_CL-CTA cluster per row), a programmatic dependent
// of the previous kernel on the stream
template <typename... KArgs, typename... Args>
static int launch_rows(const char *what, void (*kern)(KArgs...), int rows, int V, cudaStream_t st,
                       Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows * SMP_CL);
  cfg.blockDim = dim3(SMP_THREADS);
  cfg.dynamicSmemBytes = (size_t)((V + SMP_CL - 1) / SMP_CL) * sizeof(double);   // inverse-CDF staging
  if (cfg.dynamicSmemBytes > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = SMP_CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1 + pdl_enabled();
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return check_launch(what);
}

static int check_vocab(int V) {
  HS_REQUIRE(V >= 1 && V <= SMP_CL * SMP_THREADS * SEG_REG, HS_ERR_VALUE, "sampling: vocabulary size %d outside [1, %d]",
             V, SMP_CL * SMP_THREADS * SEG_REG);
  return HS_OK;
}

}  // namespace hs

extern "C" int hs_verify_token(int32_t x, const double *q, const double *p, const double *uniforms,
                               int32_t *cursor, int32_t *result, void *stream) {
  hs::verify_token_kernel<<<1, 32, 0, hs::as_stream(stream)>>>(x, q, p, uniforms, cursor, result);
  return hs::check_launch("verify_token");
}

extern "C" int hs_correct_token(const double *q, const double *p, int V, const double *uniforms,
                                int32_t *cursor, int32_t *out, void *stream) {
  int rc = hs::check_vocab(V);
  if (rc != HS_OK) return rc;
  return hs::launch_rows("correct_token", hs::correct_token_kernel, 1, V, hs::as_stream(stream), q, p, V, uniforms,
                         cursor, out);
}

extern "C" int hs_probs(const float *logits, int rows, int V, double temperature, double *probs, void *stream) {
  if (temperature < 0) return hs::set_error(HS_ERR_VALUE, "temperature must be >= 0");
  if (rows <= 0) return HS_OK;
  int rc = hs::check_vocab(V);
  if (rc != HS_OK) return rc;
  return hs::launch_rows("probs", hs::probs_kernel, rows, V, hs::as_stream(stream), logits, V, temperature, probs);
}

extern "C" int hs_sample(const double *probs, int V, const double *uniforms, int32_t *cursor, int32_t *out,
                         void *stream) {
  int rc = hs::check_vocab(V);
  if (rc != HS_OK) return rc;
  return hs::launch_rows("sample", hs::sample_kernel, 1, V, hs::as_stream(stream), probs, V, uniforms, cursor, out);
}

extern "C" int hs_draft_sample(const float *logits, int V, double temperature, double *probs_out,
                               const double *uniforms, int32_t *cursor, int32_t *out, void *stream) {
  if (temperature < 0) return hs::set_error(HS_ERR_VALUE, "temperature must be >= 0");
  if (!probs_out) return hs::set_error(HS_ERR_VALUE, "draft_sample: probs_out required");
  int rc = hs::check_vocab(V);
  if (rc != HS_OK) return rc;
  return hs::launch_rows("draft_sample", hs::draft_sample_kernel, 1, V, hs::as_stream(stream), logits, V, temperature,
                         probs_out, uniforms, cursor, out, (int32_t *)nullptr, 0, 0);
}

static int graph_launch(void *graph_exec, int n_launch, cudaStream_t st) {
  if (!graph_exec) return HS_OK;
  const cudaError_t e = cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(graph_exec), st);
  if (e != cudaSuccess) return hs::set_error(HS_ERR_CUDA, "step graph launch: %s", cudaGetErrorString(e));
  hs::count_launch(n_launch);
  return HS_OK;
}

// small host -> device uploads (token ids of a step) through a pinned ring:
// one call, stream-ordered, no synchronisation (a slot is reused only after
// its previous copy ran); n <= 1024 int32 per call
namespace {
struct UploadRing {
  static constexpr int kSlots = 64, kCap = 1024;
  int32_t *host = nullptr;
  cudaEvent_t ev[kSlots];
  bool used[kSlots] = {};
  int next = 0;
};
thread_local UploadRing g_up;
}  // namespace

extern "C" int hs_upload_i32(int32_t *dst, const int32_t *src, int n, void *stream) {
  if (n < 0 || n > UploadRing::kCap) return hs::set_error(HS_ERR_VALUE, "upload: %d values (max %d)", n, UploadRing::kCap);
  if (n == 0) return HS_OK;
  UploadRing &r = g_up;
  if (!r.host) {
    if (cudaMallocHost(&r.host, sizeof(int32_t) * UploadRing::kSlots * UploadRing::kCap) != cudaSuccess)
      return hs::set_error(HS_ERR_CUDA, "upload: pinned ring allocation failed");
    for (int i = 0; i < UploadRing::kSlots; ++i) cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming);
  }
  const int slot = r.next;
  r.next = (r.next + 1) % UploadRing::kSlots;
  if (r.used[slot]) cudaEventSynchronize(r.ev[slot]);
  int32_t *h = r.host + (size_t)slot * UploadRing::kCap;
  memcpy(h, src, sizeof(int32_t) * n);
  cudaStream_t st = hs::as_stream(stream);
  cudaError_t e = cudaMemcpyAsync(dst, h, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return hs::set_error(HS_ERR_CUDA, "upload: %s", cudaGetErrorString(e));
  cudaEventRecord(r.ev[slot], st);
  r.used[slot] = true;
  return HS_OK;
}

extern "C" int hs_draft_step(const float *logits, int V, double temperature, double *probs_out,
                             const double *uniforms, int32_t *cursor, int32_t *out, int32_t *dyn, int frontier, int lo,
                             void *graph_exec, int n_launch, void *stream) {
  if (temperature < 0) return hs::set_error(HS_ERR_VALUE, "temperature must be >= 0");
  if (!probs_out) return hs::set_error(HS_ERR_VALUE, "draft_step: probs_out required");
  if (!dyn) return hs::set_error(HS_ERR_VALUE, "draft_step: null step slot");
  int rc = hs::check_vocab(V);
  if (rc != HS_OK) return rc;
  cudaStream_t st = hs::as_stream(stream);
  rc = hs::launch_rows("draft_sample", hs::draft_sample_kernel, 1, V, st, logits, V, temperature, probs_out, uniforms,
                       cursor, out, dyn, frontier, lo);
  if (rc != HS_OK) return rc;
  return graph_launch(graph_exec, n_launch, st);
}

extern "C" int hs_graph_step(int32_t *dyn, int frontier, int lo, int token, int32_t *also, void *graph_exec,
                             int n_launch, void *stream) {
  if (!dyn) return hs::set_error(HS_ERR_VALUE, "graph_step: null step slot");
  cudaStream_t st = hs::as_stream(stream);
  hs::graph_step_kernel<<<1, 1, 0, st>>>(dyn, frontier, lo, token, also);
  int rc = hs::check_launch("graph_step");
  if (rc != HS_OK) return rc;
  return graph_launch(graph_exec, n_launch, st);
}

extern "C" int hs_verify_chain(const int32_t *tokens, int n, const double *qd, const double *pd, int V,
                               const double *uniforms, int32_t *cursor, int32_t *result, void *stream) {
  if (n < 0) return hs::set_error(HS_ERR_VALUE, "verify_chain: n < 0");
  int rc = hs::check_vocab(V);
  if (rc != HS_OK) return rc;
  return hs::launch_rows("verify_chain", hs::verify_chain_kernel, 1, V, hs::as_stream(stream), tokens, n, qd, pd, V,
                         uniforms, cursor, result);
}
