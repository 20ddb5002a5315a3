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
#include "hs_common.cuh"

namespace hs {

constexpr int SMP_THREADS = 1024;

struct ArgMax { double v; int i; };

__device__ __forceinline__ ArgMax amax(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ ArgMax block_argmax(ArgMax x) {
  __shared__ double sv[SMP_THREADS / 32];
  __shared__ int si[SMP_THREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
    x = amax(x, y);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) { sv[w] = x.v; si[w] = x.i; }
  __syncthreads();
  ArgMax r = {sv[0], si[0]};
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = amax(r, ArgMax{sv[k], si[k]});
  return r;
}

__device__ double block_sum(double x) {
  __shared__ double sw[SMP_THREADS / 32];
  x = warp_sum(x);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sw[w] = x;
  __syncthreads();
  double r = 0.0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r += sw[k];
  return r;
}

__device__ int block_count(int x) {
  __shared__ int sc[SMP_THREADS / 32];
  x = warp_sum(x);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sc[w] = x;
  __syncthreads();
  int r = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r += sc[k];
  return r;
}

// probs of one logits row into p (fp64); whole block participates
__device__ void row_probs(const float *logits, int V, double T, double *p) {
  if (T == 0.0) {
    ArgMax best = {-INFINITY, 0x7fffffff};
    for (int j = threadIdx.x; j < V; j += blockDim.x) best = amax(best, ArgMax{(double)logits[j], j});
    best = block_argmax(best);
    for (int j = threadIdx.x; j < V; j += blockDim.x) p[j] = (j == best.i) ? 1.0 : 0.0;
    __syncthreads();
    return;
  }
  ArgMax mx = {-INFINITY, 0};
  for (int j = threadIdx.x; j < V; j += blockDim.x) mx = amax(mx, ArgMax{(double)logits[j] / T, j});
  mx = block_argmax(mx);
  double s = 0.0;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const double e = exp((double)logits[j] / T - mx.v);
    p[j] = e;
    s += e;
  }
  s = block_sum(s);
  for (int j = threadIdx.x; j < V; j += blockDim.x) p[j] = p[j] / s;
  __syncthreads();
}

// inverse CDF: min(#{j : cumsum(w/scale)_j <= u}, V-1); w optionally the
// residual max(p - q, 0) (computed on the fly); whole block participates.
// Each thread owns a contiguous segment of up to SEG_REG entries held in
// registers (one pass over memory, loads all in flight); the cumulative sum
// is segment-sequential after an exclusive block scan of segment totals --
// a fixed order, so the draw is deterministic.
constexpr int SEG_REG = 32;

__device__ int inv_cdf(const double *p, const double *q, double scale, int V, double u) {
  __shared__ double seg[64];
  const int per = (V + blockDim.x - 1) / blockDim.x;
  const int j0 = threadIdx.x * per, j1 = min(V, j0 + per);
  auto w = [&](int j) {
    double x = q ? fmax(p[j] - q[j], 0.0) : p[j];
    return scale == 1.0 ? x : x / scale;
  };
  double wr[SEG_REG];
  double local = 0.0;
  if (per <= SEG_REG) {
#pragma unroll
    for (int i = 0; i < SEG_REG; ++i) wr[i] = (i < per && j0 + i < j1) ? w(j0 + i) : 0.0;
#pragma unroll
    for (int i = 0; i < SEG_REG; ++i) local += wr[i];
  } else {
    for (int j = j0; j < j1; ++j) local += w(j);
  }
  // exclusive scan of the segment totals: warp scan, then scan of warp totals
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) seg[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    double wt = (lane < (int)(blockDim.x >> 5)) ? seg[lane] : 0.0;
    double wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    double we = __shfl_up_sync(0xffffffffu, wi, 1);
    seg[32 + lane] = (lane == 0) ? 0.0 : we;   // exclusive warp base
  }
  __syncthreads();
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.0;
  double c = seg[32 + wid] + excl;
  int cnt = 0;
  if (per <= SEG_REG) {
#pragma unroll
    for (int i = 0; i < SEG_REG; ++i) {
      if (i < per && j0 + i < j1) {
        c += wr[i];
        cnt += (c <= u) ? 1 : 0;
      }
    }
  } else {
    for (int j = j0; j < j1; ++j) {
      c += w(j);
      cnt += (c <= u) ? 1 : 0;
    }
  }
  cnt = block_count(cnt);
  return cnt < V - 1 ? cnt : V - 1;
}

__global__ void __launch_bounds__(SMP_THREADS) probs_kernel(const float *logits, int V, double T, double *probs) {
  row_probs(logits + (size_t)blockIdx.x * V, V, T, probs + (size_t)blockIdx.x * V);
}

__global__ void __launch_bounds__(SMP_THREADS) sample_kernel(const double *probs, int V, const double *U,
                                                             int32_t *cursor, int32_t *out) {
  const int cur = *cursor;
  const int tok = inv_cdf(probs, nullptr, 1.0, V, U[cur]);
  __syncthreads();
  if (threadIdx.x == 0) { *out = tok; *cursor = cur + 1; }
}

__global__ void __launch_bounds__(SMP_THREADS) draft_sample_kernel(const float *logits, int V, double T,
                                                                   double *probs, const double *U,
                                                                   int32_t *cursor, int32_t *out) {
  const int cur = *cursor;
  if (T == 0.0) {
    // one-hot argmax row; its inverse CDF at any u in [0, 1) is the argmax
    // itself (model.py:198-202 with a one-hot p), so skip the scan
    ArgMax best = {-INFINITY, 0x7fffffff};
    for (int j = threadIdx.x; j < V; j += blockDim.x) best = amax(best, ArgMax{(double)logits[j], j});
    best = block_argmax(best);
    for (int j = threadIdx.x; j < V; j += blockDim.x) probs[j] = (j == best.i) ? 1.0 : 0.0;
    if (threadIdx.x == 0) { *out = best.i < V ? best.i : V - 1; *cursor = cur + 1; }
    return;
  }
  row_probs(logits, V, T, probs);
  const int tok = inv_cdf(probs, nullptr, 1.0, V, U[cur]);
  __syncthreads();
  if (threadIdx.x == 0) { *out = tok; *cursor = cur + 1; }
}

// _verify_chain: result[0..n] tokens, [n+1] count, [n+2] accepted, [n+3] status
__global__ void __launch_bounds__(SMP_THREADS) verify_chain_kernel(const int32_t *tokens, int n, const double *qd,
                                                                   const double *pd, int V, const double *U,
                                                                   int32_t *cursor, int32_t *result) {
  int cur = *cursor;
  int i = 0;
  int status = 0;
  for (; i < n; ++i) {
    const int x = tokens[i];
    const double qx = qd[(size_t)i * V + x];
    const double px = pd[(size_t)i * V + x];
    if (!(qx > 0.0)) { status = HS_ERR_CONTRACT; break; }
    const double ratio = px / qx;
    const double u = U[cur++];
    if (u < fmin(1.0, ratio)) {
      if (threadIdx.x == 0) result[i] = x;
      continue;
    }
    // correct_token: residual max(p - q, 0); Z <= 1e-12 -> sample p
    const double *p = pd + (size_t)i * V, *q = qd + (size_t)i * V;
    double z = 0.0;
    for (int j = threadIdx.x; j < V; j += blockDim.x) z += fmax(p[j] - q[j], 0.0);
    z = block_sum(z);
    const double u2 = U[cur++];
    const int tok = (z <= 1e-12) ? inv_cdf(p, nullptr, 1.0, V, u2) : inv_cdf(p, q, z, V, u2);
    if (threadIdx.x == 0) { result[i] = tok; result[n + 1] = i + 1; result[n + 2] = i; }
    break;
  }
  if (status == 0 && i == n) {
    const double u = U[cur++];
    const int tok = inv_cdf(pd + (size_t)n * V, nullptr, 1.0, V, u);
    if (threadIdx.x == 0) { result[n] = tok; result[n + 1] = n + 1; result[n + 2] = n; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    result[n + 3] = status;
    *cursor = cur;
  }
}

__global__ void __launch_bounds__(SMP_THREADS) verify_token_kernel(int x, const double *q, const double *p,
                                                                   const double *U, int32_t *cursor,
                                                                   int32_t *result) {
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
  const int cur = *cursor;
  double z = 0.0;
  for (int j = threadIdx.x; j < V; j += blockDim.x) z += fmax(p[j] - q[j], 0.0);
  z = block_sum(z);
  const int tok = (z <= 1e-12) ? inv_cdf(p, nullptr, 1.0, V, U[cur]) : inv_cdf(p, q, z, V, U[cur]);
  __syncthreads();
  if (threadIdx.x == 0) { *out = tok; *cursor = cur + 1; }
}

}  // namespace hs

extern "C" int hs_verify_token(int32_t x, const double *q, const double *p, const double *uniforms,
                               int32_t *cursor, int32_t *result, void *stream) {
  hs::verify_token_kernel<<<1, 32, 0, hs::as_stream(stream)>>>(x, q, p, uniforms, cursor, result);
  return hs::check_launch("verify_token");
}

extern "C" int hs_correct_token(const double *q, const double *p, int V, const double *uniforms,
                                int32_t *cursor, int32_t *out, void *stream) {
  hs::correct_token_kernel<<<1, hs::SMP_THREADS, 0, hs::as_stream(stream)>>>(q, p, V, uniforms, cursor, out);
  return hs::check_launch("correct_token");
}

extern "C" int hs_probs(const float *logits, int rows, int V, double temperature, double *probs, void *stream) {
  if (temperature < 0) return hs::set_error(HS_ERR_VALUE, "temperature must be >= 0");
  if (rows <= 0) return HS_OK;
  hs::probs_kernel<<<rows, hs::SMP_THREADS, 0, hs::as_stream(stream)>>>(logits, V, temperature, probs);
  return hs::check_launch("probs");
}

extern "C" int hs_sample(const double *probs, int V, const double *uniforms, int32_t *cursor, int32_t *out,
                         void *stream) {
  hs::sample_kernel<<<1, hs::SMP_THREADS, 0, hs::as_stream(stream)>>>(probs, V, uniforms, cursor, out);
  return hs::check_launch("sample");
}

extern "C" int hs_draft_sample(const float *logits, int V, double temperature, double *probs_out,
                               const double *uniforms, int32_t *cursor, int32_t *out, void *stream) {
  if (temperature < 0) return hs::set_error(HS_ERR_VALUE, "temperature must be >= 0");
  if (!probs_out) return hs::set_error(HS_ERR_VALUE, "draft_sample: probs_out required");
  hs::draft_sample_kernel<<<1, hs::SMP_THREADS, 0, hs::as_stream(stream)>>>(logits, V, temperature, probs_out,
                                                                           uniforms, cursor, out);
  return hs::check_launch("draft_sample");
}

extern "C" int hs_verify_chain(const int32_t *tokens, int n, const double *qd, const double *pd, int V,
                               const double *uniforms, int32_t *cursor, int32_t *result, void *stream) {
  if (n < 0) return hs::set_error(HS_ERR_VALUE, "verify_chain: n < 0");
  hs::verify_chain_kernel<<<1, hs::SMP_THREADS, 0, hs::as_stream(stream)>>>(tokens, n, qd, pd, V, uniforms,
                                                                           cursor, result);
  return hs::check_launch("verify_chain");
}
