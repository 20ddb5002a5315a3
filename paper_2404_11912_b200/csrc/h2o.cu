// Attention probabilities as a by-product of a forward (model.py:294-313):
//  * H2O feedback (caches.py:291-396, model.py:306-307): per layer, every query
//    row's softmax probabilities over the exposed entries, summed over all
//    heads -- what H2OCache.observe_attention accumulates;
//  * attention probes (ForwardRecorder(record_probs=True), model.py:308-312,
//    attention_probe model.py:381-393): per layer and head, the last query
//    row's probabilities over the exposed entries.
// Follows the reference's rounding points: fp64 dot products rounded to fp32
// scores, fp64 softmax, fp32 probabilities, fp64 head sums (fixed head
// order).  Visibility is the attention kernels' rule (slot positions, causal,
// sinks + window).
#include "hs_common.cuh"

namespace hs {
namespace {

struct ProbView {
  const int32_t *pos;   // layer [cap] slot positions, or null: slot + pos_base
  int pos_base, window, n_sink, win_lo;
};

__device__ __forceinline__ bool probe_visible(int kp, int qp, const ProbView &v) {
  if (kp < 0 || kp > qp) return false;
  if (v.window == 0 || kp < v.n_sink) return true;
  const int lo = max(qp - v.window + 1, v.win_lo);
  return kp >= lo;
}

// grid (t, H): one row's probabilities for one head over slots [0, n)
__global__ void h2o_head_probs_kernel(const uint16_t *k, ProbView pv, int cap, int n, int KVH, int g, int dh,
                                      const float *q, int H, int pos0, double scale, float *hp) {
  const int i = blockIdx.x, h = blockIdx.y, kv = h / g;
  const int qp = pos0 + i;
  const float *qh = q + ((size_t)i * H + h) * dh;
  float *out = hp + ((size_t)i * H + h) * n;
  extern __shared__ double h2o_z[];   // [n]
  __shared__ double red[32];
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int kp = pv.pos ? pv.pos[j] : j + pv.pos_base;
    double z = -INFINITY;
    if (probe_visible(kp, qp, pv)) {
      const uint16_t *kr = k + ((size_t)kv * cap + j) * dh;
      double acc = 0.0;
      for (int d = 0; d < dh; ++d) acc += (double)qh[d] * (double)bf16_to_f(kr[d]);
      z = (double)(float)acc * scale;            // fp32 scores, fp64 softmax (model.py:294-302)
    }
    h2o_z[j] = z;
    mx = fmax(mx, z);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = -INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    red[0] = m;
  }
  __syncthreads();
  const double M = red[0];
  __syncthreads();
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) s += h2o_z[j] == -INFINITY ? 0.0 : exp(h2o_z[j] - M);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    red[0] = tot;
  }
  __syncthreads();
  const double S = red[0];
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    out[j] = h2o_z[j] == -INFINITY ? 0.f : (float)(exp(h2o_z[j] - M) / S);
}

// probs[i][j] = sum over heads (in head order) of hp[i][h][j], fp64
__global__ void h2o_head_sum_kernel(const float *hp, int t, int H, int n, double *probs) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (j >= n) return;
  double acc = 0.0;
  for (int h = 0; h < H; ++h) acc += (double)hp[((size_t)i * H + h) * n + j];
  probs[(size_t)i * n + j] = acc;
}

}  // namespace

// layer `layer`: q [t][H][dh] (roped) at positions pos0.. over the slots
// [0, n) of a slotted cache -> probs [t][n] fp64 (scratch hp [t][H][n] fp32)
int launch_h2o_probs(const HsCache *c, int layer, int H, const float *q, int t, int pos0, int n, double *probs,
                     float *hp, cudaStream_t st) {
  HS_REQUIRE(c->kind == HS_KV_SLOTTED && c->pos != nullptr, HS_ERR_VALUE, "h2o probs: needs a slotted cache");
  HS_REQUIRE((size_t)n * 8 <= 96 * 1024, HS_ERR_CAPACITY, "h2o probs: %d entries exceed the shared-memory row", n);
  ProbView pv = {c->pos + (size_t)layer * c->cap, 0, 0, 0, 0};
  const int KVH = c->n_kv_heads, dh = c->head_dim;
  const size_t lay = (size_t)layer * KVH * c->cap * dh;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(h2o_head_probs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  h2o_head_probs_kernel<<<dim3(t, H), 256, (size_t)n * 8, st>>>(c->k + lay, pv, c->cap, n, KVH, H / KVH, dh, q, H,
                                                                pos0, 1.0 / sqrt((double)dh), hp);
  h2o_head_sum_kernel<<<dim3((n + 255) / 256, t), 256, 0, st>>>(hp, t, H, n, probs);
  return check_launch("h2o probs", 2);
}

// attention probe: the last of t query rows (q [t][H][dh]) at positions
// st->pos0.., per head, over the view [0, st->n_view) -> probe [H][n_view] fp32
int launch_probe_probs(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t, float *probe,
                       cudaStream_t s) {
  const int n = st->n_view;
  HS_REQUIRE((size_t)n * 8 <= 96 * 1024, HS_ERR_CAPACITY, "attention probe: %d entries exceed the shared-memory row",
             n);
  HS_REQUIRE(st->dyn == nullptr, HS_ERR_VALUE, "attention probe: run-time positions unsupported");
  const int KVH = c->n_kv_heads, dh = c->head_dim;
  const size_t lay = (size_t)layer * KVH * c->cap * dh;
  ProbView pv = {c->kind == HS_KV_SLOTTED ? c->pos + (size_t)layer * c->cap : nullptr, st->pos_base, st->window,
                 st->n_sink, st->win_lo};
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(h2o_head_probs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  h2o_head_probs_kernel<<<dim3(1, H), 256, (size_t)n * 8, s>>>(c->k + lay, pv, c->cap, n, KVH, H / KVH, dh,
                                                              q + (size_t)(t - 1) * H * dh, H, st->pos0 + t - 1,
                                                              1.0 / sqrt((double)dh), probe);
  return check_launch("attention probe");
}

}  // namespace hs
