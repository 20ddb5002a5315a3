// Top-k attention exposure for the TopKCache pairing (caches.py:568-652,
// SURVEY §8(f) row 4): for one decode query per layer, the exact per-kv-group
// mean softmax weight of every stored key (fp64, TopKCache.group_weights,
// caches.py:601-615), the `budget` heaviest keys per group (ties to the lower
// position, caches.py:617-627), gathered into a compact view that the
// ordinary attention kernels then attend over (keys kept in position order).
//
//   topk_scores_kernel   s[h][key] = (q_h . k_key) / sqrt(dh)      fp64, exact products
//   topk_norm_kernel     per head: max_key s, z = sum exp(s - max)  fp64
//   topk_weight_kernel   w[kv][key] = mean_{h in group} exp(s - max_h) / z_h
//   topk_select_kernel   one CTA per kv group: bitonic sort of (w desc, key asc)
//                        in shared memory, first `budget` keys flagged, then
//                        compacted in key order
//   topk_gather_kernel   K/V rows of the chosen keys -> compact [KVH][budget][dh]
#include "hs_common.cuh"

namespace hs {

int launch_attention(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t, float *out,
                     float *packed, void *ws, size_t ws_bytes, cudaStream_t stream, uint16_t *xs, int ldxs,
                     int clean_hi, const FusedRope *fr);
size_t attention_ws(int t, int H, int DH, int n_view, int split);

namespace {

constexpr int TK_MAX_KEYS = 8192;   // keys one select CTA sorts in shared memory

__global__ void topk_scores_kernel(const uint16_t *k, int cap, int n, int KVH, int g, int dh, const float *q,
                                   double inv_sqrt_dh, double *s) {
  const int key = blockIdx.x * blockDim.x + threadIdx.x, kv = blockIdx.y;
  if (key >= n) return;
  const uint16_t *kr = k + ((size_t)kv * cap + key) * dh;
  for (int j = 0; j < g; ++j) {
    const float *qh = q + (size_t)(kv * g + j) * dh;
    double acc = 0.0;
    for (int d = 0; d < dh; ++d) acc += (double)qh[d] * (double)bf16_to_f(kr[d]);
    s[(size_t)(kv * g + j) * n + key] = acc * inv_sqrt_dh;
  }
}

__global__ void topk_norm_kernel(const double *s, int n, double *mz) {
  const int h = blockIdx.x;
  const double *sh = s + (size_t)h * n;
  __shared__ double red[32];
  double mx = -INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, sh[i]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const double M = red[0];
  __syncthreads();
  double z = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) z += exp(sh[i] - M);
  z = warp_sum(z);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = z;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    mz[2 * h] = M;
    mz[2 * h + 1] = tot;
  }
}

__global__ void topk_weight_kernel(const double *s, const double *mz, int n, int g, double *w) {
  const int key = blockIdx.x * blockDim.x + threadIdx.x, kv = blockIdx.y;
  if (key >= n) return;
  double acc = 0.0;
  for (int j = 0; j < g; ++j) {
    const int h = kv * g + j;
    acc += exp(s[(size_t)h * n + key] - mz[2 * h]) / mz[2 * h + 1];
  }
  w[(size_t)kv * n + key] = acc / (double)g;
}

// (w desc, key asc): true when a must come before b
__device__ __forceinline__ bool before(double wa, int ka, double wb, int kb) {
  return wa > wb || (wa == wb && ka < kb);
}

__global__ void topk_select_kernel(const double *w, int n, int budget, int *chosen) {
  extern __shared__ __align__(16) unsigned char tk_smem[];
  const int kv = blockIdx.x;
  int npow = 1;
  while (npow < n) npow <<= 1;
  double *sw = reinterpret_cast<double *>(tk_smem);
  int *sk = reinterpret_cast<int *>(sw + npow);
  for (int i = threadIdx.x; i < npow; i += blockDim.x) {
    sw[i] = i < n ? w[(size_t)kv * n + i] : -INFINITY;
    sk[i] = i < n ? i : 0x7fffffff;
  }
  __syncthreads();
  for (int size = 2; size <= npow; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < npow; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;   // ascending in "before" order
          const bool swap = up ? before(sw[j], sk[j], sw[i], sk[i]) : before(sw[i], sk[i], sw[j], sk[j]);
          if (swap) {
            const double tw = sw[i]; sw[i] = sw[j]; sw[j] = tw;
            const int tk = sk[i]; sk[i] = sk[j]; sk[j] = tk;
          }
        }
      }
      __syncthreads();
    }
  }
  // the first `budget` entries are the chosen keys: flag them, then emit in key order
  int *flag = sk + npow;                 // reuse: [n] flags after the sort
  for (int i = threadIdx.x; i < n; i += blockDim.x) flag[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < budget; i += blockDim.x) flag[sk[i]] = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    for (int i = 0; i < n; ++i)
      if (flag[i]) chosen[(size_t)kv * budget + c++] = i;
  }
}

__global__ void topk_gather_kernel(const uint16_t *k, const uint16_t *v, int cap, int dh, const int *chosen,
                                   int budget, int ccap, uint16_t *ck, uint16_t *cv) {
  const int i = blockIdx.x, kv = blockIdx.y;
  const int key = chosen[(size_t)kv * budget + i];
  const uint16_t *ks = k + ((size_t)kv * cap + key) * dh, *vs = v + ((size_t)kv * cap + key) * dh;
  uint16_t *kd = ck + ((size_t)kv * ccap + i) * dh, *vd = cv + ((size_t)kv * ccap + i) * dh;
  for (int d = threadIdx.x; d < dh; d += blockDim.x) {
    kd[d] = ks[d];
    vd[d] = vs[d];
  }
}

inline size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

}  // namespace

size_t topk_ws_bytes(const HsModel *m, int n, int budget) {
  const int H = m->n_heads, KVH = m->n_kv_heads, dh = m->head_dim;
  const int ccap = (budget + 127) / 128 * 128;
  return al((size_t)H * n * 8) + al((size_t)H * 16) + al((size_t)KVH * n * 8) + al((size_t)KVH * budget * 4) +
         2 * al((size_t)KVH * ccap * dh * 2) + al(attention_ws(1, H, dh, budget, 512));
}

// layer attention of the single query q [H][dh] over the `budget` heaviest keys
// of each kv group among the cache's slots [0, n) (slot == position)
int launch_topk_attention(const HsModel *m, const HsCache *c, int layer, int n, int pos, int budget, const float *q,
                          uint16_t *xs, int ldxs, void *ws, size_t ws_bytes, cudaStream_t st) {
  const int H = m->n_heads, KVH = m->n_kv_heads, dh = m->head_dim, g = H / KVH;
  HS_REQUIRE(n <= TK_MAX_KEYS, HS_ERR_CAPACITY, "top-k exposure: %d keys > %d", n, TK_MAX_KEYS);
  HS_REQUIRE(budget >= 1 && budget < n, HS_ERR_VALUE, "top-k exposure: budget %d outside [1, %d)", budget, n);
  HS_REQUIRE(ws_bytes >= topk_ws_bytes(m, n, budget), HS_ERR_VALUE, "top-k exposure: workspace too small");
  const int ccap = (budget + 127) / 128 * 128;
  char *p = reinterpret_cast<char *>(ws);
  double *s = reinterpret_cast<double *>(p); p += al((size_t)H * n * 8);
  double *mz = reinterpret_cast<double *>(p); p += al((size_t)H * 16);
  double *w = reinterpret_cast<double *>(p); p += al((size_t)KVH * n * 8);
  int *chosen = reinterpret_cast<int *>(p); p += al((size_t)KVH * budget * 4);
  uint16_t *ck = reinterpret_cast<uint16_t *>(p); p += al((size_t)KVH * ccap * dh * 2);
  uint16_t *cv = reinterpret_cast<uint16_t *>(p); p += al((size_t)KVH * ccap * dh * 2);
  void *att_ws = p;
  const size_t att_bytes = attention_ws(1, H, dh, budget, 512);
  const size_t lay = (size_t)layer * KVH * c->cap * dh;
  topk_scores_kernel<<<dim3((n + 127) / 128, KVH), 128, 0, st>>>(c->k + lay, c->cap, n, KVH, g, dh, q,
                                                                  1.0 / sqrt((double)dh), s);
  topk_norm_kernel<<<H, 256, 0, st>>>(s, n, mz);
  topk_weight_kernel<<<dim3((n + 255) / 256, KVH), 256, 0, st>>>(s, mz, n, g, w);
  int npow = 1;
  while (npow < n) npow <<= 1;
  const size_t smem = (size_t)npow * (8 + 4) + (size_t)n * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(topk_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((size_t)TK_MAX_KEYS * 16));
    attr = true;
  }
  topk_select_kernel<<<KVH, 1024, smem, st>>>(w, n, budget, chosen);
  topk_gather_kernel<<<dim3(budget, KVH), 64, 0, st>>>(c->k + lay, c->v + lay, c->cap, dh, chosen, budget, ccap, ck, cv);
  {
    const int rc = check_launch("top-k exposure", 5);
    if (rc != HS_OK) return rc;
  }
  HsCache cc = *c;
  cc.kind = HS_KV_LINEAR;
  cc.n_layers = 1;
  cc.cap = ccap;
  cc.k = ck;
  cc.v = cv;
  cc.pos = nullptr;
  HsStep sv = {};
  sv.pos0 = pos;
  sv.n_view = budget;
  sv.split = 512;
  return launch_attention(&cc, 0, &sv, H, q, 1, nullptr, nullptr, att_ws, att_bytes, st, xs, ldxs, -1, nullptr);
}

}  // namespace hs
