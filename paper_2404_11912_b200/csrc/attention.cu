// Split-KV ("flash-decoding") attention over a KV-cache view, CUDA cores.
//
// Replaces the attention core of the reference forward (model.py:290-315):
// grouped scores q.K^T, causal / exposure masks, softmax with 1/sqrt(dh),
// P.V.  The cache is never materialised (no expose()): the kernel scans the
// view's slots [0, n_view) and applies the exposure rule per query:
//   visible(qp, kp) = kp >= 0 && kp <= qp &&
//                     (window == 0 || kp < n_sink || kp >= max(win_lo, qp - window + 1))
// which is FullCache (window 0), RetrievalCache (sel + spec tail, window 0)
// and the per-step StreamingCache exposure (caches.py:246-256).
//
// Grid: (n_splits, kv_heads, query-row blocks of 16).  Splits are fixed-size
// ranges of slots, so a query's partial state never depends on how many
// other queries share the launch; the combine walks splits in index order.
#include <vector>

#include "hs_common.cuh"

namespace hs {

HS_TRACE_TU
int trace_set_attn(void *p, unsigned cap) { return trace_set_tu(p, cap); }

constexpr int ATT_THREADS = 128;
constexpr int ATT_TILE = 64;     // keys per smem tile
constexpr int ATT_QROWS = 16;    // query rows per CTA

struct AttnArgs {
  const float *q;       // [t][H][DH]
  int t, H, KVH, g;
  const uint16_t *k;    // layer base [KVH][cap][DH]
  const uint16_t *v;
  const int32_t *pos;   // layer [cap] or null (slot == position)
  int cap, n_view, pos0, window, win_lo, n_sink, split, n_splits, pos_base;
  const int32_t *dyn;   // HsStep.dyn: run-time frontier / win_lo (graph replay)
  float scale;
  float *part_m, *part_l, *part_o;   // [n_splits][t*H], [n_splits][t*H][DH]
};

__device__ __forceinline__ bool visible(int kp, int qp, const AttnArgs &a) {
  if (kp < 0 || kp > qp) return false;
  if (a.window == 0 || kp < a.n_sink) return true;
  int lo = qp - a.window + 1;
  if (a.win_lo > lo) lo = a.win_lo;
  return kp >= lo;
}

template <int DH>
__global__ void __launch_bounds__(ATT_THREADS) attn_partial_kernel(AttnArgs a) {
  HS_TRACE_BEGIN
  pdl_trigger();   // the combine kernel is scheduled once every CTA here has started
  pdl_wait();      // q and the appended K/V rows come from the rope kernel
  HS_TRACE_RESTART
  if (a.dyn) { a.pos0 += a.dyn[0]; a.win_lo = a.dyn[1]; }
  constexpr int KP = DH + 8;                 // padded K row (bf16) -> conflict-free 16B reads
  constexpr int NDP = DH / 2;                // dim pairs
  constexpr int NRG = ATT_THREADS / NDP > ATT_QROWS ? ATT_QROWS : ATT_THREADS / NDP;
  constexpr int RPT = (ATT_QROWS + NRG - 1) / NRG;   // rows per thread in PV
  __shared__ __align__(16) uint16_t Ks[ATT_TILE * KP];
  __shared__ __align__(16) uint16_t Vs[ATT_TILE * DH];
  __shared__ __align__(16) float qs[ATT_QROWS * DH];
  __shared__ float S[ATT_QROWS][ATT_TILE];
  __shared__ int kpos[ATT_TILE];
  __shared__ float m_s[ATT_QROWS], l_s[ATT_QROWS], f_s[ATT_QROWS];
  __shared__ int qp_s[ATT_QROWS], head_s[ATT_QROWS], tok_s[ATT_QROWS];

  const int split = blockIdx.x, kh = blockIdx.y, rb = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nrows_total = a.g * a.t;
  const int r0 = rb * ATT_QROWS;
  const int nrows = min(ATT_QROWS, nrows_total - r0);

  const int s_lo = split * a.split;
  const int s_hi = min(a.n_view, s_lo + a.split);
  const uint16_t *kbase = a.k + (size_t)kh * a.cap * DH;
  const uint16_t *vbase = a.v + (size_t)kh * a.cap * DH;
  constexpr int VPR = DH / 8;  // 16B vectors per row
  constexpr int VPT = (ATT_TILE * VPR + ATT_THREADS - 1) / ATT_THREADS;
  uint4 kv4[VPT], vv4[VPT];
  // all of this thread's K / V vectors of a tile in flight at once
  auto load_tile = [&](int tile, int nk) {
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int e = tid + u * ATT_THREADS, kr = e / VPR, c = e % VPR;
      kv4[u] = make_uint4(0, 0, 0, 0);
      vv4[u] = make_uint4(0, 0, 0, 0);
      if (e < ATT_TILE * VPR && kr < nk) {
        kv4[u] = ld_stream(kbase + (size_t)(tile + kr) * DH + c * 8);
        vv4[u] = ld_stream(vbase + (size_t)(tile + kr) * DH + c * 8);
      }
    }
  };

  // query rows: rr = i*g + gi  ->  token i, head kh*g + gi
  if (tid < ATT_QROWS) {
    int rr = r0 + tid;
    if (tid < nrows) {
      int i = rr / a.g, gi = rr % a.g;
      tok_s[tid] = i; head_s[tid] = kh * a.g + gi; qp_s[tid] = a.pos0 + i;
    } else {
      tok_s[tid] = 0; head_s[tid] = 0; qp_s[tid] = -1;
    }
    m_s[tid] = -INFINITY; l_s[tid] = 0.f; f_s[tid] = 1.f;
  }
  __syncthreads();
  {
    // every load of the query rows and of the first K / V tile in flight at
    // once (a step's first round trip), then the shared-memory stores
    constexpr int QPT = ATT_QROWS * DH / ATT_THREADS;
    float qv[QPT];
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
      const int e = tid + u * ATT_THREADS, rr = e / DH, d = e % DH;
      qv[u] = rr < nrows ? a.q[((size_t)tok_s[rr] * a.H + head_s[rr]) * DH + d] : 0.f;
    }
    if (s_lo < s_hi) load_tile(s_lo, min(ATT_TILE, s_hi - s_lo));   // (the first tile's K / V too)
#pragma unroll
    for (int u = 0; u < QPT; ++u) qs[tid + u * ATT_THREADS] = qv[u];
  }

  float acc[RPT][2];
#pragma unroll
  for (int i = 0; i < RPT; ++i) acc[i][0] = acc[i][1] = 0.f;
  const int dp = tid % NDP, rg = tid / NDP;

  for (int tile = s_lo; tile < s_hi; tile += ATT_TILE) {
    const int nk = min(ATT_TILE, s_hi - tile);
    __syncthreads();   // previous tile fully consumed
    // ---- stage K, V (16-byte vectors) and positions ------------------------
    if (tile != s_lo) load_tile(tile, nk);
    {
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const int e = tid + u * ATT_THREADS, kr = e / VPR, c = e % VPR;
        if (e < ATT_TILE * VPR) {
          *reinterpret_cast<uint4 *>(&Ks[kr * KP + c * 8]) = kv4[u];
          *reinterpret_cast<uint4 *>(&Vs[kr * DH + c * 8]) = vv4[u];
        }
      }
    }
    if (tid < ATT_TILE) {
      int j = tile + tid;
      kpos[tid] = (tid < nk) ? (a.pos ? a.pos[j] : j + a.pos_base) : -1;
    }
    __syncthreads();
    // ---- scores: thread = (key, half of the rows) ---------------------------
    {
      const int key = tid & (ATT_TILE - 1), half = tid >> 6;   // ATT_THREADS == 2*ATT_TILE
      float dot[ATT_QROWS / 2];
#pragma unroll
      for (int i = 0; i < ATT_QROWS / 2; ++i) dot[i] = 0.f;
#pragma unroll 4
      for (int d = 0; d < DH; d += 8) {
        float kf[8];
        unpack8(*reinterpret_cast<const uint4 *>(&Ks[key * KP + d]), kf);
#pragma unroll
        for (int i = 0; i < ATT_QROWS / 2; ++i) {
          const int rr = half + 2 * i;
          if (rr >= nrows) break;   // (warp-uniform: half is a function of the warp)
          const float4 qa = *reinterpret_cast<const float4 *>(&qs[rr * DH + d]);
          const float4 qb = *reinterpret_cast<const float4 *>(&qs[rr * DH + d + 4]);
          float s = dot[i];
          s = fmaf(qa.x, kf[0], s); s = fmaf(qa.y, kf[1], s);
          s = fmaf(qa.z, kf[2], s); s = fmaf(qa.w, kf[3], s);
          s = fmaf(qb.x, kf[4], s); s = fmaf(qb.y, kf[5], s);
          s = fmaf(qb.z, kf[6], s); s = fmaf(qb.w, kf[7], s);
          dot[i] = s;
        }
      }
      const int kp = kpos[key];
#pragma unroll
      for (int i = 0; i < ATT_QROWS / 2; ++i) {
        const int rr = half + 2 * i;
        S[rr][key] = (rr < nrows && key < nk && visible(kp, qp_s[rr], a)) ? dot[i] * a.scale : -INFINITY;
      }
    }
    __syncthreads();
    // ---- online softmax: one warp per row -------------------------------------
    for (int rr = warp; rr < nrows; rr += ATT_THREADS / 32) {   // (rows past nrows are never written)
      float s0 = S[rr][lane], s1 = S[rr][lane + 32];
      float tmax = warp_max(fmaxf(s0, s1));
      float m_old = m_s[rr];
      float m_new = fmaxf(m_old, tmax);
      float p0 = 0.f, p1 = 0.f, fac = 1.f;
      if (m_new != -INFINITY) {
        p0 = (s0 == -INFINITY) ? 0.f : expf(s0 - m_new);
        p1 = (s1 == -INFINITY) ? 0.f : expf(s1 - m_new);
        fac = (m_old == -INFINITY) ? 0.f : expf(m_old - m_new);
      }
      float ps = warp_sum(p0 + p1);
      __syncwarp();   // every lane's reads of this row (and of m_s / l_s) precede the writes
      S[rr][lane] = p0; S[rr][lane + 32] = p1;
      if (lane == 0) {
        f_s[rr] = fac; m_s[rr] = m_new; l_s[rr] = l_s[rr] * fac + ps;
      }
    }
    __syncthreads();
    // ---- P.V: thread = (dim pair, row group) -----------------------------------
    if (rg < NRG) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int rr = rg + NRG * i;
        if (rr < ATT_QROWS) { const float f = f_s[rr]; acc[i][0] *= f; acc[i][1] *= f; }
      }
      // (unrolled: the shared-memory loads of the next keys issue ahead of
      // the accumulator chain, which stays in key order)
#pragma unroll 8
      for (int key = 0; key < nk; ++key) {
        const uint32_t vw = *reinterpret_cast<const uint32_t *>(&Vs[key * DH + 2 * dp]);
        const float v0 = bf16_lo(vw), v1 = bf16_hi(vw);
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int rr = rg + NRG * i;
          if (rr < nrows) {
            const float p = S[rr][key];
            acc[i][0] = fmaf(p, v0, acc[i][0]);
            acc[i][1] = fmaf(p, v1, acc[i][1]);
          }
        }
      }
    }
  }
  __syncthreads();
  // ---- write partial state ------------------------------------------------------
  const size_t base = (size_t)split * a.t * a.H;
  if (tid < nrows) {
    const size_t row = (size_t)tok_s[tid] * a.H + head_s[tid];
    a.part_m[base + row] = m_s[tid];
    a.part_l[base + row] = l_s[tid];
  }
  if (rg < NRG) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int rr = rg + NRG * i;
      if (rr < nrows) {
        const size_t row = (size_t)tok_s[rr] * a.H + head_s[rr];
        float *o = a.part_o + (base + row) * DH + 2 * dp;
        o[0] = acc[i][0];
        o[1] = acc[i][1];
      }
    }
  }
  HS_TRACE_END(8)
}

// out[i][h*DH + d] = sum_s w_s o_s / sum_s w_s l_s,  w_s = exp(m_s - M), splits in order.
// packed != nullptr: write the view's partial state (M, l, o unnormalised)
// as [rows][2 + DH] instead (sequence-shard input, hs_attention_partial).
// Latency-shaped: the CTA loads the row's (m, l) of up to CHUNK splits once
// into shared memory while every thread's o column of every split is in
// flight, so a view of <= CHUNK splits costs one L2 round trip (CHUNK 16 for
// the retrieval / streaming views, 64 for the full cache up to 131,072 keys);
// longer views take one max pass and one sum pass per chunk.  The sums run in
// split order with the same operations as shard_merge_kernel.
template <int COMB_CHUNK>
__global__ void __launch_bounds__(128) attn_combine_kernel(const float *pm, const float *pl, const float *po, int n_splits,
                                    int rows, int DH, float *out, float *packed, uint16_t *xs, int ldxs, int H) {
  HS_TRACE_BEGIN
  // the next GEMV (wo, PDL-launched) may start streaming its weights now
  pdl_trigger();
  pdl_wait();      // partial states of the attention kernel
  HS_TRACE_RESTART
  const int row = blockIdx.x, d = threadIdx.x;
  const size_t ostride = (size_t)rows * DH;
  const float *pd = po + (size_t)row * DH + d;
  float M = -INFINITY, l = 0.f, o = 0.f;
  if (n_splits <= COMB_CHUNK) {
    // one round trip: the row's (m, l) of every split are loaded once per CTA
    // into shared memory (not by every thread) while each thread's o column
    // of every split is in flight; M, the split weights and l are computed
    // once per CTA, so a thread's work is its o chain alone
    __shared__ float ms[COMB_CHUNK], ls[COMB_CHUNK], ws[COMB_CHUNK];
    __shared__ float Ml[2];
    for (int u = d; u < COMB_CHUNK; u += blockDim.x) {
      ms[u] = u < n_splits ? __ldcg(pm + (size_t)u * rows + row) : -INFINITY;
      ls[u] = u < n_splits ? __ldcg(pl + (size_t)u * rows + row) : 0.f;
    }
    float ov[COMB_CHUNK];
    if (n_splits > 0) {
      const int last = n_splits - 1;
#pragma unroll
      for (int u = 0; u < COMB_CHUNK; ++u) ov[u] = __ldcg(pd + (size_t)(u < last ? u : last) * ostride);   // (clamped: weight 0)
    } else {
#pragma unroll
      for (int u = 0; u < COMB_CHUNK; ++u) ov[u] = 0.f;
    }
    __syncthreads();
    const int nw = blockDim.x < 32 ? (int)blockDim.x : 32;   // the first warp (all of a small block)
    if (d < nw) {
      float mx = -INFINITY;
      for (int u = d; u < COMB_CHUNK; u += nw) mx = fmaxf(mx, ms[u]);
      if (nw == 32) {
        mx = warp_max(mx);   // max: order-free
      } else {
        __shared__ float mred[32];
        mred[d] = mx;
        __syncwarp((1u << nw) - 1);
        mx = -INFINITY;
        for (int k = 0; k < nw; ++k) mx = fmaxf(mx, mred[k]);
      }
      for (int u = d; u < COMB_CHUNK; u += nw) ws[u] = (ms[u] == -INFINITY) ? 0.f : expf(ms[u] - mx);
      __syncwarp(nw == 32 ? 0xffffffffu : (1u << nw) - 1);
      if (d == 0) {
        float lsum = 0.f;
        for (int u = 0; u < n_splits; ++u) {
          const float w = ws[u];
          if (w != 0.f) lsum = fmaf(w, ls[u], lsum);
        }
        Ml[0] = mx;
        Ml[1] = lsum;
      }
    }
    __syncthreads();
    M = Ml[0];
    l = Ml[1];
#pragma unroll
    for (int u = 0; u < COMB_CHUNK; ++u) {
      const float w = ws[u];
      o = (w != 0.f) ? fmaf(w, ov[u], o) : o;   // splits in order, as shard_merge_kernel
    }
  } else {
    // longer views: one max pass and one sum pass per chunk of splits
    float mv[COMB_CHUNK], lv[COMB_CHUNK], ov[COMB_CHUNK];
    for (int s0 = 0; s0 < n_splits; s0 += COMB_CHUNK) {
#pragma unroll
      for (int u = 0; u < COMB_CHUNK; ++u) mv[u] = s0 + u < n_splits ? __ldcg(pm + (size_t)(s0 + u) * rows + row) : -INFINITY;
#pragma unroll
      for (int u = 0; u < COMB_CHUNK; ++u) M = fmaxf(M, mv[u]);
    }
    for (int s0 = 0; s0 < n_splits; s0 += COMB_CHUNK) {
#pragma unroll
      for (int u = 0; u < COMB_CHUNK; ++u) {
        const int sp = s0 + u;
        mv[u] = sp < n_splits ? __ldcg(pm + (size_t)sp * rows + row) : -INFINITY;
        lv[u] = sp < n_splits ? __ldcg(pl + (size_t)sp * rows + row) : 0.f;
        ov[u] = sp < n_splits ? __ldcg(pd + sp * ostride) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < COMB_CHUNK; ++u) {
        const float w = (mv[u] == -INFINITY) ? 0.f : expf(mv[u] - M);
        if (w != 0.f) {
          l = fmaf(w, lv[u], l);
          o = fmaf(w, ov[u], o);
        }
      }
    }
  }
  if (packed) {
    packed[(size_t)row * (DH + 2) + 2 + d] = o;
    if (d == 0) {
      packed[(size_t)row * (DH + 2)] = M;
      packed[(size_t)row * (DH + 2) + 1] = l;
    }
  } else {
    const float v = o / l;
    if (out) out[(size_t)row * DH + d] = v;
    if (xs) store_split(xs, ldxs, row / H, (row % H) * DH + d, v);
  }
  HS_TRACE_END(5)
}

// rank-ordered merge of packed partial states [G][rows][2 + DH];
// the same arithmetic as attn_combine_kernel, so a 1-rank merge of a packed
// partial reproduces the unsharded output bit for bit.
__global__ void shard_merge_kernel(const float *parts, int G, int rows, int DH, float *out, uint16_t *xs, int ldxs,
                                   int H) {
  const int row = blockIdx.x;
  const size_t stride = (size_t)rows * (DH + 2);
  float M = -INFINITY;
  for (int g = 0; g < G; ++g) M = fmaxf(M, parts[g * stride + (size_t)row * (DH + 2)]);
  for (int d = threadIdx.x; d < DH; d += blockDim.x) {
    float l = 0.f, o = 0.f;
    for (int g = 0; g < G; ++g) {
      const float *p = parts + g * stride + (size_t)row * (DH + 2);
      const float m = p[0];
      if (m == -INFINITY) continue;
      const float w = expf(m - M);
      l = fmaf(w, p[1], l);
      o = fmaf(w, p[2 + d], o);
    }
    const float v = o / l;
    if (out) out[(size_t)row * DH + d] = v;
    if (xs) store_split(xs, ldxs, row / H, (row % H) * DH + d, v);
  }
}

int launch_shard_merge(const float *parts, int G, int rows, int DH, float *out, uint16_t *xs, int ldxs, int H,
                       cudaStream_t st) {
  HS_REQUIRE(G >= 1 && rows >= 1, HS_ERR_VALUE, "shard_merge: empty");
  shard_merge_kernel<<<rows, DH < 128 ? DH : 128, 0, st>>>(parts, G, rows, DH, out, xs, ldxs, H > 0 ? H : 1);
  return check_launch("shard_merge");
}

size_t attention_ws(int t, int H, int DH, int n_view, int split) {
  size_t ns = (size_t)ceil_div(n_view, split);
  return ns * t * H * (2 + DH) * sizeof(float) + 256;
}

int launch_attention_tc(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t, float *part_m,
                        float *part_l, float *part_o, int n_splits, cudaStream_t stream, int clean_hi,
                        const FusedRope *fr);

// ---- live timing of the dominant kernel (bench.py roofline) --------------------
// When enabled, every attention launch over a view of >= min_view keys is
// bracketed by CUDA events on its own stream; bench.py reads the summed
// durations and algorithmic bytes after its timed region.
struct ProfPair { cudaEvent_t a, b; long long bytes; };
static std::vector<ProfPair> g_prof;
static size_t g_prof_used = 0;
static int g_prof_on = 0, g_prof_min = 0, g_prof_dropped = 0;

static ProfPair *prof_begin(const HsCache *c, const HsStep *st, cudaStream_t stream) {
  if (!g_prof_on || st->n_view < g_prof_min) return nullptr;
  if (g_prof_used == g_prof.size()) { ++g_prof_dropped; return nullptr; }
  ProfPair *p = &g_prof[g_prof_used++];
  p->bytes = (long long)st->n_view * c->n_kv_heads * c->head_dim * 2 * 2;
  cudaEventRecord(p->a, stream);
  return p;
}

int launch_attention(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t,
                     float *out, float *packed, void *ws, size_t ws_bytes, cudaStream_t stream,
                     uint16_t *xs = nullptr, int ldxs = 0, int clean_hi = -1, const FusedRope *fr = nullptr);

int launch_attention_timed(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t,
                           float *out, float *packed, void *ws, size_t ws_bytes, cudaStream_t stream,
                           uint16_t *xs, int ldxs, int clean_hi, const FusedRope *fr) {
  ProfPair *p = prof_begin(c, st, stream);
  const int rc = launch_attention(c, layer, st, H, q, t, out, packed, ws, ws_bytes, stream, xs, ldxs, clean_hi, fr);
  if (p) cudaEventRecord(p->b, stream);
  return rc;
}

// out: normalised rows [t][H*DH] fp32 (may be null when xs is given);
// xs: additionally the exact 3-way split operand [24][ldxs] of the next GEMV
// (t <= 8), so no separate split kernel runs before wo
// clean_hi: slots below it are not written by any kernel of the current
// programmatic-dependency chain (>= 0 only from the forward, which knows where
// its RoPE kernel appends); the tensor-core kernel may load them before its
// griddepcontrol.wait
int launch_attention(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t,
                     float *out, float *packed, void *ws, size_t ws_bytes, cudaStream_t stream,
                     uint16_t *xs, int ldxs, int clean_hi, const FusedRope *fr) {
  const int DH = c->head_dim, KVH = c->n_kv_heads;
  HS_REQUIRE(H % KVH == 0, HS_ERR_SHAPE, "attention: H %% KVH != 0");
  HS_REQUIRE(st->split > 0 && st->split % ATT_TILE == 0, HS_ERR_VALUE, "attention: split must be a multiple of %d", ATT_TILE);
  HS_REQUIRE(st->n_view >= (packed ? 0 : 1) && st->n_view <= c->cap, HS_ERR_CAPACITY,
             "attention: view %d outside [1, capacity %d]", st->n_view, c->cap);
  const int n_splits = ceil_div(st->n_view, st->split);
  HS_REQUIRE(ws_bytes >= attention_ws(t, H, DH, st->n_view, st->split), HS_ERR_VALUE, "attention: workspace too small");
  AttnArgs a;
  a.q = q; a.t = t; a.H = H; a.KVH = KVH; a.g = H / KVH;
  size_t lay = (size_t)layer * KVH * c->cap * DH;
  a.k = c->k + lay; a.v = c->v + lay;
  a.pos = (c->kind == HS_KV_SLOTTED) ? c->pos + (size_t)layer * c->cap : nullptr;
  a.cap = c->cap; a.n_view = st->n_view; a.pos0 = st->pos0; a.window = st->window;
  a.win_lo = st->win_lo; a.n_sink = st->n_sink; a.split = st->split; a.n_splits = n_splits;
  a.pos_base = st->pos_base;
  a.dyn = st->dyn;
  a.scale = (float)(1.0 / sqrt((double)DH));
  float *wsf = reinterpret_cast<float *>(ws);
  a.part_m = wsf;
  a.part_l = wsf + (size_t)n_splits * t * H;
  a.part_o = wsf + (size_t)2 * n_splits * t * H;
  dim3 grid(n_splits, KVH, ceil_div(a.g * t, ATT_QROWS));
  if (n_splits == 0) {   // empty shard view: partial state (-inf, 0, 0) for every row
    cudaError_t e = launch_pdl(attn_combine_kernel<16>, dim3(t * H), dim3(DH), 0, stream,
                               (const float *)a.part_m, (const float *)a.part_l, (const float *)a.part_o, 0, t * H,
                               DH, (float *)nullptr, packed, (uint16_t *)nullptr, 0, H);
    if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "attention(empty) launch: %s", cudaGetErrorString(e));
    return check_launch("attention(empty)");
  }
  // head_dim 128 (the Llama-family targets) runs on the tensor cores; the
  // small-head draft model and the test-size models use the CUDA-core kernel
  HS_REQUIRE(fr == nullptr || DH == 128, HS_ERR_VALUE, "attention: fused RoPE needs head_dim 128");
  cudaError_t le = cudaSuccess;
  switch (DH) {
    case 8: le = launch_pdl(attn_partial_kernel<8>, grid, dim3(ATT_THREADS), 0, stream, a); break;
    case 16: le = launch_pdl(attn_partial_kernel<16>, grid, dim3(ATT_THREADS), 0, stream, a); break;
    case 32: le = launch_pdl(attn_partial_kernel<32>, grid, dim3(ATT_THREADS), 0, stream, a); break;
    case 64: le = launch_pdl(attn_partial_kernel<64>, grid, dim3(ATT_THREADS), 0, stream, a); break;
    case 128: {
      HS_REQUIRE(st->split % 128 == 0, HS_ERR_VALUE, "attention: split must be a multiple of 128 for head_dim 128");
      int rc = launch_attention_tc(c, layer, st, H, q, t, a.part_m, a.part_l, a.part_o, n_splits, stream,
                                   clean_hi, fr);
      if (rc != HS_OK) return rc;
      break;
    }
    default: return set_error(HS_ERR_SHAPE, "attention: head_dim %d unsupported (8/16/32/64/128)", DH);
  }
  if (le != cudaSuccess) return set_error(HS_ERR_CUDA, "attention launch: %s", cudaGetErrorString(le));
  auto comb = (n_splits > 16 && n_splits <= 64) ? attn_combine_kernel<64> : attn_combine_kernel<16>;
  le = launch_pdl(comb, dim3(t * H), dim3(DH), 0, stream,
                  (const float *)a.part_m, (const float *)a.part_l, (const float *)a.part_o, n_splits, t * H, DH, out,
                  packed, xs, ldxs, H);
  if (le != cudaSuccess) return set_error(HS_ERR_CUDA, "attention combine launch: %s", cudaGetErrorString(le));
  return check_launch("attention", 2);
}

}  // namespace hs

extern "C" int hs_profile_attention(int enable, int min_view) {
  using namespace hs;
  if (enable) {
    if (g_prof.empty()) {
      g_prof.resize(16384);
      for (auto &p : g_prof) {
        if (cudaEventCreate(&p.a) != cudaSuccess || cudaEventCreate(&p.b) != cudaSuccess)
          return set_error(HS_ERR_CUDA, "profile: cudaEventCreate failed");
      }
    }
    g_prof_used = 0;
    g_prof_dropped = 0;
    g_prof_min = min_view;
  }
  g_prof_on = enable;
  return HS_OK;
}

extern "C" int hs_profile_attention_read(double *ms_total, long long *bytes_total, int *launches) {
  using namespace hs;
  double ms = 0.0;
  long long bytes = 0;
  for (size_t i = 0; i < g_prof_used; ++i) {
    float e = 0.f;
    if (cudaEventSynchronize(g_prof[i].b) != cudaSuccess || cudaEventElapsedTime(&e, g_prof[i].a, g_prof[i].b) != cudaSuccess)
      return set_error(HS_ERR_CUDA, "profile: event read failed");
    ms += e;
    bytes += g_prof[i].bytes;
  }
  *ms_total = ms;
  *bytes_total = bytes;
  *launches = (int)g_prof_used;
  return g_prof_dropped ? set_error(HS_ERR_VALUE, "profile: %d launches not recorded (pool full)", g_prof_dropped)
                        : HS_OK;
}

extern "C" size_t hs_attention_workspace_bytes(int t, int n_heads, int head_dim, int n_view, int split) {
  return hs::attention_ws(t, n_heads, head_dim, n_view, split);
}

extern "C" int hs_attention(const HsCache *c, int layer, const HsStep *st, int n_heads, const float *q,
                            int t, float *out, void *workspace, size_t ws_bytes, void *stream) {
  return hs::launch_attention(c, layer, st, n_heads, q, t, out, nullptr, workspace, ws_bytes, hs::as_stream(stream));
}

extern "C" int hs_attention_partial(const HsCache *c, int layer, const HsStep *st, int n_heads, const float *q,
                                    int t, float *packed, void *workspace, size_t ws_bytes, void *stream) {
  return hs::launch_attention(c, layer, st, n_heads, q, t, nullptr, packed, workspace, ws_bytes,
                              hs::as_stream(stream));
}

extern "C" int hs_shard_merge(const float *parts, int n_shards, int rows, int head_dim, float *out, void *stream) {
  return hs::launch_shard_merge(parts, n_shards, rows, head_dim, out, nullptr, 0, 1, hs::as_stream(stream));
}
