// Batched prefill: the prompt's dense projections as
// tensor-core GEMMs instead of t/8 weight-streaming GEMV passes.
//
// Replaces the batched `_forward` of `prefill` (model.py:334-354) for long
// prompts.  The decode path (hs_forward) keeps every row bit-identical
// whatever the batch (the chunk == step-sequence contract, model.py:366-378);
// prefill only has to be fp32-accurate, so each projection here is
//     Y (+)= W . (hi + mid + lo)      -- one tcgen05 GEMM (gemm_tc.cu) whose
// three bf16 activation planes accumulate into one fp32 TMEM accumulator:
// the exact 3-way bf16 split of the fp32 activations, so every product is
// exact and the sums are fp32, like the GEMV.  RMSNorm, RoPE + cache append
// and attention are the decode path's kernels (attention runs causally over
// all t query rows).  Rows go through the dense layers in blocks of up to
// PF_ROWS so the GEMM scratch stays bounded.
#include "hs_common.cuh"

namespace hs {

int launch_embed(const uint16_t *emb, int ld, int d, const int32_t *tokens, int t, float *x, cudaStream_t st);
int launch_rope_append(const HsModel *m, const HsCache *c, const HsStep *s, int layer, const float *qkv, int t,
                       float *q_out, float *q_stash, cudaStream_t st);
int launch_attention_timed(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t, float *out,
                           float *packed, void *ws, size_t ws_bytes, cudaStream_t stream, uint16_t *xs, int ldxs,
                           int clean_hi = -1, const FusedRope *fr = nullptr);
size_t attention_ws(int t, int H, int DH, int n_view, int split);
int launch_prefill_attention(const HsCache *c, int layer, int H, const float *q, int t, int pos0, int pos_base,
                             int n_keys, float *out, float *packed, cudaStream_t stream);
int launch_shard_merge(const float *parts, int G, int rows, int DH, float *out, uint16_t *xs, int ldxs, int H,
                       cudaStream_t st);
int shard_all_gather(const HsShard *sh, const void *send, void *recv, size_t bytes, cudaStream_t st);
int launch_gemm3_tc(const uint16_t *s0, const uint16_t *s1, const uint16_t *s2, int ldk, int R, const uint16_t *W,
                    int ld, int N, float *Y, int ldy, int accumulate, cudaStream_t st, int blocked);

namespace {

#ifndef HS_PF_ROWS
#define HS_PF_ROWS 2048
#endif
constexpr int PF_ROWS = HS_PF_ROWS;   // rows per dense block (bounded GEMM scratch)
constexpr int PF_QROWS = 1024;   // query rows per attention call (bounded partial-state scratch)

// RMSNorm (optional gain) + exact 3-way split of rows [0, R) into three
// [R][ldk] bf16 planes; grid (ceil(ldk / 1024), R)
__global__ void __launch_bounds__(256) pf_split_kernel(const float *x, int ldx, int K, int ldk, const float *gain,
                                                       float eps, uint16_t *hi, uint16_t *mid, uint16_t *lo) {
  const int r = blockIdx.y;
  const float *xr = x + (size_t)r * ldx;
  __shared__ double red[8];
  double scale = 1.0;
  if (gain != nullptr) {
    double ss = 0.0;
    for (int k = threadIdx.x; k < K; k += 256) ss += (double)xr[k] * xr[k];
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[w];
    scale = sqrt(tot / (double)K + (double)eps);   // rms_norm, model.py:282-284
  }
  for (int j = 0; j < 4; ++j) {
    const int k = blockIdx.x * 1024 + j * 256 + threadIdx.x;
    if (k >= ldk) break;
    float h = 0.f;
    if (k < K) h = gain ? (float)(((double)xr[k] / scale) * (double)gain[k]) : xr[k];
    uint16_t a, b, c;
    split3(h, a, b, c);
    hi[(size_t)r * ldk + k] = a;
    mid[(size_t)r * ldk + k] = b;
    lo[(size_t)r * ldk + k] = c;
  }
}

// act[r][i] = silu(g) * u for the interleaved gate/up rows (model.py:320-322)
__global__ void pf_swiglu_kernel(const float *gu, int R, int ff, float *act) {
  const size_t n = (size_t)R * ff;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const size_t r = e / ff, i = e % ff;
    const double g = (double)gu[r * 2 * ff + 2 * i];
    act[e] = (float)(g * (0.5 * (tanh(0.5 * g) + 1.0))) * gu[r * 2 * ff + 2 * i + 1];
  }
}

struct PfWs {
  float *x, *qkv, *q, *attn, *gu, *act;
  uint16_t *s0, *s1, *s2;   // split planes [PF_ROWS][max(ld_d, ld_ff)]
  void *att_ws;
  size_t att_bytes;
  float *send, *recv;       // sequence shards: packed partial states of PF_SQROWS query rows, own / all ranks
};

constexpr int PF_SQROWS = 4096;   // query rows per sharded attention exchange

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t carve(const HsModel *m, int t, int n_view, int split, int world, char *base, PfWs *w) {
  const int d = m->d_model, H = m->n_heads, KVH = m->n_kv_heads, dh = m->head_dim;
  const int R = t < PF_ROWS ? t : PF_ROWS;
  const int ldk = m->ld_d > m->ld_ff ? m->ld_d : m->ld_ff;
  size_t off = 0;
  auto take = [&](size_t bytes) { char *p = base ? base + off : nullptr; off += align256(bytes); return p; };
  w->x = (float *)take((size_t)t * d * 4);
  w->qkv = (float *)take((size_t)t * (H + 2 * KVH) * dh * 4);
  w->q = (float *)take((size_t)t * H * dh * 4);
  w->attn = (float *)take((size_t)t * d * 4);
  const size_t gu_cols = (size_t)(2 * m->d_ff > m->vocab_size ? 2 * m->d_ff : m->vocab_size);
  w->gu = (float *)take((size_t)R * gu_cols * 4);
  w->act = (float *)take((size_t)R * m->d_ff * 4);
  w->s0 = (uint16_t *)take((size_t)R * ldk * 2);
  w->s1 = (uint16_t *)take((size_t)R * ldk * 2);
  w->s2 = (uint16_t *)take((size_t)R * ldk * 2);
  w->att_bytes = attention_ws(t < PF_QROWS ? t : PF_QROWS, H, dh, n_view, split);
  w->att_ws = take(w->att_bytes);
  const size_t part = (size_t)(t < PF_SQROWS ? t : PF_SQROWS) * H * (dh + 2) * 4;
  w->send = world > 0 ? (float *)take(part) : nullptr;
  w->recv = world > 0 ? (float *)take(part * world) : nullptr;
  return off;
}

// Y[R][N] (ldy) (+)= W[N][ld] . (s0 + s1 + s2)[R][ld]^T, fp32 accumulate (tcgen05)
// (split_rows_n wrote the planes at row stride ld)
int gemm3(const uint16_t *W, int ld, int N, const PfWs &w, int R, int accumulate, float *Y, int ldy, cudaStream_t s,
          int blocked) {
  return launch_gemm3_tc(w.s0, w.s1, w.s2, ld, R, W, ld, N, Y, ldy, accumulate, s, blocked);
}

int split_rows_n(const float *x, int ldx, int R, int K, int ldk, const float *gain, float eps, const PfWs &w,
                 cudaStream_t s) {
  dim3 grid((ldk + 1023) / 1024, R);
  pf_split_kernel<<<grid, 256, 0, s>>>(x, ldx, K, ldk, gain, eps, w.s0, w.s1, w.s2);
  return check_launch("prefill split");
}

}  // namespace
}  // namespace hs

extern "C" size_t hs_prefill_workspace_bytes(const HsModel *m, int t, int n_view, int split) {
  hs::PfWs w;
  return hs::carve(m, t, n_view, split, 0, nullptr, &w);
}

extern "C" size_t hs_prefill_sharded_workspace_bytes(const HsModel *m, int t, int n_view, int split, int world) {
  hs::PfWs w;
  return hs::carve(m, t, n_view, split, world, nullptr, &w);
}

static int prefill_impl(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh,
                        const int32_t *tokens, int t, float *logits, float *q_stash, void *workspace,
                        size_t workspace_bytes, void *stream);

extern "C" int hs_prefill(const HsModel *m, const HsCache *c, const HsStep *st, const int32_t *tokens, int t,
                          float *logits, float *q_stash, void *workspace, size_t workspace_bytes, void *stream) {
  return prefill_impl(m, c, st, nullptr, tokens, t, logits, q_stash, workspace, workspace_bytes, stream);
}

extern "C" int hs_prefill_sharded(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh,
                                  const int32_t *tokens, int t, float *logits, float *q_stash, void *workspace,
                                  size_t workspace_bytes, void *stream) {
  HS_REQUIRE(sh != nullptr && sh->comm != nullptr && sh->world >= 1 && sh->rank >= 0 && sh->rank < sh->world,
             HS_ERR_VALUE, "prefill: bad shard descriptor");
  HS_REQUIRE(m->head_dim == 128 && c->kind == HS_KV_LINEAR && st->append_mode == HS_APPEND_POS, HS_ERR_VALUE,
             "prefill: the sharded prefill needs head_dim 128 and a full (linear) cache");
  return prefill_impl(m, c, st, sh, tokens, t, logits, q_stash, workspace, workspace_bytes, stream);
}

static int prefill_impl(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh,
                        const int32_t *tokens, int t, float *logits, float *q_stash, void *workspace,
                        size_t workspace_bytes, void *stream) {
  using namespace hs;
  HS_REQUIRE(t >= 1, HS_ERR_VALUE, "empty token sequence");
  HS_REQUIRE(c->n_layers == m->n_layers && c->n_kv_heads == m->n_kv_heads && c->head_dim == m->head_dim,
             HS_ERR_SHAPE, "prefill: cache geometry does not match the model");
  HS_REQUIRE(st->pos0 + t <= m->max_seq, HS_ERR_CAPACITY, "sequence of %d exceeds max_seq %d", st->pos0 + t,
             m->max_seq);
  PfWs w;
  const size_t need = carve(m, t, st->n_view, st->split, sh ? sh->world : 0, (char *)workspace, &w);
  HS_REQUIRE(workspace_bytes >= need, HS_ERR_VALUE, "prefill: workspace %zu < %zu", workspace_bytes, need);
  cudaStream_t s = as_stream(stream);
  const int d = m->d_model, H = m->n_heads, KVH = m->n_kv_heads, dh = m->head_dim, ff = m->d_ff;
  const int nqkv = (H + 2 * KVH) * dh;
  const float eps = m->norm_eps;
  int rc;
#define HS_TRY(call) do { if ((rc = (call)) != HS_OK) return rc; } while (0)
  HS_TRY(launch_embed(m->emb, m->ld_d, d, tokens, t, w.x, s));
  for (int l = 0; l < m->n_layers; ++l) {
    const uint16_t *wqkv = m->wqkv + (size_t)l * nqkv * m->ld_d;
    const uint16_t *wo = m->wo + (size_t)l * d * m->ld_d;
    const uint16_t *wgu = m->wgu + (size_t)l * 2 * ff * m->ld_d;
    const uint16_t *wdn = m->wdown + (size_t)l * d * m->ld_ff;
    const float *an = m->attn_norm + (size_t)l * d, *mn = m->mlp_norm + (size_t)l * d;
    for (int r0 = 0; r0 < t; r0 += PF_ROWS) {
      const int R = t - r0 < PF_ROWS ? t - r0 : PF_ROWS;
      HS_TRY(split_rows_n(w.x + (size_t)r0 * d, d, R, d, m->ld_d, an, eps, w, s));
      HS_TRY(gemm3(wqkv, m->ld_d, nqkv, w, R, 0, w.qkv + (size_t)r0 * nqkv, nqkv, s, m->blocked & 1));
    }
    HS_TRY(launch_rope_append(m, c, st, l, w.qkv, t, w.q, q_stash, s));
    // causal attention: head_dim 128 on the 128-row tensor-core prefill kernel
    // (prefill_attn.cu); other head sizes in blocks of query rows on the
    // decode kernels, a block seeing keys up to its last row
    static const bool tc_prefill = getenv("HS_PREFILL_DECODE_ATTN") == nullptr;   // A/B hook
    if (sh) {
      // sequence shards: every rank attends all query rows over its own key
      // slots, the packed partial states go to all ranks and are merged in
      // rank order (the decode path's exchange), PF_SQROWS rows
      // at a time
      for (int a0 = 0; a0 < t; a0 += PF_SQROWS) {
        const int tq = t - a0 < PF_SQROWS ? t - a0 : PF_SQROWS;
        HS_TRY(launch_prefill_attention(c, l, H, w.q + (size_t)a0 * H * dh, tq, st->pos0 + a0, st->pos_base,
                                        st->n_view, nullptr, w.send, s));
        HS_TRY(shard_all_gather(sh, w.send, w.recv, (size_t)tq * H * (dh + 2) * 4, s));
        HS_TRY(launch_shard_merge(w.recv, sh->world, tq * H, dh, w.attn + (size_t)a0 * d, nullptr, 0, H, s));
      }
    } else if (tc_prefill && dh == 128 && st->pos_base == 0 && st->window == 0 && c->kind == HS_KV_LINEAR) {
      HS_TRY(launch_prefill_attention(c, l, H, w.q, t, st->pos0, 0,
                                      st->n_view < st->pos0 + t ? st->n_view : st->pos0 + t, w.attn, nullptr, s));
    } else
    for (int a0 = 0; a0 < t; a0 += PF_QROWS) {
      const int tq = t - a0 < PF_QROWS ? t - a0 : PF_QROWS;
      HsStep sa = *st;
      sa.pos0 = st->pos0 + a0;
      const int vis = st->pos0 + a0 + tq - st->pos_base;
      sa.n_view = vis < st->n_view ? vis : st->n_view;
      HS_TRY(launch_attention_timed(c, l, &sa, H, w.q + (size_t)a0 * H * dh, tq, w.attn + (size_t)a0 * d, nullptr,
                                    w.att_ws, w.att_bytes, s, nullptr, 0));
    }
    for (int r0 = 0; r0 < t; r0 += PF_ROWS) {
      const int R = t - r0 < PF_ROWS ? t - r0 : PF_ROWS;
      float *xr = w.x + (size_t)r0 * d;
      HS_TRY(split_rows_n(w.attn + (size_t)r0 * d, d, R, d, m->ld_d, nullptr, 0.f, w, s));
      HS_TRY(gemm3(wo, m->ld_d, d, w, R, 1, xr, d, s, m->blocked & 1));                  // x += wo . attn
      HS_TRY(split_rows_n(xr, d, R, d, m->ld_d, mn, eps, w, s));
      HS_TRY(gemm3(wgu, m->ld_d, 2 * ff, w, R, 0, w.gu, 2 * ff, s, m->blocked & 1));
      pf_swiglu_kernel<<<592, 256, 0, s>>>(w.gu, R, ff, w.act);
      HS_TRY(check_launch("prefill swiglu"));
      HS_TRY(split_rows_n(w.act, ff, R, ff, m->ld_ff, nullptr, 0.f, w, s));
      HS_TRY(gemm3(wdn, m->ld_ff, d, w, R, 1, xr, d, s, m->blocked & 1));                // x += w_down . act
    }
  }
  for (int r0 = 0; r0 < t; r0 += PF_ROWS) {
    const int R = t - r0 < PF_ROWS ? t - r0 : PF_ROWS;
    HS_TRY(split_rows_n(w.x + (size_t)r0 * d, d, R, d, m->ld_d, m->final_norm, eps, w, s));
    HS_TRY(gemm3(m->head, m->ld_d, m->vocab_size, w, R, 0, logits + (size_t)r0 * m->vocab_size,
                 m->vocab_size, s, (m->blocked >> 1) & 1));
  }
#undef HS_TRY
  return HS_OK;
}
