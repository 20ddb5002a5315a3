// Native forward driver: one C call runs a whole lane step (model.py:247-331)
// so the host never pays per-layer launch overhead from Python, and the
// sequence can be captured into a CUDA graph by the caller.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gemv_norm.h"
#include "hs_common.cuh"

namespace hs {

int launch_embed(const uint16_t *emb, int ld, int d, const int32_t *tokens, int t, float *x, cudaStream_t st);
int launch_embed_norm(const uint16_t *emb, int ld, int d, const int32_t *tokens, int t, float *x, const float *gain,
                      uint16_t *xs, int ldk, cudaStream_t st);
int launch_rope_append(const HsModel *m, const HsCache *c, const HsStep *s, int layer, const float *qkv, int t,
                       float *q_out, float *q_stash, cudaStream_t st);
int launch_attention_timed(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t, float *out,
                           float *packed, void *ws, size_t ws_bytes, cudaStream_t stream, uint16_t *xs, int ldxs,
                           int clean_hi = -1, const FusedRope *fr = nullptr);
int launch_shard_merge(const float *parts, int G, int rows, int DH, float *out, uint16_t *xs, int ldxs, int H,
                       cudaStream_t st);
int shard_all_gather(const HsShard *sh, const void *send, void *recv, size_t bytes, cudaStream_t st);
size_t attention_ws(int t, int H, int DH, int n_view, int split);
size_t topk_ws_bytes(const HsModel *m, int n, int budget);
int launch_topk_attention(const HsModel *m, const HsCache *c, int layer, int n, int pos, int budget, const float *q,
                          uint16_t *xs, int ldxs, void *ws, size_t ws_bytes, cudaStream_t st);
int launch_h2o_probs(const HsCache *c, int layer, int H, const float *q, int t, int pos0, int n, double *probs,
                     float *hp, cudaStream_t st);
int launch_probe_probs(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t, float *probe,
                       cudaStream_t s);

// ---- error state -------------------------------------------------------------
static thread_local char g_err[512] = "";

int set_error(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// kernels launched by this library since load (gpu_launches evidence for bench.py)
static unsigned long long g_launches = 0;

int pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("HS_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v;
}

void count_launch(int n) { __atomic_add_fetch(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }

int check_launch(const char *what, int n_kernels) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  count_launch(n_kernels);
  return HS_OK;
}

int launch_split_rows(const float *x, int ldx, int t, int K, int ldk, const float *gain, float eps, uint16_t *xs,
                      cudaStream_t st);
int launch_gemv_tc(const uint16_t *xs, int t, const uint16_t *w, int ldw, int N, int epilogue, float *y, int ldy,
                   uint16_t *xs_out, int ld_xs_out, void *ws, size_t ws_bytes, cudaStream_t st,
                   const GemvNorm *norm = nullptr, const float *yin = nullptr, int ldyin = 0, int blocked = 0);
int launch_norm_prep(const float *x, int ldx, int t, int K, const float *gain, uint16_t *xs, int ldk,
                     cudaStream_t st);
size_t gemv_tc_ws_bytes(int N, int nkb);
void gemv_set_keep_l2(int keep);

// weights of a model small enough to stay L2-resident between its steps (the
// draft: 88 MB at the JF68M shape against a 126 MB L2; HS_L2_KEEP_MB overrides)
static int keep_weights_in_l2(const HsModel *m) {
  static const long long lim = getenv("HS_L2_KEEP_MB") ? atoll(getenv("HS_L2_KEEP_MB")) : 100;
  const long long nqkv = (long long)(m->n_heads + 2 * m->n_kv_heads) * m->head_dim;
  const long long bytes = 2LL * ((long long)m->n_layers * ((nqkv + m->d_model + 2LL * m->d_ff) * m->ld_d +
                                                         (long long)m->d_model * m->ld_ff) +
                                 (long long)m->vocab_size * m->ld_d);
  return bytes <= lim * 1000000LL;
}

// ---- tensor-parallel dense layers ("TP-shard the dense
// weights"): every projection is split by output rows in whole 128-row tiles
// (rank r of G computes tiles [T*r/G, T*(r+1)/G)); the rank's block goes to a
// packed send buffer [rows][wmax], an all-gather (NCCL, or the loopback
// group's device copies) replicates every block, and tp_unpack_kernel
// scatters them into the replicated activation.  The RMSNorm operand and row
// statistics of the next projection are rebuilt by norm_prep (bit-identical
// to the GEMV epilogue that produces them in the replicated forward).  Each
// rank streams 1/G of the weight bytes; the K split of a block follows its
// own row count, so results equal the G = 1 forward to fp32 rounding (and
// are bitwise identical on every rank).
__host__ __device__ inline void tp_rows(int N, int rank, int world, int &r0, int &n) {
  const int tiles = (N + 127) / 128;
  const int t0 = (int)((long long)tiles * rank / world), t1 = (int)((long long)tiles * (rank + 1) / world);
  r0 = t0 * 128;
  const int r1 = t1 * 128 < N ? t1 * 128 : N;
  n = r1 > r0 ? r1 - r0 : 0;
}
inline int tp_wmax(int N, int world) { return ((N + 127) / 128 + world - 1) / world * 128; }

// recv [world][rows][wm] elements of es bytes -> dst [rows][ld]: rank g's
// block lands at its columns (half: SwiGLU output, act column = row / 2)
__global__ void tp_unpack_kernel(const unsigned char *recv, int world, int rows, int wm, int es, int N, int half,
                                 unsigned char *dst, int ld) {
  const int row = blockIdx.x, g = blockIdx.y;
  int r0, n;
  tp_rows(N, g, world, r0, n);
  if (half) { r0 >>= 1; n >>= 1; }
  const unsigned char *src = recv + ((size_t)g * rows + row) * wm * es;
  unsigned char *d = dst + ((size_t)row * ld + r0) * es;
  if (es == 4) {
    for (int c = threadIdx.x; c < n; c += blockDim.x) reinterpret_cast<float *>(d)[c] = reinterpret_cast<const float *>(src)[c];
  } else {
    for (int c = threadIdx.x; c < n; c += blockDim.x)
      reinterpret_cast<uint16_t *>(d)[c] = reinterpret_cast<const uint16_t *>(src)[c];
  }
}

static int tp_exchange(const HsShard *tp, const void *send, void *recv, int rows, int wm, int es, int N, int half,
                       void *dst, int ld, cudaStream_t s) {
  int rc = shard_all_gather(tp, send, recv, (size_t)rows * wm * es, s);
  if (rc != HS_OK) return rc;
  tp_unpack_kernel<<<dim3(rows, tp->world), 256, 0, s>>>((const unsigned char *)recv, tp->world, rows, wm, es, N,
                                                         half, (unsigned char *)dst, ld);
  return check_launch("tp_unpack");
}

static size_t tp_send_bytes(const HsModel *m, int t, int world) {
  if (world <= 0) return 0;
  const int d = m->d_model, nqkv = (m->n_heads + 2 * m->n_kv_heads) * m->head_dim;
  size_t b = (size_t)t * tp_wmax(nqkv, world) * 4;
  const size_t cand[3] = {(size_t)t * tp_wmax(d, world) * 4, (size_t)24 * (tp_wmax(2 * m->d_ff, world) / 2) * 2,
                          (size_t)t * tp_wmax(m->vocab_size, world) * 4};
  for (size_t c : cand) b = c > b ? c : b;
  return b;
}

// Workspace layout.  The head is position-independent so that the regions
// which must stay zero/clean between calls never move:
//   [gemv counters + partials (max over the model's matrices)]
//   [Xd: 24 x ld_d bf16 split operand][Xf: 24 x ld_ff bf16]
//   then per-call regions: x, qkv, q, attn, attention partials and, when
//   sharded, the packed per-rank partial states (send) and their gather (recv).
struct FwdWs {
  void *gemv_ws;
  size_t gemv_bytes;
  uint16_t *xd, *xf, *xa;   // split operands: normed input (xd), act (xf), attention output (xa)
  float *x, *qkv, *q, *attn;
  void *att_ws;
  size_t att_bytes;
  float *send, *recv;
  void *tsend, *trecv;      // tensor-parallel block exchange
};

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static size_t gemv_region(const HsModel *m) {
  const int d = m->d_model, kv = m->n_kv_heads * m->head_dim;
  size_t g = 0;
  const int Ns[5] = {d + 2 * kv, d, 2 * m->d_ff, d, m->vocab_size};
  const int Ks[5] = {m->ld_d, m->ld_d, m->ld_d, m->ld_ff, m->ld_d};
  for (int i = 0; i < 5; ++i) {
    // the whole matrix and every row block a tensor-parallel rank can own
    for (int tiles = (Ns[i] + 127) / 128; tiles >= 1; --tiles) {
      const int n = tiles * 128 < Ns[i] ? tiles * 128 : Ns[i];
      size_t b = gemv_tc_ws_bytes(n, Ks[i] / 64);
      if (b > g) g = b;
    }
  }
  return align256(g);
}

static size_t carve(const HsModel *m, int t, int n_view, int split, int world, char *base, FwdWs *w,
                    int tp_world = 0) {
  const int d = m->d_model, H = m->n_heads, KVH = m->n_kv_heads, dh = m->head_dim;
  size_t off = 0;
  auto take = [&](size_t bytes) { char *p = base ? base + off : nullptr; off += align256(bytes); return p; };
  w->gemv_bytes = gemv_region(m);
  w->gemv_ws = take(w->gemv_bytes);
  w->xd = (uint16_t *)take((size_t)24 * m->ld_d * 2);
  w->xf = (uint16_t *)take((size_t)24 * m->ld_ff * 2);
  w->xa = (uint16_t *)take((size_t)24 * m->ld_d * 2);
  w->x = (float *)take((size_t)t * d * 4);
  w->qkv = (float *)take((size_t)t * (H + 2 * KVH) * dh * 4);
  w->q = (float *)take((size_t)t * H * dh * 4);
  w->attn = (float *)take((size_t)t * d * 4);
  w->att_bytes = attention_ws(t, H, dh, n_view, split);
  w->att_ws = take(w->att_bytes);
  const size_t part = (size_t)t * H * (dh + 2) * 4;
  w->send = world > 0 ? (float *)take(part) : nullptr;
  w->recv = world > 0 ? (float *)take(part * world) : nullptr;
  const size_t tb = tp_send_bytes(m, t, tp_world);
  w->tsend = tp_world > 0 ? take(tb) : nullptr;
  w->trecv = tp_world > 0 ? take(tb * tp_world) : nullptr;
  return off;
}

}  // namespace hs

namespace hs {
int trace_set_gemv(void *p, unsigned cap);
int trace_set_kv(void *p, unsigned cap);
int trace_set_attn(void *p, unsigned cap);
int trace_set_attntc(void *p, unsigned cap);
int trace_set_gemv_phases(void *p, unsigned cap);
}  // namespace hs

/* debugging/profiling aid (not part of hs_abi.h): per-CTA timeline of the
 * forward's kernels.  buf holds 4 regions of `cap` records of 3 u64 (kernel
 * id << 32 | SM, globaltimer start, end); NULL turns tracing off.           */
extern "C" int hs_cta_trace(void *buf, unsigned cap) {
  unsigned long long *b = reinterpret_cast<unsigned long long *>(buf);
  const size_t r = (size_t)cap * 3;
  // regions of cap x 3 u64 each; the fifth holds the GEMV phase records (16 u64 per CTA)
  int (*set[5])(void *, unsigned) = {hs::trace_set_gemv, hs::trace_set_kv, hs::trace_set_attn, hs::trace_set_attntc,
                                     hs::trace_set_gemv_phases};
  for (int i = 0; i < 5; ++i)
    if (set[i](b ? b + i * r : nullptr, b ? (i == 4 ? cap * 3 / 16 : cap) : 0) != 0)
      return hs::set_error(HS_ERR_VALUE, "cta trace unavailable (build with HS_TRACE_BUILD=1)");
  return HS_OK;
}

extern "C" const char *hs_last_error(void) { return hs::g_err; }
extern "C" int hs_stream_sync(void *stream) {
  const cudaError_t e = cudaStreamSynchronize(hs::as_stream(stream));
  return e == cudaSuccess ? HS_OK : hs::set_error(HS_ERR_CUDA, "stream sync: %s", cudaGetErrorString(e));
}
extern "C" int hs_abi_version(void) { return HS_ABI_VERSION; }
extern "C" unsigned long long hs_launch_count(void) { return __atomic_load_n(&hs::g_launches, __ATOMIC_RELAXED); }
extern "C" void hs_note_launches(unsigned long long n) { hs::count_launch((int)n); }
extern "C" int hs_device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

extern "C" size_t hs_forward_workspace_bytes(const HsModel *m, int t, int n_view, int split, int world) {
  hs::FwdWs w;
  return hs::carve(m, t, n_view, split, world, nullptr, &w);
}

extern "C" size_t hs_forward_workspace_clean_bytes(const HsModel *m) {
  // bytes at the head of the workspace that must be zero before the first call
  return hs::gemv_region(m) + hs::align256((size_t)24 * m->ld_d * 2) + hs::align256((size_t)24 * m->ld_ff * 2) +
         hs::align256((size_t)24 * m->ld_d * 2);
}

static int forward_impl(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh,
                        const int32_t *tokens, int t, float *logits, float *q_stash, void *workspace,
                        size_t workspace_bytes, void *stream, int topk_budget, double *probs = nullptr,
                        float *hprobs = nullptr, float *probe = nullptr, const HsShard *tp = nullptr);

extern "C" int hs_forward(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh,
                          const int32_t *tokens, int t, float *logits, float *q_stash, void *workspace,
                          size_t workspace_bytes, void *stream) {
  return forward_impl(m, c, st, sh, tokens, t, logits, q_stash, workspace, workspace_bytes, stream, 0);
}

extern "C" size_t hs_forward_tp_workspace_bytes(const HsModel *m, int t, int n_view, int split, int world,
                                                int tp_world) {
  hs::FwdWs w;
  return hs::carve(m, t, n_view, split, world, nullptr, &w, tp_world);
}

// hs_forward with tensor-parallel dense layers over `tp` (rank / world of
// its communicator; may be the same communicator as the sequence shards
// `sh`, or sh == NULL for a replicated cache such as the retrieval lane's)
extern "C" int hs_forward_tp(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh,
                             const HsShard *tp, const int32_t *tokens, int t, float *logits, float *q_stash,
                             void *workspace, size_t workspace_bytes, void *stream) {
  HS_REQUIRE(tp != nullptr && tp->comm != nullptr && tp->world >= 1 && tp->rank >= 0 && tp->rank < tp->world,
             HS_ERR_VALUE, "forward: bad tensor-parallel descriptor");
  HS_REQUIRE(t <= 8, HS_ERR_VALUE, "forward: tensor-parallel layers run decode / verify blocks of <= 8 rows");
  return forward_impl(m, c, st, sh, tokens, t, logits, q_stash, workspace, workspace_bytes, stream, 0, nullptr,
                      nullptr, nullptr, tp);
}

extern "C" size_t hs_forward_topk_workspace_bytes(const HsModel *m, int n_view, int budget) {
  return hs_forward_workspace_bytes(m, 1, n_view, 512, 0) + 256 + hs::topk_ws_bytes(m, n_view, budget);
}

// one decode position with TopKCache exposure (caches.py:617-634): every
// layer attends over the `budget` heaviest keys of each kv group
extern "C" int hs_forward_topk(const HsModel *m, const HsCache *c, const HsStep *st, int budget,
                               const int32_t *tokens, float *logits, float *q_stash, void *workspace,
                               size_t workspace_bytes, void *stream) {
  HS_REQUIRE(c->kind == HS_KV_LINEAR && st->append_mode == HS_APPEND_POS && st->pos_base == 0, HS_ERR_VALUE,
             "top-k forward: needs an unsharded linear cache");
  return forward_impl(m, c, st, nullptr, tokens, 1, logits, q_stash, workspace, workspace_bytes, stream, budget);
}

// one forward that also reports, per layer, every query row's attention
// probabilities over the exposed slots summed over heads (model.py:306-307,
// H2OCache.observe_attention): probs [L][t][n_view] fp64, head_scratch
// [t][H][n_view] fp32
extern "C" int hs_forward_attn_probs(const HsModel *m, const HsCache *c, const HsStep *st, const int32_t *tokens,
                                     int t, float *logits, float *q_stash, double *probs, float *head_scratch,
                                     void *workspace, size_t workspace_bytes, void *stream) {
  HS_REQUIRE(probs != nullptr && head_scratch != nullptr, HS_ERR_VALUE, "forward: null probability buffers");
  HS_REQUIRE(c->kind == HS_KV_SLOTTED, HS_ERR_VALUE, "forward: attention probabilities need a slotted cache");
  return forward_impl(m, c, st, nullptr, tokens, t, logits, q_stash, workspace, workspace_bytes, stream, 0, probs,
                      head_scratch);
}

// hs_forward that also records, per layer and head, the last query row's
// attention probabilities over the view (ForwardRecorder(record_probs=True),
// model.py:308-312): probe [L][H][n_view] fp32, 0 for invisible slots
extern "C" int hs_forward_probe(const HsModel *m, const HsCache *c, const HsStep *st, const int32_t *tokens, int t,
                                float *logits, float *q_stash, float *probe, void *workspace, size_t workspace_bytes,
                                void *stream) {
  HS_REQUIRE(probe != nullptr, HS_ERR_VALUE, "forward: null probe buffer");
  return forward_impl(m, c, st, nullptr, tokens, t, logits, q_stash, workspace, workspace_bytes, stream, 0, nullptr,
                      nullptr, probe);
}

static int forward_impl(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh,
                        const int32_t *tokens, int t, float *logits, float *q_stash, void *workspace,
                        size_t workspace_bytes, void *stream, int topk_budget, double *probs, float *hprobs,
                        float *probe, const HsShard *tp) {
  using namespace hs;
  HS_REQUIRE(t >= 1, HS_ERR_VALUE, "empty token sequence");
  HS_REQUIRE(c->n_layers == m->n_layers && c->n_kv_heads == m->n_kv_heads && c->head_dim == m->head_dim,
             HS_ERR_SHAPE, "forward: cache geometry does not match the model");
  HS_REQUIRE(st->pos0 + t <= m->max_seq, HS_ERR_CAPACITY, "sequence of %d exceeds max_seq %d", st->pos0 + t,
             m->max_seq);
  const bool sharded = sh != nullptr;
  if (sharded) {
    HS_REQUIRE(sh->comm != nullptr && sh->world >= 1 && sh->rank >= 0 && sh->rank < sh->world, HS_ERR_VALUE,
               "forward: bad shard descriptor (rank %d of %d)", sh->rank, sh->world);
    HS_REQUIRE(c->kind == HS_KV_LINEAR && st->append_mode == HS_APPEND_POS, HS_ERR_VALUE,
               "forward: only a full (linear) cache can be sequence-sharded");
  }
  FwdWs w;
  const size_t need = carve(m, t, st->n_view, st->split, sharded ? sh->world : 0, (char *)workspace, &w,
                            tp ? tp->world : 0);
  HS_REQUIRE(workspace_bytes >= need, HS_ERR_VALUE, "forward: workspace %zu < %zu", workspace_bytes, need);
  void *topk_ws = nullptr;
  size_t topk_bytes = 0;
  if (topk_budget > 0) {
    topk_ws = (char *)workspace + align256(need);
    topk_bytes = topk_ws_bytes(m, st->n_view, topk_budget);
    HS_REQUIRE(workspace_bytes >= align256(need) + topk_bytes, HS_ERR_VALUE, "forward: top-k workspace too small");
  }
  cudaStream_t s = as_stream(stream);
  gemv_set_keep_l2(keep_weights_in_l2(m));
  const int d = m->d_model, H = m->n_heads, KVH = m->n_kv_heads, dh = m->head_dim, ff = m->d_ff;
  const int nqkv = (H + 2 * KVH) * dh;
  const float eps = m->norm_eps;
  // slots below clean_hi are not appended to by this forward's RoPE kernels,
  // so the attention kernel may stream them before its dependency wait
  const int clean_hi = st->dyn ? -1
                       : st->append_mode == HS_APPEND_POS    ? st->pos0 - st->pos_base
                       : st->append_mode == HS_APPEND_LINEAR ? st->append_base
                                                             : -1;
  const bool fused_split = t <= 8;   // one row block: folded norms, no split kernels
  HS_REQUIRE(tp == nullptr || (fused_split && topk_budget == 0 && probs == nullptr && probe == nullptr), HS_ERR_VALUE,
             "forward: tensor-parallel layers need a plain forward of <= 8 rows");
  int rc;
#define HS_TRY(call) do { if ((rc = (call)) != HS_OK) return rc; } while (0)
  if (fused_split) {
    // ---- one row block (decode / verify): every RMSNorm is folded into the
    // GEMVs -- the residual producer (embedding, wo, w_down) writes the next
    // operand split(x * gain) and per-tile row sums of squares, the consumer
    // (wqkv, gate|up, lm_head) scales its result by 1 / rms -- so no split /
    // normalise kernel runs between the weight streams.
    static const bool fused_rope_ok = getenv("HS_NO_FUSED_ROPE") == nullptr;   // A/B hook
    const bool fuse_rope = fused_rope_ok && topk_budget == 0 && probs == nullptr && probe == nullptr &&
                           dh == 128 && st->dyn == nullptr && st->n_view > 0 &&   // (an empty shard view launches no
                           // attention kernel, so it could not write q_stash / the rows)
                           (st->append_mode == HS_APPEND_POS || st->append_mode == HS_APPEND_LINEAR);
    HS_TRY(launch_embed_norm(m->emb, m->ld_d, d, tokens, t, w.x, m->attn_norm, w.xd, m->ld_d, s));
    for (int l = 0; l < m->n_layers; ++l) {
      const uint16_t *wqkv = m->wqkv + (size_t)l * nqkv * m->ld_d;
      const uint16_t *wo = m->wo + (size_t)l * d * m->ld_d;
      const uint16_t *wgu = m->wgu + (size_t)l * 2 * ff * m->ld_d;
      const uint16_t *wdn = m->wdown + (size_t)l * d * m->ld_ff;
      const bool last = l + 1 == m->n_layers;
      GemvNorm in_qkv = {w.x, d, d, eps, nullptr, nullptr, 0};
      if (tp) {
        int r0, n;
        tp_rows(nqkv, tp->rank, tp->world, r0, n);
        const int wm = tp_wmax(nqkv, tp->world);
        if (n > 0)
          HS_TRY(launch_gemv_tc(w.xd, t, wqkv + (size_t)r0 * m->ld_d, m->ld_d, n, 0, (float *)w.tsend, wm, nullptr,
                                0, w.gemv_ws, w.gemv_bytes, s, &in_qkv, nullptr, 0, m->blocked & 1));
        HS_TRY(tp_exchange(tp, w.tsend, w.trecv, t, wm, 4, nqkv, 0, w.qkv, nqkv, s));
      } else {
        HS_TRY(launch_gemv_tc(w.xd, t, wqkv, m->ld_d, nqkv, 0, w.qkv, nqkv, nullptr, 0, w.gemv_ws, w.gemv_bytes, s,
                              &in_qkv, nullptr, 0, m->blocked & 1));
      }
      if (fuse_rope) {
        // RoPE + K/V append inside the tensor-core attention (its q staging
        // reads the qkv rows; the CTA covering the appended slots writes them)
        const FusedRope fr = {w.qkv, nqkv, m->rope_cos, m->rope_sin,
                              q_stash ? q_stash + (size_t)l * H * dh : nullptr};
        if (sharded) {
          const size_t part = (size_t)t * H * (dh + 2) * 4;
          HS_TRY(launch_attention_timed(c, l, st, H, nullptr, t, nullptr, w.send, w.att_ws, w.att_bytes, s, nullptr,
                                        0, clean_hi, &fr));
          HS_TRY(shard_all_gather(sh, w.send, w.recv, part, s));
          HS_TRY(launch_shard_merge(w.recv, sh->world, t * H, dh, nullptr, w.xa, m->ld_d, H, s));
        } else {
          HS_TRY(launch_attention_timed(c, l, st, H, nullptr, t, nullptr, nullptr, w.att_ws, w.att_bytes, s, w.xa,
                                        m->ld_d, clean_hi, &fr));
        }
      } else {
      HS_TRY(launch_rope_append(m, c, st, l, w.qkv, t, w.q, q_stash, s));
      if (sharded) {
        const size_t part = (size_t)t * H * (dh + 2) * 4;
        HS_TRY(launch_attention_timed(c, l, st, H, w.q, t, nullptr, w.send, w.att_ws, w.att_bytes, s, nullptr, 0, clean_hi));
        HS_TRY(shard_all_gather(sh, w.send, w.recv, part, s));
        HS_TRY(launch_shard_merge(w.recv, sh->world, t * H, dh, nullptr, w.xa, m->ld_d, H, s));
      } else if (topk_budget > 0) {
        HS_TRY(launch_topk_attention(m, c, l, st->n_view, st->pos0, topk_budget, w.q, w.xa, m->ld_d, topk_ws,
                                     topk_bytes, s));
      } else {
        HS_TRY(launch_attention_timed(c, l, st, H, w.q, t, nullptr, nullptr, w.att_ws, w.att_bytes, s, w.xa,
                                      m->ld_d, clean_hi));
      }
      if (probs)
        HS_TRY(launch_h2o_probs(c, l, H, w.q, t, st->pos0, st->n_view, probs + (size_t)l * t * st->n_view, hprobs,
                                s));
      if (probe) HS_TRY(launch_probe_probs(c, l, st, H, w.q, t, probe + (size_t)l * H * st->n_view, s));
      }
      const float *gain_next = last ? m->final_norm : m->attn_norm + (size_t)(l + 1) * d;
      GemvNorm in_gu = {w.x, d, d, eps, nullptr, nullptr, 0};
      if (tp) {
        int r0, n, wm;
        // w_o: residual block -> all ranks; the mlp_norm operand is rebuilt replicated
        tp_rows(d, tp->rank, tp->world, r0, n);
        wm = tp_wmax(d, tp->world);
        if (n > 0)
          HS_TRY(launch_gemv_tc(w.xa, t, wo + (size_t)r0 * m->ld_d, m->ld_d, n, 1, (float *)w.tsend, wm, nullptr, 0,
                                w.gemv_ws, w.gemv_bytes, s, nullptr, w.x + r0, d, m->blocked & 1));
        HS_TRY(tp_exchange(tp, w.tsend, w.trecv, t, wm, 4, d, 0, w.x, d, s));
        HS_TRY(launch_norm_prep(w.x, d, t, d, m->mlp_norm + (size_t)l * d, w.xd, m->ld_d, s));
        // gate|up: SwiGLU act block (split operand rows) -> all ranks
        tp_rows(2 * ff, tp->rank, tp->world, r0, n);
        wm = tp_wmax(2 * ff, tp->world);
        if (n > 0)
          HS_TRY(launch_gemv_tc(w.xd, t, wgu + (size_t)r0 * m->ld_d, m->ld_d, n, 2, nullptr, 0, (uint16_t *)w.tsend,
                                wm / 2, w.gemv_ws, w.gemv_bytes, s, &in_gu, nullptr, 0, m->blocked & 1));
        HS_TRY(tp_exchange(tp, w.tsend, w.trecv, 3 * 8, wm / 2, 2, 2 * ff, 1, w.xf, m->ld_ff, s));
        // w_down: residual block -> all ranks; next norm operand rebuilt
        tp_rows(d, tp->rank, tp->world, r0, n);
        wm = tp_wmax(d, tp->world);
        if (n > 0)
          HS_TRY(launch_gemv_tc(w.xf, t, wdn + (size_t)r0 * m->ld_ff, m->ld_ff, n, 1, (float *)w.tsend, wm, nullptr,
                                0, w.gemv_ws, w.gemv_bytes, s, nullptr, w.x + r0, d, m->blocked & 1));
        HS_TRY(tp_exchange(tp, w.tsend, w.trecv, t, wm, 4, d, 0, w.x, d, s));
        HS_TRY(launch_norm_prep(w.x, d, t, d, gain_next, w.xd, m->ld_d, s));
        continue;
      }
      GemvNorm out_wo = {nullptr, 0, 1, 0.f, m->mlp_norm + (size_t)l * d, w.xd, m->ld_d};
      HS_TRY(launch_gemv_tc(w.xa, t, wo, m->ld_d, d, 1, w.x, d, nullptr, 0, w.gemv_ws, w.gemv_bytes, s, &out_wo, nullptr, 0, m->blocked & 1));
      HS_TRY(launch_gemv_tc(w.xd, t, wgu, m->ld_d, 2 * ff, 2, nullptr, 0, w.xf, m->ld_ff, w.gemv_ws, w.gemv_bytes, s,
                            &in_gu, nullptr, 0, m->blocked & 1));
      GemvNorm out_dn = {nullptr, 0, 1, 0.f, gain_next, w.xd, m->ld_d};
      HS_TRY(launch_gemv_tc(w.xf, t, wdn, m->ld_ff, d, 1, w.x, d, nullptr, 0, w.gemv_ws, w.gemv_bytes, s, &out_dn, nullptr, 0, m->blocked & 1));
    }
    GemvNorm in_head = {w.x, d, d, eps, nullptr, nullptr, 0};
    if (tp) {
      int r0, n;
      tp_rows(m->vocab_size, tp->rank, tp->world, r0, n);
      const int wm = tp_wmax(m->vocab_size, tp->world);
      if (n > 0)
        HS_TRY(launch_gemv_tc(w.xd, t, m->head + (size_t)r0 * m->ld_d, m->ld_d, n, 0, (float *)w.tsend, wm, nullptr,
                              0, w.gemv_ws, w.gemv_bytes, s, &in_head, nullptr, 0, (m->blocked >> 1) & 1));
      HS_TRY(tp_exchange(tp, w.tsend, w.trecv, t, wm, 4, m->vocab_size, 0, logits, m->vocab_size, s));
      return HS_OK;
    }
    HS_TRY(launch_gemv_tc(w.xd, t, m->head, m->ld_d, m->vocab_size, 0, logits, m->vocab_size, nullptr, 0, w.gemv_ws,
                          w.gemv_bytes, s, &in_head, nullptr, 0, (m->blocked >> 1) & 1));
    return HS_OK;
  }
  // ---- several row blocks (prefill-sized batches through the decode path):
  // the same folded-norm GEMVs per block of 8 rows, the operand and row
  // statistics prepared by norm_prep (bit-identical to the producing GEMV
  // epilogue of the single-block path), so every row equals a decode step.
  HS_TRY(launch_embed(m->emb, m->ld_d, d, tokens, t, w.x, s));
  for (int l = 0; l < m->n_layers; ++l) {
    const uint16_t *wqkv = m->wqkv + (size_t)l * nqkv * m->ld_d;
    const uint16_t *wo = m->wo + (size_t)l * d * m->ld_d;
    const uint16_t *wgu = m->wgu + (size_t)l * 2 * ff * m->ld_d;
    const uint16_t *wdn = m->wdown + (size_t)l * d * m->ld_ff;
    const float *an = m->attn_norm + (size_t)l * d, *mn = m->mlp_norm + (size_t)l * d;
    for (int r0 = 0; r0 < t; r0 += 8) {
      const int tp = t - r0 < 8 ? t - r0 : 8;
      const GemvNorm in_n = {w.x + (size_t)r0 * d, d, d, eps, nullptr, nullptr, 0};
      HS_TRY(launch_norm_prep(w.x + (size_t)r0 * d, d, tp, d, an, w.xd, m->ld_d, s));
      HS_TRY(launch_gemv_tc(w.xd, tp, wqkv, m->ld_d, nqkv, 0, w.qkv + (size_t)r0 * nqkv, nqkv, nullptr, 0, w.gemv_ws,
                            w.gemv_bytes, s, &in_n, nullptr, 0, m->blocked & 1));
    }
    HS_TRY(launch_rope_append(m, c, st, l, w.qkv, t, w.q, q_stash, s));
    if (sharded) {
      // this rank's partial softmax state -> all ranks -> rank-ordered merge
      const size_t part = (size_t)t * H * (dh + 2) * 4;
      HS_TRY(launch_attention_timed(c, l, st, H, w.q, t, nullptr, w.send, w.att_ws, w.att_bytes, s, nullptr, 0, clean_hi));
      HS_TRY(shard_all_gather(sh, w.send, w.recv, part, s));
      HS_TRY(launch_shard_merge(w.recv, sh->world, t * H, dh, w.attn, nullptr, m->ld_d, H, s));
    } else {
      HS_TRY(launch_attention_timed(c, l, st, H, w.q, t, w.attn, nullptr, w.att_ws, w.att_bytes, s, nullptr, 0, clean_hi));
    }
    if (probs)
      HS_TRY(launch_h2o_probs(c, l, H, w.q, t, st->pos0, st->n_view, probs + (size_t)l * t * st->n_view, hprobs, s));
    if (probe) HS_TRY(launch_probe_probs(c, l, st, H, w.q, t, probe + (size_t)l * H * st->n_view, s));
    for (int r0 = 0; r0 < t; r0 += 8) {
      const int tp = t - r0 < 8 ? t - r0 : 8;
      float *xr = w.x + (size_t)r0 * d;
      const GemvNorm in_n = {xr, d, d, eps, nullptr, nullptr, 0};
      HS_TRY(launch_split_rows(w.attn + (size_t)r0 * d, d, tp, d, m->ld_d, nullptr, 0.f, w.xd, s));
      HS_TRY(launch_gemv_tc(w.xd, tp, wo, m->ld_d, d, 1, xr, d, nullptr, 0, w.gemv_ws, w.gemv_bytes, s, nullptr, nullptr,
                            0, m->blocked & 1));
      HS_TRY(launch_norm_prep(xr, d, tp, d, mn, w.xd, m->ld_d, s));
      HS_TRY(launch_gemv_tc(w.xd, tp, wgu, m->ld_d, 2 * ff, 2, nullptr, 0, w.xf, m->ld_ff, w.gemv_ws, w.gemv_bytes, s,
                            &in_n, nullptr, 0, m->blocked & 1));
      HS_TRY(launch_gemv_tc(w.xf, tp, wdn, m->ld_ff, d, 1, xr, d, nullptr, 0, w.gemv_ws, w.gemv_bytes, s, nullptr,
                            nullptr, 0, m->blocked & 1));
    }
  }
  for (int r0 = 0; r0 < t; r0 += 8) {
    const int tp = t - r0 < 8 ? t - r0 : 8;
    const GemvNorm in_n = {w.x + (size_t)r0 * d, d, d, eps, nullptr, nullptr, 0};
    HS_TRY(launch_norm_prep(w.x + (size_t)r0 * d, d, tp, d, m->final_norm, w.xd, m->ld_d, s));
    HS_TRY(launch_gemv_tc(w.xd, tp, m->head, m->ld_d, m->vocab_size, 0, logits + (size_t)r0 * m->vocab_size,
                          m->vocab_size, nullptr, 0, w.gemv_ws, w.gemv_bytes, s, &in_n, nullptr, 0,
                          (m->blocked >> 1) & 1));
  }
#undef HS_TRY
  return HS_OK;
}

