/*
 * hs_abi.h -- C ABI of the B200 TriForce decode hot path (libhs_b200.so).
 *
 * Plain C: device pointers, sizes and a cudaStream_t passed as void*.  No
 * allocation crosses the boundary (callers own every buffer, including the
 * workspace), no exceptions: every entry point returns HS_OK or a negative
 * status whose message is available from hs_last_error().  Statuses map 1:1
 * onto the reference's exception types (hierspec/errors.py:4-39).
 *
 * Each entry point cites the reference operation it replaces
 * (paths relative to /root/reference/pkg/src/hierspec/).
 *
 * Storage model:
 *   weights   bf16, [out][in] row-major ("K-major"), row stride padded to 64
 *   norms     fp32
 *   acts      fp32
 *   KV        bf16, head-major  [layer][kv_head][slot][head_dim]
 *   probs     fp64 (matches prob_from_logits, model.py:182-195)
 */
#ifndef HS_ABI_H
#define HS_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_ABI_VERSION 2

/* ---- status codes (errors.py) ----------------------------------------- */
#define HS_OK            0
#define HS_ERR_SHAPE    -1   /* ShapeError      errors.py:4   */
#define HS_ERR_CONTRACT -2   /* ContractError   errors.py:18  */
#define HS_ERR_CAPACITY -3   /* CapacityError   errors.py:14  */
#define HS_ERR_FINITE   -4   /* FiniteError     errors.py:8   */
#define HS_ERR_VALUE    -5   /* ValueError                    */
#define HS_ERR_CUDA    -10   /* launch / runtime failure      */

const char *hs_last_error(void);
int hs_abi_version(void);
/* block the host until the stream's work is done (the per-round read-back) */
int hs_stream_sync(void *stream);
int hs_device_sm_count(int device);
/* number of kernels this library has launched since it was loaded */
unsigned long long hs_launch_count(void);
/* add n to that count (kernels launched by replaying a captured CUDA graph) */
void hs_note_launches(unsigned long long n);

/* ---- model descriptor --------------------------------------------------
 * Replaces ModelWeights.runtime() (model.py:116-143): fused wqkv, fused
 * gate|up (rows interleaved gate_i, up_i so the SwiGLU epilogue sees both),
 * transposed to [out][in] bf16.  All pointers are device pointers; layer
 * tensors are packed with a fixed per-layer stride.                        */
typedef struct {
  int n_layers, n_heads, n_kv_heads, head_dim, d_ff, vocab_size, max_seq;
  int d_model;         /* n_heads * head_dim                         */
  int ld_d, ld_ff;     /* padded row strides (elements) for K=d, K=d_ff */
  float norm_eps;
  const uint16_t *emb;        /* [V][ld_d]                  bf16       */
  const uint16_t *head;       /* [V][ld_d]   lm_head^T or emb (tied)   */
  const float *final_norm;    /* [d]                                   */
  const float *attn_norm;     /* [L][d]                                */
  const float *mlp_norm;      /* [L][d]                                */
  const uint16_t *wqkv;       /* [L][(H+2KVH)dh][ld_d]                 */
  const uint16_t *wo;         /* [L][d][ld_d]                          */
  const uint16_t *wgu;        /* [L][2 d_ff][ld_d] interleaved         */
  const uint16_t *wdown;      /* [L][d][ld_ff]                         */
  const float *rope_cos;      /* [max_seq][dh/2] fp32 (tensor.py:66-76)*/
  const float *rope_sin;
  int blocked;         /* weight layout: bit 0 -- wqkv / wo / wgu / wdown,
                          bit 1 -- head, stored tile-blocked: [N/128][ld/64]
                          [128][64] (every 128 x 64 GEMV tile one contiguous
                          16 KB block; N a multiple of 128); 0 = row-major  */
} HsModel;

/* ---- KV cache descriptor ------------------------------------------------
 * One struct covers the three policies of the hot path:
 *   FullCache       (caches.py:176-221)  kind=HS_KV_LINEAR, slot == position
 *   RetrievalCache  (caches.py:439-565)  kind=HS_KV_SLOTTED, pos[] per slot
 *   StreamingCache  (caches.py:224-288)  kind=HS_KV_SLOTTED, ring of slots   */
#define HS_KV_LINEAR  0
#define HS_KV_SLOTTED 1

typedef struct {
  int kind;
  int n_layers, n_kv_heads, head_dim;
  int cap;              /* slots per (layer, kv head)                        */
  uint16_t *k;          /* [L][KVH][cap][dh] bf16                           */
  uint16_t *v;
  int32_t *pos;         /* SLOTTED: [L][cap] absolute position, -1 = empty   */
} HsCache;

/* Per-forward description of where new rows go and what attention sees.
 *   append: HS_APPEND_POS   slot = position                 (full)
 *           HS_APPEND_LINEAR slot = append_base + i          (retrieval tail)
 *           HS_APPEND_RING  slot = p < n_sink ? p : n_sink + (p-n_sink)%ring
 *   view:   slots [0, n_view) are scanned; a key at position kp is visible
 *           to the query at position qp iff kp >= 0 && kp <= qp &&
 *           (window == 0 || kp < n_sink || kp >= max(win_lo, qp-window+1))
 *           -- the sequential exposure rule of StreamingCache.expose
 *           (caches.py:246-256) evaluated per query.                         */
#define HS_APPEND_POS    0
#define HS_APPEND_LINEAR 1
#define HS_APPEND_RING   2

typedef struct {
  int pos0;          /* absolute position of the first new token (frontier) */
  int append_mode;
  int append_base;
  int n_sink;
  int ring;
  int n_view;
  int window;
  int win_lo;
  int split;         /* keys per attention split (fixed => t-invariant)    */
  int pos_base;      /* LINEAR caches: absolute position of slot 0 (start of
                        this rank's sequence shard; 0 when unsharded)       */
  int own_hi;        /* HS_APPEND_POS: rows at positions < pos_base or >=
                        own_hi are not stored on this rank (0 = no bound)   */
  const int32_t *dyn;  /* optional device int32[2] read at run time: the
                          frontier (added to pos0) and win_lo -- lets a
                          captured CUDA graph replay a lane step at any
                          position; NULL = use pos0 / win_lo as given       */
} HsStep;

/* ---- sequence sharding of the full cache -----------------
 * Rank r stores the full-cache positions [pos_base, own_hi); every rank runs
 * the same forward, attends over its own slots, and the per-rank partial
 * softmax states (m, l, unnormalised o) of every query row are all-gathered
 * over NCCL and merged in rank order, so all ranks hold bit-identical
 * attention outputs.  comm is an ncclComm_t made by hs_comm_init.          */
typedef struct {
  void *comm;
  int rank, world;
} HsShard;

size_t hs_comm_id_bytes(void);
int hs_comm_unique_id(void *id);                       /* rank 0; ship id to the others */
int hs_comm_init(void **comm, const void *id, int world, int rank);
int hs_comm_destroy(void *comm);
/* recv [world][bytes] <- every rank's send [bytes], rank order            */
int hs_all_gather(void *comm, const void *send, void *recv, size_t bytes, void *stream);
/* in-place sum; dtype 0 bf16, 1 f32, 2 f64, 3 i32                          */
int hs_all_reduce_sum(void *comm, void *buf, size_t count, int dtype, void *stream);
/* recv = every rank's send block of bytes_per_rank[r] bytes, concatenated in
 * rank order (variable-size all-gather: grouped NCCL broadcasts)           */
int hs_all_gather_v(void *comm, int rank, int world, const void *send, void *recv,
                    const size_t *bytes_per_rank, void *stream);
/* HS_OK, or the communicator's asynchronous error (NCCL) / a broken
 * loopback group.  NCCL communicators are created non-blocking and every
 * call is bounded by HS_NCCL_TIMEOUT_S seconds (default 300): a peer that
 * never arrives aborts the communicator and returns HS_ERR_CUDA.          */
int hs_comm_check(void *comm);
/* abort: a failing rank releases its peers (NCCL: ncclCommAbort; loopback:
 * every pending and later collective of the group fails at once)            */
int hs_comm_abort(void *comm);
/* In-process loopback group of `world` ranks on one device: comms[r] is rank
 * r's communicator (use it in HsShard.comm from rank r's host thread and
 * stream).  Collectives are device-to-device copies with the NCCL calls'
 * semantics, so G-shard sessions run (and are tested) on one GPU.         */
int hs_loopback_create(int world, void **comms);
int hs_loopback_destroy(void *any_comm_of_the_group);
/* Replicated retrieval cache after a sharded build (caches.py:458-502 over
 * a sequence-sharded source): ranges [layer][rank][2] (host int32) are the
 * slot ranges each rank filled from its own shard; per layer every rank's
 * K/V block is all-gathered (variable sizes) and unpacked into its slots.  */
size_t hs_retrieval_exchange_workspace_bytes(const HsCache *c);
int hs_retrieval_exchange(const HsShard *sh, const HsCache *c, const int32_t *ranges, void *workspace,
                          size_t ws_bytes, void *stream);

/* ---- fused forward (model.py:247-331) -----------------------------------
 * t tokens (device int32) at st->pos0 through all layers: RMSNorm+QKV GEMV,
 * RoPE + KV append, split-KV attention, wo+residual, RMSNorm+gate|up with a
 * SwiGLU epilogue, down+residual, final norm + head.  Writes t logits rows
 * (fp32) and, if q_stash != NULL, the last row's post-RoPE queries per layer
 * ([L][H][dh], the ForwardRecorder.last_queries of model.py:309).
 * Row results are independent of t (bitwise), so a batched verify equals a
 * sequence of decode steps (model.py:366-378 contract).                     */
size_t hs_forward_workspace_bytes(const HsModel *m, int t, int n_view, int split, int world);
/* leading bytes of the forward workspace that must be zero before first use */
size_t hs_forward_workspace_clean_bytes(const HsModel *m);
/* sh == NULL: unsharded.  Otherwise c is this rank's shard of a FULL cache
 * (kind LINEAR, st->pos_base / st->own_hi set) and attention is merged
 * across sh->world ranks per layer.                                          */
int hs_forward(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh,
               const int32_t *tokens, int t, float *logits, float *q_stash,
               void *workspace, size_t workspace_bytes, void *stream);

/* hs_forward with tensor-parallel dense layers (the
 * projections of model.py:285,316,320-323,328 split by output rows in
 * 128-row tiles over tp->world ranks, each block all-gathered over tp->comm
 * and the next RMSNorm operand rebuilt replicated).  sh: the sequence
 * shards of a full cache (may share tp's communicator) or NULL for a
 * replicated cache (the retrieval lane).  t <= 8 (decode / verify blocks).
 * Logits and every activation end up identical on all ranks.               */
size_t hs_forward_tp_workspace_bytes(const HsModel *m, int t, int n_view, int split, int world, int tp_world);
int hs_forward_tp(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh, const HsShard *tp,
                  const int32_t *tokens, int t, float *logits, float *q_stash,
                  void *workspace, size_t workspace_bytes, void *stream);

/* one decode position over a TopKCache (caches.py:568-652; the oracle
 * upper-bound pairing of analytics.measure_acceptance): like hs_forward with
 * t = 1 on an unsharded full cache, but each layer attends only over the
 * `budget` keys of each kv group with the largest exact group-mean softmax
 * weight (fp64; ties to the lower position).  st->n_view must exceed budget. */
size_t hs_forward_topk_workspace_bytes(const HsModel *m, int n_view, int budget);
int hs_forward_topk(const HsModel *m, const HsCache *c, const HsStep *st, int budget, const int32_t *tokens,
                    float *logits, float *q_stash, void *workspace, size_t workspace_bytes, void *stream);

/* hs_forward on a slotted cache that also reports the attention feedback of
 * H2OCache.observe_attention (caches.py:335-345, model.py:306-307): probs
 * [L][t][n_view] fp64 = per query row, the softmax probabilities over the
 * exposed slots summed over all heads (0 for invisible slots), with the
 * reference's rounding points; head_scratch [t][H][n_view] fp32.           */
int hs_forward_attn_probs(const HsModel *m, const HsCache *c, const HsStep *st, const int32_t *tokens, int t,
                          float *logits, float *q_stash, double *probs, float *head_scratch, void *workspace,
                          size_t workspace_bytes, void *stream);

/* hs_forward (unsharded) that also records the attention probe of
 * ForwardRecorder(record_probs=True) (model.py:308-312): probe
 * [L][H][n_view] fp32 = per layer and head, the last query row's softmax
 * probabilities over the view's slots (0 where a slot is not visible).     */
int hs_forward_probe(const HsModel *m, const HsCache *c, const HsStep *st, const int32_t *tokens, int t,
                     float *logits, float *q_stash, float *probe, void *workspace, size_t workspace_bytes,
                     void *stream);

/* ---- batched prefill (model.py:334-354) --------------
 * Same contract as hs_forward for an unsharded cache, for long prompts: the
 * dense projections run as tensor-core GEMMs (cuBLAS, three bf16 GEMMs over
 * the exact split of the fp32 activations, fp32 accumulation) in blocks of
 * 2048 rows; causal attention on the 128-query-row tensor-core prefill kernel
 * (head_dim 128) or the decode kernels in blocks of 1024 query rows.
 * fp32-accurate but not bit-identical to a decode_step sequence (use
 * hs_forward for that).                                                     */
size_t hs_prefill_workspace_bytes(const HsModel *m, int t, int n_view, int split);
int hs_prefill(const HsModel *m, const HsCache *c, const HsStep *st, const int32_t *tokens, int t,
               float *logits, float *q_stash, void *workspace, size_t workspace_bytes, void *stream);
/* the same over a sequence-sharded full cache (head_dim 128): dense layers on
 * every rank, each rank's attention over its own key slots as packed partial
 * states, exchanged with sh's communicator and merged in rank order         */
size_t hs_prefill_sharded_workspace_bytes(const HsModel *m, int t, int n_view, int split, int world);
int hs_prefill_sharded(const HsModel *m, const HsCache *c, const HsStep *st, const HsShard *sh,
                       const int32_t *tokens, int t, float *logits, float *q_stash, void *workspace,
                       size_t workspace_bytes, void *stream);

/* ---- building blocks (also used by tests and the per-layer cache API) ---- */

/* Tensor-core GEMV (tcgen05 + TMA, swap-AB): y (+)= W . x for one pass of
 * t <= 8 activation rows held as an exact 3-way bf16 split xs [24][ldw]
 * (rows split*8 + r; see hs_split_rows).  epilogue 0 store, 1 accumulate,
 * 2 SwiGLU pairs (output split of act written to xs_out [24][ld_xs_out] and,
 * if y != NULL, fp32 act to y).  The workspace head (hs_gemv_tc_workspace_bytes)
 * must be zero before the first call; kernels leave it zero.              */
size_t hs_gemv_tc_workspace_bytes(int N, int ldw);
int hs_gemv_tc(const uint16_t *xs, int t, const uint16_t *w, int ldw, int N, int epilogue, float *y, int ldy,
               uint16_t *xs_out, int ld_xs_out, void *workspace, size_t ws_bytes, void *stream);

/* Tensor-core GEMM of the batched prefill (tcgen05 + TMA, gemm_tc.cu):
 * y[r][n] (+)= sum_k w[n][k] * (s0 + s1 + s2)[r][k] for rows r < rows, with
 * s0/s1/s2 the exact 3-way bf16 split planes of fp32 activations ([rows][ldk],
 * ldk >= ldw, K = ldw a multiple of 64) and w bf16 [n][ldw]; all three planes
 * accumulate into one fp32 accumulator (model.py:281-285,316-328 matmuls for
 * long prompts).  accumulate = 1 adds into y (residual updates).             */
/* row-major [N][ld] bf16 -> tile-blocked [N/128][ld/64][128][64] in place
 * (tmp: N x ld scratch), or back (inverse = 1); N % 128 == 0, ld % 64 == 0 */
int hs_weights_block(uint16_t *w, uint16_t *tmp, int N, int ld, int inverse, void *stream);

int hs_gemm3_tc(const uint16_t *s0, const uint16_t *s1, const uint16_t *s2, int ldk, int rows,
                const uint16_t *w, int ldw, int n, float *y, int ldy, int accumulate, void *stream);

/* activation prep for hs_gemv_tc: optional RMSNorm (gain != NULL,
 * model.py:282-284) then exact split h = hi + mid + lo into xs [24][ldk]    */
int hs_split_rows(const float *x, int ldx, int t, int K, int ldk, const float *gain, float eps,
                  uint16_t *xs, void *stream);

/* embedding lookup (model.py:274): x[r] = float(emb[tokens[r]])            */
int hs_embed(const uint16_t *emb, int ld, int d, const int32_t *tokens, int t, float *x,
             void *stream);

/* RoPE (model.py:235-244) on q,k rows of qkv [t][(H+2KVH)dh] at positions
 * pos0.., K/V appended to `layer` per st (caches.py append hooks); q written
 * to q_out [t][H][dh]; last row's q to q_stash[layer] if non-NULL.          */
int hs_rope_append(const HsModel *m, const HsCache *c, const HsStep *st, int layer,
                   const float *qkv, int t, float *q_out, float *q_stash, void *stream);

/* raw KV row write for the per-layer cache API (KVCache.append, caches.py:136)
 * rows [t][KVH][dh] fp32 -> bf16 at slots[i], positions pos[i]             */
int hs_kv_write(const HsCache *c, int layer, const float *k, const float *v, int t,
                const int32_t *slots, const int32_t *pos, void *stream);

/* split-KV attention over a cache view (model.py:290-315):
 * q [t][H][dh] fp32 -> out [t][H*dh] fp32                                   */
size_t hs_attention_workspace_bytes(int t, int n_heads, int head_dim, int n_view, int split);
int hs_attention(const HsCache *c, int layer, const HsStep *st, int n_heads,
                 const float *q, int t, float *out, void *workspace, size_t ws_bytes,
                 void *stream);
/* same, but writes this view's partial softmax state per query row instead
 * of the normalised output: packed [t*H][2 + dh] = (m, l, o[dh]) with o
 * unnormalised and m = -inf, l = 0 for rows that see no key (shard input). */
int hs_attention_partial(const HsCache *c, int layer, const HsStep *st, int n_heads,
                         const float *q, int t, float *packed, void *workspace, size_t ws_bytes,
                         void *stream);
/* causal prefill attention (head_dim 128, linear cache; model.py:290-315 for
 * a prompt block): t query rows at positions st->pos0.. over the cache slots
 * [0, st->n_view), slot s holding position s + st->pos_base.  Exactly one of
 * out ([t][H*dh] normalised) / packed ([t*H][2 + dh] partial state) is set. */
int hs_prefill_attention(const HsCache *c, int layer, const HsStep *st, int n_heads, const float *q, int t,
                         float *out, float *packed, void *stream);

/* live timing of the dominant kernel for bench.py: while enabled, every
 * attention launch of hs_forward over a view of >= min_view keys is
 * bracketed by CUDA events on its stream; read returns the summed device
 * time, the algorithmic K+V bytes and the launch count (enable resets).     */
int hs_profile_attention(int enable, int min_view);
int hs_profile_attention_read(double *ms_total, long long *bytes_total, int *launches);

/* chunk scoring, score_chunks (caches.py:414-436), all layers at once.
 * keys: layer l, kv head h, token i at  keys + l*ls + h*hs + i*ts  (bf16 if
 * key_bf16 else fp32); queries [L][H][dh] fp32; scores [L][n_chunks] fp64.  */
int hs_chunk_score(const void *keys, int key_bf16, long long layer_stride, long long head_stride,
                   long long token_stride, int n_layers, int n_kv_heads, int head_dim, int upto,
                   int chunk, const float *queries, int n_heads, double *scores, void *stream);

/* chunk selection of RetrievalCache.build (caches.py:474-495) per layer:
 * top (quota-1) non-last chunks by (-score, id) + the last chunk (all chunks
 * if clamped).  importance [L][quota] ([last] + rest), chosen [L][quota]
 * ascending, ring [L][budget]: victim FIFO as slot indices.  n_chosen and
 * n_exposed are written to out_counts[0..1].                                */
size_t hs_chunk_select_workspace_bytes(int n_layers, int n_chunks);
int hs_chunk_select(const double *scores, int n_layers, int n_chunks, int upto, int chunk,
                    int budget, int32_t *importance, int32_t *chosen, int32_t *ring,
                    int32_t *out_counts, void *workspace, size_t ws_bytes, void *stream);

/* gather of the chosen chunks into the retrieval cache slots, position order
 * (st.push(K[sel_idx], ...) caches.py:490-493).  src is a LINEAR cache
 * holding positions [src_lo, src_hi) (a sequence shard; 0, 0 = unsharded);
 * the K/V slots of chunks outside it are left untouched (positions are
 * written for every chunk); hs_retrieval_exchange then fills them from their
 * owner ranks.                                                              */
int hs_retrieval_gather(const HsCache *src, const HsCache *dst, const int32_t *chosen,
                        int chosen_stride, int n_chosen, int chunk, int upto, int src_lo, int src_hi,
                        void *stream);

/* RetrievalCache.commit / _overwrite (caches.py:529-555) for all layers:
 * spec slots [n_sel, n_sel+n_spec) -- the first `take` move into the victim
 * slots ring[(head+i) % n_sel]; the rest shift down.                         */
int hs_retrieval_commit(const HsCache *c, const int32_t *ring, int ring_stride, int n_sel, int ring_head,
                        int n_spec, int take, void *stream);

/* copy a cache's live slots (clone(), caches.py:216-221 / 283-288 / 557-565) */
int hs_cache_copy(const HsCache *dst, const HsCache *src, int n_slots, void *stream);

/* ---- sampling & verification (model.py:182-206, speculation.py:52-72,187-208)
 * probs [rows][V] fp64: temperature 0 -> one-hot argmax (lowest index wins) */
int hs_probs(const float *logits, int rows, int V, double temperature, double *probs,
             void *stream);

/* inverse-CDF draw consuming one uniform: token = min(#{c_j <= u}, V-1),
 * u = uniforms[*cursor]; (*cursor)++ (device int).  Writes token to out.    */
int hs_sample(const double *probs, int V, const double *uniforms, int32_t *cursor,
              int32_t *out, void *stream);

/* draft step fused: probs of one logits row + sample (draft_round,
 * speculation.py:221-226).  probs_out may be NULL only if temperature == 0. */
int hs_draft_sample(const float *logits, int V, double temperature, double *probs_out,
                    const double *uniforms, int32_t *cursor, int32_t *out, void *stream);

/* one draft step through a captured one-token step graph (draft_round,
 * speculation.py:221-226, without a host round trip per token): draft_sample
 * of the lane's frontier row, the token also written with the step's
 * positions into the graph's slot dyn = [frontier, window watermark, token],
 * then the graph (cudaGraphExec_t, NULL: none) is launched on the stream;
 * n_launch = kernels in the graph (launch accounting).                      */
int hs_draft_step(const float *logits, int V, double temperature, double *probs_out,
                  const double *uniforms, int32_t *cursor, int32_t *out, int32_t *dyn, int frontier,
                  int lo, void *graph_exec, int n_launch, void *stream);

/* n <= 1024 int32 host values (src, pageable) -> device dst, stream-ordered
 * through a pinned ring (no synchronisation): a step's token ids.           */
int hs_upload_i32(int32_t *dst, const int32_t *src, int n, void *stream);

/* positions (+ token >= 0, also copied to *also when non-NULL) of a step
 * graph's slot, then the graph: the lane's catch-up over a host token.      */
int hs_graph_step(int32_t *dyn, int frontier, int lo, int token, int32_t *also, void *graph_exec,
                  int n_launch, void *stream);

/* _verify_chain (speculation.py:187-208).  tokens[n] (device), qd [n][V],
 * pd [n+1][V].  result[0..n]: emitted tokens; result[n+1] = count emitted;
 * result[n+2] = accepted; result[n+3] = status (0 ok, HS_ERR_CONTRACT when
 * q[x] <= 0, verify_token speculation.py:58-60).                             */
int hs_verify_chain(const int32_t *tokens, int n, const double *qd, const double *pd, int V,
                    const double *uniforms, int32_t *cursor, int32_t *result, void *stream);

/* verify_token alone (speculation.py:52-62): result[0] = accepted (0/1),
 * result[1] = status; one uniform.                                          */
int hs_verify_token(int32_t x, const double *q, const double *p, const double *uniforms,
                    int32_t *cursor, int32_t *result, void *stream);

/* correct_token alone (speculation.py:65-72): one uniform.                  */
int hs_correct_token(const double *q, const double *p, int V, const double *uniforms,
                     int32_t *cursor, int32_t *out, void *stream);

/* ---- sequence sharding ----------------------------------
 * merge per-shard packed partial states [G][rows][2 + dh] in rank order:
 * M = max m_s, out = sum_s e^{m_s-M} o_s / sum_s e^{m_s-M} l_s.            */
int hs_shard_merge(const float *parts, int n_shards, int rows, int head_dim, float *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HS_ABI_H */
