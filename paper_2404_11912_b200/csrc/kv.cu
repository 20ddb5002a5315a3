// KV-cache maintenance kernels: embedding, RoPE + append, raw row writes,
// retrieval overwrite-on-commit, cache clone.
#include "hs_common.cuh"

namespace hs {

HS_TRACE_TU
int trace_set_kv(void *p, unsigned cap) { return trace_set_tu(p, cap); }

// ---- embedding (model.py:274) ----------------------------------------------
__global__ void embed_kernel(const uint16_t *emb, int ld, int d, const int32_t *tokens, float *x) {
  HS_TRACE_BEGIN
  const int r = blockIdx.x;
  const uint16_t *row = emb + (size_t)tokens[r] * ld;
  for (int c = threadIdx.x; c < d; c += blockDim.x) x[(size_t)r * d + c] = bf16_to_f(row[c]);
  HS_TRACE_END(6)
}

int launch_embed(const uint16_t *emb, int ld, int d, const int32_t *tokens, int t, float *x,
                 cudaStream_t st) {
  embed_kernel<<<t, 256, 0, st>>>(emb, ld, d, tokens, x);
  return check_launch("embed");
}

// embedding rows + the first layer's folded-RMSNorm operand in one kernel
// (the single-block forward): x[r] = emb[token r] and xs = split(x * gain),
// norm_prep's arithmetic on the same fp32 values.  grid (tiles of 128
// columns, t).  A programmatic dependent of the previous forward's last
// kernel: scheduled while it drains, everything after griddepcontrol.wait
// (the tokens come from the sampler, x is still read by that kernel).
__global__ void __launch_bounds__(128) embed_norm_kernel(const uint16_t *emb, int ld, int d, const int32_t *tokens,
                                                         float *x, const float *gain, uint16_t *xs, int ldk) {
  HS_TRACE_BEGIN
  pdl_wait();
  pdl_trigger();
  HS_TRACE_RESTART
  const int r = blockIdx.y, col = blockIdx.x * 128 + threadIdx.x;
  if (col < d) {
    const float v = bf16_to_f(emb[(size_t)tokens[r] * ld + col]);
    x[(size_t)r * d + col] = v;
    store_split(xs, ldk, r, col, __fmul_rn(v, gain[col]));
  }
  HS_TRACE_END(6)
}

int launch_embed_norm(const uint16_t *emb, int ld, int d, const int32_t *tokens, int t, float *x, const float *gain,
                      uint16_t *xs, int ldk, cudaStream_t st) {
  HS_REQUIRE(t >= 1 && t <= 8, HS_ERR_SHAPE, "embed_norm: t=%d outside [1,8]", t);
  cudaError_t e = launch_pdl(embed_norm_kernel, dim3((d + 127) / 128, t), dim3(128), 0, st, emb, ld, d, tokens, x,
                             gain, xs, ldk);
  if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "embed_norm launch: %s", cudaGetErrorString(e));
  return check_launch("embed_norm");
}

// slot of the i-th new row at position p, or -1 when this rank does not store
// it (sequence shard of a full cache: positions [pos_base, own_hi))
__device__ __forceinline__ int append_slot(const HsStep &s, int i, int p) {
  if (s.append_mode == HS_APPEND_POS) {
    if (p < s.pos_base || (s.own_hi > 0 && p >= s.own_hi)) return -1;
    return p - s.pos_base;
  }
  if (s.append_mode == HS_APPEND_LINEAR) return s.append_base + i;
  return p < s.n_sink ? p : s.n_sink + (p - s.n_sink) % s.ring;
}

// ---- RoPE + append (model.py:286-289, _rope_rows model.py:235-244) ---------
// grid (t, H + 2*KVH); thread = rotation pair.  Rotation in fp64 from the
// fp32-rounded table, rounded to fp32 (q) and then bf16 (cached k), exactly
// the reference's rounding points plus the bf16 storage.
__global__ void rope_append_kernel(HsModel m, HsCache c, HsStep s, int layer, const float *qkv,
                                   float *q_out, float *q_stash, int t) {
  HS_TRACE_BEGIN
  pdl_trigger();   // the attention kernel may set up (barriers, TMEM, tensor maps) meanwhile
  pdl_wait();      // qkv comes from the preceding GEMV
  HS_TRACE_RESTART
  const int i = blockIdx.x, hh = blockIdx.y, pr = threadIdx.x;
  const int H = m.n_heads, KVH = m.n_kv_heads, DH = m.head_dim, half = DH / 2;
  if (pr >= half) return;
  const int p = (s.dyn ? s.dyn[0] : 0) + s.pos0 + i;
  const int ncols = (H + 2 * KVH) * DH;
  const float *row = qkv + (size_t)i * ncols;
  if (hh < H + KVH) {
    const int col = hh * DH + 2 * pr;
    const double e = (double)row[col], o = (double)row[col + 1];
    const double cs = (double)m.rope_cos[(size_t)p * half + pr];
    const double sn = (double)m.rope_sin[(size_t)p * half + pr];
    const float y0 = (float)(e * cs - o * sn);
    const float y1 = (float)(e * sn + o * cs);
    if (hh < H) {
      float *qo = q_out + ((size_t)i * H + hh) * DH + 2 * pr;
      qo[0] = y0; qo[1] = y1;
      if (q_stash && i == t - 1) {
        float *qs = q_stash + ((size_t)layer * H + hh) * DH + 2 * pr;
        qs[0] = y0; qs[1] = y1;
      }
    } else {
      const int kh = hh - H;
      const int slot = append_slot(s, i, p);
      if (slot < 0) return;
      uint16_t *kd = c.k + (((size_t)layer * KVH + kh) * c.cap + slot) * DH + 2 * pr;
      kd[0] = f_to_bf16(y0); kd[1] = f_to_bf16(y1);
      if (kh == 0 && pr == 0 && c.kind == HS_KV_SLOTTED) c.pos[(size_t)layer * c.cap + slot] = p;
    }
  } else {
    const int kh = hh - H - KVH;
    const int slot = append_slot(s, i, p);
    if (slot < 0) return;
    const int col = (H + KVH + kh) * DH + 2 * pr;
    uint16_t *vd = c.v + (((size_t)layer * KVH + kh) * c.cap + slot) * DH + 2 * pr;
    vd[0] = f_to_bf16(row[col]); vd[1] = f_to_bf16(row[col + 1]);
  }
  HS_TRACE_END(7)
}

int launch_rope_append(const HsModel *m, const HsCache *c, const HsStep *s, int layer, const float *qkv,
                       int t, float *q_out, float *q_stash, cudaStream_t st) {
  HS_REQUIRE(m->head_dim % 2 == 0 && m->head_dim <= 256, HS_ERR_SHAPE, "rope: bad head_dim");
  HS_REQUIRE(s->pos0 + t <= m->max_seq, HS_ERR_CAPACITY, "sequence of %d exceeds max_seq %d", s->pos0 + t, m->max_seq);
  if (s->append_mode == HS_APPEND_POS) {
    const int hi = s->own_hi > 0 && s->own_hi < s->pos0 + t ? s->own_hi : s->pos0 + t;
    HS_REQUIRE(hi - s->pos_base <= c->cap, HS_ERR_CAPACITY, "full cache overflow past %d", s->pos_base + c->cap);
  }
  if (s->append_mode == HS_APPEND_LINEAR)
    HS_REQUIRE(s->append_base + t <= c->cap, HS_ERR_CAPACITY, "retrieval spec tail overflow (%d slots)", c->cap);
  if (s->append_mode == HS_APPEND_RING)
    HS_REQUIRE(s->ring > 0 && s->n_sink + s->ring <= c->cap, HS_ERR_CAPACITY, "ring exceeds capacity");
  dim3 grid(t, m->n_heads + 2 * m->n_kv_heads);
  cudaError_t e = launch_pdl(rope_append_kernel, grid, dim3(m->head_dim / 2), 0, st, *m, *c, *s, layer, qkv, q_out,
                             q_stash, t);
  if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "rope_append launch: %s", cudaGetErrorString(e));
  return check_launch("rope_append");
}

// ---- raw row writes for the per-layer API ------------------------------------
__global__ void kv_write_kernel(HsCache c, int layer, const float *k, const float *v, int t,
                                const int32_t *slots, const int32_t *pos) {
  const int i = blockIdx.x, kh = blockIdx.y, DH = c.head_dim;
  const int slot = slots[i];
  const size_t dst = (((size_t)layer * c.n_kv_heads + kh) * c.cap + slot) * DH;
  const size_t src = ((size_t)i * c.n_kv_heads + kh) * DH;
  for (int d = threadIdx.x; d < DH; d += blockDim.x) {
    c.k[dst + d] = f_to_bf16(k[src + d]);
    c.v[dst + d] = f_to_bf16(v[src + d]);
  }
  if (kh == 0 && threadIdx.x == 0 && c.kind == HS_KV_SLOTTED) c.pos[(size_t)layer * c.cap + slot] = pos[i];
}

// ---- RetrievalCache.commit (caches.py:529-555) --------------------------------
// grid (L, KVH); every thread owns fixed dims, so the sequential FIFO order of
// overwrites (including wrap-around when take > n_sel) is preserved per dim.
__global__ void retrieval_commit_kernel(HsCache c, const int32_t *ring, int ring_stride, int n_sel, int head,
                                        int n_spec, int take) {
  const int l = blockIdx.x, kh = blockIdx.y, DH = c.head_dim;
  const size_t rowbase = ((size_t)l * c.n_kv_heads + kh) * c.cap;
  int32_t *pos = c.pos + (size_t)l * c.cap;
  const int32_t *rg = ring + (size_t)l * ring_stride;
  for (int i = 0; i < take; ++i) {
    const int dst = rg[(head + i) % n_sel];
    const int src = n_sel + i;
    for (int d = threadIdx.x; d < DH; d += blockDim.x) {
      c.k[(rowbase + dst) * DH + d] = c.k[(rowbase + src) * DH + d];
      c.v[(rowbase + dst) * DH + d] = c.v[(rowbase + src) * DH + d];
    }
    if (kh == 0 && threadIdx.x == 0) pos[dst] = pos[src];
  }
  for (int i = take; i < n_spec; ++i) {
    const int src = n_sel + i, dst = n_sel + i - take;
    for (int d = threadIdx.x; d < DH; d += blockDim.x) {
      c.k[(rowbase + dst) * DH + d] = c.k[(rowbase + src) * DH + d];
      c.v[(rowbase + dst) * DH + d] = c.v[(rowbase + src) * DH + d];
    }
    if (kh == 0 && threadIdx.x == 0) pos[dst] = pos[src];
  }
  __syncthreads();
  if (kh == 0) {
    for (int i = n_spec - take + threadIdx.x; i < n_spec; i += blockDim.x) pos[n_sel + i] = -1;
  }
}

}  // namespace hs

extern "C" int hs_embed(const uint16_t *emb, int ld, int d, const int32_t *tokens, int t, float *x,
                        void *stream) {
  return hs::launch_embed(emb, ld, d, tokens, t, x, hs::as_stream(stream));
}

extern "C" int hs_rope_append(const HsModel *m, const HsCache *c, const HsStep *st, int layer,
                              const float *qkv, int t, float *q_out, float *q_stash, void *stream) {
  return hs::launch_rope_append(m, c, st, layer, qkv, t, q_out, q_stash, hs::as_stream(stream));
}

extern "C" int hs_kv_write(const HsCache *c, int layer, const float *k, const float *v, int t,
                           const int32_t *slots, const int32_t *pos, void *stream) {
  if (t <= 0) return HS_OK;
  dim3 grid(t, c->n_kv_heads);
  hs::kv_write_kernel<<<grid, c->head_dim < 128 ? c->head_dim : 128, 0, hs::as_stream(stream)>>>(
      *c, layer, k, v, t, slots, pos);
  return hs::check_launch("kv_write");
}

extern "C" int hs_retrieval_commit(const HsCache *c, const int32_t *ring, int ring_stride, int n_sel, int ring_head,
                                   int n_spec, int take, void *stream) {
  if (take < 0 || take > n_spec) return hs::set_error(HS_ERR_CONTRACT, "retrieval commit: take %d outside [0,%d]", take, n_spec);
  if (take > 0 && n_sel < 1) return hs::set_error(HS_ERR_CONTRACT, "retrieval cache has no slots");
  if (n_spec == 0) return HS_OK;
  dim3 grid(c->n_layers, c->n_kv_heads);
  hs::retrieval_commit_kernel<<<grid, c->head_dim < 128 ? c->head_dim : 128, 0, hs::as_stream(stream)>>>(
      *c, ring, ring_stride, n_sel, ring_head, n_spec, take);
  return hs::check_launch("retrieval_commit");
}

extern "C" int hs_cache_copy(const HsCache *dst, const HsCache *src, int n_slots, void *stream) {
  if (n_slots <= 0) return HS_OK;
  if (dst->head_dim != src->head_dim || dst->n_kv_heads != src->n_kv_heads || dst->n_layers != src->n_layers ||
      n_slots > dst->cap || n_slots > src->cap)
    return hs::set_error(HS_ERR_SHAPE, "cache_copy: geometry mismatch");
  cudaStream_t st = hs::as_stream(stream);
  const size_t rows = (size_t)src->n_layers * src->n_kv_heads;
  const size_t w = (size_t)n_slots * src->head_dim * 2;
  cudaError_t e = cudaMemcpy2DAsync(dst->k, (size_t)dst->cap * dst->head_dim * 2, src->k,
                                    (size_t)src->cap * src->head_dim * 2, w, rows, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(dst->v, (size_t)dst->cap * dst->head_dim * 2, src->v,
                          (size_t)src->cap * src->head_dim * 2, w, rows, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && src->kind == HS_KV_SLOTTED && dst->kind == HS_KV_SLOTTED)
    e = cudaMemcpy2DAsync(dst->pos, (size_t)dst->cap * 4, src->pos, (size_t)src->cap * 4, (size_t)n_slots * 4,
                          src->n_layers, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return hs::set_error(HS_ERR_CUDA, "cache_copy: %s", cudaGetErrorString(e));
  return HS_OK;
}
