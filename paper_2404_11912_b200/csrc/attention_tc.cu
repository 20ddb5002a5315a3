// Tensor-core split-KV attention for head_dim 128 (tcgen05 + TMA).
//
// Replaces the attention core of the reference forward (model.py:290-315)
// for the target model's lanes: the multi-token verify over the full cache
// (outer_verify, speculation.py:264-275), autoregressive decode, and the
// retrieval view.  Same exposure rule and partial-state layout as the
// CUDA-core kernel in attention.cu (see there), so attn_combine_kernel merges
// either.
//
// Per CTA work item (split of 2048/512 slots, kv head, block of <= 16 query
// rows), per 128-key tile:
//   S^T[128 keys x 48] = K_tile[128 x 128] . Qsplit^T        (8 x tcgen05.mma K16)
//   softmax in registers (thread = key = TMEM lane), online max/sum across
//   the 4 warps, P split exactly into 3 bf16 terms -> smem (K-major, SW128)
//   O^T[128 dh x 48]   = V_tile^T (MN-major) . Psplit^T      (8 x tcgen05.mma K16)
//   thread = dh lane accumulates o = o*fac + (hi + mid + lo) in registers.
// q and p enter the tensor core as exact 3-way bf16 splits, so every product
// is exact and accumulation is fp32: numerics match the fp32 CUDA-core path.
// Each query row is its own MMA column: a row's result does not depend on
// the other rows in the launch (t-invariance of the verify forward).
//
// Warp roles: warps 0-3 own TMEM lane quarters (softmax / accumulate), thread
// 0 issues the MMAs at the points where the four warps are synchronised;
// warp 4 is the TMA producer (one K stage + one V stage, 32 KB each), so the
// next tile's K streams while the current tile's P.V runs.  Two CTAs per SM,
// persistent over work items.
#include "hs_common.cuh"
#include "tc_util.cuh"

namespace hs {

int get_tmap_bf16(const void *ptr, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes, uint32_t box_rows,
                  CUtensorMap *out);

namespace {

constexpr int AT_KT = 128;              // keys per tile (MMA M of S^T)
constexpr int AT_DH = 128;
constexpr int AT_QR = 16;               // query rows per work item
constexpr int AT_N = 3 * AT_QR;         // MMA N (3-way split)
constexpr int AT_HALF = 128 * 64 * 2;   // one [128 rows x 64] bf16 SW128 tile = 16 KB
constexpr int AT_QP = AT_N * 128;       // one [48 rows x 64] bf16 SW128 atom column = 6 KB
constexpr int AT_THREADS = 160;
constexpr int AT_SMEM = 2 * AT_HALF /*K*/ + 2 * AT_HALF /*V*/ + 2 * AT_QP /*Q*/ + 2 * AT_QP /*P*/ + 2048 + 1024;

struct AttTcArgs {
  const float *q;       // [t][H][128]
  int t, H, KVH, g;
  const int32_t *pos;   // layer [cap] or null
  int cap, layer, n_view, pos0, window, win_lo, n_sink, split, n_splits, n_qb, n_items;
  float scale;
  float *part_m, *part_l, *part_o;
};

__device__ __forceinline__ bool visible_tc(int kp, int qp, const AttTcArgs &a) {
  if (kp < 0 || kp > qp) return false;
  if (a.window == 0 || kp < a.n_sink) return true;
  int lo = qp - a.window + 1;
  if (a.win_lo > lo) lo = a.win_lo;
  return kp >= lo;
}

// byte offset of element (row n, col k) in a K-major SW128 operand made of
// 64-column atoms of `rows` rows each
__device__ __forceinline__ uint32_t sw128_off(int n, int k, int rows) {
  const int atom = k >> 6, kk = k & 63;
  return (uint32_t)(atom * rows * 128 + n * 128 + ((((kk >> 3) ^ (n & 7)) & 7) << 4) + ((kk & 7) << 1));
}

__device__ __forceinline__ void named_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__global__ void __launch_bounds__(AT_THREADS, 2) attn_tc_kernel(const __grid_constant__ CUtensorMap tmK,
                                                              const __grid_constant__ CUtensorMap tmV, AttTcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *sK = base;                        // 2 x 16 KB (dh halves)
  unsigned char *sV = sK + 2 * AT_HALF;            // 2 x 16 KB
  unsigned char *sQ = sV + 2 * AT_HALF;            // 2 x 6 KB
  unsigned char *sP = sQ + 2 * AT_QP;              // 2 x 6 KB (key halves)
  uint64_t *bars = reinterpret_cast<uint64_t *>(sP + 2 * AT_QP);
  uint64_t *kfull = bars + 0, *kempty = bars + 1, *vfull = bars + 2, *vempty = bars + 3, *sdone = bars + 4,
           *odone = bars + 5;
  uint32_t *tmem_base = reinterpret_cast<uint32_t *>(bars + 8);
  float *red = reinterpret_cast<float *>(bars + 16);          // [4][AT_QR]
  int *qp_s = reinterpret_cast<int *>(red + 4 * AT_QR);        // [AT_QR]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  if (tid == 0) {
    tc::tma_prefetch(&tmK);
    tc::tma_prefetch(&tmV);
    tc::mbar_init(kfull, 1); tc::mbar_init(kempty, 1); tc::mbar_init(vfull, 1); tc::mbar_init(vempty, 1);
    tc::mbar_init(sdone, 1); tc::mbar_init(odone, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<128>(tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_base;
  const uint32_t tS = tmem, tO = tmem + 64;

  // ---------------------------------------------------------------- producer
  if (warp == 4) {
    if (tc::elect_one()) {
      uint32_t g = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        const int split = item % a.n_splits, kh = (item / a.n_splits) % a.KVH;
        const int lo = split * a.split, hi = min(a.n_view, lo + a.split);
        const int row0 = (a.layer * a.KVH + kh) * a.cap;
        for (int tile = lo; tile < hi; tile += AT_KT, ++g) {
          tc::mbar_wait(kempty, (g & 1) ^ 1);
          tc::mbar_expect_tx(kfull, 2 * AT_HALF);
          tc::tma_load_2d(sK, &tmK, kfull, 0, row0 + tile);
          tc::tma_load_2d(sK + AT_HALF, &tmK, kfull, 64, row0 + tile);
          tc::mbar_wait(vempty, (g & 1) ^ 1);
          tc::mbar_expect_tx(vfull, 2 * AT_HALF);
          tc::tma_load_2d(sV, &tmV, vfull, 0, row0 + tile);
          tc::tma_load_2d(sV + AT_HALF, &tmV, vfull, 64, row0 + tile);
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers (warps 0-3)
  constexpr uint32_t idS = tc::idesc_bf16(128, AT_N, 0, 0);
  constexpr uint32_t idO = tc::idesc_bf16(128, AT_N, 1, 0);
  const uint32_t tl = (uint32_t)(warp * 32) << 16;   // this warp's TMEM lane quarter
  uint32_t g = 0;
  for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
    const int split = item % a.n_splits, kh = (item / a.n_splits) % a.KVH, qb = item / (a.n_splits * a.KVH);
    const int lo = split * a.split, hi = min(a.n_view, lo + a.split);
    const int r0 = qb * AT_QR;
    const int nrows = min(AT_QR, a.g * a.t - r0);
    // ---- stage the query split (rows n = s*16 + rr) -------------------------------
    if (tid < AT_QR) qp_s[tid] = tid < nrows ? a.pos0 + (r0 + tid) / a.g : -1;
    for (int e = tid; e < AT_QR * AT_DH; e += 128) {
      const int rr = e >> 7, d = e & 127;
      float v = 0.f;
      if (rr < nrows) {
        const int i = (r0 + rr) / a.g, head = kh * a.g + (r0 + rr) % a.g;
        v = a.q[((size_t)i * a.H + head) * AT_DH + d];
      }
      const __nv_bfloat16 h0 = __float2bfloat16_rn(v);
      const float r1 = v - __bfloat162float(h0);
      const __nv_bfloat16 h1 = __float2bfloat16_rn(r1);
      const __nv_bfloat16 h2 = __float2bfloat16_rn(r1 - __bfloat162float(h1));
      *reinterpret_cast<__nv_bfloat16 *>(sQ + sw128_off(rr, d, AT_N)) = h0;
      *reinterpret_cast<__nv_bfloat16 *>(sQ + sw128_off(AT_QR + rr, d, AT_N)) = h1;
      *reinterpret_cast<__nv_bfloat16 *>(sQ + sw128_off(2 * AT_QR + rr, d, AT_N)) = h2;
    }
    tc::fence_async_smem();
    named_sync();
    float m_run[AT_QR], l_run[AT_QR], o_acc[AT_QR];
#pragma unroll
    for (int r = 0; r < AT_QR; ++r) { m_run[r] = -INFINITY; l_run[r] = 0.f; o_acc[r] = 0.f; }

    for (int tile = lo; tile < hi; tile += AT_KT, ++g) {
      const uint32_t ph = g & 1;
      // ---- S^T = K . Qsplit^T ---------------------------------------------------
      if (tid == 0) {
        tc::mbar_wait(kfull, ph);
        tc::fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_DH / 16; ++kk) {
          const uint64_t da = tc::desc_k_sw128(sK + (kk >> 2) * AT_HALF) + 2 * (kk & 3);
          const uint64_t db = tc::desc_k_sw128(sQ + (kk >> 2) * AT_QP) + 2 * (kk & 3);
          tc::mma_bf16(tS, da, db, idS, kk != 0);
        }
        tc::mma_commit(kempty);
        tc::mma_commit(sdone);
      }
      const int key = tile + tid;               // this thread's key slot
      const bool in_range = key < hi;
      const int kp = in_range ? (a.pos ? a.pos[key] : key) : -1;
      tc::mbar_wait(sdone, ph);
      tc::fence_after();
      float s[AT_N];
#pragma unroll
      for (int c = 0; c < AT_N; c += 8) tc::tmem_ld8(tS + tl + c, s + c);
      tc::tmem_ld_wait();
      // ---- masked scores, tile max across the 128 keys ---------------------------
      float x[AT_QR];
#pragma unroll
      for (int r = 0; r < AT_QR; ++r) {
        const bool vis = r < nrows && visible_tc(kp, qp_s[r], a);
        x[r] = vis ? ((s[r] + s[AT_QR + r]) + s[2 * AT_QR + r]) * a.scale : -INFINITY;
        float mx = warp_max(x[r]);
        if (lane == 0) red[warp * AT_QR + r] = mx;
      }
      named_sync();
      float fac[AT_QR], p[AT_QR];
#pragma unroll
      for (int r = 0; r < AT_QR; ++r) {
        const float tmax = fmaxf(fmaxf(red[r], red[AT_QR + r]), fmaxf(red[2 * AT_QR + r], red[3 * AT_QR + r]));
        const float m_new = fmaxf(m_run[r], tmax);
        fac[r] = 1.f;
        p[r] = 0.f;
        if (m_new != -INFINITY) {
          p[r] = (x[r] == -INFINITY) ? 0.f : expf(x[r] - m_new);
          fac[r] = (m_run[r] == -INFINITY) ? 0.f : expf(m_run[r] - m_new);
        }
        m_run[r] = m_new;
      }
      named_sync();   // everyone read red[] (max) before it is reused for sums
#pragma unroll
      for (int r = 0; r < AT_QR; ++r) {
        const float ps = warp_sum(p[r]);
        if (lane == 0) red[warp * AT_QR + r] = ps;
        // P split into smem (K-major over keys): rows r, 16+r, 32+r
        const __nv_bfloat16 h0 = __float2bfloat16_rn(p[r]);
        const float r1 = p[r] - __bfloat162float(h0);
        const __nv_bfloat16 h1 = __float2bfloat16_rn(r1);
        const __nv_bfloat16 h2 = __float2bfloat16_rn(r1 - __bfloat162float(h1));
        *reinterpret_cast<__nv_bfloat16 *>(sP + sw128_off(r, tid, AT_N)) = h0;
        *reinterpret_cast<__nv_bfloat16 *>(sP + sw128_off(AT_QR + r, tid, AT_N)) = h1;
        *reinterpret_cast<__nv_bfloat16 *>(sP + sw128_off(2 * AT_QR + r, tid, AT_N)) = h2;
      }
      tc::fence_async_smem();
      tc::fence_before();
      named_sync();
#pragma unroll
      for (int r = 0; r < AT_QR; ++r)
        l_run[r] = l_run[r] * fac[r] + ((red[r] + red[AT_QR + r]) + (red[2 * AT_QR + r] + red[3 * AT_QR + r]));
      // ---- O^T = V^T . Psplit^T -------------------------------------------------
      if (tid == 0) {
        tc::fence_after();
        tc::mbar_wait(vfull, ph);
        tc::fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_KT / 16; ++kk) {
          // A = V^T, MN-major: 64-dh blocks 16 KB apart (LBO), 8-key groups 1 KB apart (SBO)
          const uint64_t da = tc::desc_mn_sw128(sV + kk * 2048, AT_HALF, 1024);
          const uint64_t db = tc::desc_k_sw128(sP + (kk >> 2) * AT_QP) + 2 * (kk & 3);
          tc::mma_bf16(tO, da, db, idO, kk != 0);
        }
        tc::mma_commit(vempty);
        tc::mma_commit(odone);
      }
      tc::mbar_wait(odone, ph);
      tc::fence_after();
      float o[AT_N];
#pragma unroll
      for (int c = 0; c < AT_N; c += 8) tc::tmem_ld8(tO + tl + c, o + c);
      tc::tmem_ld_wait();
#pragma unroll
      for (int r = 0; r < AT_QR; ++r) o_acc[r] = o_acc[r] * fac[r] + ((o[r] + o[AT_QR + r]) + o[2 * AT_QR + r]);
      tc::fence_before();
      named_sync();   // TMEM S/O and smem P free for the next tile
    }
    // ---- partial state of this item ---------------------------------------------------
    const size_t pbase = (size_t)split * a.t * a.H;
#pragma unroll
    for (int r = 0; r < AT_QR; ++r) {
      if (r < nrows) {
        const int i = (r0 + r) / a.g, head = kh * a.g + (r0 + r) % a.g;
        const size_t row = (size_t)i * a.H + head;
        a.part_o[(pbase + row) * AT_DH + tid] = o_acc[r];
        if (tid == 0) { a.part_m[pbase + row] = m_run[r]; a.part_l[pbase + row] = l_run[r]; }
      }
    }
    named_sync();
  }
  tc::fence_before();
  named_sync();
  if (warp == 0) tc::tmem_dealloc<128>(tmem);
}

}  // namespace

int launch_attention_tc(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t, float *part_m,
                        float *part_l, float *part_o, int n_splits, cudaStream_t stream) {
  HS_REQUIRE(c->head_dim == AT_DH, HS_ERR_SHAPE, "attention_tc: head_dim must be 128");
  CUtensorMap mk, mv;
  const uint64_t rows = (uint64_t)c->n_layers * c->n_kv_heads * c->cap;
  int rc = get_tmap_bf16(c->k, AT_DH, rows, AT_DH * 2, AT_KT, &mk);
  if (rc != HS_OK) return rc;
  rc = get_tmap_bf16(c->v, AT_DH, rows, AT_DH * 2, AT_KT, &mv);
  if (rc != HS_OK) return rc;
  AttTcArgs a;
  a.q = q; a.t = t; a.H = H; a.KVH = c->n_kv_heads; a.g = H / c->n_kv_heads;
  a.pos = (c->kind == HS_KV_SLOTTED) ? c->pos + (size_t)layer * c->cap : nullptr;
  a.cap = c->cap; a.layer = layer; a.n_view = st->n_view; a.pos0 = st->pos0; a.window = st->window;
  a.win_lo = st->win_lo; a.n_sink = st->n_sink; a.split = st->split; a.n_splits = n_splits;
  a.n_qb = ceil_div(a.g * t, AT_QR);
  a.n_items = n_splits * a.KVH * a.n_qb;
  a.scale = (float)(1.0 / sqrt((double)AT_DH));
  a.part_m = part_m; a.part_l = part_l; a.part_o = part_o;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
    attr = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = a.n_items < 2 * sms ? a.n_items : 2 * sms;
  attn_tc_kernel<<<grid, AT_THREADS, AT_SMEM, stream>>>(mk, mv, a);
  return check_launch("attention_tc");
}

}  // namespace hs
