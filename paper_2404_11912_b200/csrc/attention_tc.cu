// Tensor-core split-KV attention for head_dim 128 (tcgen05 + TMA).
//
// Replaces the attention core of the reference forward (model.py:290-315)
// for the target model's lanes: the multi-token verify over the full cache
// (outer_verify, speculation.py:264-275), autoregressive decode, and the
// retrieval view.  Same exposure rule and partial-state layout as the
// CUDA-core kernel in attention.cu (see there), so attn_combine_kernel merges
// either.
//
// Per CTA work item (split of 2048/512 slots, kv head, block of <= 8 query
// rows -- query blocks vary fastest so items sharing a split run together),
// per 128-key tile:
//   S^T[128 keys x 24] = K_tile[128 x 128] . Qsplit^T        (8 x tcgen05.mma K16)
//   softmax in registers (thread = key = TMEM lane), tile max across the 4
//   warps of a group (redux + one named barrier), P split exactly into 3 bf16
//   terms -> smem (K-major, SW128)
//   O^T[128 dh x 24]   = V_tile^T (MN-major) . Psplit^T      (8 x tcgen05.mma K16)
//   thread = dh lane accumulates o = o*fac + (hi + mid + lo) in registers.
// q and p enter the tensor core as exact 3-way bf16 splits, so every product
// is exact and accumulation is fp32: numerics match the fp32 CUDA-core path.
// Each query row is its own MMA column: a row's result does not depend on
// the other rows in the launch (t-invariance of the verify forward).
//
// Software pipeline (S, P, O double-buffered in TMEM/smem; one K and one V
// stage per CTA, two CTAs per SM): S runs one tile ahead of P.V, O(i-1) is
// folded into the register accumulator while the tensor core and the TMA
// stream work on tile i.  Warp roles (10 warps): two softmax groups of four
// warps (the item's rows split evenly between them), warp 4 the TMA producer
// (first tile issued before griddepcontrol.wait when it holds no appended
// slot), warp 5 the MMA issuer.  Persistent over work items.  With FusedRope
// the q staging also applies RoPE to the qkv rows and the CTA covering this
// step's slots appends the new K/V rows before its producer loads them.
#include <stdlib.h>

#include "hs_common.cuh"
#include "tc_util.cuh"

namespace hs {

HS_TRACE_TU
int trace_set_attntc(void *p, unsigned cap) { return trace_set_tu(p, cap); }

int get_tmap_bf16(const void *ptr, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes, uint32_t box_rows,
                  CUtensorMap *out);

namespace {

constexpr int AT_KT = 128;              // keys per tile (MMA M of S^T)
constexpr int AT_DH = 128;
constexpr int AT_QR = 8;                // query rows per work item (more rows -> more items)
constexpr int AT_N = 3 * AT_QR;         // MMA N (3-way split)
constexpr int AT_HALF = 128 * 64 * 2;   // one [128 rows x 64] bf16 SW128 tile = 16 KB
constexpr int AT_KV = 2 * AT_HALF;      // one K or V tile (two dh halves) = 32 KB
constexpr int AT_QP = AT_N * 128;       // one [24 rows x 64] bf16 SW128 atom column = 3 KB
constexpr int AT_OPND = 2 * AT_QP;      // Q or one P buffer = 6 KB
constexpr int AT_THREADS = 320;          // 2 softmax groups x 4 warps, TMA warp, MMA warp
constexpr int AT_GR = 4;                 // query rows per softmax group
constexpr int AT_KSTAGES = 1, AT_VSTAGES = 1;
constexpr int AT_SMEM = AT_KSTAGES * AT_KV + AT_VSTAGES * AT_KV + AT_OPND + 2 * AT_OPND + 1024;

struct AttTcArgs {
  const float *q;       // [t][H][128]
  int t, H, KVH, g;
  const int32_t *pos;   // layer [cap] or null
  int cap, layer, n_view, pos0, window, win_lo, n_sink, split, n_splits, n_qb, n_items, pos_base;
  int clean_hi;         // slots < clean_hi are not written by the preceding kernels (see launch_attention)
  int l2_prefetch;      // prefetch the first item's clean tiles to L2 before the dependency wait
  // fused RoPE + append (forward path, FusedRope): q and this step's K/V rows
  // come straight from the qkv GEMV output; qkv == null: q given, rows appended
  const float *qkv;
  int ncols;
  const float *rope_cos, *rope_sin;   // [max_seq][64] fp32
  float *q_stash;                     // this layer's [H][128], or null
  uint16_t *k_app, *v_app;            // this layer's cache rows [KVH][cap][128]
  int32_t *pos_app;                   // slotted: this layer's pos [cap], else null
  int app_mode, app_base, own_hi;     // HsStep append rule (positions or linear tail)
  int dirty_lo, dirty_hi;             // slots this step appends
  const int32_t *dyn;   // HsStep.dyn: run-time frontier offset / win_lo (graph replay), or null
  float scale_log2;     // log2(e) / sqrt(dh)
  float *part_m, *part_l, *part_o;
};

// work item -> (split, kv head, query block).  Query blocks vary fastest, so
// the items sharing one K/V split run side by side and read it through L2
// (a long prefill block has up to 128 query blocks per split; decode and
// verify have one).
__device__ __forceinline__ void item_coords(int item, const AttTcArgs &a, int &split, int &kh, int &qb) {
  qb = item % a.n_qb;
  split = (item / a.n_qb) % a.n_splits;
  kh = item / (a.n_qb * a.n_splits);
}

__device__ __forceinline__ bool visible_tc(int kp, int qp, const AttTcArgs &a, int win_lo) {
  if (kp < 0 || kp > qp) return false;
  if (a.window == 0 || kp < a.n_sink) return true;
  int lo = qp - a.window + 1;
  if (win_lo > lo) lo = win_lo;
  return kp >= lo;
}

// byte offset of element (row n, col k) in a K-major SW128 operand made of
// 64-column atoms of AT_N rows each
__device__ __forceinline__ uint32_t sw128_off(int n, int k) {
  const int atom = k >> 6, kk = k & 63;
  return (uint32_t)(atom * AT_QP + n * 128 + ((((kk >> 3) ^ (n & 7)) & 7) << 4) + ((kk & 7) << 1));
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// all 8 softmax warps / the 4 warps of one softmax group
__device__ __forceinline__ void softmax_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void group_sync(int grp) { asm volatile("bar.sync %0, 128;" ::"r"(2 + grp) : "memory"); }

// order-preserving float <-> int for redux.sync max
__device__ __forceinline__ int f2o(float f) { const int i = __float_as_int(f); return i ^ ((i >> 31) & 0x7fffffff); }
__device__ __forceinline__ float o2f(int i) { return __int_as_float(i ^ ((i >> 31) & 0x7fffffff)); }

__device__ __forceinline__ void split3_store(unsigned char *buf, int n, int k, float v) {
  const __nv_bfloat16 h0 = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(h0);
  const __nv_bfloat16 h1 = __float2bfloat16_rn(r1);
  const __nv_bfloat16 h2 = __float2bfloat16_rn(r1 - __bfloat162float(h1));
  *reinterpret_cast<__nv_bfloat16 *>(buf + sw128_off(n, k)) = h0;
  *reinterpret_cast<__nv_bfloat16 *>(buf + sw128_off(AT_QR + n, k)) = h1;
  *reinterpret_cast<__nv_bfloat16 *>(buf + sw128_off(2 * AT_QR + n, k)) = h2;
}

__global__ void __launch_bounds__(AT_THREADS, 2) attn_tc_kernel(const __grid_constant__ CUtensorMap tmK,
                                                              const __grid_constant__ CUtensorMap tmV, AttTcArgs a) {
  HS_TRACE_BEGIN
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *sK = base;                        // AT_KSTAGES x 32 KB
  unsigned char *sV = sK + AT_KSTAGES * AT_KV;     // AT_VSTAGES x 32 KB
  unsigned char *sQ = sV + AT_VSTAGES * AT_KV;     // 12 KB
  unsigned char *sP = sQ + AT_OPND;                // 2 buffers x 12 KB
  // TMA <-> MMA: kfull/kempty/vfull/vempty; MMA <-> softmax warps: sfull/sfree,
  // pfull, ofull/ofree, qfull (per item).  Per-tile barriers alternate on
  // buffer b = g & 1 with phase (g >> 1) & 1.
  __shared__ uint64_t kfull[2], kempty[2], vfull[2], vempty[2], sfull[2], sfree[2], pfull[2], ofull[2], ofree[2];
  __shared__ uint64_t qfull, dready;
  __shared__ uint32_t tmem_base;
  __shared__ int red[2][4][AT_QR];
  __shared__ float redl[4][AT_QR];
  __shared__ int qp_s[AT_QR];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  tc::grid_dep_launch();             // the combine kernel is scheduled once every CTA here has started
  if (tid == 0) {
    tc::tma_prefetch(&tmK);
    tc::tma_prefetch(&tmV);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&kfull[s], 1); tc::mbar_init(&kempty[s], 1); tc::mbar_init(&vfull[s], 1);
      tc::mbar_init(&vempty[s], 1); tc::mbar_init(&sfull[s], 1); tc::mbar_init(&sfree[s], 8);
      tc::mbar_init(&pfull[s], 8); tc::mbar_init(&ofull[s], 1); tc::mbar_init(&ofree[s], 8);
    }
    tc::mbar_init(&qfull, 8);
    tc::mbar_init(&dready, 8);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<128>(&tmem_base);   // S[b] at b*32, O[b] at 64 + b*32
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  // ---------------------------------------------------------------- TMA producer (warp 4)
  if (warp == 4) {
    if (tc::elect_one()) {
      // K / V are streamed once: evict-first, so they do not push the split
      // states (read back by the combine) out of L2
      const uint64_t kv_pol = tc::policy_evict_first();
      auto load_kv = [&](uint32_t g, int row) {
        const int ks = g % AT_KSTAGES, vs = g % AT_VSTAGES;
        const uint32_t kph = (g / AT_KSTAGES) & 1, vph = (g / AT_VSTAGES) & 1;
        tc::mbar_wait(&kempty[ks], kph ^ 1);
        tc::mbar_expect_tx(&kfull[ks], AT_KV);
        tc::tma_load_2d_hint(sK + ks * AT_KV, &tmK, &kfull[ks], 0, row, kv_pol);
        tc::tma_load_2d_hint(sK + ks * AT_KV + AT_HALF, &tmK, &kfull[ks], 64, row, kv_pol);
        tc::mbar_wait(&vempty[vs], vph ^ 1);
        tc::mbar_expect_tx(&vfull[vs], AT_KV);
        tc::tma_load_2d_hint(sV + vs * AT_KV, &tmV, &vfull[vs], 0, row, kv_pol);
        tc::tma_load_2d_hint(sV + vs * AT_KV + AT_HALF, &tmV, &vfull[vs], 64, row, kv_pol);
      };
      // Programmatic dependent launch: the first tile of this CTA's first item
      // streams in while the RoPE kernel (and the GEMV before it) drain, when
      // none of its slots is one the current step appends
      bool pre = false;
      if (blockIdx.x < a.n_items) {
        int split, kh, qb;
        item_coords(blockIdx.x, a, split, kh, qb);
        const int lo = split * a.split;
        const int row0 = (a.layer * a.KVH + kh) * a.cap;
        if (lo + AT_KT <= a.clean_hi) {
          load_kv(0, row0 + lo);
          pre = true;
        }
        // small views (the retrieval lane): the rest of the first item's
        // clean tiles go to L2 at once, so the single-stage ring refills
        // from L2 instead of paying an HBM round trip per tile
        if (a.l2_prefetch) {
          const int hi = min(a.n_view, lo + a.split);
          for (int tile = lo + AT_KT; tile < hi && tile + AT_KT <= a.clean_hi; tile += AT_KT) {
            tc::tma_prefetch_l2_2d(&tmK, 0, row0 + tile);
            tc::tma_prefetch_l2_2d(&tmK, 64, row0 + tile);
            tc::tma_prefetch_l2_2d(&tmV, 0, row0 + tile);
            tc::tma_prefetch_l2_2d(&tmV, 64, row0 + tile);
          }
        }
      }
      tc::grid_dep_wait();             // K/V rows appended by the previous kernel
      uint32_t g = 0, nitem = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x, ++nitem) {
        int split, kh, qb;
        item_coords(item, a, split, kh, qb);
        const int lo = split * a.split, hi = min(a.n_view, lo + a.split);
        const int row0 = (a.layer * a.KVH + kh) * a.cap;
        bool waited = false;
        for (int tile = lo; tile < hi; tile += AT_KT, ++g) {
          // fused append: the softmax warps write this step's rows first
          if (a.qkv && !waited && tile < a.dirty_hi && tile + AT_KT > a.dirty_lo) {
            tc::mbar_wait(&dready, nitem & 1);
            waited = true;
          }
          if (g > 0 || !pre) load_kv(g, row0 + tile);
        }
      }
    }
    return;
  }
  tc::grid_dep_wait();               // q, positions and the appended K/V rows
  HS_TRACE_RESTART
  // query positions: host values, or (graph replay) offset by the device frontier
  const int pos0 = a.dyn ? a.pos0 + a.dyn[0] : a.pos0;
  const int win_lo = a.dyn ? a.dyn[1] : a.win_lo;

  // ---------------------------------------------------------------- MMA issuer (warp 5)
  if (warp == 5) {
    if (tc::elect_one()) {
      constexpr uint32_t idS = tc::idesc_bf16(128, AT_N, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16(128, AT_N, 1, 0);
      auto issue_S = [&](uint32_t g) {
        const int s = g & 1, ks = g % AT_KSTAGES;
        const uint32_t ph = (g >> 1) & 1;
        tc::mbar_wait(&kfull[ks], (g / AT_KSTAGES) & 1);
        tc::mbar_wait(&sfree[s], ph ^ 1);
        tc::fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_DH / 16; ++kk) {
          const uint64_t da = tc::desc_k_sw128(sK + ks * AT_KV + (kk >> 2) * AT_HALF) + 2 * (kk & 3);
          const uint64_t db = tc::desc_k_sw128(sQ + (kk >> 2) * AT_QP) + 2 * (kk & 3);
          tc::mma_bf16(tmem + s * 32, da, db, idS, kk != 0);
        }
        tc::mma_commit(&kempty[ks]);
        tc::mma_commit(&sfull[s]);
      };
      auto issue_PV = [&](uint32_t g) {
        const int s = g & 1, vs = g % AT_VSTAGES;
        const uint32_t ph = (g >> 1) & 1;
        tc::mbar_wait(&pfull[s], ph);
        tc::mbar_wait(&vfull[vs], (g / AT_VSTAGES) & 1);
        tc::mbar_wait(&ofree[s], ph ^ 1);
        tc::fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_KT / 16; ++kk) {
          // A = V^T, MN-major: 64-dh blocks 16 KB apart (LBO), 8-key groups 1 KB apart (SBO)
          const uint64_t da = tc::desc_mn_sw128(sV + vs * AT_KV + kk * 2048, AT_HALF, 1024);
          const uint64_t db = tc::desc_k_sw128(sP + s * AT_OPND + (kk >> 2) * AT_QP) + 2 * (kk & 3);
          tc::mma_bf16(tmem + 64 + s * 32, da, db, idO, kk != 0);
        }
        tc::mma_commit(&vempty[vs]);
        tc::mma_commit(&ofull[s]);
      };
      uint32_t g = 0, nitem = 0;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x, ++nitem) {
        int split, kh, qb;
        item_coords(item, a, split, kh, qb);
        const int lo = split * a.split, hi = min(a.n_view, lo + a.split);
        const int ntiles = (hi - lo + AT_KT - 1) / AT_KT;
        tc::mbar_wait(&qfull, nitem & 1);          // this item's query split is staged
        issue_S(g);
        for (int it = 0; it < ntiles; ++it) {       // S runs one tile ahead of P.V
          if (it + 1 < ntiles) issue_S(g + it + 1);
          issue_PV(g + it);
        }
        g += ntiles;
      }
    }
    return;
  }

  // ------------------------------------------------ softmax warps 0-3 and 6-9 (two row groups)
  // Two groups of four warps split the (up to) 8 query rows of a work item,
  // halving each thread's per-tile softmax work; warp w reads TMEM lane
  // quarter w % 4, so thread ltid = key (S) / head dim (O) index.
  const int grp = warp < 4 ? 0 : 1;
  const int ltid = (warp & 3) * 32 + lane;
  const int stid = grp * 128 + ltid;                 // 0..255 over both groups
  const uint32_t tl = (uint32_t)((warp & 3) * 32) << 16;   // this warp's TMEM lane quarter
  uint32_t g = 0;
  for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
    int split, kh, qb;
    item_coords(item, a, split, kh, qb);
    const int lo = split * a.split, hi = min(a.n_view, lo + a.split);
    const int r0 = qb * AT_QR;
    const int nrows = min(AT_QR, a.g * a.t - r0);
    // the item's rows split as evenly as possible between the two groups
    // (t = 5: 3 + 2, not 4 + 1): the softmax of the busier group paces the tile
    const int half = (nrows + 1) >> 1;
    const int rb = grp ? half : 0, re = grp ? nrows : half;   // this group's rows [rb, re)
    const bool active = rb < re;                     // uniform per group
    const int ntiles = (hi - lo + AT_KT - 1) / AT_KT;
    // ---- stage the query split; zero both P buffers (rows >= nrows stay 0) ----------
    // (all S/P.V MMAs of the previous item completed: its tiles were all consumed)
    if (stid < AT_QR) qp_s[stid] = stid < nrows ? pos0 + (r0 + stid) / a.g : -1;
    if (a.qkv == nullptr) {
      for (int e = stid; e < AT_QR * AT_DH; e += 256) {
        const int rr = e >> 7, d = e & 127;
        float v = 0.f;
        if (rr < nrows) {
          const int i = (r0 + rr) / a.g, head = kh * a.g + (r0 + rr) % a.g;
          v = a.q[((size_t)i * a.H + head) * AT_DH + d];
        }
        split3_store(sQ, rr, d, v);
      }
    } else {
      // RoPE of the query pairs (rope_append_kernel's fp64 rotation, model.py:235-244)
      for (int e = stid; e < AT_QR * (AT_DH / 2); e += 256) {
        const int rr = e >> 6, pr = e & 63;
        float y0 = 0.f, y1 = 0.f;
        if (rr < nrows) {
          const int i = (r0 + rr) / a.g, head = kh * a.g + (r0 + rr) % a.g;
          const int p = pos0 + i;
          const float *row = a.qkv + (size_t)i * a.ncols + head * AT_DH + 2 * pr;
          const double ev = (double)row[0], ov = (double)row[1];
          const double cs = (double)a.rope_cos[(size_t)p * (AT_DH / 2) + pr];
          const double sn = (double)a.rope_sin[(size_t)p * (AT_DH / 2) + pr];
          y0 = (float)(ev * cs - ov * sn);
          y1 = (float)(ev * sn + ov * cs);
          if (a.q_stash && split == 0 && i == a.t - 1) {
            a.q_stash[head * AT_DH + 2 * pr] = y0;
            a.q_stash[head * AT_DH + 2 * pr + 1] = y1;
          }
        }
        split3_store(sQ, rr, 2 * pr, y0);
        split3_store(sQ, rr, 2 * pr + 1, y1);
      }
      // this step's K (rotated) and V rows of kv head kh that fall in the item's slots
      if (lo < a.dirty_hi && hi > a.dirty_lo) {
        for (int e = stid; e < a.t * (AT_DH / 2); e += 256) {
          const int i = e >> 6, pr = e & 63;
          const int p = pos0 + i;
          int slot;
          if (a.app_mode == HS_APPEND_POS)
            slot = (p < a.pos_base || (a.own_hi > 0 && p >= a.own_hi)) ? -1 : p - a.pos_base;
          else
            slot = a.app_base + i;
          if (slot < lo || slot >= hi) continue;
          const float *row = a.qkv + (size_t)i * a.ncols;
          const float *kr = row + (a.H + kh) * AT_DH + 2 * pr;
          const double ev = (double)kr[0], ov = (double)kr[1];
          const double cs = (double)a.rope_cos[(size_t)p * (AT_DH / 2) + pr];
          const double sn = (double)a.rope_sin[(size_t)p * (AT_DH / 2) + pr];
          uint16_t *kd = a.k_app + ((size_t)kh * a.cap + slot) * AT_DH + 2 * pr;
          kd[0] = f_to_bf16((float)(ev * cs - ov * sn));
          kd[1] = f_to_bf16((float)(ev * sn + ov * cs));
          const float *vr = row + (a.H + a.KVH + kh) * AT_DH + 2 * pr;
          uint16_t *vd = a.v_app + ((size_t)kh * a.cap + slot) * AT_DH + 2 * pr;
          vd[0] = f_to_bf16(vr[0]);
          vd[1] = f_to_bf16(vr[1]);
          if (a.pos_app && pr == 0) a.pos_app[slot] = p;   // every reader of the slot writes it (same value)
        }
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");   // the TMA reads these rows next
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dready);
    }
    for (int e = stid; e < 2 * AT_OPND / 16; e += 256) reinterpret_cast<uint4 *>(sP)[e] = make_uint4(0, 0, 0, 0);
    tc::fence_async_smem();
    softmax_sync();
    if (lane == 0) tc::mbar_arrive(&qfull);

    float m_run[AT_GR], l_run[AT_GR], o_acc[AT_GR], fac_prev[AT_GR];
#pragma unroll
    for (int r = 0; r < AT_GR; ++r) { m_run[r] = -INFINITY; l_run[r] = 0.f; o_acc[r] = 0.f; fac_prev[r] = 1.f; }

    const int qmin = pos0 + r0 / a.g;   // smallest query position of this block
    for (int it = 0; it <= ntiles; ++it) {
      if (it < ntiles) {
        const uint32_t gi = g + it;
        const int s = gi & 1;
        const uint32_t ph = (gi >> 1) & 1;
        const int key = lo + it * AT_KT + ltid;
        const int kp = key < hi ? (a.pos ? a.pos[key] : key + a.pos_base) : -1;
        tc::mbar_wait(&sfull[s], ph);
        tc::fence_after();
        float sv[3 * AT_GR];
        if (active) {
#pragma unroll
          for (int c = 0; c < 3; ++c) tc::tmem_ld4(tmem + s * 32 + tl + c * AT_QR + rb, sv + c * AT_GR);
          tc::tmem_ld_wait();
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sfree[s]);
        float fac[AT_GR];
#pragma unroll
        for (int r = 0; r < AT_GR; ++r) fac[r] = 1.f;
        if (active) {
          // masked scores and tile max across the 128 keys; a full tile of a
          // linear (full-cache) view entirely below every query needs no mask
          const int tile_last = lo + it * AT_KT + AT_KT - 1;
          const bool allvis = a.pos == nullptr && a.window == 0 && tile_last < hi && tile_last + a.pos_base <= qmin;
          float x[AT_GR];
#pragma unroll
          for (int r = 0; r < AT_GR; ++r) {
            if (rb + r < re) {
              const float sc = ((sv[r] + sv[AT_GR + r]) + sv[2 * AT_GR + r]) * a.scale_log2;
              x[r] = (allvis || visible_tc(kp, qp_s[rb + r], a, win_lo)) ? sc : -INFINITY;
              const int mx = __reduce_max_sync(0xffffffffu, f2o(x[r]));
              if (lane == 0) red[s][warp & 3][rb + r] = mx;
            }
          }
          group_sync(grp);
#pragma unroll
          for (int r = 0; r < AT_GR; ++r) {
            const int rr = rb + r;
            if (rr < re) {
              const int mi = max(max(red[s][0][rr], red[s][1][rr]), max(red[s][2][rr], red[s][3][rr]));
              const float m_new = fmaxf(m_run[r], o2f(mi));
              float p = 0.f;
              if (m_new != -INFINITY) {
                // exp(s - m) in the log2 domain; ex2(-inf) = +0 covers masked keys
                // and the first visible tile (m_run = -inf)
                p = ex2(x[r] - m_new);
                fac[r] = ex2(m_run[r] - m_new);
              }
              m_run[r] = m_new;
              l_run[r] = l_run[r] * fac[r] + p;   // per-thread partial; reduced once per item
              split3_store(sP + s * AT_OPND, rr, ltid, p);
            }
          }
          tc::fence_async_smem();
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&pfull[s]);
        if (it > 0) {   // fold O(it-1) with the previous tile's rescale factor
          const uint32_t gp = gi - 1;
          const int sp = gp & 1;
          tc::mbar_wait(&ofull[sp], (gp >> 1) & 1);
          tc::fence_after();
          float ov[3 * AT_GR];
          if (active) {
#pragma unroll
            for (int c = 0; c < 3; ++c) tc::tmem_ld4(tmem + 64 + sp * 32 + tl + c * AT_QR + rb, ov + c * AT_GR);
            tc::tmem_ld_wait();
          }
          tc::fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&ofree[sp]);
#pragma unroll
          for (int r = 0; r < AT_GR; ++r)
            if (rb + r < re)
              o_acc[r] = o_acc[r] * fac_prev[r] + ((ov[r] + ov[AT_GR + r]) + ov[2 * AT_GR + r]);
        }
#pragma unroll
        for (int r = 0; r < AT_GR; ++r) fac_prev[r] = fac[r];
      } else {        // drain O(last)
        const uint32_t gp = g + ntiles - 1;
        const int sp = gp & 1;
        tc::mbar_wait(&ofull[sp], (gp >> 1) & 1);
        tc::fence_after();
        float ov[3 * AT_GR];
        if (active) {
#pragma unroll
          for (int c = 0; c < 3; ++c) tc::tmem_ld4(tmem + 64 + sp * 32 + tl + c * AT_QR + rb, ov + c * AT_GR);
          tc::tmem_ld_wait();
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&ofree[sp]);
#pragma unroll
        for (int r = 0; r < AT_GR; ++r)
          if (rb + r < re)
            o_acc[r] = o_acc[r] * fac_prev[r] + ((ov[r] + ov[AT_GR + r]) + ov[2 * AT_GR + r]);
      }
    }
    g += ntiles;
    // ---- l: sum of the per-thread partials (fixed order), then write partial state ----
#pragma unroll
    for (int r = 0; r < AT_GR; ++r) {
      if (rb + r < re) {
        float v = l_run[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) redl[warp & 3][rb + r] = v;
      }
    }
    group_sync(grp);
    const size_t pbase = (size_t)split * a.t * a.H;
    // the split states stay in L2 (evict-last) for the combine that follows
    const uint64_t st_pol = tc::policy_evict_last();
#pragma unroll
    for (int r = 0; r < AT_GR; ++r) {
      const int rr = rb + r;
      if (rr < re) {
        const int i = (r0 + rr) / a.g, head = kh * a.g + (r0 + rr) % a.g;
        const size_t row = (size_t)i * a.H + head;
        tc::st_hint_f32(a.part_o + (pbase + row) * AT_DH + ltid, o_acc[r], st_pol);
        if (ltid == 0) {
          // m back to natural-log units
          tc::st_hint_f32(a.part_m + pbase + row, m_run[r] * 0.69314718055994530942f, st_pol);
          tc::st_hint_f32(a.part_l + pbase + row, (redl[0][rr] + redl[1][rr]) + (redl[2][rr] + redl[3][rr]), st_pol);
        }
      }
    }
    softmax_sync();
  }
  tc::fence_before();
  softmax_sync();
  if (warp == 0) tc::tmem_dealloc<128>(tmem);
  HS_TRACE_END(4)
}

}  // namespace

int launch_attention_tc(const HsCache *c, int layer, const HsStep *st, int H, const float *q, int t, float *part_m,
                        float *part_l, float *part_o, int n_splits, cudaStream_t stream, int clean_hi,
                        const FusedRope *fr) {
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
  a.pos_base = st->pos_base;
  a.n_qb = ceil_div(a.g * t, AT_QR);
  a.n_items = n_splits * a.KVH * a.n_qb;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)AT_DH));
  a.part_m = part_m; a.part_l = part_l; a.part_o = part_o;
  a.clean_hi = st->dyn ? -1 : clean_hi;
  // experiment hook (off: measured 3.38 vs 3.28 ms per retrieval forward with it on)
  static const int l2pf = getenv("HS_ATT_L2PF") ? atoi(getenv("HS_ATT_L2PF")) : 0;
  a.l2_prefetch = l2pf && st->split <= 512;   // one item per CTA: its whole split fits the prefetch
  a.dyn = st->dyn;
  a.qkv = nullptr;
  a.dirty_lo = a.dirty_hi = 0;
  if (fr) {
    HS_REQUIRE(st->append_mode == HS_APPEND_POS || st->append_mode == HS_APPEND_LINEAR, HS_ERR_VALUE,
               "attention: fused RoPE needs a position or linear-tail append");
    HS_REQUIRE(st->dyn == nullptr, HS_ERR_VALUE, "attention: fused RoPE needs host positions");
    const size_t lay = (size_t)layer * c->n_kv_heads * c->cap * AT_DH;
    a.qkv = fr->qkv; a.ncols = fr->ncols; a.rope_cos = fr->rope_cos; a.rope_sin = fr->rope_sin;
    a.q_stash = fr->q_stash;
    a.k_app = c->k + lay; a.v_app = c->v + lay;
    a.pos_app = c->kind == HS_KV_SLOTTED ? c->pos + (size_t)layer * c->cap : nullptr;
    a.app_mode = st->append_mode; a.app_base = st->append_base; a.own_hi = st->own_hi;
    if (st->append_mode == HS_APPEND_POS) {
      a.dirty_lo = st->pos0 - st->pos_base;
      a.dirty_hi = a.dirty_lo + t;
    } else {
      a.dirty_lo = st->append_base;
      a.dirty_hi = st->append_base + t;
    }
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
    attr = true;
  }
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = a.n_items < 2 * sms ? a.n_items : 2 * sms;
  cudaError_t e = launch_pdl(attn_tc_kernel, dim3(grid), dim3(AT_THREADS), AT_SMEM, stream, mk, mv, a);
  if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "attention_tc launch: %s", cudaGetErrorString(e));
  return check_launch("attention_tc");
}

}  // namespace hs
