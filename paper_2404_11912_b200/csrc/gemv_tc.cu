// Tensor-core weight-streaming GEMV (tcgen05 + TMA), the projection engine of
// every decode / verify forward (model.py:285, 316, 320-323, 328).
//
// Swap-AB: the weight tile is the MMA's A operand (M = 128 output rows, bf16
// [out][in] = K-major), the activations are B (N = 24 columns).  fp32
// activations are split EXACTLY into three bf16 terms, x = hi + mid + lo
// (round-to-nearest splitting captures 8+8+8 significand bits, the full fp32
// mantissa), laid out as rows [split*8 + r] of a [24][K] bf16 operand; the
// tensor core forms the exact bf16 x bf16 products and accumulates in fp32
// in TMEM, so the result matches an fp32 CUDA-core GEMV to rounding.  The
// epilogue sums the three column groups in a fixed order.
//
// Pipeline per CTA (128 threads): warp 0 issues TMA loads of [128 x 64]
// weight tiles + [24 x 64] activation tiles into a 5-stage ring (the weight
// tiles of the first stages before griddepcontrol.wait), warp 1 issues
// tcgen05.mma (4 x K16 per stage) and tcgen05.commit frees the stage, all four
// warps drain TMEM (tcgen05.ld) in the epilogue.  K is split over gridDim.y
// CTAs (about one CTA per SM, gemv_tc_ksplit); the split CTAs of a tile form a
// thread-block cluster and the split-0 CTA sums their partials over DSMEM in
// split order (deterministic; the split depends only on N and K, never on t,
// so a row's result does not depend on the batch size).
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "gemv_norm.h"
#include "hs_common.cuh"
#include "tc_util.cuh"

namespace hs {

HS_TRACE_TU
int trace_set_gemv(void *p, unsigned cap) { return trace_set_tu(p, cap); }

// per-CTA phase stamps of the GEMV (trace builds only, tools/gemv_phases.py):
// [id: tile | split << 16 | sm << 32 | n_tiles << 48, start, release, first
// stage landed, last stage landed, accumulator complete, reduced/finalised,
// TMEM read, residual loaded, cluster barrier 1, DSMEM partials loaded,
// finalize done, -, -, -, end]  (16 u64)
#ifdef HS_CTA_TRACE
static __device__ unsigned long long *g_gph = nullptr;
static __device__ unsigned int g_gph_n = 0, g_gph_cap = 0;
int trace_set_gemv_phases(void *p, unsigned cap) {
  unsigned long long *q = reinterpret_cast<unsigned long long *>(p);
  unsigned zero = 0;
  if (cudaMemcpyToSymbol(g_gph, &q, sizeof(q)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(g_gph_n, &zero, sizeof(zero)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(g_gph_cap, &cap, sizeof(cap)) != cudaSuccess) return -1;
  return 0;
}
#define GPH_STAMP(slot) if (g_gph != nullptr) gph[slot] = gtime();
#else
int trace_set_gemv_phases(void *, unsigned) { return -1; }
#define GPH_STAMP(slot)
#endif

constexpr int TC_BM = 128;        // output rows per tile (MMA M)
constexpr int TC_BK = 64;         // K per stage (one 128-byte swizzle row)
constexpr int TC_XN = 24;         // activation columns: 3 splits x 8 rows
constexpr int TC_T = 8;           // activation rows per pass
#ifndef HS_TC_STAGES
#define HS_TC_STAGES 5
#endif
constexpr int TC_STAGES = HS_TC_STAGES;   // 5 x 19 KB: two CTAs per SM (a GEMV + the next one's prefetch)
constexpr int TC_W_BYTES = TC_BM * TC_BK * 2;    // 16 KB
constexpr int TC_X_BYTES = TC_XN * TC_BK * 2;    // 3 KB
constexpr int TC_SMEM = TC_STAGES * (TC_W_BYTES + TC_X_BYTES) + 1024 + 256;   // with the worst-case alignment slack
// + the split-0 CTA's landing area for the partials of splits 1..ks-1 (cluster split-K)
constexpr int TC_SMEM_MAX = TC_SMEM + 7 * TC_BM * TC_T * 4;
constexpr int TC_COUNTER_INTS = 16384;           // per-tile arrival counters at the workspace head

// ---------------------------------------------------------------------------
// host: tensor-map cache
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::mutex g_map_mu;
struct MapKey {
  const void *p; uint64_t inner, rows, stride; uint32_t box_rows;
  bool operator==(const MapKey &o) const {
    return p == o.p && inner == o.inner && rows == o.rows && stride == o.stride && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey &k) const {
    return std::hash<const void *>()(k.p) ^ (k.inner * 1315423911u) ^ (k.rows << 7) ^ k.box_rows;
  }
};
static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

int get_tmap_bf16(const void *ptr, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes, uint32_t box_rows,
                  CUtensorMap *out) {
  std::lock_guard<std::mutex> lock(g_map_mu);
  MapKey key{ptr, inner, rows, row_stride_bytes, box_rows};
  auto it = g_maps.find(key);
  if (it != g_maps.end()) { *out = it->second; return HS_OK; }
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return set_error(HS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(HS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps.emplace(key, m);
  *out = m;
  return HS_OK;
}

// ---------------------------------------------------------------------------
// activation prep: optional RMSNorm, then exact 3-way bf16 split

// grid (column blocks of SPLIT_COLS, TC_T rows); rows >= t are written as zeros.
// With a gain, every CTA of a row recomputes the row's sum of squares over
// the whole row (16-byte loads, all in flight at once, fixed reduction order:
// identical in every CTA and independent of t), so the RMSNorm needs no
// second pass and the kernel is one memory round trip deep.
constexpr int SPLIT_THREADS = 256;
constexpr int SPLIT_COLS = 1024;

__global__ void __launch_bounds__(SPLIT_THREADS) split_rows_kernel(const float *x, int ldx, int t, int K, int ldk,
                                                                   const float *gain, float eps, uint16_t *xs) {
  HS_TRACE_BEGIN
  tc::grid_dep_launch();
  tc::grid_dep_wait();
  const int r = blockIdx.y;
  __shared__ double red[SPLIT_THREADS / 32];
  double scale = 1.0;
  const float *xr = x + (size_t)r * ldx;
  if (gain != nullptr && r < t) {
    double ss = 0.0;
    if ((K & 3) == 0 && (ldx & 3) == 0 && ((uintptr_t)x & 15) == 0) {
      const float4 *x4 = reinterpret_cast<const float4 *>(xr);
#pragma unroll 4
      for (int k = threadIdx.x; k < K / 4; k += SPLIT_THREADS) {
        const float4 v = x4[k];
        ss += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
      }
    } else {
      for (int k = threadIdx.x; k < K; k += SPLIT_THREADS) ss += (double)xr[k] * xr[k];
    }
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < SPLIT_THREADS / 32; ++w) tot += red[w];
    scale = sqrt(tot / (double)K + (double)eps);   // rms_norm, model.py:282-284
  }
  const int c0 = blockIdx.x * SPLIT_COLS;
#pragma unroll
  for (int j = 0; j < SPLIT_COLS / SPLIT_THREADS; ++j) {
    const int k = c0 + j * SPLIT_THREADS + threadIdx.x;
    if (k >= ldk) break;
    float h = 0.f;
    if (r < t && k < K) {
      const float v = xr[k];
      h = gain ? (float)(((double)v / scale) * (double)gain[k]) : v;
    }
    uint16_t a, b, c;
    split3(h, a, b, c);
    xs[(size_t)r * ldk + k] = a;
    xs[(size_t)(TC_T + r) * ldk + k] = b;
    xs[(size_t)(2 * TC_T + r) * ldk + k] = c;
  }
  HS_TRACE_END(2)
}

// Folded-RMSNorm operand prep for rows [0, t) of x: split(fp32(x * gain))
// into xs [24][ldk] -- the operand the residual GEMV epilogue writes in the
// single-block forward (its consumer computes the RMS itself, gemv_rms).
// grid (tiles of 128 columns, t), 128 threads.
__global__ void __launch_bounds__(128) norm_prep_kernel(const float *x, int ldx, int K, const float *gain,
                                                        uint16_t *xs, int ldk) {
  HS_TRACE_BEGIN
  const int r = blockIdx.y, col = blockIdx.x * 128 + threadIdx.x;
  if (col < K) store_split(xs, ldk, r, col, __fmul_rn(x[(size_t)r * ldx + col], gain[col]));
  HS_TRACE_END(3)
}

int launch_norm_prep(const float *x, int ldx, int t, int K, const float *gain, uint16_t *xs, int ldk,
                     cudaStream_t st) {
  HS_REQUIRE(t >= 1 && t <= TC_T, HS_ERR_SHAPE, "norm_prep: t=%d outside [1,%d]", t, TC_T);
  norm_prep_kernel<<<dim3((K + 127) / 128, t), 128, 0, st>>>(x, ldx, K, gain, xs, ldk);
  return check_launch("norm_prep");
}

struct GemvTcArgs {
  int N, nkb, ks, t, epilogue, n_tiles;
  int cluster;        // 1: the ks split CTAs of a tile are one cluster, partials reduced through DSMEM
  int push;           // cluster reduction by pushes into the split-0 CTA (its landing area fits two CTAs per SM)
  int nrow;           // pushed floats per row (4 when t <= 4, else 8)
  // folded RMSNorm (model.py:282-284) of this GEMV's input rows: the operand
  // is split(x * gain) and the result is scaled by 1 / rms(x) here, the RMS
  // computed from the un-normalised rows x_in [t][ldx_in] (gemv_rms)
  const float *x_in;
  int ldx_in, norm_K;
  float eps;
  // residual producer (epilogue 1): also write the next GEMV's operand
  // split(x_new * gnext)
  const float *gnext;
  uint16_t *xs_next;
  int ld_next;
  float *y;
  int ldy;
  // residual source of epilogue 1 (null: y itself, updated in place); the
  // tensor-parallel forward reads x[:, block] and writes the block to a send
  // buffer
  const float *yin;
  int ldyin;
  uint16_t *xs_out;   // swiglu epilogue: split of act written here ([24][ld_xs_out]) if non-null
  int ld_xs_out;
  float *partial;     // [ks][n_tiles*128][8]
  int *counters;      // [n_tiles]
  int trig_late;      // signal programmatic launch completion after the last weight load is issued
  int blocked;        // weights stored tile-blocked [N/128][K/64][128][64] (HsModel.blocked)
  int l2pf;           // experiment hook: weight tiles past the ring prefetched to L2 before the dependency wait
  int *align_probe;   // non-null: thread 0 reports the dynamic shared memory's misalignment and the CTA exits
  int keep_l2;        // weights loaded evict-last (a small model re-read every step) instead of evict-first
};

// all 128 threads of the CTA call finalize (uniform control flow: the residual
// producer reduces its tile's row sums of squares across the CTA)
// yres: the residual rows y[r][o] (epilogue 1), loaded by the caller ahead of
// the split-K handshake so they are not one more round trip on the tail
template <int EPI>
__device__ __forceinline__ void finalize(const GemvTcArgs &a, int o, const float *vin, const float *yres, float gn,
                                         int lane, int tile, const double *inv_rms, double (*red)[TC_T],
                                         unsigned long long *gst) {
  float v[TC_T];
#pragma unroll
  for (int r = 0; r < TC_T; ++r) v[r] = a.x_in ? (float)((double)vin[r] * inv_rms[r]) : vin[r];
  if constexpr (EPI == 2) {
    float up[TC_T];
#pragma unroll
    for (int r = 0; r < TC_T; ++r) up[r] = __shfl_down_sync(0xffffffffu, v[r], 1);
    if ((o & 1) == 0 && o + 1 < a.N) {
      const int i = o >> 1;
#pragma unroll
      for (int r = 0; r < TC_T; ++r) {
        if (r < a.t) {
          const double g = (double)v[r];
          const float act = (float)(g * (0.5 * (tanh(0.5 * g) + 1.0))) * up[r];   // model.py:321-322
          if (a.y) a.y[(size_t)r * a.ldy + i] = act;
          if (a.xs_out) store_split(a.xs_out, a.ld_xs_out, r, i, act);
        }
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < TC_T; ++r) {
      if (r < a.t && o < a.N) {
        const float nv = (EPI == 1) ? (yres[r] + v[r]) : v[r];
        a.y[(size_t)r * a.ldy + o] = nv;
        // the exact product of two floats fits a double, so the fp32 product
        // (one rounding) equals the reference's (float)((double)x * (double)g)
        if (a.xs_next) store_split(a.xs_next, a.ld_next, r, o, __fmul_rn(nv, gn));
      }
    }
#ifdef HS_CTA_TRACE
    if (gst && threadIdx.x == 0) gst[12] = gtime();
#endif
  }
  (void)lane; (void)tile; (void)red;
}

// 1 / sqrt(mean(x^2) + eps) of rows [0, t) of x (model.py:282-284), computed
// by the 64 threads of warps 2-3 while the main loop streams the weights:
// thread j sums float4 columns 4j + 256i in fp64, then the two warps' xor
// trees, warp 2 + warp 3.  Every consumer of a row (and every path: single
// block, multi-block, tensor-parallel) sums in this same order.
__device__ __forceinline__ double sq4(const float4 v) {
  return (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
}
__device__ __forceinline__ void gemv_rms(const GemvTcArgs &a, int j, double *inv_rms, double (*red)[TC_T]) {
  const int lane = j & 31, w = j >> 5;
  const int K4 = a.norm_K & ~3;
  // rows in pairs (more loads in flight for the longer verify batches); every
  // row accumulates its chunks in the same order either way
  for (int r = 0; r < a.t; r += 2) {
    const bool two = r + 1 < a.t;
    const float *x0 = a.x_in + (size_t)r * a.ldx_in, *x1 = x0 + a.ldx_in;
    double s0 = 0.0, s1 = 0.0;
    for (int c = 4 * j; c < K4; c += 256) {
      const float4 v0 = __ldcg(reinterpret_cast<const float4 *>(x0 + c));
      const float4 v1 = two ? __ldcg(reinterpret_cast<const float4 *>(x1 + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      s0 += sq4(v0);
      s1 += sq4(v1);
    }
    for (int c = K4 + j; c < a.norm_K; c += 64) {
      const float u0 = __ldcg(x0 + c), u1 = two ? __ldcg(x1 + c) : 0.f;
      s0 += (double)u0 * u0;
      s1 += (double)u1 * u1;
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (lane == 0) {
      red[w][r] = s0;
      if (two) red[w][r + 1] = s1;
    }
  }
  asm volatile("bar.sync 3, 64;" ::: "memory");
  if (j < a.t) inv_rms[j] = 1.0 / sqrt((red[0][j] + red[1][j]) / (double)a.norm_K + (double)a.eps);
}

// EPI: 0 store (optionally scaled by the folded RMSNorm), 1 residual
// accumulate (+ next operand and row statistics), 2 SwiGLU -- one
// instantiation per epilogue keeps each kernel's code (and its instruction
// cache footprint on the tail) small
template <int EPI>
__global__ void __launch_bounds__(128, 2) gemv_tc_kernel(const __grid_constant__ CUtensorMap tmW,
                                                         const __grid_constant__ CUtensorMap tmX, GemvTcArgs a) {
  HS_TRACE_BEGIN
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  if (a.align_probe) {
    if (threadIdx.x == 0) *a.align_probe = (int)(reinterpret_cast<uintptr_t>(smem_raw) & 1023);
    return;
  }
  unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *sW = base;
  unsigned char *sX = base + TC_STAGES * TC_W_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(sX + TC_STAGES * TC_X_BYTES);
  uint64_t *empty = full + TC_STAGES;
  uint64_t *accum = empty + TC_STAGES;
  uint64_t *redbar = accum + 1;   // split-0 CTA: the other splits' pushed partials have landed
  uint32_t *tmem_base = reinterpret_cast<uint32_t *>(redbar + 1);
  int *flag = reinterpret_cast<int *>(tmem_base + 1);
  // split-0 CTA of a cluster: partials pushed by splits 1..ks-1, [ks-1][128][nrow] fp32
  float *pushed = reinterpret_cast<float *>(base + TC_STAGES * (TC_W_BYTES + TC_X_BYTES) + 256);
#ifdef HS_CTA_TRACE
  __shared__ unsigned long long gph[16];
  if (threadIdx.x == 0 && g_gph != nullptr) {
    for (int j = 0; j < 16; ++j) gph[j] = 0;
    gph[1] = gtime();
  }
#endif

  if (!a.trig_late) tc::grid_dep_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int per = a.nkb / a.ks, rem = a.nkb % a.ks;
  const int kb0 = split * per + min(split, rem);
  const int nk = per + (split < rem ? 1 : 0);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmW);
    tc::tma_prefetch(&tmX);
    for (int s = 0; s < TC_STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    tc::mbar_init(accum, 1);
    tc::mbar_init(redbar, 1);
    tc::fence_mbar_init();
    // split-0 CTA: the pushed partials arrive as transaction bytes
    if (a.cluster && a.push && split == 0) tc::mbar_expect_tx(redbar, (a.ks - 1) * TC_BM * a.nrow * 4);
  }
  if (warp == 1) tc::tmem_alloc<32>(tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t taddr = *tmem_base;
  // the split CTAs push into the split-0 CTA's shared memory at the end: its
  // reduction barrier must be initialised cluster-wide first (waited below)
  if (a.cluster && a.push) tc::cluster_arrive_relaxed();

  if (warp == 0) {
    if (tc::elect_one()) {
      // Programmatic dependent launch: the weights never depend on the
      // previous kernel, so the first stages' weight tiles stream in while
      // that kernel drains; only the activation tiles wait for it.
      // large models' weights are streamed exactly once per forward (evict-first);
      // a small model's (the draft) stay in L2 between its steps
      const uint64_t pol = a.keep_l2 ? tc::policy_evict_last() : tc::policy_evict_first();
      const int npre = nk < TC_STAGES ? nk : TC_STAGES;
      for (int i = 0; i < npre; ++i) {
        tc::mbar_expect_tx(&full[i], TC_W_BYTES + TC_X_BYTES);
        if (a.blocked) tc::tma_load_2d_hint(sW + i * TC_W_BYTES, &tmW, &full[i], 0, (tile * a.nkb + kb0 + i) * TC_BM, pol);
        else tc::tma_load_2d_hint(sW + i * TC_W_BYTES, &tmW, &full[i], (kb0 + i) * TC_BK, tile * TC_BM, pol);
      }
      for (int i = npre; i < nk && i < npre + a.l2pf; ++i)   // experiment hook (HS_GEMV_L2PF)
        tc::tma_prefetch_l2_2d(&tmW, (kb0 + i) * TC_BK, tile * TC_BM);
      tc::grid_dep_wait();
      HS_TRACE_RESTART
      GPH_STAMP(2)
      for (int i = 0; i < npre; ++i) tc::tma_load_2d(sX + i * TC_X_BYTES, &tmX, &full[i], (kb0 + i) * TC_BK, 0);
      for (int i = npre; i < nk; ++i) {
        const int s = i % TC_STAGES;
        const uint32_t ph = (i / TC_STAGES) & 1;
        tc::mbar_wait(&empty[s], ph ^ 1);
        tc::mbar_expect_tx(&full[s], TC_W_BYTES + TC_X_BYTES);
        const int k = (kb0 + i) * TC_BK;
        if (a.blocked) tc::tma_load_2d_hint(sW + s * TC_W_BYTES, &tmW, &full[s], 0, (tile * a.nkb + kb0 + i) * TC_BM, pol);
        else tc::tma_load_2d_hint(sW + s * TC_W_BYTES, &tmW, &full[s], k, tile * TC_BM, pol);
        tc::tma_load_2d(sX + s * TC_X_BYTES, &tmX, &full[s], k, 0);
      }
      if (a.trig_late) tc::grid_dep_launch();
    } else {
      tc::grid_dep_wait();
      HS_TRACE_RESTART
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      constexpr uint32_t idesc = tc::idesc_bf16(TC_BM, TC_XN, 0, 0);
      for (int i = 0; i < nk; ++i) {
        const int s = i % TC_STAGES;
        const uint32_t ph = (i / TC_STAGES) & 1;
        tc::mbar_wait(&full[s], ph);
        tc::fence_after();
#ifdef HS_CTA_TRACE
        if (i == 0) GPH_STAMP(3)
        if (i == nk - 1) GPH_STAMP(4)
#endif
        const uint64_t da = tc::desc_k_sw128(sW + s * TC_W_BYTES);
        const uint64_t db = tc::desc_k_sw128(sX + s * TC_X_BYTES);
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; ++kk)   // +32 bytes per K16 step inside the swizzle row
          tc::mma_bf16(taddr, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(accum);
    }
  }
  if (warp != 0) tc::grid_dep_wait();   // epilogue reads y written by earlier kernels
  __syncwarp();
  __shared__ double inv_rms[TC_T];
  __shared__ double red[4][TC_T];
  if (a.x_in && warp >= 2) gemv_rms(a, threadIdx.x - 64, inv_rms, red);   // folded RMSNorm of the input rows
  const int row = warp * 32 + lane;
  const int o = tile * TC_BM + row;
  // operands of the epilogue that do not depend on the accumulator (residual
  // rows, next norm's gain) are loaded while the main loop still runs, so
  // they are not a memory round trip on the tail; only the finalising CTA
  // of a cluster needs them
  const bool fin_cta = a.ks == 1 || !a.cluster || split == 0;
  float yres[TC_T];
#pragma unroll
  for (int r = 0; r < TC_T; ++r)
    yres[r] = (fin_cta && EPI == 1 && r < a.t && o < a.N)
                  ? __ldcg(a.yin ? a.yin + (size_t)r * a.ldyin + o : a.y + (size_t)r * a.ldy + o)
                  : 0.f;
  const float gn = (fin_cta && EPI == 1 && a.xs_next && o < a.N) ? __ldg(a.gnext + o) : 0.f;

  // ---- epilogue: TMEM -> registers ---------------------------------------------------
  tc::mbar_wait(accum, 0);
  tc::fence_after();
  if (a.trig_late) tc::grid_dep_launch();
#ifdef HS_CTA_TRACE
  if (threadIdx.x == 0) GPH_STAMP(5)
#endif
  __syncthreads();   // inv_rms visible
  const uint32_t tl = taddr + ((uint32_t)(warp * 32) << 16);
  float h[8], m[8], l[8], v[TC_T];
  tc::tmem_ld8(tl + 0, h);
  tc::tmem_ld8(tl + 8, m);
  tc::tmem_ld8(tl + 16, l);
  tc::tmem_ld_wait();
#ifdef HS_CTA_TRACE
  if (threadIdx.x == 0) GPH_STAMP(7)
#endif
#pragma unroll
  for (int r = 0; r < TC_T; ++r) v[r] = nk > 0 ? (h[r] + m[r]) + l[r] : 0.f;
#ifdef HS_CTA_TRACE
  if (threadIdx.x == 0 && g_gph != nullptr) {
    float sy = 0.f;
    for (int r = 0; r < TC_T; ++r) sy += yres[r];
    if (sy == -1.2345e-30f) gph[0] = 1;
    GPH_STAMP(8)
  }
#endif

  // split-K reduction into acc (split order, the finalising CTA's own
  // partial first), then ONE finalize call site for every reduction mode
  float acc[TC_T];
  bool do_fin = true;   // CTA-uniform
  if (a.ks == 1) {
#pragma unroll
    for (int r = 0; r < TC_T; ++r) acc[r] = v[r];
  } else if (a.cluster && a.push) {
    // push style: splits 1..ks-1 store their partial rows straight into the
    // split-0 CTA's shared memory with st.async, each store completing its
    // transaction bytes on the split-0 CTA's reduction barrier, then exit
    // without waiting; the split-0 CTA waits for all bytes and sums locally
    tc::cluster_wait();   // the split-0 CTA's barrier is initialised
#ifdef HS_CTA_TRACE
    if (threadIdx.x == 0) GPH_STAMP(9)
#endif
    const int nrow = a.nrow;   // rows >= t are zero
    if (split != 0) {
      float *dst = pushed + ((size_t)(split - 1) * TC_BM + row) * nrow;
      const uint32_t ra = tc::mapa_u32(dst, 0), rb = tc::mapa_u32(redbar, 0);
      tc::st_async_f4(ra, make_float4(v[0], v[1], v[2], v[3]), rb);
      if (nrow > 4) tc::st_async_f4(ra + 16, make_float4(v[4], v[5], v[6], v[7]), rb);
      do_fin = false;
    } else {
      tc::mbar_wait_cluster(redbar, 0);
#pragma unroll
      for (int r = 0; r < TC_T; ++r) acc[r] = 0.f + v[r];
      for (int s2 = 1; s2 < a.ks; ++s2) {
        const float *src = pushed + ((size_t)(s2 - 1) * TC_BM + row) * nrow;
        const float4 x0 = *reinterpret_cast<const float4 *>(src);
        acc[0] += x0.x; acc[1] += x0.y; acc[2] += x0.z; acc[3] += x0.w;
        if (nrow > 4) {
          const float4 x1 = *reinterpret_cast<const float4 *>(src + 4);
          acc[4] += x1.x; acc[5] += x1.y; acc[6] += x1.z; acc[7] += x1.w;
        }
      }
#ifdef HS_CTA_TRACE
      if (threadIdx.x == 0) GPH_STAMP(10)
#endif
    }
  } else if (a.cluster) {
    // pull style (the landing area would not fit): every CTA parks its
    // partial in its idle stage buffers, the split-0 CTA reads them over
    // DSMEM between two cluster barriers
    float *ps = reinterpret_cast<float *>(sW) + row * TC_T;
    *reinterpret_cast<float4 *>(ps) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4 *>(ps + 4) = make_float4(v[4], v[5], v[6], v[7]);
    tc::cluster_sync();
    do_fin = split == 0;
    if (do_fin) {
#pragma unroll
      for (int r = 0; r < TC_T; ++r) acc[r] = 0.f;
      float4 x0[8], x1[8];   // all splits' partials in flight at once
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        if (s2 < a.ks) {
          x0[s2] = tc::ld_dsmem_f4(ps, s2);
          x1[s2] = tc::ld_dsmem_f4(ps + 4, s2);
        }
      }
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        if (s2 < a.ks) {
          acc[0] += x0[s2].x; acc[1] += x0[s2].y; acc[2] += x0[s2].z; acc[3] += x0[s2].w;
          acc[4] += x1[s2].x; acc[5] += x1[s2].y; acc[6] += x1[s2].z; acc[7] += x1[s2].w;
        }
      }
    }
  } else {
    // global partials + arrival counter (> 8 splits, or clusters disabled)
    float *pp = a.partial + ((size_t)split * a.n_tiles * TC_BM + o) * TC_T;
    *reinterpret_cast<float4 *>(pp) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4 *>(pp + 4) = make_float4(v[4], v[5], v[6], v[7]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int old = atomicAdd(&a.counters[tile], 1);
      *flag = (old == a.ks - 1);
    }
    __syncthreads();
    do_fin = *flag != 0;
    if (do_fin) {
      __threadfence();
#pragma unroll
      for (int r = 0; r < TC_T; ++r) acc[r] = 0.f;
      constexpr int KS_MAX = 16;   // all split partials in flight at once, then summed in split order
      float4 x0[KS_MAX], x1[KS_MAX];
#pragma unroll
      for (int s2 = 0; s2 < KS_MAX; ++s2) {
        if (s2 < a.ks) {
          const float *q = a.partial + ((size_t)s2 * a.n_tiles * TC_BM + o) * TC_T;
          x0[s2] = __ldcg(reinterpret_cast<const float4 *>(q));
          x1[s2] = __ldcg(reinterpret_cast<const float4 *>(q + 4));
        }
      }
#pragma unroll
      for (int s2 = 0; s2 < KS_MAX; ++s2) {
        if (s2 < a.ks) {
          acc[0] += x0[s2].x; acc[1] += x0[s2].y; acc[2] += x0[s2].z; acc[3] += x0[s2].w;
          acc[4] += x1[s2].x; acc[5] += x1[s2].y; acc[6] += x1[s2].z; acc[7] += x1[s2].w;
        }
      }
      if (threadIdx.x == 0) a.counters[tile] = 0;   // self-cleaning for the next launch
    }
  }
  if (do_fin) {
#ifdef HS_CTA_TRACE
    finalize<EPI>(a, o, acc, yres, gn, lane, tile, inv_rms, red, g_gph ? gph : nullptr);
#else
    finalize<EPI>(a, o, acc, yres, gn, lane, tile, inv_rms, red, nullptr);
#endif
#ifdef HS_CTA_TRACE
    if (threadIdx.x == 0) GPH_STAMP(11)
#ifdef HS_GEMV_FIN_TWICE
    // experiment: the same (idempotent) finalize again -- warm caches
    __syncthreads();
    if (threadIdx.x == 0 && g_gph != nullptr) gph[3] = gtime();
    finalize<EPI>(a, o, acc, yres, gn, lane, tile, inv_rms, red, nullptr);
    if (threadIdx.x == 0 && g_gph != nullptr) gph[4] = gtime();
#endif
#endif
  }
  if (a.cluster && !a.push) tc::cluster_sync();   // pull style: partials stay readable until the leader is done
#ifdef HS_CTA_TRACE
  if (threadIdx.x == 0) GPH_STAMP(6)
#endif
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<32>(taddr);
#ifdef HS_CTA_TRACE
  if (threadIdx.x == 0 && g_gph != nullptr) {
    const unsigned i_ = atomicAdd(&g_gph_n, 1u);
    if (i_ < g_gph_cap) {
      unsigned sm_;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));
      unsigned long long *o = g_gph + (size_t)i_ * 16;
      o[0] = (unsigned long long)tile | ((unsigned long long)split << 16) | ((unsigned long long)sm_ << 32) |
             ((unsigned long long)a.n_tiles << 48);
      for (int j = 1; j < 15; ++j) o[j] = gph[j];
      o[15] = gtime();
    }
  }
#endif
  HS_TRACE_END(1 | (a.n_tiles << 8))
}

// K split: a function of (N, K) only.  About one CTA per SM: the smallest
// split that gives every SM a CTA (at most one wave of 2 per SM, >= 4
// K-blocks per CTA).  Measured (tools/fwdbench.py, Llama2-7B shapes): long
// weight streams per CTA beat wave-filling splits -- gate|up as 172 whole-K
// CTAs runs the retrieval forward 8% faster than as 860 CTAs in 2.9 waves,
// and more, shorter CTAs lose monotonically.
// split-K reduction through a thread-block cluster (default; HS_GEMV_NO_CLUSTER=1
// uses the global-memory partials + arrival counter path for every split)
static int gemv_use_cluster() {
  static const int on = [] {
    const char *e = getenv("HS_GEMV_NO_CLUSTER");
    return !(e != nullptr && e[0] == '1');
  }();
  return on;
}

// alignment slack the ring needs: 0 when the kernel's dynamic shared memory
// already starts 1024-byte aligned (probed once per process on every
// instantiation, outside stream capture), else 1024
template <int EPI>
__global__ void __launch_bounds__(128, 2) gemv_tc_kernel(const __grid_constant__ CUtensorMap tmW,
                                                         const __grid_constant__ CUtensorMap tmX, GemvTcArgs a);
static int gemv_smem_slack(cudaStream_t st) {
  static int slack = -1;
  if (slack >= 0) return slack;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return 1024;
  int *d = nullptr, h[3] = {1, 1, 1};
  if (cudaMalloc(&d, sizeof(int) * 3) != cudaSuccess) { slack = 1024; return slack; }
  CUtensorMap m;
  memset(&m, 0, sizeof(m));
  void (*kerns[3])(const CUtensorMap, const CUtensorMap, GemvTcArgs) = {gemv_tc_kernel<0>, gemv_tc_kernel<1>,
                                                                          gemv_tc_kernel<2>};
  for (int k = 0; k < 3; ++k) {
    GemvTcArgs a;
    memset(&a, 0, sizeof(a));
    a.align_probe = d + k;
    kerns[k]<<<1, 128, TC_SMEM, st>>>(m, m, a);
  }
  cudaMemcpyAsync(h, d, sizeof(int) * 3, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(d);
  slack = (h[0] == 0 && h[1] == 0 && h[2] == 0) ? 0 : 1024;
  if (getenv("HS_GEMV_DEBUG")) fprintf(stderr, "gemv_tc: dynamic smem misalignment %d %d %d -> slack %d\n", h[0], h[1], h[2], slack);
  return slack;
}

// dynamic shared memory one GEMV CTA may use while two fit per SM (a GEMV
// and its programmatic dependent's prefetching CTA)
static int gemv_smem_budget() {
  static const int b = [] {
    int dev = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, gemv_tc_kernel<1>) != cudaSuccess) return TC_SMEM;
    const int reserved = 1024;   // per-CTA system reservation
    const int r = per_sm / 2 - reserved - (int)fa.sharedSizeBytes;
    if (getenv("HS_GEMV_DEBUG")) fprintf(stderr, "gemv_tc: smem budget %d (per SM %d, static %zu)\n", r, per_sm, fa.sharedSizeBytes);
    return r;
  }();
  return b;
}

int gemv_tc_ksplit(int N, int nkb) {
  const int tiles = (N + TC_BM - 1) / TC_BM;
  if (const char *e = getenv("HS_GEMV_KS")) {   // experiment hook: "N/nkb:ks,..."
    for (const char *q = e; *q;) {
      const int n = atoi(q);
      const char *sl = strchr(q, '/');
      const char *c = strchr(q, ':');
      if (!c || !sl) break;
      if (n == N && atoi(sl + 1) == nkb) return atoi(c + 1);
      const char *nx = strchr(c, ',');
      if (!nx) break;
      q = nx + 1;
    }
  }
  constexpr int SMS = 148;
  int ks = (SMS + tiles - 1) / tiles;
  const int cap = nkb / 4 < 8 ? nkb / 4 : 8;   // <= 8: the split CTAs of a tile fit one (portable) cluster
  if (ks > cap) ks = cap;
  return ks < 1 ? 1 : ks;
}

size_t gemv_tc_ws_bytes(int N, int nkb) {
  const int tiles = (N + TC_BM - 1) / TC_BM;
  const int ks = gemv_tc_ksplit(N, nkb);
  return (size_t)TC_COUNTER_INTS * 4 + (ks > 1 ? (size_t)ks * tiles * TC_BM * TC_T * 4 : 0);
}

int launch_split_rows(const float *x, int ldx, int t, int K, int ldk, const float *gain, float eps, uint16_t *xs,
                      cudaStream_t st) {
  HS_REQUIRE(t >= 1 && t <= TC_T, HS_ERR_SHAPE, "split_rows: t=%d outside [1,%d]", t, TC_T);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((ldk + SPLIT_COLS - 1) / SPLIT_COLS, TC_T, 1);
  cfg.blockDim = dim3(SPLIT_THREADS, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled();
  cudaError_t e = cudaLaunchKernelEx(&cfg, split_rows_kernel, x, ldx, t, K, ldk, gain, eps, xs);
  if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "split_rows launch: %s", cudaGetErrorString(e));
  return check_launch("split_rows");
}

// L2 policy of the weight tiles for the GEMVs this host thread launches next
// (set per forward: forward.cu)
static thread_local int g_gemv_keep_l2 = 0;
void gemv_set_keep_l2(int keep) { g_gemv_keep_l2 = keep; }

// y (+)= W . x for one pass of <= 8 rows whose split operand is in xs [24][ldw]
int launch_gemv_tc(const uint16_t *xs, int t, const uint16_t *w, int ldw, int N, int epilogue, float *y, int ldy,
                   uint16_t *xs_out, int ld_xs_out, void *ws, size_t ws_bytes, cudaStream_t st,
                   const GemvNorm *norm, const float *yin, int ldyin, int blocked) {
  HS_REQUIRE(t >= 1 && t <= TC_T, HS_ERR_SHAPE, "gemv_tc: t=%d outside [1,%d]", t, TC_T);
  HS_REQUIRE(ldw % TC_BK == 0, HS_ERR_SHAPE, "gemv_tc: ldw %d not a multiple of %d", ldw, TC_BK);
  HS_REQUIRE(((uintptr_t)w % 16) == 0 && ((uintptr_t)xs % 16) == 0, HS_ERR_VALUE, "gemv_tc: operands must be 16B aligned");
  HS_REQUIRE(epilogue >= 0 && epilogue <= 2, HS_ERR_VALUE, "gemv_tc: epilogue %d not in {0, 1, 2}", epilogue);
  HS_REQUIRE(epilogue != 2 || N % 2 == 0, HS_ERR_SHAPE, "gemv_tc: swiglu needs an even N");
  const int nkb = ldw / TC_BK;
  const int tiles = (N + TC_BM - 1) / TC_BM;
  HS_REQUIRE(tiles <= TC_COUNTER_INTS, HS_ERR_SHAPE, "gemv_tc: N too large");
  HS_REQUIRE(ws_bytes >= gemv_tc_ws_bytes(N, nkb), HS_ERR_VALUE, "gemv_tc: workspace too small");
  CUtensorMap mw, mx;
  HS_REQUIRE(!blocked || N % TC_BM == 0, HS_ERR_SHAPE, "gemv_tc: a blocked matrix needs N %% 128 == 0 (N %d)", N);
  const bool blk = blocked != 0;
  int rc = blk ? get_tmap_bf16(w, (uint64_t)TC_BK, (uint64_t)N * nkb, (uint64_t)TC_BK * 2, TC_BM, &mw)
               : get_tmap_bf16(w, (uint64_t)ldw, (uint64_t)N, (uint64_t)ldw * 2, TC_BM, &mw);
  if (rc != HS_OK) return rc;
  rc = get_tmap_bf16(xs, (uint64_t)ldw, (uint64_t)TC_XN, (uint64_t)ldw * 2, TC_XN, &mx);
  if (rc != HS_OK) return rc;
  GemvTcArgs a;
  a.N = N; a.nkb = nkb; a.ks = gemv_tc_ksplit(N, nkb); a.t = t; a.epilogue = epilogue; a.n_tiles = tiles;
  a.blocked = blk ? 1 : 0;
  a.cluster = (a.ks > 1 && a.ks <= 8 && gemv_use_cluster()) ? 1 : 0;
  static const int push_mode = getenv("HS_GEMV_PUSH") ? atoi(getenv("HS_GEMV_PUSH")) : 1;   // A/B hook
  a.nrow = (t <= 4 && push_mode != 2) ? 4 : TC_T;
  const int land = a.cluster ? (a.ks - 1) * TC_BM * a.nrow * 4 : 0;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemv_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_MAX);
    cudaFuncSetAttribute(gemv_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_MAX);
    cudaFuncSetAttribute(gemv_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_MAX);
    attr_set = true;
  }
  const int smem_base = TC_SMEM - 1024 + gemv_smem_slack(st);
  a.push = (a.cluster && push_mode && (push_mode == 2 || smem_base + land <= gemv_smem_budget())) ? 1 : 0;
  a.y = y; a.ldy = ldy; a.xs_out = xs_out; a.ld_xs_out = ld_xs_out;
  a.yin = yin; a.ldyin = ldyin;
  a.x_in = nullptr; a.ldx_in = 0; a.norm_K = 1; a.eps = 0.f;
  a.gnext = nullptr; a.xs_next = nullptr; a.ld_next = 0;
  if (norm) {
    a.x_in = norm->x_in; a.ldx_in = norm->ldx_in; a.norm_K = norm->norm_K; a.eps = norm->eps;
    a.gnext = norm->gnext; a.xs_next = norm->xs_next; a.ld_next = norm->ld_next;
    HS_REQUIRE(a.x_in == nullptr || ((uintptr_t)a.x_in % 16 == 0 && a.ldx_in % 4 == 0), HS_ERR_VALUE,
               "gemv_tc: norm input rows must be 16-byte aligned");
    HS_REQUIRE(a.xs_next == nullptr || epilogue == 1, HS_ERR_VALUE, "gemv_tc: next-operand output needs epilogue 1");
  }
  // programmatic launch completion once the weight stream is issued (the
  // dependent's CTAs then start together; HS_GEMV_TRIG=0: at CTA start)
  static const int trig_late = getenv("HS_GEMV_TRIG") ? atoi(getenv("HS_GEMV_TRIG")) : 1;
  a.trig_late = trig_late;
  a.align_probe = nullptr;
  a.keep_l2 = g_gemv_keep_l2;
  static const int l2pf = getenv("HS_GEMV_L2PF") ? atoi(getenv("HS_GEMV_L2PF")) : 0;
  a.l2pf = l2pf;
  a.counters = reinterpret_cast<int *>(ws);
  a.partial = reinterpret_cast<float *>(reinterpret_cast<char *>(ws) + (size_t)TC_COUNTER_INTS * 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles, a.ks, 1);
  cfg.blockDim = dim3(128, 1, 1);
  cfg.dynamicSmemBytes = smem_base + (a.push ? land : 0);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (a.cluster) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = a.ks;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  auto kern = epilogue == 2 ? gemv_tc_kernel<2> : epilogue == 1 ? gemv_tc_kernel<1> : gemv_tc_kernel<0>;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mw, mx, a);
  if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "gemv_tc launch: %s", cudaGetErrorString(e));
  return check_launch("gemv_tc");
}

// row-major [N][ld] <-> tile-blocked [N/128][ld/64][128][64] (one 16-byte
// unit per thread; dst index space)
__global__ void relayout_blocked_kernel(const uint16_t *src, uint16_t *dst, int N, int ld, int inverse) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nkb = ld / 64;
  const size_t total = (size_t)N * ld / 8;
  if (i >= total) return;
  const size_t e = i * 8;   // element of the blocked layout
  const int c = (int)(e % 64);
  const size_t r_in_tile = (e / 64) % 128;
  const size_t kb = (e / (64 * 128)) % nkb;
  const size_t tile = e / ((size_t)64 * 128 * nkb);
  const size_t rm = (tile * 128 + r_in_tile) * ld + kb * 64 + c;   // element of the row-major layout
  if (inverse) *reinterpret_cast<uint4 *>(dst + rm) = *reinterpret_cast<const uint4 *>(src + e);
  else *reinterpret_cast<uint4 *>(dst + e) = *reinterpret_cast<const uint4 *>(src + rm);
}

}  // namespace hs

extern "C" int hs_weights_block(uint16_t *w, uint16_t *tmp, int N, int ld, int inverse, void *stream) {
  HS_REQUIRE(N % 128 == 0 && ld % 64 == 0 && N > 0, HS_ERR_SHAPE, "weights_block: N %d / ld %d", N, ld);
  const size_t units = (size_t)N * ld / 8;
  cudaStream_t st = hs::as_stream(stream);
  cudaError_t e = cudaMemcpyAsync(tmp, w, (size_t)N * ld * 2, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return hs::set_error(HS_ERR_CUDA, "weights_block: %s", cudaGetErrorString(e));
  hs::relayout_blocked_kernel<<<(unsigned)((units + 255) / 256), 256, 0, st>>>(tmp, w, N, ld, inverse);
  return hs::check_launch("weights_block");
}

extern "C" size_t hs_gemv_tc_workspace_bytes(int N, int ldw) { return hs::gemv_tc_ws_bytes(N, ldw / hs::TC_BK); }

extern "C" int hs_split_rows(const float *x, int ldx, int t, int K, int ldk, const float *gain, float eps,
                             uint16_t *xs, void *stream) {
  return hs::launch_split_rows(x, ldx, t, K, ldk, gain, eps, xs, hs::as_stream(stream));
}

extern "C" int hs_gemv_tc(const uint16_t *xs, int t, const uint16_t *w, int ldw, int N, int epilogue, float *y, int ldy,
                          uint16_t *xs_out, int ld_xs_out, void *workspace, size_t ws_bytes, void *stream) {
  return hs::launch_gemv_tc(xs, t, w, ldw, N, epilogue, y, ldy, xs_out, ld_xs_out, workspace, ws_bytes,
                            hs::as_stream(stream), nullptr, nullptr, 0, 0);
}
