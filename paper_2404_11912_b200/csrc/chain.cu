// Persistent dense chain: several dependent weight-streaming GEMVs of a
// decode / verify forward in ONE kernel (model.py:282-285, 316-328).
//
// Per layer the forward runs rope+append and attention as their own kernels
// and everything dense in between as one chain launch:
//     wo (+residual) -> RMSNorm + gate|up (+SwiGLU) -> down (+residual)
//     -> RMSNorm + wqkv of the next layer   (or final norm + lm_head)
// Every phase is a swap-AB tcgen05 GEMV exactly like gemv_tc.cu (weight tile
// = A, M = 128 rows, K-major SW128; the t <= 8 activation rows enter as an
// exact 3-way bf16 split, B = 24 columns, fp32 accumulation in TMEM).  What
// the chain adds:
//   * one persistent CTA per SM owns the work items b, b + G, ... of the
//     whole chain (item = (phase, 128-row tile, K split)); its TMA producer
//     streams the weight tiles of ALL its items through one ring, so HBM keeps
//     streaming across phase boundaries while the CTA waits for the phase's
//     activations -- no kernel boundary, no launch gap, no pipeline drain;
//   * the activation operand is built in shared memory by the epilogue warps
//     straight from the fp32 rows (RMSNorm scale, gain, exact split), so no
//     separate split/normalise kernels exist;
//   * phases are separated by a grid-wide barrier (all CTAs are co-resident:
//     one per SM); the RMSNorm row statistics of the residual stream are
//     produced by the finalising CTAs of the residual phases as per-tile fp64
//     sums of squares and reduced in tile order by the consumers;
//   * K-split partial tiles are reduced by the last-arriving CTA in split
//     order (deterministic; splits depend only on (N, K), never on t, so a
//     row's result does not depend on the batch: the chunk == step-sequence
//     contract of model.py:366-378).
#include <stdlib.h>
#include <string.h>

#include "hs_common.cuh"
#include "tc_util.cuh"

namespace hs {

int get_tmap_bf16(const void *ptr, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes, uint32_t box_rows,
                  CUtensorMap *out);

namespace {

constexpr int CH_BM = 128;                      // output rows per tile (MMA M)
constexpr int CH_BK = 64;                       // K per stage / per B atom
constexpr int CH_T = 8;                         // activation rows per launch
constexpr int CH_XN = 24;                       // B columns: 3 splits x 8 rows
constexpr int CH_STAGES = 7;
constexpr int CH_MAXNK = 16;                    // K blocks per item (B resident in smem)
constexpr int CH_W_BYTES = CH_BM * CH_BK * 2;   // 16 KB
constexpr int CH_ATOM = CH_XN * 128;            // one 64-column B atom: 24 rows x 128 B
constexpr int CH_B_BYTES = CH_MAXNK * CH_ATOM;  // 36 KB
constexpr int CH_IQ = 256;                      // item queue entries per launch
constexpr int CH_QMAX = CH_T * CH_MAXNK * CH_BK / 4 / 128;   // float4 activation loads per builder thread
constexpr int CH_THREADS = 320;   // producer, MMA, 4 epilogue, 4 builder warps
constexpr int CH_SMEM = CH_STAGES * CH_W_BYTES + 2 * CH_B_BYTES + 1024 + 512;

}  // namespace

struct ChainPhase {
  int N, K, nkb, ks, n_tiles, n_items, item0;
  int epilogue;          // 0 store, 1 residual accumulate (+ row sums of squares), 2 SwiGLU pairs
  const float *src;      // fp32 activation rows [t][ld_src]
  int ld_src;
  const float *gain;     // RMSNorm gain (nullptr: no norm)
  int ssq_parts;         // >0: norm statistics = sum of ssq[0..parts) ; 0: computed from src
  float *y;
  int ldy;
};

constexpr int CH_MAXPH = 4;

struct ChainArgs {
  ChainPhase ph[CH_MAXPH];
  int n_phases, t, total_items, blocked;
  float eps;
  float *partial;        // [ks][n_tiles * 128][8]
  int *counters;         // [tiles] K-split arrivals (self-cleaning)
  int *bar;              // [CH_MAXPH + 1] phase barriers + exit counter (self-cleaning)
  int *claim;            // [CH_MAXPH][64] per-(phase, split) tile claim counters (self-cleaning)
  double *ssq;           // [tiles][8] per-tile row sums of squares of the residual stream
};

namespace {

__device__ __forceinline__ uint32_t b_off(int n, int k) {   // K-major SW128, 24-row atoms
  const int atom = k >> 6, kk = k & 63;
  return (uint32_t)(atom * CH_ATOM + n * 128 + ((((kk >> 3) ^ (n & 7)) & 7) << 4) + ((kk & 7) << 1));
}

__device__ __forceinline__ void split3f(float h, uint16_t &a, uint16_t &b, uint16_t &c) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(h);
  const float r1 = h - __bfloat162float(hi);
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  const float r2 = r1 - __bfloat162float(mid);
  a = __bfloat16_as_ushort(hi);
  b = __bfloat16_as_ushort(mid);
  c = __bfloat16_as_ushort(__float2bfloat16_rn(r2));
}

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void bld_sync() { asm volatile("bar.sync 2, 128;" ::: "memory"); }

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Work assignment of a phase: CTAs are dealt into ks groups (b % ks); group s
// owns K split s of every 128-row tile, its CTAs take the tiles round-robin.
// A CTA therefore keeps ONE K range -- and one activation operand -- for the
// whole phase.
struct PhaseWork { int split, kb0, nk, tile0, tstep; };

__device__ __forceinline__ PhaseWork work_of(const ChainPhase &ph, int b, int G) {
  PhaseWork w;
  w.split = b % ph.ks;
  w.tile0 = b / ph.ks;
  w.tstep = (G - w.split + ph.ks - 1) / ph.ks;   // CTAs in this split group
  const int per = ph.nkb / ph.ks, rem = ph.nkb % ph.ks;
  w.kb0 = w.split * per + min(w.split, rem);
  w.nk = per + (w.split < rem ? 1 : 0);
  return w;
}

// optional event trace (hs_chain_trace): 128 slots per CTA, globaltimer ns
__device__ unsigned long long *g_chain_trace = nullptr;
__device__ __forceinline__ void trace(int slot, int code) {
  unsigned long long *t = g_chain_trace;
  if (t == nullptr || slot >= 128) return;
  unsigned long long ns;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ns));
  t[((size_t)blockIdx.x * 128 + slot) * 2] = (unsigned long long)code;
  t[((size_t)blockIdx.x * 128 + slot) * 2 + 1] = ns;
}

// every CTA's producer (after its last claim) and builders (after its last
// barrier) have checked in: nobody touches the sync counters any more
__device__ void reset_sync(const ChainArgs &a) {
  for (int p = 0; p < CH_MAXPH; ++p) a.bar[p] = 0;
  for (int i = 0; i < CH_MAXPH * 64; ++i) a.claim[i] = 0;
  a.bar[CH_MAXPH] = 0;
  __threadfence();
}

// finalize one output row o of a tile (all 128 epilogue threads call it)
__device__ void chain_finalize(const ChainArgs &a, const ChainPhase &ph, int tile, int o, const float *v, int lane,
                               int etid, double (*red)[CH_T]) {
  if (ph.epilogue == 2) {
    float up[CH_T];
#pragma unroll
    for (int r = 0; r < CH_T; ++r) up[r] = __shfl_down_sync(0xffffffffu, v[r], 1);
    if ((o & 1) == 0 && o + 1 < ph.N) {
      const int i = o >> 1;
#pragma unroll
      for (int r = 0; r < CH_T; ++r) {
        if (r < a.t) {
          const double g = (double)v[r];
          ph.y[(size_t)r * ph.ldy + i] = (float)(g * (0.5 * (tanh(0.5 * g) + 1.0))) * up[r];   // model.py:321-322
        }
      }
    }
    return;
  }
  double sq[CH_T];
#pragma unroll
  for (int r = 0; r < CH_T; ++r) {
    sq[r] = 0.0;
    if (r < a.t && o < ph.N) {
      float *p = ph.y + (size_t)r * ph.ldy + o;
      const float nv = ph.epilogue == 1 ? (*p + v[r]) : v[r];
      *p = nv;
      sq[r] = (double)nv * (double)nv;
    }
  }
  if (ph.epilogue != 1) return;
  // per-tile row sums of squares (fixed order: lanes, then warps in order)
#pragma unroll
  for (int r = 0; r < CH_T; ++r) {
    const double s = warp_sum(sq[r]);
    if (lane == 0) red[etid >> 5][r] = s;
  }
  epi_sync();
  if (etid < CH_T) {
    const int q = etid;
    a.ssq[(size_t)tile * CH_T + q] = (red[0][q] + red[1][q]) + (red[2][q] + red[3][q]);
  }
  epi_sync();
}

__global__ void __launch_bounds__(CH_THREADS, 1) chain_kernel(const __grid_constant__ CUtensorMap tm0,
                                                              const __grid_constant__ CUtensorMap tm1,
                                                              const __grid_constant__ CUtensorMap tm2,
                                                              const __grid_constant__ CUtensorMap tm3,
                                                              const ChainArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *sW = base;
  unsigned char *sB = base + CH_STAGES * CH_W_BYTES;            // 2 x B buffers
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + 2 * CH_B_BYTES);
  uint64_t *full = bars, *empty = bars + CH_STAGES;
  uint64_t *bfull = empty + CH_STAGES, *bempty = bfull + 2, *tfull = bempty + 2, *tempty = tfull + 2;
  uint32_t *tmem_base = reinterpret_cast<uint32_t *>(tempty + 2);
  int *flag = reinterpret_cast<int *>(tmem_base + 1);
  __shared__ double red_e[4][CH_T];   // epilogue: per-warp row sums of squares
  __shared__ double red_b[4][CH_T];   // builders: per-warp row statistics
  __shared__ double inv_s[CH_T];      // builders: 1 / RMS of each row
  __shared__ int iq_tile[CH_IQ];      // producer -> MMA / epilogue: claimed tiles, -1 ends a phase
  __shared__ volatile int iq_flag[CH_IQ];
  auto item_wait = [&](int k) -> int {
    if (k >= CH_IQ) __trap();
    while (iq_flag[k] == 0) { }
    __threadfence_block();
    return iq_tile[k];
  };

  tc::grid_dep_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  for (int i = threadIdx.x; i < CH_IQ; i += blockDim.x) iq_flag[i] = 0;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm0);
    if (a.n_phases > 1) tc::tma_prefetch(&tm1);
    if (a.n_phases > 2) tc::tma_prefetch(&tm2);
    if (a.n_phases > 3) tc::tma_prefetch(&tm3);
    for (int s = 0; s < CH_STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&bfull[b], 4); tc::mbar_init(&bempty[b], 1);
      tc::mbar_init(&tfull[b], 1); tc::mbar_init(&tempty[b], 4);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc<64>(tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t taddr = *tmem_base;

  if (warp == 0) {
    // ---- TMA producer: claims tiles of its split group dynamically (faster
    // CTAs take more), publishes each claim to the MMA and epilogue warps
    // through the item queue, streams the weight tiles through one ring.
    // (weights never depend on earlier kernels: no grid dependency wait)
    if (tc::elect_one()) {
      const uint64_t pol = tc::policy_evict_first();
      const CUtensorMap *maps[4] = {&tm0, &tm1, &tm2, &tm3};
      uint32_t g = 0;
      int k = 0;
      trace(0, 1);
      // the claim counters are reset by the previous chain launch's last CTA:
      // wait for that grid before the first claim
      tc::grid_dep_wait();
      for (int p = 0; p < a.n_phases; ++p) {
        const ChainPhase &ph = a.ph[p];
        const PhaseWork w = work_of(ph, cta, G);
        const CUtensorMap *m = maps[p];
        int *ctr = a.claim + p * 64 + w.split;
        if (p < 4) trace(1 + p, 100 + p);
        while (true) {
          // claim only when about to stream it (the ring hides the atomic's
          // latency); no claim ahead, so a slow SM never sits on spare work
          const int tile = atomicAdd(ctr, 1);
          iq_tile[k] = tile < ph.n_tiles ? tile : -1;
          __threadfence_block();
          iq_flag[k] = 1;
          ++k;
          if (tile >= ph.n_tiles) break;
          for (int i = 0; i < w.nk; ++i, ++g) {
            const int s = g % CH_STAGES;
            tc::mbar_wait(&empty[s], ((g / CH_STAGES) & 1) ^ 1);
            tc::mbar_expect_tx(&full[s], CH_W_BYTES);
            if (a.blocked)
              tc::tma_load_2d_hint(sW + s * CH_W_BYTES, m, &full[s], 0, (tile * ph.nkb + w.kb0 + i) * CH_BM, pol);
            else
              tc::tma_load_2d_hint(sW + s * CH_W_BYTES, m, &full[s], (w.kb0 + i) * CH_BK, tile * CH_BM, pol);
          }
        }
      }
      // all claims done: count toward the reset of the sync counters
      if (atomicAdd(&a.bar[CH_MAXPH], 1) == 2 * G - 1) reset_sync(a);
    }
  } else if (warp == 1) {
    // ---- MMA issuer -------------------------------------------------------------
    if (tc::elect_one()) {
      constexpr uint32_t idesc = tc::idesc_bf16(CH_BM, CH_XN, 0, 0);
      uint32_t g = 0, j = 0;
      int k = 0;
      for (int p = 0; p < a.n_phases; ++p) {
        const PhaseWork w = work_of(a.ph[p], cta, G);
        const int b = p & 1;
        tc::mbar_wait(&bfull[b], (p >> 1) & 1);   // this phase's activation operand
        tc::fence_after();
        if (p < 4) trace(40 + p, 200 + p);
        unsigned char *bb = sB + b * CH_B_BYTES;
        while (true) {
          const int tile = item_wait(k++);
          if (tile < 0) break;
          const int tb = j & 1;
          tc::mbar_wait(&tempty[tb], ((j >> 1) & 1) ^ 1);
          tc::fence_after();
          for (int i = 0; i < w.nk; ++i, ++g) {
            const int s = g % CH_STAGES;
            tc::mbar_wait(&full[s], (g / CH_STAGES) & 1);
            tc::fence_after();
            const uint64_t da = tc::desc_k_sw128(sW + s * CH_W_BYTES);
            const uint64_t db = tc::desc_k_sw128(bb + i * CH_ATOM);
#pragma unroll
            for (int kk = 0; kk < CH_BK / 16; ++kk)
              tc::mma_bf16(taddr + tb * 32, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
            tc::mma_commit(&empty[s]);
          }
          tc::mma_commit(&tfull[tb]);
          ++j;
        }
        tc::mma_commit(&bempty[b]);
      }
    }
  } else if (warp >= 6) {
    // ---- warps 6-9: activation builders: one split operand per phase ----------------
    tc::grid_dep_wait();   // the first phase's activations come from earlier kernels
    const int btid = threadIdx.x - 192;   // 0..127
    const int bq = warp - 6;
    for (int p = 0; p < a.n_phases; ++p) {
      const ChainPhase &ph = a.ph[p];
      const PhaseWork w = work_of(ph, cta, G);
      if (p > 0) {   // grid barrier: phase p-1's outputs complete everywhere
        if (btid == 0) {
          while (ld_acquire(&a.bar[p - 1]) < G) __nanosleep(20);
          trace(48 + p, 400 + p);
        }
        bld_sync();
      }
      // (1) this CTA's activation slice, rows [0, t) x its K range: every load
      //     in flight at once (rows >= t are never read back -- their MMA
      //     columns are ignored by the epilogue)
      const int nq = (w.nk * CH_BK) >> 2, c0 = w.kb0 * CH_BK;
      const int total = a.t * nq;
      float4 fv[CH_QMAX];
#pragma unroll
      for (int i = 0; i < CH_QMAX; ++i) {
        const int e = btid + i * 128;
        fv[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e < total) {
          const int r = e / nq, col = c0 + ((e - r * nq) << 2);
          const float *sp = ph.src + (size_t)r * ph.ld_src + col;
          if (col + 3 < ph.K && (((uintptr_t)sp) & 15) == 0) {
            fv[i] = __ldcg(reinterpret_cast<const float4 *>(sp));
          } else {
            fv[i].x = col < ph.K ? __ldcg(sp) : 0.f;
            fv[i].y = col + 1 < ph.K ? __ldcg(sp + 1) : 0.f;
            fv[i].z = col + 2 < ph.K ? __ldcg(sp + 2) : 0.f;
            fv[i].w = col + 3 < ph.K ? __ldcg(sp + 3) : 0.f;
          }
        }
      }
      // (2) RMSNorm row scales (model.py:282-284): 1 / sqrt(mean(x^2) + eps)
      if (ph.gain != nullptr) {
        if (ph.ssq_parts > 0) {   // per-tile sums: 16 lanes per row, fixed tree order
          const int r = btid >> 4, l16 = btid & 15;
          double s = 0.0;
          for (int k = l16; k < ph.ssq_parts; k += 16) s += __ldcg(&a.ssq[(size_t)k * CH_T + r]);
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (l16 == 0) inv_s[r] = 1.0 / sqrt(s / (double)ph.K + (double)a.eps);
        } else {   // statistics straight from the rows (first phase of a forward)
#pragma unroll 1
          for (int r = 0; r < a.t; ++r) {
            double s = 0.0;
            for (int c = btid * 4; c < ph.K; c += 512) {
              const float *sp = ph.src + (size_t)r * ph.ld_src + c;
              if (c + 3 < ph.K && ((((uintptr_t)sp) & 15) == 0)) {
                const float4 f = __ldcg(reinterpret_cast<const float4 *>(sp));
                s += (double)f.x * f.x + (double)f.y * f.y + (double)f.z * f.z + (double)f.w * f.w;
              } else {
                for (int u = 0; u < 4 && c + u < ph.K; ++u) {
                  const double v = (double)__ldcg(sp + u);
                  s += v * v;
                }
              }
            }
            s = warp_sum(s);
            if (lane == 0) red_b[bq][r] = s;
          }
          bld_sync();
          if (btid < a.t)
            inv_s[btid] = 1.0 / sqrt(((red_b[0][btid] + red_b[1][btid]) + (red_b[2][btid] + red_b[3][btid])) /
                                     (double)ph.K + (double)a.eps);
        }
        bld_sync();
      }
      // (3) scale, exact 3-way bf16 split, swizzled stores into the B buffer
      const int b = p & 1;
      tc::mbar_wait(&bempty[b], ((p >> 1) & 1) ^ 1);
      unsigned char *bb = sB + b * CH_B_BYTES;
#pragma unroll
      for (int i = 0; i < CH_QMAX; ++i) {
        const int e = btid + i * 128;
        if (e < total) {
          const int r = e / nq, cc = (e - r * nq) << 2;
          const int col = c0 + cc;
          float v[4] = {fv[i].x, fv[i].y, fv[i].z, fv[i].w};
          if (ph.gain) {
            const double is = inv_s[r];
            if (col + 3 < ph.K && ((col & 3) == 0)) {
              const float4 gg = __ldg(reinterpret_cast<const float4 *>(ph.gain + col));
              v[0] = (float)(((double)v[0] * is) * (double)gg.x);
              v[1] = (float)(((double)v[1] * is) * (double)gg.y);
              v[2] = (float)(((double)v[2] * is) * (double)gg.z);
              v[3] = (float)(((double)v[3] * is) * (double)gg.w);
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (col + u < ph.K) v[u] = (float)(((double)v[u] * is) * (double)__ldg(ph.gain + col + u));
            }
          }
          uint16_t h[3][4];
#pragma unroll
          for (int u = 0; u < 4; ++u) split3f(v[u], h[0][u], h[1][u], h[2][u]);
#pragma unroll
          for (int sp3 = 0; sp3 < 3; ++sp3) {
            uint2 wv;
            wv.x = (uint32_t)h[sp3][0] | ((uint32_t)h[sp3][1] << 16);
            wv.y = (uint32_t)h[sp3][2] | ((uint32_t)h[sp3][3] << 16);
            *reinterpret_cast<uint2 *>(bb + b_off(sp3 * CH_T + r, cc)) = wv;
          }
        }
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bfull[b]);
      if (btid == 0) trace(56 + p, 300 + p);
    }
    // past every barrier: count toward the reset of the sync counters
    if (btid == 0 && atomicAdd(&a.bar[CH_MAXPH], 1) == 2 * G - 1) reset_sync(a);
  } else {
    // ---- warps 2-5: epilogue (warp w reads TMEM lanes 32 * (w % 4) ..) --------------
    tc::grid_dep_wait();   // y / partials / counters are touched by earlier kernels
    const int q = warp & 3, etid = threadIdx.x - 64;
    const int row = q * 32 + lane;
    uint32_t j = 0;
    int k = 0;
    for (int p = 0; p < a.n_phases; ++p) {
      const ChainPhase &ph = a.ph[p];
      const PhaseWork w = work_of(ph, cta, G);
      while (true) {
        const int tile = item_wait(k++);
        if (tile < 0) break;
        const int tb = j & 1;
        tc::mbar_wait(&tfull[tb], (j >> 1) & 1);
        tc::fence_after();
        const uint32_t tl = taddr + tb * 32 + ((uint32_t)(q * 32) << 16);
        float hh[8], mm[8], ll[8], v[CH_T];
        tc::tmem_ld8(tl + 0, hh);
        tc::tmem_ld8(tl + 8, mm);
        tc::tmem_ld8(tl + 16, ll);
        tc::tmem_ld_wait();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[tb]);
#pragma unroll
        for (int r = 0; r < CH_T; ++r) v[r] = (hh[r] + mm[r]) + ll[r];
        const int o = tile * CH_BM + row;
        if (ph.ks == 1) {
          chain_finalize(a, ph, tile, o, v, lane, etid, red_e);
          ++j;
          continue;
        }
        float *pp = a.partial + ((size_t)w.split * ph.n_tiles * CH_BM + o) * CH_T;
        *reinterpret_cast<float4 *>(pp) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4 *>(pp + 4) = make_float4(v[4], v[5], v[6], v[7]);
        epi_sync();   // the CTA's partial tile is written; one cumulative fence publishes it
        if (etid == 0) {
          __threadfence();
          *flag = (atomicAdd(&a.counters[tile], 1) == ph.ks - 1);
        }
        epi_sync();
        if (*flag) {
          __threadfence();
#pragma unroll
          for (int r = 0; r < CH_T; ++r) v[r] = 0.f;
          const float *q0 = a.partial + (size_t)o * CH_T;
          const size_t sstride = (size_t)ph.n_tiles * CH_BM * CH_T;
          int s2 = 0;
          for (; s2 + 8 <= ph.ks; s2 += 8) {   // 8 splits' loads in flight, summed in split order
            float4 x[8][2];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              x[u][0] = __ldcg(reinterpret_cast<const float4 *>(q0 + (s2 + u) * sstride));
              x[u][1] = __ldcg(reinterpret_cast<const float4 *>(q0 + (s2 + u) * sstride + 4));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              v[0] += x[u][0].x; v[1] += x[u][0].y; v[2] += x[u][0].z; v[3] += x[u][0].w;
              v[4] += x[u][1].x; v[5] += x[u][1].y; v[6] += x[u][1].z; v[7] += x[u][1].w;
            }
          }
          for (; s2 < ph.ks; ++s2) {
            const float4 x0 = __ldcg(reinterpret_cast<const float4 *>(q0 + s2 * sstride));
            const float4 x1 = __ldcg(reinterpret_cast<const float4 *>(q0 + s2 * sstride + 4));
            v[0] += x0.x; v[1] += x0.y; v[2] += x0.z; v[3] += x0.w;
            v[4] += x1.x; v[5] += x1.y; v[6] += x1.z; v[7] += x1.w;
          }
          chain_finalize(a, ph, tile, o, v, lane, etid, red_e);
          if (etid == 0) a.counters[tile] = 0;   // self-cleaning
        }
        epi_sync();   // flag is rewritten by the next item
        if (etid == 0 && j < 40) trace(64 + j, 500 + p);
        ++j;
      }
      if (p + 1 < a.n_phases) {   // arrive: this CTA's phase-p outputs are complete
        __threadfence();
        epi_sync();
        if (etid == 0) { atomicAdd(&a.bar[p], 1); trace(120 + p, 600 + p); }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<64>(taddr);
}

}  // namespace

// K split of one phase: a function of (N, K) only (t-invariance).  Minimises
// the busiest CTA's K blocks plus a small per-split finalisation cost.
int chain_ksplit(int N, int nkb, int G) {
  const int tiles = (N + CH_BM - 1) / CH_BM;
  int best = 1;
  double best_cost = 1e30;
  for (int ks = 1; ks <= 64 && ks <= nkb && ks <= G; ++ks) {
    const int nk = (nkb + ks - 1) / ks;
    if (nk > CH_MAXNK) continue;
    const int gs = G / ks;                        // smallest split group
    // busiest CTA: its items stream nk K blocks each but cost at least ~5
    // blocks of epilogue latency (partial store + arrival atomic); the
    // last-arriving CTA of a tile then reads ks partials (~2.5 blocks per 8)
    const int items = (tiles + gs - 1) / gs;
    const double cost = (double)items * (nk > 5 ? nk : 5) + (ks > 1 ? 2.5 * ((ks + 7) / 8) : 0.0);
    if (cost < best_cost - 1e-9) { best_cost = cost; best = ks; }
  }
  return best;
}

struct ChainSpec {
  const uint16_t *w;
  int ldw, N, K, epilogue;
  const float *src;
  int ld_src;
  const float *gain;
  int ssq_parts;
  float *y;
  int ldy;
};

static int g_chain_sms = 0;

int chain_grid() {
  if (!g_chain_sms) cudaDeviceGetAttribute(&g_chain_sms, cudaDevAttrMultiProcessorCount, 0);
  return g_chain_sms;
}

constexpr size_t CH_WS_SYNC = 16384 * 4 + 2048;   // counters | barriers + claims (zero at rest)

size_t chain_ws_bytes(int max_n_tiles_ks) {   // partials + counters + barriers + ssq
  return (size_t)max_n_tiles_ks * CH_BM * CH_T * 4 + CH_WS_SYNC + 4096 * CH_T * 8;
}

// ws layout: [counters 16384 ints][bar 16 ints][ssq 4096 x 8 doubles][partials]
int launch_chain(const ChainSpec *ps, int n, int t, float eps, void *ws, size_t ws_bytes, cudaStream_t st) {
  HS_REQUIRE(n >= 1 && n <= CH_MAXPH, HS_ERR_VALUE, "chain: %d phases", n);
  HS_REQUIRE(t >= 1 && t <= CH_T, HS_ERR_SHAPE, "chain: t=%d outside [1,%d]", t, CH_T);
  const int G = chain_grid();
  ChainArgs a = {};
  CUtensorMap maps[CH_MAXPH];
  memset(maps, 0, sizeof(maps));
  int item0 = 0;
  size_t need_part = 0;
  for (int i = 0; i < n; ++i) {
    const ChainSpec &s = ps[i];
    HS_REQUIRE(s.ldw % CH_BK == 0 && s.K <= s.ldw, HS_ERR_SHAPE, "chain: bad K %d / ld %d", s.K, s.ldw);
    HS_REQUIRE(s.epilogue != 2 || s.N % 2 == 0, HS_ERR_SHAPE, "chain: swiglu needs an even N");
    static int blocked_test = -1;
    if (blocked_test < 0) { const char *e = getenv("HS_GEMV_BLOCKED_TEST"); blocked_test = e && e[0] == '1'; }
    a.blocked = blocked_test;
    int rc = blocked_test ? get_tmap_bf16(s.w, (uint64_t)CH_BK, (uint64_t)s.N * (s.ldw / CH_BK), (uint64_t)CH_BK * 2, CH_BM, &maps[i])
                          : get_tmap_bf16(s.w, (uint64_t)s.ldw, (uint64_t)s.N, (uint64_t)s.ldw * 2, CH_BM, &maps[i]);
    if (rc != HS_OK) return rc;
    ChainPhase &ph = a.ph[i];
    ph.N = s.N; ph.K = s.K; ph.nkb = s.ldw / CH_BK; ph.n_tiles = (s.N + CH_BM - 1) / CH_BM;
    HS_REQUIRE(ph.n_tiles <= 16384, HS_ERR_SHAPE, "chain: N too large");
    ph.ks = chain_ksplit(s.N, ph.nkb, G);
    ph.n_items = ph.n_tiles * ph.ks;
    ph.item0 = item0;
    item0 += ph.n_items;
    ph.epilogue = s.epilogue; ph.src = s.src; ph.ld_src = s.ld_src; ph.gain = s.gain; ph.ssq_parts = s.ssq_parts;
    ph.y = s.y; ph.ldy = s.ldy;
    HS_REQUIRE(s.epilogue != 1 || ph.n_tiles <= 4096, HS_ERR_SHAPE, "chain: residual too wide");
    if (ph.ks > 1) need_part = need_part > (size_t)ph.ks * ph.n_tiles ? need_part : (size_t)ph.ks * ph.n_tiles;
  }
  HS_REQUIRE(ws_bytes >= chain_ws_bytes((int)need_part), HS_ERR_VALUE, "chain: workspace too small");
  char *w = reinterpret_cast<char *>(ws);
  a.counters = reinterpret_cast<int *>(w);
  a.bar = reinterpret_cast<int *>(w + 16384 * 4);
  a.claim = a.bar + 64;
  a.ssq = reinterpret_cast<double *>(w + CH_WS_SYNC);
  a.partial = reinterpret_cast<float *>(w + CH_WS_SYNC + 4096 * CH_T * 8);
  a.n_phases = n; a.t = t; a.total_items = item0; a.eps = eps;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, CH_SMEM);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(CH_THREADS, 1, 1);
  cfg.dynamicSmemBytes = CH_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl_enabled();
  cudaError_t e = cudaLaunchKernelEx(&cfg, chain_kernel, maps[0], maps[1], maps[2], maps[3], a);
  if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "chain launch: %s", cudaGetErrorString(e));
  return check_launch("chain");
}

int chain_set_trace(void *buf) {
  unsigned long long *p = reinterpret_cast<unsigned long long *>(buf);
  cudaError_t e = cudaMemcpyToSymbol(g_chain_trace, &p, sizeof(p));
  return e == cudaSuccess ? HS_OK : set_error(HS_ERR_CUDA, "chain trace: %s", cudaGetErrorString(e));
}

size_t chain_ws_for_model(const HsModel *m) {
  const int G = chain_grid() ? chain_grid() : 148;
  const int d = m->d_model, kv = m->n_kv_heads * m->head_dim;
  const int Ns[5] = {d + 2 * kv, d, 2 * m->d_ff, d, m->vocab_size};
  const int Ks[5] = {m->ld_d, m->ld_d, m->ld_d, m->ld_ff, m->ld_d};
  size_t mx = 0;
  for (int i = 0; i < 5; ++i) {
    const int ks = chain_ksplit(Ns[i], Ks[i] / CH_BK, G);
    const size_t v = (size_t)ks * ((Ns[i] + CH_BM - 1) / CH_BM);
    if (ks > 1 && v > mx) mx = v;
  }
  return chain_ws_bytes((int)mx);
}

}  // namespace hs

/* debugging aid: per-CTA event trace of the chain kernel (128 slots x
 * (code, globaltimer ns) per CTA); NULL disables.  Not part of hs_abi.h.  */
extern "C" int hs_chain_trace(void *buf) { return hs::chain_set_trace(buf); }
