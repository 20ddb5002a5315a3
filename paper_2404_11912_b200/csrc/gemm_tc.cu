// Tensor-core GEMM for the batched prefill's dense layers (tcgen05 + TMA).
//
// Replaces the batched matmuls of `prefill` (model.py:334-354 through
// `_forward`, model.py:281-285,316-328) for long prompts:
//
//     Y[r][n] (+)= sum_k W[n][k] * (s0 + s1 + s2)[r][k]
//
// where s0 + s1 + s2 is the exact 3-way bf16 split of the fp32 activation
// row (pf_split_kernel): every product is exact in the tensor core and all
// three planes accumulate into ONE fp32 TMEM accumulator, so the result is
// an fp32-accumulated dot product of the fp32 activations with the bf16
// weights -- the GEMV's numerics at GEMM throughput.
//
// Tiling: D[128 activation rows x BN weight rows] in TMEM (A = activation
// planes, K-major SW128; B = weight rows, K-major SW128), K in 64-element
// steps; one stage = 3 A tiles + 1 B tile.  Persistent CTAs (one per SM)
// walk the tiles activation-row-tile fastest, so the CTAs running together
// share weight tiles through L2 while the activation planes stay
// L2-resident.  Warp roles: warp 0 TMA producer, warp 1 MMA issuer, warps
// 2-5 epilogue (TMEM -> registers -> Y, optional accumulate); the TMEM
// accumulator is double-buffered so a tile's epilogue overlaps the next
// tile's main loop.
#include "hs_common.cuh"
#include "tc_util.cuh"

namespace hs {

int get_tmap_bf16(const void *ptr, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes, uint32_t box_rows,
                  CUtensorMap *out);

namespace {

constexpr int GM_M = 128;                  // activation rows per tile (MMA M, TMEM lanes)
constexpr int GM_BN = 192;                 // weight rows per tile (MMA N)
constexpr int GM_KS = 64;                  // K elements per stage (one SW128 atom)
constexpr int GM_STAGES = 3;
constexpr int GM_A = GM_M * GM_KS * 2;     // one activation plane tile: 16 KB
constexpr int GM_B = GM_BN * GM_KS * 2;    // weight tile: 24 KB
constexpr int GM_STAGE = 3 * GM_A + GM_B;  // 72 KB
constexpr int GM_SMEM = GM_STAGES * GM_STAGE + 1024;
constexpr int GM_THREADS = 192;            // TMA warp, MMA warp, 4 epilogue warps
constexpr int GM_TMEM_COLS = 512;          // two BN-column accumulators

struct GemmArgs {
  int R, N, nk;            // activation rows, weight rows, K steps
  int n_mt, n_nt, tiles;
  float *y;
  int ldy, accumulate;
  int blocked;             // W tile-blocked [N/128][K/64][128][64] (HsModel.blocked): loaded as 3 x 64-row boxes
};

__global__ void __launch_bounds__(GM_THREADS, 1) gemm3_tc_kernel(const __grid_constant__ CUtensorMap tA0,
                                                                 const __grid_constant__ CUtensorMap tA1,
                                                                 const __grid_constant__ CUtensorMap tA2,
                                                                 const __grid_constant__ CUtensorMap tW, GemmArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[GM_STAGES], empty[GM_STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tA0);
    tc::tma_prefetch(&tA1);
    tc::tma_prefetch(&tA2);
    tc::tma_prefetch(&tW);
    for (int s = 0; s < GM_STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 4);   // one arrive per epilogue warp
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc<GM_TMEM_COLS>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  tc::grid_dep_wait();   // the split planes / Y of the preceding kernels

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (tc::elect_one()) {
      uint32_t g = 0;
      for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
        const int mt = tile % a.n_mt, nt = tile / a.n_mt;
        for (int ks = 0; ks < a.nk; ++ks, ++g) {
          const int s = g % GM_STAGES;
          tc::mbar_wait(&empty[s], ((g / GM_STAGES) & 1) ^ 1);
          unsigned char *st = base + s * GM_STAGE;
          tc::mbar_expect_tx(&full[s], GM_STAGE);
          tc::tma_load_2d(st, &tA0, &full[s], ks * GM_KS, mt * GM_M);
          tc::tma_load_2d(st + GM_A, &tA1, &full[s], ks * GM_KS, mt * GM_M);
          tc::tma_load_2d(st + 2 * GM_A, &tA2, &full[s], ks * GM_KS, mt * GM_M);
          if (a.blocked) {
            // the 192 weight rows of this tile as three 64-row halves of 128-row blocks
#pragma unroll
            for (int c = 0; c < GM_BN / 64; ++c) {
              const int r = nt * GM_BN + c * 64;
              tc::tma_load_2d(st + 3 * GM_A + c * 64 * 128, &tW, &full[s], 0, ((r >> 7) * a.nk + ks) * 128 + (r & 127));
            }
          } else {
            tc::tma_load_2d(st + 3 * GM_A, &tW, &full[s], ks * GM_KS, nt * GM_BN);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (tc::elect_one()) {
      constexpr uint32_t idesc = tc::idesc_bf16(GM_M, GM_BN, 0, 0);
      uint32_t g = 0, it = 0;
      for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
        const int b = it & 1;
        tc::mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);   // the epilogue drained this accumulator
        tc::fence_after();
        const uint32_t d = tmem + b * 256;
        for (int ks = 0; ks < a.nk; ++ks, ++g) {
          const int s = g % GM_STAGES;
          tc::mbar_wait(&full[s], (g / GM_STAGES) & 1);
          tc::fence_after();
          unsigned char *st = base + s * GM_STAGE;
#pragma unroll
          for (int p = 0; p < 3; ++p) {
#pragma unroll
            for (int kk = 0; kk < GM_KS / 16; ++kk) {
              const uint64_t da = tc::desc_k_sw128(st + p * GM_A) + 2 * kk;
              const uint64_t db = tc::desc_k_sw128(st + 3 * GM_A) + 2 * kk;
              tc::mma_bf16(d, da, db, idesc, (ks | p | kk) != 0);
            }
          }
          tc::mma_commit(&empty[s]);   // frees the stage once these MMAs have read it
        }
        tc::mma_commit(&tfull[b]);     // accumulator complete
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2-5)
    const int q = warp & 3;                     // TMEM lane quarter this warp may read
    const int lane = threadIdx.x & 31;
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      const int b = it & 1;
      const int mt = tile % a.n_mt, nt = tile / a.n_mt;
      tc::mbar_wait_sleep(&tfull[b], (it >> 1) & 1);
      tc::fence_after();
      const int row = mt * GM_M + q * 32 + lane;
      const uint32_t taddr = tmem + b * 256 + ((uint32_t)(q * 32) << 16);
      float *yr = a.y + (size_t)row * a.ldy + (size_t)nt * GM_BN;
      const int ncols = min(GM_BN, a.N - nt * GM_BN);
#pragma unroll 1
      for (int c0 = 0; c0 < GM_BN; c0 += 8) {
        float v[8];
        tc::tmem_ld8(taddr + c0, v);
        tc::tmem_ld_wait();
        if (row < a.R && c0 < ncols) {
          if (c0 + 8 <= ncols && (reinterpret_cast<uintptr_t>(yr + c0) & 15) == 0) {
            float4 *p4 = reinterpret_cast<float4 *>(yr + c0);
            if (a.accumulate) {
              const float4 o0 = p4[0], o1 = p4[1];
              v[0] += o0.x; v[1] += o0.y; v[2] += o0.z; v[3] += o0.w;
              v[4] += o1.x; v[5] += o1.y; v[6] += o1.z; v[7] += o1.w;
            }
            p4[0] = make_float4(v[0], v[1], v[2], v[3]);
            p4[1] = make_float4(v[4], v[5], v[6], v[7]);
          } else {
            for (int j = 0; j < 8 && c0 + j < ncols; ++j) yr[c0 + j] = a.accumulate ? yr[c0 + j] + v[j] : v[j];
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[b]);
    }
  }
  __syncthreads();
  tc::grid_dep_launch();
  if (warp == 1) tc::tmem_dealloc<GM_TMEM_COLS>(tmem);
}

}  // namespace

// Y[R][N] (ldy) (+)= W[N][ld] . (s0 + s1 + s2)[R][ld]^T with the split planes
// at row stride ldk (elements); fp32 accumulate in TMEM
int launch_gemm3_tc(const uint16_t *s0, const uint16_t *s1, const uint16_t *s2, int ldk, int R, const uint16_t *W,
                    int ld, int N, float *Y, int ldy, int accumulate, cudaStream_t st, int blocked) {
  HS_REQUIRE(ld % GM_KS == 0 && ldk >= ld && R >= 1 && N >= 1, HS_ERR_SHAPE, "gemm3_tc: bad shape (ld %d, ldk %d)", ld,
             ldk);
  HS_REQUIRE(!blocked || N % 128 == 0, HS_ERR_SHAPE, "gemm3_tc: a blocked W needs N %% 128 == 0 (N %d)", N);
  CUtensorMap m0, m1, m2, mw;
  int rc;
  if ((rc = get_tmap_bf16(s0, ld, R, (uint64_t)ldk * 2, GM_M, &m0)) != HS_OK) return rc;
  if ((rc = get_tmap_bf16(s1, ld, R, (uint64_t)ldk * 2, GM_M, &m1)) != HS_OK) return rc;
  if ((rc = get_tmap_bf16(s2, ld, R, (uint64_t)ldk * 2, GM_M, &m2)) != HS_OK) return rc;
  if (blocked) {
    if ((rc = get_tmap_bf16(W, GM_KS, (uint64_t)N * (ld / GM_KS), GM_KS * 2, 64, &mw)) != HS_OK) return rc;
  } else if ((rc = get_tmap_bf16(W, ld, N, (uint64_t)ld * 2, GM_BN, &mw)) != HS_OK) {
    return rc;
  }
  GemmArgs a;
  a.R = R; a.N = N; a.nk = ld / GM_KS;
  a.n_mt = ceil_div(R, GM_M);
  a.n_nt = ceil_div(N, GM_BN);
  a.tiles = a.n_mt * a.n_nt;
  a.y = Y; a.ldy = ldy; a.accumulate = accumulate; a.blocked = blocked;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GM_SMEM);
    attr = true;
  }
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = a.tiles < sms ? a.tiles : sms;
  cudaError_t e = launch_pdl(gemm3_tc_kernel, dim3(grid), dim3(GM_THREADS), GM_SMEM, st, m0, m1, m2, mw, a);
  if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "gemm3_tc launch: %s", cudaGetErrorString(e));
  return check_launch("gemm3_tc");
}

}  // namespace hs

extern "C" int hs_gemm3_tc(const uint16_t *s0, const uint16_t *s1, const uint16_t *s2, int ldk, int rows,
                           const uint16_t *w, int ldw, int n, float *y, int ldy, int accumulate, void *stream) {
  return hs::launch_gemm3_tc(s0, s1, s2, ldk, rows, w, ldw, n, y, ldy, accumulate, hs::as_stream(stream), 0);
}
