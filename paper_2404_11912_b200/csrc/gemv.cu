// Weight-streaming GEMV for the decode/verify forwards (M = t <= 8 rows per pass).
//
// Replaces the fp64-accumulate projections of the reference forward
// (model.py:285, 316, 320-323, 328; tensor.py:26-36).  Weights are bf16
// [out][in] rows ("K-major"), activations fp32, accumulation fp32.
//
// Layout of the work:
//   * a CTA owns ROWS = 32*RL output rows and a contiguous K range; the K
//     range is split across a thread-block CLUSTER of KS CTAs (1..8) whose
//     partial sums are reduced through distributed shared memory in rank
//     order -- deterministic, no atomics, no second launch;
//   * a warp is 4 groups of 8 lanes; a group owns RL rows and reads one
//     128-byte line of each row per step (coalesced), lanes j of the group
//     cover k = 64*it + 8*j .. +8;
//   * the CTA's slice of x is staged once in shared memory (fp32) with the
//     optional RMSNorm prologue applied; all groups of a warp read the same
//     x addresses (broadcast).
// Every output's reduction order depends only on (N, K), never on t, so a
// row's result is bit-identical whether it is computed alone (decode) or in a
// batch (verify) -- the chunk == step-sequence contract of model.py:366-378.
#include <cooperative_groups.h>

#include "hs_common.cuh"

namespace cg = cooperative_groups;

namespace hs {

constexpr int GEMV_THREADS = 256;
constexpr int GEMV_MAXT = 8;
constexpr int GEMV_UNROLL = 4;

struct GemvArgs {
  const float *x;
  int ldx, t, K;
  const uint16_t *w;
  int ldw, N;
  int prologue;
  const float *gain;
  float eps;
  int epilogue;
  float *y;
  int ldy;
  int ks;         // cluster size along K
  int nkb;        // number of 64-wide K blocks (ldw / 64)
  int kr_max;     // smem K capacity per CTA (elements)
};

__device__ __forceinline__ void kblock_range(int nkb, int ks, int q, int &b0, int &b1) {
  int base = nkb / ks, rem = nkb % ks;
  b0 = q * base + min(q, rem);
  b1 = b0 + base + (q < rem ? 1 : 0);
}

template <int T, int RL>
__global__ void __launch_bounds__(GEMV_THREADS) gemv_kernel(GemvArgs a) {
  constexpr int ROWS = 32 * RL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *xs = reinterpret_cast<float *>(smem_raw);                       // [T][kr_max]
  float *red = xs + T * a.kr_max;                                        // [ROWS][T]
  double *ss = reinterpret_cast<double *>(red + ROWS * T);               // [T]
  double *wsum = ss + T;                                                 // [8][T]
  double *scale = wsum + 8 * T;                                          // [T]

  cg::cluster_group cluster = cg::this_cluster();
  const int q = (int)cluster.block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  int b0, b1;
  kblock_range(a.nkb, a.ks, q, b0, b1);
  const int k0 = b0 * 64, kr = (b1 - b0) * 64;

  // ---- stage x[0:T][k0:k0+kr) ; partial sum of squares per row (fp64) ----
  double ssl[T];
#pragma unroll
  for (int r = 0; r < T; ++r) ssl[r] = 0.0;
  for (int kk = tid; kk < kr; kk += GEMV_THREADS) {
    int k = k0 + kk;
#pragma unroll
    for (int r = 0; r < T; ++r) {
      float v = (k < a.K) ? a.x[(size_t)r * a.ldx + k] : 0.f;
      xs[r * a.kr_max + kk] = v;
      ssl[r] += (double)v * (double)v;
    }
  }
  if (a.prologue == 1) {
#pragma unroll
    for (int r = 0; r < T; ++r) {
      double v = warp_sum(ssl[r]);
      if (lane == 0) wsum[warp * T + r] = v;
    }
    __syncthreads();
    if (tid < T) {
      double s = 0.0;
      for (int w = 0; w < GEMV_THREADS / 32; ++w) s += wsum[w * T + tid];
      ss[tid] = s;
    }
    cluster.sync();
    if (tid < T) {
      double tot = 0.0;
      for (int r2 = 0; r2 < a.ks; ++r2) tot += cluster.map_shared_rank(ss, r2)[tid];
      // rms_norm: x / sqrt(mean(x^2) + eps) * gain  (model.py:282-284)
      scale[tid] = sqrt(tot / (double)a.K + (double)a.eps);
    }
    __syncthreads();
    for (int kk = tid; kk < kr; kk += GEMV_THREADS) {
      int k = k0 + kk;
      double g = (k < a.K) ? (double)a.gain[k] : 0.0;
#pragma unroll
      for (int r = 0; r < T; ++r) {
        float *p = &xs[r * a.kr_max + kk];
        *p = (float)(((double)*p / scale[r]) * g);
      }
    }
  }
  __syncthreads();

  // ---- main loop ------------------------------------------------------------
  const int grp = lane >> 3, j = lane & 7;
  const int row_local0 = (warp * 4 + grp) * RL;
  const int row0 = blockIdx.x * ROWS + row_local0;
  const uint16_t *wrow[RL];
  bool rok[RL];
#pragma unroll
  for (int rl = 0; rl < RL; ++rl) {
    rok[rl] = (row0 + rl) < a.N;
    wrow[rl] = a.w + (size_t)(rok[rl] ? row0 + rl : 0) * a.ldw + k0 + j * 8;
  }
  float acc[RL][T];
#pragma unroll
  for (int rl = 0; rl < RL; ++rl)
#pragma unroll
    for (int r = 0; r < T; ++r) acc[rl][r] = 0.f;

  const int n_it = kr / 64;
  for (int it = 0; it < n_it; it += GEMV_UNROLL) {
    uint4 wv[GEMV_UNROLL][RL];
#pragma unroll
    for (int u = 0; u < GEMV_UNROLL; ++u)
#pragma unroll
      for (int rl = 0; rl < RL; ++rl)
        wv[u][rl] = (it + u < n_it && rok[rl]) ? ld_stream(wrow[rl] + (size_t)(it + u) * 64)
                                               : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < GEMV_UNROLL; ++u) {
      if (it + u < n_it) {
        float wf[RL][8];
#pragma unroll
        for (int rl = 0; rl < RL; ++rl) unpack8(wv[u][rl], wf[rl]);
        const int kk = (it + u) * 64 + j * 8;
#pragma unroll
        for (int r = 0; r < T; ++r) {
          const float4 xa = *reinterpret_cast<const float4 *>(&xs[r * a.kr_max + kk]);
          const float4 xb = *reinterpret_cast<const float4 *>(&xs[r * a.kr_max + kk + 4]);
#pragma unroll
          for (int rl = 0; rl < RL; ++rl) {
            float s = acc[rl][r];
            s = fmaf(wf[rl][0], xa.x, s);
            s = fmaf(wf[rl][1], xa.y, s);
            s = fmaf(wf[rl][2], xa.z, s);
            s = fmaf(wf[rl][3], xa.w, s);
            s = fmaf(wf[rl][4], xb.x, s);
            s = fmaf(wf[rl][5], xb.y, s);
            s = fmaf(wf[rl][6], xb.z, s);
            s = fmaf(wf[rl][7], xb.w, s);
            acc[rl][r] = s;
          }
        }
      }
    }
  }
  // reduce the 8 lanes of the group (fixed butterfly)
#pragma unroll
  for (int rl = 0; rl < RL; ++rl)
#pragma unroll
    for (int r = 0; r < T; ++r) {
      float v = acc[rl][r];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (j == 0) red[(row_local0 + rl) * T + r] = v;
    }
  cluster.sync();

  // ---- cluster reduction in rank order + epilogue ----------------------------
  // rank q finalises rows [q*ROWS/ks, (q+1)*ROWS/ks) (pairs kept together)
  const int per = ((ROWS / a.ks) + 1) & ~1;
  const int lo = q * per, hi = min(ROWS, lo + per);
  const int npairs = (hi - lo + 1) / 2;
  for (int idx = tid; idx < npairs * T; idx += GEMV_THREADS) {
    const int pr = idx / T, r = idx % T;
    const int rl0 = lo + 2 * pr;
    float v0 = 0.f, v1 = 0.f;
    for (int r2 = 0; r2 < a.ks; ++r2) {
      const float *rr = cluster.map_shared_rank(red, r2);
      v0 += rr[rl0 * T + r];
      if (rl0 + 1 < hi) v1 += rr[(rl0 + 1) * T + r];
    }
    const int o = blockIdx.x * ROWS + rl0;
    if (a.epilogue == 2) {
      // SwiGLU pair (gate_i, up_i): act = fp32(silu64(gate)) * up  (model.py:321-322)
      if (o + 1 < a.N) {
        double g = (double)v0;
        float act = (float)(g * (0.5 * (tanh(0.5 * g) + 1.0)));
        a.y[(size_t)r * a.ldy + (o >> 1)] = act * v1;
      }
    } else {
      float *y0 = a.y + (size_t)r * a.ldy + o;
      if (o < a.N) {
        if (a.epilogue == 1) y0[0] = y0[0] + v0; else y0[0] = v0;
      }
      if (rl0 + 1 < hi && o + 1 < a.N) {
        if (a.epilogue == 1) y0[1] = y0[1] + v1; else y0[1] = v1;
      }
    }
  }
  cluster.sync();  // keep shared memory alive until every rank has read it
}

template <int T, int RL>
static cudaError_t launch_gemv_t(const GemvArgs &a, int row_blocks, size_t smem, cudaStream_t st) {
  auto kern = gemv_kernel<T, RL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(row_blocks, a.ks, 1);
  cfg.blockDim = dim3(GEMV_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = a.ks;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int RL>
static cudaError_t launch_gemv_rl(const GemvArgs &a, int row_blocks, cudaStream_t st) {
  auto smem_for = [&](int T) {
    return (size_t)T * a.kr_max * 4 + (size_t)32 * RL * T * 4 + (size_t)(T + 8 * T + T) * 8;
  };
  switch (a.t) {
    case 1: return launch_gemv_t<1, RL>(a, row_blocks, smem_for(1), st);
    case 2: return launch_gemv_t<2, RL>(a, row_blocks, smem_for(2), st);
    case 3: return launch_gemv_t<3, RL>(a, row_blocks, smem_for(3), st);
    case 4: return launch_gemv_t<4, RL>(a, row_blocks, smem_for(4), st);
    case 5: return launch_gemv_t<5, RL>(a, row_blocks, smem_for(5), st);
    case 6: return launch_gemv_t<6, RL>(a, row_blocks, smem_for(6), st);
    case 7: return launch_gemv_t<7, RL>(a, row_blocks, smem_for(7), st);
    default: return launch_gemv_t<8, RL>(a, row_blocks, smem_for(8), st);
  }
}

// K split depends only on (N, K): keeps every row's result independent of t.
int gemv_ksplit(int N, int ldw, int RL) {
  int nkb = ldw / 64;
  int ks = 1;
  while (ks < 8 && (nkb + ks - 1) / ks > 32) ks *= 2;   // <= 2048 K per CTA
  int row_blocks = (N + 32 * RL - 1) / (32 * RL);
  while (ks < 8 && row_blocks * ks < 2 * 148 && nkb / (2 * ks) >= 4) ks *= 2;
  return ks;
}

int gemv_rows_per_lane(int N, int epilogue) {
  if (epilogue == 2) return 2;
  return N >= 8192 ? 2 : 1;
}

int launch_gemv(const float *x, int ldx, int t, int K, const uint16_t *w, int ldw, int N,
                int prologue, const float *gain, float eps, int epilogue, float *y, int ldy,
                cudaStream_t st) {
  HS_REQUIRE(t >= 1 && K >= 1 && N >= 1, HS_ERR_SHAPE, "gemv: empty operand");
  HS_REQUIRE(ldw % 64 == 0 && ldw >= K, HS_ERR_SHAPE, "gemv: ldw %d must be a multiple of 64 >= K %d", ldw, K);
  HS_REQUIRE(epilogue != 2 || N % 2 == 0, HS_ERR_SHAPE, "gemv: swiglu needs an even N");
  const int RL = gemv_rows_per_lane(N, epilogue);
  GemvArgs a;
  a.ldx = ldx; a.K = K; a.w = w; a.ldw = ldw; a.N = N; a.prologue = prologue; a.gain = gain;
  a.eps = eps; a.epilogue = epilogue; a.ldy = ldy;
  a.nkb = ldw / 64;
  a.ks = gemv_ksplit(N, ldw, RL);
  a.kr_max = ((a.nkb + a.ks - 1) / a.ks) * 64;
  const int row_blocks = (N + 32 * RL - 1) / (32 * RL);
  for (int r0 = 0; r0 < t; r0 += GEMV_MAXT) {
    a.t = (t - r0) < GEMV_MAXT ? (t - r0) : GEMV_MAXT;
    a.x = x + (size_t)r0 * ldx;
    a.y = y + (size_t)r0 * ldy;
    cudaError_t e = RL == 2 ? launch_gemv_rl<2>(a, row_blocks, st) : launch_gemv_rl<1>(a, row_blocks, st);
    if (e != cudaSuccess) return set_error(HS_ERR_CUDA, "gemv launch: %s", cudaGetErrorString(e));
    count_launch(1);
  }
  return HS_OK;
}

}  // namespace hs

extern "C" int hs_gemv(const float *x, int ldx, int t, int K, const uint16_t *w, int ldw, int N,
                       int prologue, const float *gain, float eps, int epilogue, float *y, int ldy,
                       void *stream) {
  return hs::launch_gemv(x, ldx, t, K, w, ldw, N, prologue, gain, eps, epilogue, y, ldy,
                         hs::as_stream(stream));
}
