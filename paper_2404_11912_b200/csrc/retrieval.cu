// Retrieval-cache builder: chunk scoring, top-k chunk selection, gather.
//
// Replaces score_chunks (caches.py:414-436) and RetrievalCache.build
// (caches.py:458-502).  Selection is per LAYER (scores averaged over all query
// heads), the last -- possibly partial -- chunk is always kept, ties go to the
// lower chunk id, and the victim FIFO is the reversed importance order with
// positions ascending inside a chunk.  Scores are fp64 like the reference;
// products of bf16/fp32 keys and fp32 queries are exact in fp64, so rankings
// agree with the reference except for sub-1e-16 near-ties.
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "hs_common.cuh"
#include "tc_util.cuh"

namespace hs {

constexpr int SCORE_THREADS = 256;
constexpr int SEL_THREADS = 1024;
constexpr int SEL_MAX = 8192;   // max chunks kept per layer (quota)

// grid (n_chunks, n_layers); thread = VW consecutive head dims of one kv head.
// Keys are read in batches of SB rows per (head, dims) group with every load
// of the batch -- for all of the thread's groups -- issued before any is
// consumed: a 64 KB chunk (8 keys x 32 heads x 128 dims bf16) is in flight at
// once instead of one 16-byte load per dependent step.
constexpr int SB = 8;
template <typename KT, int VW>
__global__ void __launch_bounds__(SCORE_THREADS) chunk_score_kernel(
    const KT *keys, long long ls, long long hs_, long long ts, int KVH, int DH, int upto, int chunk,
    const float *queries, int H, double *scores, int n_chunks) {
  const int c = blockIdx.x, l = blockIdx.y;
  const int b0 = c * chunk, b1 = min(upto, b0 + chunk);
  const int g = H / KVH;
  const int groups = KVH * (DH / VW);
  constexpr int GPT = 2;   // groups per thread per pass (KVH 32 x 16 vectors = 512 = 2 x 256 threads)
  double part = 0.0;
  for (int e0 = threadIdx.x; e0 < groups; e0 += GPT * SCORE_THREADS) {
    double sum[GPT][VW];
#pragma unroll
    for (int j = 0; j < GPT; ++j)
#pragma unroll
      for (int u = 0; u < VW; ++u) sum[j][u] = 0.0;
    for (int i0 = b0; i0 < b1; i0 += SB) {
      float f[GPT][SB][VW];
#pragma unroll
      for (int j = 0; j < GPT; ++j) {
        const int e = e0 + j * SCORE_THREADS;
        const int kh = e / (DH / VW), d0 = (e % (DH / VW)) * VW;
        const KT *kp = keys + l * ls + kh * hs_ + d0;
#pragma unroll
        for (int s = 0; s < SB; ++s) {
          const int i = i0 + s;
          const bool ok = e < groups && i < b1;
          if constexpr (VW == 8 && sizeof(KT) == 2) {
            const uint4 w = ok ? *reinterpret_cast<const uint4 *>(kp + (size_t)i * ts) : make_uint4(0, 0, 0, 0);
            unpack8(w, f[j][s]);
          } else if constexpr (VW == 8) {
            const float4 a = ok ? *reinterpret_cast<const float4 *>(kp + (size_t)i * ts) : make_float4(0, 0, 0, 0);
            const float4 b = ok ? *reinterpret_cast<const float4 *>(kp + (size_t)i * ts + 4) : make_float4(0, 0, 0, 0);
            f[j][s][0] = a.x; f[j][s][1] = a.y; f[j][s][2] = a.z; f[j][s][3] = a.w;
            f[j][s][4] = b.x; f[j][s][5] = b.y; f[j][s][6] = b.z; f[j][s][7] = b.w;
          } else if constexpr (sizeof(KT) == 2) {
            f[j][s][0] = ok ? bf16_to_f(kp[(size_t)i * ts]) : 0.f;
          } else {
            f[j][s][0] = ok ? kp[(size_t)i * ts] : 0.f;
          }
        }
      }
      // the reference's per-chunk key sum, in key order (caches.py:431)
#pragma unroll
      for (int j = 0; j < GPT; ++j)
#pragma unroll
        for (int s = 0; s < SB; ++s)
#pragma unroll
          for (int u = 0; u < VW; ++u) sum[j][u] += (double)f[j][s][u];
    }
    const double cnt = (double)(b1 - b0);
#pragma unroll
    for (int j = 0; j < GPT; ++j) {
      const int e = e0 + j * SCORE_THREADS;
      if (e >= groups) continue;
      const int kh = e / (DH / VW), d0 = (e % (DH / VW)) * VW;
      for (int gi = 0; gi < g; ++gi) {
        const float *qh = queries + ((size_t)l * H + kh * g + gi) * DH + d0;
#pragma unroll
        for (int u = 0; u < VW; ++u) part += (double)qh[u] * (sum[j][u] / cnt);
      }
    }
  }
  __shared__ double red[SCORE_THREADS / 32];
  part = warp_sum(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < SCORE_THREADS / 32; ++w) tot += red[w];
    double s = tot / (double)H / sqrt((double)DH);
    if (s == 0.0) s = 0.0;   // fold -0.0 so ties compare like Python floats
    scores[(size_t)l * n_chunks + c] = s;
  }
}

// ---- TMA-staged chunk scoring (bf16 keys, the build path) -------------------
// grid (ceil(n_chunks / CS_NB), n_layers), 8 consumer warps + 1 TMA warp, two
// CTAs per SM.  Each stage is one 3-D tensor-map box {dh, chunk keys, hb kv
// heads} of one chunk (hb chosen so a stage is <= 32 KB: 16 heads at chunk 8,
// dh 128), streamed through a CS_STAGES-deep ring; a chunk is KVH / hb
// stages.  Thread = (head of the stage, 8 consecutive dims): fp64 sum of the
// chunk's keys in key order (caches.py:431, exact for bf16 inputs), then the
// fp64 dot with the group's queries, accumulated over the chunk's stages;
// per chunk the 8 warp partials are summed in warp order (deterministic; the
// same arithmetic as chunk_score_kernel up to the order of the final sum).
constexpr int CS_STAGES = 3;
constexpr int CS_STAGE_BYTES = 32768;
constexpr int CS_NB = 16;            // chunks per CTA
constexpr int CS_CONSUMERS = 256;
constexpr int CS_THREADS = CS_CONSUMERS + 32;
constexpr int CS_SMEM = CS_STAGES * CS_STAGE_BYTES + 1024;

struct CsArgs {
  int KVH, DH, H, g, upto, chunk, n_chunks, hb, spc;
  const float *q;     // [L][H][DH]
  double *scores;     // [L][n_chunks]
};

__global__ void __launch_bounds__(CS_THREADS, 2) chunk_score_tma_kernel(const __grid_constant__ CUtensorMap tm,
                                                                      CsArgs a) {
  extern __shared__ __align__(128) unsigned char cs_smem[];
  unsigned char *ring = cs_smem;
  uint64_t *full = reinterpret_cast<uint64_t *>(cs_smem + CS_STAGES * CS_STAGE_BYTES);
  uint64_t *empty = full + CS_STAGES;
  __shared__ double red[CS_NB][CS_CONSUMERS / 32];
  const int l = blockIdx.y;
  const int c0 = blockIdx.x * CS_NB;
  const int nc = min(CS_NB, a.n_chunks - c0);
  const int n_st = nc * a.spc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < CS_STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], CS_CONSUMERS / 32);
    }
    tc::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t stage_bytes = (uint32_t)a.hb * a.chunk * a.DH * 2;
  if (warp == CS_CONSUMERS / 32) {
    // TMA producer
    if (lane == 0) {
      tc::tma_prefetch(&tm);
      const uint64_t pol = tc::policy_evict_first();
      for (int i = 0; i < n_st; ++i) {
        const int slot = i % CS_STAGES;
        if (i >= CS_STAGES) tc::mbar_wait_sleep(&empty[slot], ((i / CS_STAGES) - 1) & 1);
        const int c = c0 + i / a.spc, j = i % a.spc;
        tc::mbar_expect_tx(&full[slot], stage_bytes);
        tc::tma_load_3d_hint(ring + slot * CS_STAGE_BYTES, &tm, &full[slot], 0, c * a.chunk,
                             l * a.KVH + j * a.hb, pol);
      }
    }
    return;
  }
  const int dgs = a.DH / 8;
  const int hl = threadIdx.x / dgs, dg = threadIdx.x % dgs;
  const bool active = hl < a.hb;
  double part = 0.0;
  for (int i = 0; i < n_st; ++i) {
    const int slot = i % CS_STAGES;
    const int ci = i / a.spc, j = i % a.spc;
    const int c = c0 + ci;
    const int b0 = c * a.chunk, cnt = min(a.upto, b0 + a.chunk) - b0;
    tc::mbar_wait(&full[slot], (i / CS_STAGES) & 1);
    if (active) {
      const unsigned char *src = ring + slot * CS_STAGE_BYTES + ((size_t)hl * a.chunk * a.DH + dg * 8) * 2;
      double sum[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) sum[u] = 0.0;
      for (int s = 0; s < cnt; ++s) {   // key order (caches.py:431)
        float f[8];
        unpack8(*reinterpret_cast<const uint4 *>(src + (size_t)s * a.DH * 2), f);
#pragma unroll
        for (int u = 0; u < 8; ++u) sum[u] += (double)f[u];
      }
      // the chunk mean sum / cnt: for a power-of-two count the product with
      // the exact reciprocal is the same correctly rounded value, without
      // the fp64 division sequence (the partial last chunk divides)
      const double dcnt = (double)cnt;
      if ((cnt & (cnt - 1)) == 0) {
        const double rc = 1.0 / dcnt;
#pragma unroll
        for (int u = 0; u < 8; ++u) sum[u] *= rc;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) sum[u] /= dcnt;
      }
      const int kh = j * a.hb + hl;
      for (int gi = 0; gi < a.g; ++gi) {
        const float4 *qh = reinterpret_cast<const float4 *>(a.q + ((size_t)l * a.H + kh * a.g + gi) * a.DH + dg * 8);
        const float4 x = __ldg(qh), y = __ldg(qh + 1);
        const float qv[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
        for (int u = 0; u < 8; ++u) part += (double)qv[u] * sum[u];
      }
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&empty[slot]);
    if (j == a.spc - 1) {   // chunk complete: warp partial, then start the next chunk
      const double w = warp_sum(part);
      if (lane == 0) red[ci][warp] = w;
      part = 0.0;
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(CS_CONSUMERS) : "memory");
  if (threadIdx.x < nc) {
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < CS_CONSUMERS / 32; ++w) tot += red[threadIdx.x][w];
    double sc = tot / (double)a.H / sqrt((double)a.DH);
    if (sc == 0.0) sc = 0.0;   // fold -0.0 so ties compare like Python floats
    a.scores[(size_t)l * a.n_chunks + c0 + threadIdx.x] = sc;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 cs_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess && p)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// TMA path: bf16 keys laid out [layer][kv head][slot][dh] (layer stride = KVH x
// head stride), dh a multiple of 8 up to 256, 16-byte aligned strides.
// Returns 1 when launched, 0 when the geometry needs the generic kernel.
static int launch_chunk_score_tma(const void *keys, long long ls, long long hs_, long long ts, int L, int KVH,
                                  int DH, int upto, int chunk, const float *q, int H, double *scores, int n_chunks,
                                  cudaStream_t st) {
  if (DH % 8 || DH > 256 || ts != DH || ls != (long long)KVH * hs_ || (hs_ * 2) % 16 || ((uintptr_t)keys % 16) ||
      ((uintptr_t)q % 16) || chunk > 256 || DH / 8 > CS_CONSUMERS)
    return 0;
  int hb = KVH < CS_CONSUMERS / (DH / 8) ? KVH : CS_CONSUMERS / (DH / 8);
  while (hb > 1 && ((long long)hb * chunk * DH * 2 > CS_STAGE_BYTES || KVH % hb)) --hb;
  if ((long long)hb * chunk * DH * 2 > CS_STAGE_BYTES || hb > 256) return 0;
  auto enc = cs_encode();
  if (!enc) return 0;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)DH, (cuuint64_t)upto, (cuuint64_t)L * KVH};
  cuuint64_t strides[2] = {(cuuint64_t)ts * 2, (cuuint64_t)hs_ * 2};
  cuuint32_t box[3] = {(cuuint32_t)DH, (cuuint32_t)chunk, (cuuint32_t)hb};
  cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(keys), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 0;
  CsArgs a;
  a.KVH = KVH; a.DH = DH; a.H = H; a.g = H / KVH; a.upto = upto; a.chunk = chunk; a.n_chunks = n_chunks;
  a.hb = hb; a.spc = KVH / hb; a.q = q; a.scores = scores;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(chunk_score_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, CS_SMEM);
    attr = true;
  }
  dim3 grid(ceil_div(n_chunks, CS_NB), L);
  chunk_score_tma_kernel<<<grid, CS_THREADS, CS_SMEM, st>>>(m, a);
  return 1;
}

__device__ __forceinline__ unsigned long long order_key(double s) {
  unsigned long long u = (unsigned long long)__double_as_longlong(s);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// ascending by (key desc, id asc) == "better first"
__device__ __forceinline__ bool better(unsigned long long ka, int ia, unsigned long long kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

// in-smem bitonic sort of n (power of two) (key,id) pairs, best first
__device__ void bitonic_best_first(unsigned long long *key, int *id, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const bool sw = up ? better(key[hi], id[hi], key[lo], id[lo]) : better(key[lo], id[lo], key[hi], id[hi]);
        if (sw) {
          unsigned long long tk = key[lo]; key[lo] = key[hi]; key[hi] = tk;
          int ti = id[lo]; id[lo] = id[hi]; id[hi] = ti;
        }
      }
    }
  }
  __syncthreads();
}

__device__ void bitonic_ints_ascending(int *v, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        if ((v[lo] > v[hi]) == up) { int t = v[lo]; v[lo] = v[hi]; v[hi] = t; }
      }
    }
  }
  __syncthreads();
}

// one CTA per layer
__global__ void __launch_bounds__(SEL_THREADS) chunk_select_kernel(
    const double *scores, int n, int k_sel, int chunk, int upto, int quota, int budget,
    int32_t *importance, int32_t *chosen, int32_t *ring, int32_t *counts) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned long long *skey = reinterpret_cast<unsigned long long *>(sm);   // [SEL_MAX]
  int *sid = reinterpret_cast<int *>(skey + SEL_MAX);                        // [SEL_MAX]
  int *asc = sid + SEL_MAX;                                                  // [SEL_MAX]
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long prefix_s;
  __shared__ int remaining_s, nsel_s;
  __shared__ int wscan[SEL_THREADS / 32];

  const int l = blockIdx.x, tid = threadIdx.x;
  const double *sc = scores + (size_t)l * n;
  const int ncand = n - 1;              // the last chunk is pinned
  const int last = n - 1;

  unsigned long long T = 0;             // threshold key
  int take_eq;                          // how many == T to take (lowest ids)
  bool all = (k_sel >= ncand);
  if (!all) {
    unsigned long long prefix = 0, mask = 0;
    int remaining = k_sel;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += SEL_THREADS) hist[i] = 0;
      __syncthreads();
      for (int i = tid; i < ncand; i += SEL_THREADS) {
        unsigned long long k = order_key(sc[i]);
        if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255ull], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        unsigned int cum = 0;
        int digit = 0;
        for (int d = 255; d >= 0; --d) {
          if (cum + hist[d] >= (unsigned)remaining) { digit = d; break; }
          cum += hist[d];
        }
        remaining_s = remaining - (int)cum;
        prefix_s = prefix | ((unsigned long long)digit << shift);
      }
      __syncthreads();
      remaining = remaining_s;
      prefix = prefix_s;
      mask |= 0xFFull << shift;
    }
    T = prefix;
    take_eq = remaining;
  } else {
    take_eq = 0;
  }
  if (tid == 0) nsel_s = 0;
  __syncthreads();
  // ---- collect: key > T all; key == T the take_eq lowest ids ----------------
  int eq_base = 0;
  for (int c0 = 0; c0 < ncand; c0 += SEL_THREADS) {
    const int i = c0 + tid;
    unsigned long long k = (i < ncand) ? order_key(sc[i]) : 0;
    const bool gt = (i < ncand) && (all || k > T);
    const bool eq = (i < ncand) && !all && (k == T);
    if (gt) {
      int slot = atomicAdd(&nsel_s, 1);
      skey[slot] = k; sid[slot] = i;
    }
    // ordered exclusive scan of eq flags across the block
    unsigned int ball = __ballot_sync(0xffffffffu, eq);
    int lane = tid & 31, w = tid >> 5;
    int before_in_warp = __popc(ball & ((1u << lane) - 1u));
    if (lane == 0) wscan[w] = __popc(ball);
    __syncthreads();
    int before = 0, total = 0;
    for (int ww = 0; ww < SEL_THREADS / 32; ++ww) {
      if (ww < w) before += wscan[ww];
      total += wscan[ww];
    }
    if (eq && eq_base + before + before_in_warp < take_eq) {
      int slot = atomicAdd(&nsel_s, 1);
      skey[slot] = k; sid[slot] = i;
    }
    eq_base += total;
    __syncthreads();
  }
  const int nsel = nsel_s;   // == k_sel (or ncand when all)
  int P = 1;
  while (P < nsel) P <<= 1;
  for (int i = nsel + tid; i < P; i += SEL_THREADS) { skey[i] = 0; sid[i] = 0x7fffffff; }
  bitonic_best_first(skey, sid, P);
  // importance = [last] + best-first rest
  int32_t *imp = importance + (size_t)l * quota;
  for (int i = tid; i < nsel + 1; i += SEL_THREADS) imp[i] = (i == 0) ? last : sid[i - 1];
  // chosen ascending
  int Q = 1;
  while (Q < nsel + 1) Q <<= 1;
  for (int i = tid; i < Q; i += SEL_THREADS) asc[i] = (i < nsel) ? sid[i] : (i == nsel ? last : 0x7fffffff);
  bitonic_ints_ascending(asc, Q);
  int32_t *ch = chosen + (size_t)l * quota;
  for (int i = tid; i < nsel + 1; i += SEL_THREADS) ch[i] = asc[i];
  // victim ring (slot indices): reversed importance order, ascending inside a chunk
  const int last_size = upto - last * chunk;
  int32_t *rg = ring + (size_t)l * budget;
  for (int e = tid; e <= nsel; e += SEL_THREADS) {
    const int cid = (e == nsel) ? last : sid[nsel - 1 - e];
    // slot base = rank of cid in asc * chunk (binary search)
    int lo = 0, hi = nsel;   // asc[0..nsel] valid
    while (lo < hi) { int mid = (lo + hi) >> 1; if (asc[mid] < cid) lo = mid + 1; else hi = mid; }
    const int base = lo * chunk;
    const int sz = (cid == last) ? last_size : chunk;
    for (int u = 0; u < sz; ++u) rg[e * chunk + u] = base + u;
  }
  if (l == 0 && tid == 0) {
    counts[0] = nsel + 1;
    counts[1] = nsel * chunk + last_size;
  }
}

// grid (n_chosen, KVH, L): copy chunk tokens (position order) into slots j*chunk..
// src holds positions [src_lo, src_hi) (a sequence shard; src_hi 0 = no bound);
// the K/V slots of chosen chunks outside it are left untouched (their owner
// rank ships them, hs_retrieval_exchange); positions are written for all.
__global__ void retrieval_gather_kernel(HsCache src, HsCache dst, const int32_t *chosen, int quota,
                                        int chunk, int upto, int src_lo, int src_hi) {
  const int j = blockIdx.x, kh = blockIdx.y, l = blockIdx.z, DH = src.head_dim;
  const int cid = chosen[(size_t)l * quota + j];
  const int p0 = cid * chunk, p1 = min(upto, p0 + chunk);
  const int n = p1 - p0;
  const bool mine = p0 >= src_lo && (src_hi == 0 || p0 < src_hi);
  uint16_t *kd = dst.k + (((size_t)l * dst.n_kv_heads + kh) * dst.cap + (size_t)j * chunk) * DH;
  uint16_t *vd = dst.v + (((size_t)l * dst.n_kv_heads + kh) * dst.cap + (size_t)j * chunk) * DH;
  const int nvec = n * DH / 8;
  if (mine) {
    const uint16_t *ks = src.k + (((size_t)l * src.n_kv_heads + kh) * src.cap + (p0 - src_lo)) * DH;
    const uint16_t *vs = src.v + (((size_t)l * src.n_kv_heads + kh) * src.cap + (p0 - src_lo)) * DH;
    for (int e = threadIdx.x; e < nvec; e += blockDim.x) {
      reinterpret_cast<uint4 *>(kd)[e] = ld_stream(reinterpret_cast<const uint4 *>(ks) + e);
      reinterpret_cast<uint4 *>(vd)[e] = ld_stream(reinterpret_cast<const uint4 *>(vs) + e);
    }
  }
  if (kh == 0)
    for (int u = threadIdx.x; u < n; u += blockDim.x) dst.pos[(size_t)l * dst.cap + j * chunk + u] = p0 + u;
}

}  // namespace hs

extern "C" int hs_chunk_score(const void *keys, int key_bf16, long long layer_stride, long long head_stride,
                              long long token_stride, int n_layers, int n_kv_heads, int head_dim, int upto,
                              int chunk, const float *queries, int n_heads, double *scores, void *stream) {
  if (upto < 1) return hs::set_error(HS_ERR_CONTRACT, "retrieval build needs a non-empty source prefix");
  if (chunk < 1 || n_heads % n_kv_heads != 0)
    return hs::set_error(HS_ERR_SHAPE, "chunk_score: bad geometry (chunk %d, heads %d/%d)", chunk, n_heads, n_kv_heads);
  const int n_chunks = hs::ceil_div(upto, chunk);
  dim3 grid(n_chunks, n_layers);
  cudaStream_t st = hs::as_stream(stream);
  const bool vec = head_dim % 8 == 0 && token_stride % 8 == 0 && head_stride % 8 == 0 && layer_stride % 8 == 0 &&
                   ((uintptr_t)keys % 16) == 0 && ((uintptr_t)queries % 16) == 0;
#define HS_SCORE(KT, VW)                                                                                 \
  hs::chunk_score_kernel<KT, VW><<<grid, hs::SCORE_THREADS, 0, st>>>((const KT *)keys, layer_stride,    \
      head_stride, token_stride, n_kv_heads, head_dim, upto, chunk, queries, n_heads, scores, n_chunks)
  static const bool no_tma = getenv("HS_SCORE_NO_TMA") != nullptr;   // A/B hook: the generic kernel
  if (key_bf16 && !no_tma &&
      hs::launch_chunk_score_tma(keys, layer_stride, head_stride, token_stride, n_layers, n_kv_heads, head_dim, upto,
                                 chunk, queries, n_heads, scores, n_chunks, st))
    return hs::check_launch("chunk_score");
  if (key_bf16) { if (vec) HS_SCORE(uint16_t, 8); else HS_SCORE(uint16_t, 1); }
  else { if (vec) HS_SCORE(float, 8); else HS_SCORE(float, 1); }
#undef HS_SCORE
  return hs::check_launch("chunk_score");
}

extern "C" size_t hs_chunk_select_workspace_bytes(int n_layers, int n_chunks) { return 0; }

extern "C" int hs_chunk_select(const double *scores, int n_layers, int n_chunks, int upto, int chunk,
                               int budget, int32_t *importance, int32_t *chosen, int32_t *ring,
                               int32_t *out_counts, void *workspace, size_t ws_bytes, void *stream) {
  if (budget < chunk || budget % chunk) return hs::set_error(HS_ERR_VALUE, "budget must be a multiple of chunk_size");
  const int quota = budget / chunk;
  if (quota > hs::SEL_MAX) return hs::set_error(HS_ERR_VALUE, "quota %d exceeds %d", quota, hs::SEL_MAX);
  if (n_chunks != hs::ceil_div(upto, chunk)) return hs::set_error(HS_ERR_SHAPE, "chunk_select: n_chunks mismatch");
  const bool clamped = budget >= upto;
  int k_sel = clamped ? n_chunks - 1 : quota - 1;
  if (k_sel > n_chunks - 1) k_sel = n_chunks - 1;
  const size_t smem = (size_t)hs::SEL_MAX * (8 + 4 + 4);
  auto kern = hs::chunk_select_kernel;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<n_layers, hs::SEL_THREADS, smem, hs::as_stream(stream)>>>(scores, n_chunks, k_sel, chunk, upto, quota,
                                                                  budget, importance, chosen, ring, out_counts);
  return hs::check_launch("chunk_select");
}

extern "C" int hs_retrieval_gather(const HsCache *src, const HsCache *dst, const int32_t *chosen, int chosen_stride,
                                   int n_chosen, int chunk, int upto, int src_lo, int src_hi, void *stream) {
  if (dst->kind != HS_KV_SLOTTED) return hs::set_error(HS_ERR_VALUE, "gather: destination must be slotted");
  if ((long long)n_chosen * chunk > dst->cap) return hs::set_error(HS_ERR_CAPACITY, "gather: %d chunks exceed capacity", n_chosen);
  if (src->head_dim != dst->head_dim || src->n_kv_heads != dst->n_kv_heads || src->n_layers != dst->n_layers)
    return hs::set_error(HS_ERR_SHAPE, "gather: geometry mismatch");
  if ((src_hi > 0 ? (src_hi < upto ? src_hi : upto) : upto) - src_lo > src->cap)
    return hs::set_error(HS_ERR_CONTRACT, "source cache shorter than requested build range");
  if (src_lo % chunk != 0 || (src_hi > 0 && src_hi % chunk != 0))
    return hs::set_error(HS_ERR_VALUE, "gather: shard bounds [%d, %d) not chunk-aligned", src_lo, src_hi);
  dim3 grid(n_chosen, src->n_kv_heads, src->n_layers);
  hs::retrieval_gather_kernel<<<grid, 128, 0, hs::as_stream(stream)>>>(*src, *dst, chosen, chosen_stride, chunk, upto,
                                                                        src_lo, src_hi);
  return hs::check_launch("retrieval_gather");
}
