// Causal prefill attention for head_dim 128 on the tensor cores (tcgen05 + TMA),
// 128 query rows per CTA -- the attention core of the batched prefill
// `_forward` (model.py:290-315 over model.py:348-349) for long prompts.
//
// The decode kernel (attention_tc.cu) is built for <= 8 query rows: keys on
// the MMA's M side, one thread per key, so every query row costs cross-warp
// reductions per tile.  Here the orientation is flipped:
//   S[128 q x 64 keys]   = sum_i Q_i . K^T       (Q split exactly into 3 bf16 terms)
//   softmax per row in registers: thread = query row = TMEM lane
//   O_tile[128 q x 128 dh] = sum_i P_i . V       (P split into 2 bf16 terms)
//   o += o * fac + O_tile in registers (online softmax, fp32)
// Products of the Q splits with the bf16 keys are exact, so the scores are
// fp32-accurate; P in probability units is carried to 16 significand bits
// (relative 2^-17), below the fp32 accumulation noise of a long row.
//
// Warp roles (192 threads): warps 0-3 softmax (row = 32 w + lane), warp 4 TMA
// producer (3-stage K and V rings of 64-key tiles), warp 5 MMA issuer.  S and
// O are double buffered in TMEM, so S(j+1) runs on the tensor core while the
// softmax of tile j and the fold of O(j-1) run in registers.  One CTA per SM
// (225 KB shared memory); heavy (late) query tiles are scheduled first.
#include "hs_common.cuh"
#include "tc_util.cuh"

namespace hs {

int get_tmap_bf16(const void *ptr, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes, uint32_t box_rows,
                  CUtensorMap *out);

namespace {

constexpr int PA_DH = 128;
constexpr int PA_QT = 128;                     // query rows per CTA (MMA M)
constexpr int PA_KT = 64;                      // keys per tile (MMA N of S, K of P.V)
constexpr int PA_NS = 3;                       // K and V ring stages
constexpr int PA_ATOM = 128 * 64 * 2;          // one [128 rows x 64] bf16 SW128 atom = 16 KB
constexpr int PA_OP = 2 * PA_ATOM;             // one [128 x 128] bf16 operand (a Q split) = 32 KB
constexpr int PA_KATOM = PA_KT * 64 * 2;       // [64 keys x 64 dh] half of a K or V tile = 8 KB
constexpr int PA_KV = 2 * PA_KATOM;            // one K or V stage = 16 KB
constexpr int PA_THREADS = 192;
constexpr int PA_SMEM = 3 * PA_OP /*Q*/ + 2 * PA_NS * PA_KV /*K, V*/ + 2 * PA_ATOM /*P*/ + 1024;

struct PrefillArgs {
  const float *q;       // [t][H][128] roped queries
  float *out;           // [t][H*128] normalised rows, or null
  float *packed;        // [t*H][2 + 128] partial state (m, l, o) of this key range, or null
  int t, H, KVH, g, layer, cap, pos0, n_keys, pos_base;   // key slot s holds position s + pos_base
  float scale_log2;
};

// byte offset of element (row, col) in a K-major SW128 [128 x 128] operand
__device__ __forceinline__ uint32_t chunk_off(int row, int chunk16) {   // chunk16 = col / 8
  return (uint32_t)((chunk16 >> 3) * PA_ATOM + row * 128 + ((((chunk16 & 7) ^ (row & 7)) & 7) << 4));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const uint32_t lo = __bfloat16_as_ushort(__float2bfloat16_rn(a));
  const uint32_t hi = __bfloat16_as_ushort(__float2bfloat16_rn(b));
  return lo | (hi << 16);
}

// {lo, hi} -> packed bf16x2 (round to nearest), one instruction
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 32 lanes x 32 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(PA_THREADS, 1) prefill_attn_kernel(const __grid_constant__ CUtensorMap tmK,
                                                                    const __grid_constant__ CUtensorMap tmV,
                                                                    PrefillArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *sQ = base;                  // 3 splits x 32 KB
  unsigned char *sK = sQ + 3 * PA_OP;        // PA_NS x 16 KB
  unsigned char *sV = sK + PA_NS * PA_KV;    // PA_NS x 16 KB
  unsigned char *sP = sV + PA_NS * PA_KV;    // 2 splits x [128 rows x 64 keys] = 2 x 16 KB
  __shared__ uint64_t kfull[PA_NS], kempty[PA_NS], vfull[PA_NS], vempty[PA_NS];
  __shared__ uint64_t sfull[2], sfree[2], pfull, pfree, ofull[2], ofree[2], qfull;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (a.t + PA_QT - 1) / PA_QT;
  const int qt = n_qt - 1 - (int)blockIdx.x;           // heavy (late) tiles first
  const int h = blockIdx.y, kh = h / a.g;
  const int r0 = qt * PA_QT;
  const int rows = min(PA_QT, a.t - r0);
  // slots [0, kend) are visible to some row (a sequence shard's slots may all
  // lie past the tile's queries: ntiles = 0, the rows' partial state is empty)
  const int kend = max(0, min(a.n_keys, a.pos0 + r0 + rows - a.pos_base));
  const int ntiles = (kend + PA_KT - 1) / PA_KT;
  const int qmin = a.pos0 + r0 - a.pos_base;           // first query position of the tile, in slots

  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tmK);
    tc::tma_prefetch(&tmV);
    for (int st = 0; st < PA_NS; ++st) {
      tc::mbar_init(&kfull[st], 1); tc::mbar_init(&kempty[st], 1); tc::mbar_init(&vfull[st], 1);
      tc::mbar_init(&vempty[st], 1);
    }
    tc::mbar_init(&pfull, 4); tc::mbar_init(&pfree, 1); tc::mbar_init(&qfull, 4);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&sfull[b], 1); tc::mbar_init(&sfree[b], 4); tc::mbar_init(&ofull[b], 1); tc::mbar_init(&ofree[b], 4);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);     // S[b] at 64 b, O[b] at 128 + 128 b
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  // ------------------------------------------------------------------ TMA producer
  if (warp == 4) {
    if (tc::elect_one()) {
      const int row0 = (a.layer * a.KVH + kh) * a.cap;
      for (int j = 0; j < ntiles; ++j) {
        const int st = j % PA_NS;
        const uint32_t ph = (j / PA_NS) & 1;
        tc::mbar_wait_sleep(&kempty[st], ph ^ 1);
        tc::mbar_expect_tx(&kfull[st], PA_KV);
        tc::tma_load_2d(sK + st * PA_KV, &tmK, &kfull[st], 0, row0 + j * PA_KT);
        tc::tma_load_2d(sK + st * PA_KV + PA_KATOM, &tmK, &kfull[st], 64, row0 + j * PA_KT);
        tc::mbar_wait_sleep(&vempty[st], ph ^ 1);
        tc::mbar_expect_tx(&vfull[st], PA_KV);
        tc::tma_load_2d(sV + st * PA_KV, &tmV, &vfull[st], 0, row0 + j * PA_KT);
        tc::tma_load_2d(sV + st * PA_KV + PA_KATOM, &tmV, &vfull[st], 64, row0 + j * PA_KT);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ MMA issuer
  if (warp == 5) {
    if (tc::elect_one()) {
      constexpr uint32_t idS = tc::idesc_bf16(128, PA_KT, 0, 0);
      constexpr uint32_t idO = tc::idesc_bf16(128, 128, 0, 1);
      auto issue_S = [&](int j) {
        const int b = j & 1, st = j % PA_NS;
        tc::mbar_wait_sleep(&kfull[st], (j / PA_NS) & 1);
        tc::mbar_wait_sleep(&sfree[b], ((j >> 1) & 1) ^ 1);
        tc::fence_after();
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int kk = 0; kk < PA_DH / 16; ++kk) {
            const uint64_t da = tc::desc_k_sw128(sQ + i * PA_OP + (kk >> 2) * PA_ATOM) + 2 * (kk & 3);
            const uint64_t db = tc::desc_k_sw128(sK + st * PA_KV + (kk >> 2) * PA_KATOM) + 2 * (kk & 3);
            tc::mma_bf16(tmem + b * PA_KT, da, db, idS, (i | kk) != 0);
          }
        tc::mma_commit(&kempty[st]);
        tc::mma_commit(&sfull[b]);
      };
      auto issue_PV = [&](int j) {
        const int b = j & 1, st = j % PA_NS;
        tc::mbar_wait_sleep(&pfull, j & 1);
        tc::mbar_wait_sleep(&vfull[st], (j / PA_NS) & 1);
        tc::mbar_wait_sleep(&ofree[b], ((j >> 1) & 1) ^ 1);
        tc::fence_after();
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int kk = 0; kk < PA_KT / 16; ++kk) {
            const uint64_t da = tc::desc_k_sw128(sP + i * PA_ATOM) + 2 * kk;
            // B = V [keys x dh], dh contiguous (MN-major): 64-dh blocks 8 KB apart, 8-key groups 1 KB apart
            const uint64_t db = tc::desc_mn_sw128(sV + st * PA_KV + kk * 2048, PA_KATOM, 1024);
            tc::mma_bf16(tmem + 128 + b * 128, da, db, idO, (i | kk) != 0);
          }
        tc::mma_commit(&vempty[st]);
        tc::mma_commit(&pfree);
        tc::mma_commit(&ofull[b]);
      };
      tc::mbar_wait_sleep(&qfull, 0);
      if (ntiles > 0) issue_S(0);
      for (int j = 0; j < ntiles; ++j) {
        if (j + 1 < ntiles) issue_S(j + 1);
        issue_PV(j);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ softmax warps 0-3
  const int r = warp * 32 + lane;                      // query row of this thread = TMEM lane
  const uint32_t tl = (uint32_t)(warp * 32) << 16;
  const int qp = a.pos0 + r0 + r - a.pos_base;         // its position, in slots (may be < 0 on a shard)
  {  // stage Q (3-way exact split), zero rows past t
    const float *qrow = a.q + ((size_t)(r0 + r) * a.H + h) * PA_DH;
#pragma unroll 2
    for (int c = 0; c < PA_DH / 8; ++c) {
      float v[8];
      if (r < rows) {
        const float4 x0 = *reinterpret_cast<const float4 *>(qrow + 8 * c);
        const float4 x1 = *reinterpret_cast<const float4 *>(qrow + 8 * c + 4);
        v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w; v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = 0.f;
      }
      uint32_t p0[4], p1[4], p2[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float h0[2], m0[2], l0[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float x = v[2 * e + u];
          h0[u] = __bfloat162float(__float2bfloat16_rn(x));
          const float rr = x - h0[u];
          m0[u] = __bfloat162float(__float2bfloat16_rn(rr));
          l0[u] = rr - m0[u];
        }
        p0[e] = pack_bf16(h0[0], h0[1]);
        p1[e] = pack_bf16(m0[0], m0[1]);
        p2[e] = pack_bf16(l0[0], l0[1]);
      }
      const uint32_t off = chunk_off(r, c);
      *reinterpret_cast<uint4 *>(sQ + off) = make_uint4(p0[0], p0[1], p0[2], p0[3]);
      *reinterpret_cast<uint4 *>(sQ + PA_OP + off) = make_uint4(p1[0], p1[1], p1[2], p1[3]);
      *reinterpret_cast<uint4 *>(sQ + 2 * PA_OP + off) = make_uint4(p2[0], p2[1], p2[2], p2[3]);
    }
    tc::fence_async_smem();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&qfull);
  }

  float o_acc[PA_DH];
#pragma unroll
  for (int d = 0; d < PA_DH; ++d) o_acc[d] = 0.f;
  float m_run = -INFINITY, l_run = 0.f, fac_prev = 1.f;

  auto fold = [&](int j, float fac) {   // o = o * fac + O_tile(j)
    const int b = j & 1;
    tc::mbar_wait_sleep(&ofull[b], (j >> 1) & 1);
    tc::fence_after();
#pragma unroll
    for (int c = 0; c < PA_DH / 32; ++c) {
      float ov[32];
      tmem_ld32(tmem + 128 + b * 128 + c * 32 + tl, ov);
      tc::tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) o_acc[32 * c + e] = fmaf(o_acc[32 * c + e], fac, ov[e]);
    }
    tc::fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&ofree[b]);
  };

  for (int j = 0; j < ntiles; ++j) {
    const int b = j & 1;
    const int k0 = j * PA_KT;
    const bool masked = k0 + PA_KT - 1 > qmin || k0 + PA_KT > kend;   // some key of the tile invisible to some row
    tc::mbar_wait_sleep(&sfull[b], (j >> 1) & 1);
    tc::fence_after();
    float sv[PA_KT];
    tmem_ld32(tmem + b * PA_KT + tl, sv);
    tmem_ld32(tmem + b * PA_KT + 32 + tl, sv + 32);
    tc::tmem_ld_wait();
    tc::fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&sfree[b]);         // S is in registers: the buffer is free
    // scores in the log2 domain; invisible keys -> -inf (exp2 -> +0)
    if (masked) {
#pragma unroll
      for (int e = 0; e < PA_KT; ++e) {
        const int kp = k0 + e;
        sv[e] = (kp <= qp && kp < a.n_keys) ? sv[e] * a.scale_log2 : -INFINITY;
      }
    } else {
#pragma unroll
      for (int e = 0; e < PA_KT; ++e) sv[e] *= a.scale_log2;
    }
    float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};   // independent chains
#pragma unroll
    for (int e = 0; e < PA_KT; ++e) mx4[e & 3] = fmaxf(mx4[e & 3], sv[e]);
    const float m_new = fmaxf(m_run, fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])));
    // a row with nothing visible yet (shard slots past its position) keeps m = -inf: p = 0, fac = 0
    const float m_ref = m_new == -INFINITY ? 0.f : m_new;
    const float fac = ex2f(m_run - m_ref);              // ex2(-inf) = 0 on the first tile
    // P = exp2(s - m), split into 2 bf16 terms -> smem (the previous P.V must be done with it)
    tc::mbar_wait_sleep(&pfree, (j & 1) ^ 1);
    float sm4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q8 = 0; q8 < PA_KT / 8; ++q8) {           // 8 chunks of 8 keys
      uint32_t h4[4], m4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p0 = ex2f(sv[8 * q8 + 2 * e] - m_ref), p1 = ex2f(sv[8 * q8 + 2 * e + 1] - m_ref);
        sm4[e] += p0 + p1;
        const uint32_t hp = cvt_bf16x2(p0, p1);
        const float h0 = __uint_as_float(hp << 16), h1 = __uint_as_float(hp & 0xffff0000u);
        h4[e] = hp;
        m4[e] = cvt_bf16x2(p0 - h0, p1 - h1);
      }
      const uint32_t off = chunk_off(r, q8);
      *reinterpret_cast<uint4 *>(sP + off) = make_uint4(h4[0], h4[1], h4[2], h4[3]);
      *reinterpret_cast<uint4 *>(sP + PA_ATOM + off) = make_uint4(m4[0], m4[1], m4[2], m4[3]);
    }
    const float sum = (sm4[0] + sm4[1]) + (sm4[2] + sm4[3]);
    tc::fence_async_smem();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&pfull);
    l_run = l_run * fac + sum;
    if (j > 0) fold(j - 1, fac_prev);
    fac_prev = fac;
    m_run = m_new;
  }
  if (ntiles > 0) fold(ntiles - 1, fac_prev);
  if (r < rows && a.packed) {
    float *pk = a.packed + ((size_t)(r0 + r) * a.H + h) * (PA_DH + 2);
    pk[0] = m_run == -INFINITY ? -INFINITY : m_run * 0.69314718055994530942f;   // natural-log units
    pk[1] = l_run;
#pragma unroll
    for (int d = 0; d < PA_DH; ++d) pk[2 + d] = o_acc[d];
  } else if (r < rows) {
    const float inv = 1.f / l_run;
    float *orow = a.out + (size_t)(r0 + r) * a.H * PA_DH + (size_t)h * PA_DH;
#pragma unroll
    for (int d = 0; d < PA_DH; d += 4)
      *reinterpret_cast<float4 *>(orow + d) =
          make_float4(o_acc[d] * inv, o_acc[d + 1] * inv, o_acc[d + 2] * inv, o_acc[d + 3] * inv);
  }
  tc::fence_before();
  asm volatile("bar.sync 1, 128;" ::: "memory");       // the 4 softmax warps: all TMEM reads done
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

// causal attention of t query rows at positions [pos0, pos0 + t) over the
// slots [0, n_keys) of a linear, unwindowed cache whose slot s holds position
// s + pos_base (a sequence shard; 0 for a whole cache).  out: normalised rows;
// packed: this key range's partial state per row, for the rank-ordered merge.
int launch_prefill_attention(const HsCache *c, int layer, int H, const float *q, int t, int pos0, int pos_base,
                             int n_keys, float *out, float *packed, cudaStream_t stream) {
  HS_REQUIRE(c->head_dim == PA_DH, HS_ERR_SHAPE, "prefill attention: head_dim must be 128");
  HS_REQUIRE(H % c->n_kv_heads == 0, HS_ERR_SHAPE, "prefill attention: H %% KVH != 0");
  HS_REQUIRE(c->kind == HS_KV_LINEAR, HS_ERR_VALUE, "prefill attention: needs a linear (full) cache");
  HS_REQUIRE(n_keys >= 0 && n_keys <= c->cap, HS_ERR_CAPACITY, "prefill attention: bad key range");
  HS_REQUIRE(packed != nullptr || n_keys + pos_base >= pos0 + 1, HS_ERR_VALUE,
             "prefill attention: normalised output needs every query's keys");
  HS_REQUIRE(t >= 1, HS_ERR_VALUE, "prefill attention: empty query block");
  CUtensorMap mk, mv;
  const uint64_t rows = (uint64_t)c->n_layers * c->n_kv_heads * c->cap;
  int rc = get_tmap_bf16(c->k, PA_DH, rows, PA_DH * 2, PA_KT, &mk);
  if (rc != HS_OK) return rc;
  rc = get_tmap_bf16(c->v, PA_DH, rows, PA_DH * 2, PA_KT, &mv);
  if (rc != HS_OK) return rc;
  PrefillArgs a;
  a.q = q; a.out = out; a.packed = packed; a.t = t; a.H = H; a.KVH = c->n_kv_heads; a.g = H / c->n_kv_heads;
  a.layer = layer; a.cap = c->cap; a.pos0 = pos0; a.n_keys = n_keys; a.pos_base = pos_base;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)PA_DH));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prefill_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PA_SMEM);
    attr = true;
  }
  dim3 grid((t + PA_QT - 1) / PA_QT, H);
  prefill_attn_kernel<<<grid, PA_THREADS, PA_SMEM, stream>>>(mk, mv, a);
  return check_launch("prefill_attention");
}

}  // namespace hs

// per-layer public entry (hs_abi.h): attention of t query rows at positions
// st->pos0.. over the cache's slots [0, st->n_view) (positions + st->pos_base)
extern "C" int hs_prefill_attention(const HsCache *c, int layer, const HsStep *st, int n_heads, const float *q,
                                    int t, float *out, float *packed, void *stream) {
  HS_REQUIRE(c != nullptr && st != nullptr && q != nullptr, HS_ERR_VALUE, "prefill attention: null argument");
  HS_REQUIRE((out != nullptr) != (packed != nullptr), HS_ERR_VALUE, "prefill attention: exactly one of out / packed");
  HS_REQUIRE(layer >= 0 && layer < c->n_layers, HS_ERR_VALUE, "prefill attention: layer %d out of range", layer);
  return hs::launch_prefill_attention(c, layer, n_heads, q, t, st->pos0, st->pos_base, st->n_view, out, packed,
                                      hs::as_stream(stream));
}
