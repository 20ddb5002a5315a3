// Shared device helpers for the B200 TriForce kernels (sm_100a).
#pragma once
#include <utility>

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>

#include "hs_abi.h"

namespace hs {

// ---- error state (hs_abi.cu) ---------------------------------------------
int set_error(int code, const char *fmt, ...);
int check_launch(const char *what, int n_kernels = 1);
void count_launch(int n);

#define HS_REQUIRE(cond, code, ...)                 \
  do {                                              \
    if (!(cond)) return ::hs::set_error(code, __VA_ARGS__); \
  } while (0)

// ---- optional per-CTA timeline (debugging/profiling aid, hs_cta_trace) -------
// Compiled in only with -DHS_CTA_TRACE (HS_TRACE_BUILD=1 python build.py):
// each translation unit owns a region of the trace buffer; an instrumented
// kernel's thread 0 records (kernel id, SM, globaltimer start, end) per CTA.
// Off by default: the per-CTA pointer load alone costs ~3% of a forward.
#ifdef HS_CTA_TRACE
#define HS_TRACE_TU                                                                          \
  static __device__ unsigned long long *g_ctrace = nullptr;                                  \
  static __device__ unsigned int g_ctrace_n = 0, g_ctrace_cap = 0;                           \
  static int trace_set_tu(void *p, unsigned cap) {                                           \
    unsigned long long *q = reinterpret_cast<unsigned long long *>(p);                       \
    unsigned zero = 0;                                                                        \
    if (cudaMemcpyToSymbol(g_ctrace, &q, sizeof(q)) != cudaSuccess) return -1;                \
    if (cudaMemcpyToSymbol(g_ctrace_n, &zero, sizeof(zero)) != cudaSuccess) return -1;        \
    if (cudaMemcpyToSymbol(g_ctrace_cap, &cap, sizeof(cap)) != cudaSuccess) return -1;        \
    return 0;                                                                                 \
  }
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define HS_TRACE_BEGIN unsigned long long hs_t0_ = g_ctrace ? gtime() : 0ull;
// restart the CTA's clock (e.g. after griddepcontrol.wait: time from the dependency release)
#define HS_TRACE_RESTART if (g_ctrace != nullptr) hs_t0_ = gtime();
#define HS_TRACE_END(kid)                                                                     \
  if (g_ctrace != nullptr && threadIdx.x == 0) {                                              \
    const unsigned i_ = atomicAdd(&g_ctrace_n, 1u);                                           \
    if (i_ < g_ctrace_cap) {                                                                  \
      unsigned sm_;                                                                           \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                                        \
      g_ctrace[(size_t)i_ * 3] = ((unsigned long long)(kid) << 32) | sm_;                     \
      g_ctrace[(size_t)i_ * 3 + 1] = hs_t0_;                                                  \
      g_ctrace[(size_t)i_ * 3 + 2] = gtime();                                                 \
    }                                                                                         \
  }
#else
#define HS_TRACE_TU \
  static int trace_set_tu(void *, unsigned) { return -1; }
#define HS_TRACE_BEGIN
#define HS_TRACE_RESTART
#define HS_TRACE_END(kid)
#endif

// ---- bf16 <-> fp32 -----------------------------------------------------------
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ float bf16_to_f(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }
__device__ __forceinline__ uint16_t f_to_bf16(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// exact 3-way bf16 split h = hi + mid + lo (8+8+8 significand bits: the full
// fp32 mantissa), the operand format of the tensor-core GEMV
__device__ __forceinline__ void split3(float h, uint16_t &a, uint16_t &b, uint16_t &c) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(h);
  const float r1 = h - __bfloat162float(hi);
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  const float r2 = r1 - __bfloat162float(mid);
  a = __bfloat16_as_ushort(hi);
  b = __bfloat16_as_ushort(mid);
  c = f_to_bf16(r2);
}

// element (row r <= 7, column k) of a split operand [24][ld]
__device__ __forceinline__ void store_split(uint16_t *xs, int ld, int r, int k, float v) {
  uint16_t a, b, c;
  split3(v, a, b, c);
  xs[(size_t)r * ld + k] = a;
  xs[(size_t)(8 + r) * ld + k] = b;
  xs[(size_t)(16 + r) * ld + k] = c;
}

// 16-byte streaming load that bypasses L1 allocation (weights, KV: read once)
__device__ __forceinline__ uint4 ld_stream(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ void unpack8(const uint4 &u, float *f) {
  f[0] = bf16_lo(u.x); f[1] = bf16_hi(u.x);
  f[2] = bf16_lo(u.y); f[3] = bf16_hi(u.y);
  f[4] = bf16_lo(u.z); f[5] = bf16_hi(u.z);
  f[6] = bf16_lo(u.w); f[7] = bf16_hi(u.w);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// RoPE + append fused into the tensor-core attention (forward path): the
// qkv GEMV output [t][ncols] and the model's fp32 rotation tables
struct FusedRope {
  const float *qkv;
  int ncols;
  const float *rope_cos, *rope_sin;
  float *q_stash;   // this layer's [H][dh] slice of the recorder stash, or null
};

// programmatic dependent launch on/off (HS_NO_PDL=1 disables it: debugging aid)
int pdl_enabled();

// launch `kern` as a programmatic dependent of the previous kernel on `st`:
// it may be scheduled once every CTA of that kernel has issued
// griddepcontrol.launch_dependents (or exited), and must itself execute
// griddepcontrol.wait before touching anything the predecessor writes
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled();
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace hs
