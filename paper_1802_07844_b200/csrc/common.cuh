// common.cuh -- shared device/host helpers for the sm_100a half-space Spectral-Ewald kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/hsewald_b200.h"

namespace hs {

constexpr double kPi = 3.14159265358979323846;
constexpr double kSqrtPi = 1.7724538509055160273;

// Device-side error flags (bit set) raised by kernels and checked after the stream syncs.
enum : unsigned {
  FLAG_SINGULAR = 1u,
  FLAG_OUT_OF_GRID = 2u,
  FLAG_GEOMETRY = 4u,
};

void set_error(const std::string& msg);
hs_status fail(hs_status s, const std::string& msg);

#define HS_CUDA(expr)                                                                        \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return ::hs::fail(HS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));    \
  } while (0)

#define HS_TRY(expr)                  \
  do {                                \
    hs_status _s = (expr);            \
    if (_s != HS_OK) return _s;       \
  } while (0)

// Kernel launch accounting (every launch in this library goes through HS_LAUNCHED).
extern int64_t g_launches;
#define HS_LAUNCHED(ctx)                                                            \
  do {                                                                              \
    (ctx)->launches++;                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess)                                                          \
      return ::hs::fail(HS_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(_e)); \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// --- window (_gridding.py:21-30): lo = floor((pos-origin)/h) - P/2 + 1
__device__ __forceinline__ int64_t window_lo(double pos, double origin, double h, int P) {
  return (int64_t)floor(__ddiv_rn(__dsub_rn(pos, origin), h)) - P / 2 + 1;
}
// distance of grid node (lo+a) from pos: pos - (origin + (lo+a) h)  (reference op order)
__device__ __forceinline__ double window_d(double pos, double origin, double h, int64_t idx) {
  return __dsub_rn(pos, __dadd_rn(origin, __dmul_rn((double)idx, h)));
}

// ---- checked build (make checked -> libhsewald_b200_checked.so, -DHS_CHECKED): HS_CHECK(c)
// records the first failing (translation unit, source line) and a failure count in per-TU
// device words that hs_debug_checks() collects; the production build compiles it away.
// (compute-sanitizer is closed on the GPU pool this was built on: DESIGN.md section 2.6.)
#ifdef HS_CHECKED
static __device__ unsigned long long g_chk_first;
static __device__ unsigned long long g_chk_count;
#ifndef HS_TU_ID
#define HS_TU_ID 0
#endif
#define HS_CHECK(c)                                                                               \
  do {                                                                                            \
    if (!(c)) {                                                                                   \
      atomicCAS(&::hs::g_chk_first, 0ull, ((unsigned long long)HS_TU_ID << 32) | (unsigned)__LINE__); \
      atomicAdd(&::hs::g_chk_count, 1ull);                                                        \
    }                                                                                             \
  } while (0)
#define HS_DEFINE_CHECK_COLLECT(NAME)                                                             \
  void chk_collect_##NAME(unsigned long long* first, unsigned long long* count, int reset) {       \
    unsigned long long f = 0, c = 0;                                                              \
    cudaMemcpyFromSymbol(&f, g_chk_first, sizeof(f));                                             \
    cudaMemcpyFromSymbol(&c, g_chk_count, sizeof(c));                                             \
    if (f && !*first) *first = f;                                                                 \
    *count += c;                                                                                  \
    if (reset) {                                                                                  \
      const unsigned long long z = 0;                                                             \
      cudaMemcpyToSymbol(g_chk_first, &z, sizeof(z));                                             \
      cudaMemcpyToSymbol(g_chk_count, &z, sizeof(z));                                             \
    }                                                                                             \
  }
#else
#define HS_CHECK(c) \
  do {              \
  } while (0)
#define HS_DEFINE_CHECK_COLLECT(NAME) \
  void chk_collect_##NAME(unsigned long long*, unsigned long long*, int) {}
#endif

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace hs

// Context: device, stream, scratch arenas, error flag.
struct hs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  unsigned* d_flags = nullptr;     // device error flags
  unsigned* h_flags = nullptr;     // pinned mirror
  int64_t launches = 0;
  // simple grow-only scratch arena
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
};

namespace hs {
// Grow-only scratch: returns a device pointer of at least `bytes`.
hs_status ctx_scratch(hs_ctx* ctx, size_t bytes, void** out);
// Reset device flags (async), then after sync read them; maps to a status.
hs_status ctx_reset_flags(hs_ctx* ctx);
hs_status ctx_check_flags(hs_ctx* ctx, const char* where);
}  // namespace hs
