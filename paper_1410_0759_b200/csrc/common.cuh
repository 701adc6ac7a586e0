// Device-side helpers shared by every kernel of libdnnp.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "core.h"

namespace dnnp {

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

// Exact floor(n / d) for 32-bit n through multiply-high and shift
// (reference intdiv.py:42-60: the plain and the add-corrected forms).
__device__ __forceinline__ uint32_t mdiv(uint32_t n, const MagicDiv& m) {
  if (m.d == 1) return n;
  uint32_t t = __umulhi(n, m.mul);
  return m.add ? (t + ((n - t) >> 1)) >> (m.shift - 1) : t >> m.shift;
}
__device__ __forceinline__ void mdivmod(uint32_t n, const MagicDiv& m, uint32_t& q,
                                        uint32_t& r) {
  q = mdiv(n, m);
  r = n - q * m.d;
}

// Logical (n, c, h, w) -> element offset.
__device__ __forceinline__ int64_t voff(const View4& v, int64_t n, int64_t c, int64_t h,
                                        int64_t w) {
  return n * v.sn + c * v.sc + h * v.sh + w * v.sw;
}

template <typename T>
__device__ __forceinline__ T dmul(T a, T b);
template <>
__device__ __forceinline__ float dmul<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double dmul<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T dadd(T a, T b);
template <>
__device__ __forceinline__ float dadd<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double dadd<double>(double a, double b) { return __dadd_rn(a, b); }
template <typename T>
__device__ __forceinline__ T dsub(T a, T b);
template <>
__device__ __forceinline__ float dsub<float>(float a, float b) { return __fsub_rn(a, b); }
template <>
__device__ __forceinline__ double dsub<double>(double a, double b) { return __dsub_rn(a, b); }

// Programmatic dependent launch (sm_90+): a producer lets the next kernel
// of the stream launch early (trigger); a kernel launched with the
// programmatic-serialization attribute waits for its prerequisite grid to
// complete -- memory visible -- before it touches what that grid wrote.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline unsigned grid_for(int64_t work, int threads, int waves_cap = 32) {
  int64_t blocks = ceil_div(work, threads);
  int64_t cap = int64_t(kNumSMs) * waves_cap;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return unsigned(blocks);
}

}  // namespace dnnp
