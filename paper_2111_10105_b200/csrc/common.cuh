// Shared device helpers for the dmcg sm_100a kernels.
//
// Exactness rules: the reference build has no FMA
// contraction (CMakeLists.txt:7-9), so every operation that must reproduce
// the reference bit for bit — the quantiser (src/quantize.cpp:22-38), the
// float range widening (src/codec.cpp:31-41) and the delta SpMM
// (src/laplacian.cpp:45) — is written with explicit round-to-nearest
// intrinsics (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn), which nvcc
// never fuses.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dmcg {

constexpr int kCB = 4;  // CG column-block width (32 B of f64 per row)

// src/quantize.cpp:22-29 (UniformQuantizer::quantize).
__device__ __forceinline__ uint32_t quantize_level(double min_, double width, uint32_t levels,
                                                   bool degenerate, double x) {
  if (degenerate) return 0u;
  const double t = floor(__ddiv_rn(__dsub_rn(x, min_), width));
  if (t <= 0.0) return 0u;
  if (t >= (double)(levels - 1u)) return levels - 1u;
  return (uint32_t)t;
}

// src/quantize.cpp:31-38 (UniformQuantizer::dequantize), no FMA.
__device__ __forceinline__ double dequantize_level(double min_, double width, bool degenerate,
                                                   uint32_t level) {
  if (degenerate) return min_;
  return __dadd_rn(min_, __dmul_rn(__dadd_rn((double)level, 0.5), width));
}

// Quantiser parameters of a float range (quantize.cpp:15-20).
struct QParams {
  double min_, width;
  uint32_t levels;
  bool degenerate;
};
__device__ __forceinline__ QParams make_qparams(float mn, float mx, int bits) {
  QParams q;
  q.levels = 1u << bits;
  q.min_ = (double)mn;
  q.degenerate = (mn == mx);
  q.width = q.degenerate ? 0.0 : __ddiv_rn(__dsub_rn((double)mx, q.min_), (double)q.levels);
  return q;
}

// src/codec.cpp:31-41 (widened_range).
__device__ __forceinline__ void widened_range(double lo, double hi, float* flo, float* fhi) {
  float a = __double2float_rn(lo);
  if ((double)a > lo) a = nextafterf(a, -INFINITY);
  float b = __double2float_rn(hi);
  if ((double)b < hi) b = nextafterf(b, INFINITY);
  *flo = a;
  *fhi = b;
}

// Order-preserving map double -> uint64 so that atomicMin/atomicMax on the
// key equals min/max on the value (finite inputs).
__device__ __forceinline__ unsigned long long ordered_key(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_to_double(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

template <typename T>
__device__ __forceinline__ double to_f64(T v) {
  return (double)v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace dmcg
