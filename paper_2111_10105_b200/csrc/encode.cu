// Encode-side kernels that must reproduce the reference arithmetic exactly.
// Compiled with --fmad=false (and explicit _rn intrinsics) because the
// reference Release build has no FMA contraction (CMakeLists.txt:7-9).
#include <cfloat>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace dmcg {

namespace {

// K1 — delta coordinates (src/laplacian.cpp:39-46, called at codec.cpp:419).
// One warp per vertex row; lanes stride the F frames (coalesced 256 B /
// 128 B per warp access).  The row's CSR column list is sorted with the
// diagonal in place, so accumulating in list order reproduces Eigen's
// column-major sparse x dense product order; L's values are implicit
// (degree on the diagonal, -1 off it: laplacian.cpp:27-30).
constexpr int kDeltaWarps = 8;
constexpr int kDeltaChunk = 8;  // 8 x 32 = 256 frames per pass

template <typename T>
__global__ void __launch_bounds__(kDeltaWarps * 32)
    k_delta(int n, int F, const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
            const T* __restrict__ x0, const T* __restrict__ x1, const T* __restrict__ x2,
            double* __restrict__ delta, int* flags, int a0) {
  const int a = blockIdx.y + a0;
  const T* __restrict__ X = a == 0 ? x0 : (a == 1 ? x1 : x2);
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kDeltaWarps + (threadIdx.x >> 5);
  if (i >= n) return;
  const uint32_t pb = rp[i], pe = rp[i + 1];
  const double deg = (double)(pe - pb - 1);
  double* out = delta + ((size_t)a * n + i) * F;
  bool bad = false;
  for (int f0 = 0; f0 < F; f0 += 32 * kDeltaChunk) {
    double acc[kDeltaChunk];
#pragma unroll
    for (int c = 0; c < kDeltaChunk; ++c) acc[c] = 0.0;
    for (uint32_t p = pb; p < pe; ++p) {
      const uint32_t j = ci[p];
      const double v = (j == (uint32_t)i) ? deg : -1.0;
      const T* xr = X + (size_t)j * F;
#pragma unroll
      for (int c = 0; c < kDeltaChunk; ++c) {
        const int f = f0 + c * 32 + lane;
        if (f < F) {
          const double xv = (double)xr[f];
          if (j == (uint32_t)i && !isfinite(xv)) bad = true;
          acc[c] = __dadd_rn(acc[c], __dmul_rn(v, xv));
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kDeltaChunk; ++c) {
      const int f = f0 + c * 32 + lane;
      if (f < F) out[f] = acc[c];
    }
  }
  if (bad) atomicOr(flags, 1 << a);
}

// K1, vectorised (the default when every row starts 16-byte aligned): one
// warp per vertex row, each lane 16-byte loads of VEC consecutive frames,
// CH chunks per pass (256 frames per pass); the row's
// neighbour indices are loaded once (lane t holds entry t) and broadcast by
// shuffles, and neighbour p + 1's loads are issued before neighbour p's
// adds, so two rows' worth of loads are in flight per warp.  The additions
// run in the CSR order with _rn intrinsics, as k_delta (bit-identical).
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using V = float4;
  static constexpr int N = 4;
  __device__ static void get(const V& v, double* o) {
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
};
template <>
struct Vec16<double> {
  using V = double2;
  static constexpr int N = 2;
  __device__ static void get(const V& v, double* o) {
    o[0] = v.x; o[1] = v.y;
  }
};

// chunks per pass: 8 accumulators per lane either way (f32: 256 frames,
// f64: 256 frames per pass)
template <typename T>
constexpr int delta_vec_ch() { return sizeof(T) == 4 ? 2 : 4; }

template <typename T>
__global__ void __launch_bounds__(kDeltaWarps * 32)
    k_delta_vec(int n, int F, const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                const T* __restrict__ x0, const T* __restrict__ x1, const T* __restrict__ x2,
                double* __restrict__ delta, int* flags, int a0) {
  using VT = Vec16<T>;
  using V = typename VT::V;
  constexpr int VEC = VT::N, CH = delta_vec_ch<T>(), PASS = 32 * VEC * CH;
  const int a = blockIdx.y + a0;  // a0: first axis of this launch
  const T* __restrict__ X = a == 0 ? x0 : (a == 1 ? x1 : x2);
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kDeltaWarps + (threadIdx.x >> 5);
  if (i >= n) return;
  const uint32_t pb = rp[i], pe = rp[i + 1];
  const int cnt = (int)(pe - pb);
  const double deg = (double)(cnt - 1);
  const uint32_t my_ci = lane < cnt ? ci[pb + lane] : 0u;
  double* out = delta + ((size_t)a * n + i) * F;
  bool bad = false;
  const int nv = F / VEC;  // vectors per row
  for (int f0 = 0; f0 < F; f0 += PASS) {
    const int v0 = f0 / VEC;
    double acc[CH * VEC];
#pragma unroll
    for (int c = 0; c < CH * VEC; ++c) acc[c] = 0.0;
    auto col = [&](int p) -> uint32_t {
      return p < 32 ? __shfl_sync(0xffffffffu, my_ci, p) : ci[pb + p];
    };
    V nxt[CH];
    uint32_t jn = col(0);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int v = v0 + c * 32 + lane;
      if (v < nv) nxt[c] = reinterpret_cast<const V*>(X + (size_t)jn * F)[v];
    }
    for (int p = 0; p < cnt; ++p) {
      V cur[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) cur[c] = nxt[c];
      const uint32_t j = jn;
      if (p + 1 < cnt) {
        jn = col(p + 1);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int v = v0 + c * 32 + lane;
          if (v < nv) nxt[c] = reinterpret_cast<const V*>(X + (size_t)jn * F)[v];
        }
      }
      // warp-uniform split: off the diagonal acc + (-1 * x) is acc - x (the
      // product is exact), one DADD per element; the diagonal entry carries the
      // degree product and validate_sequence's finiteness check
      if (j != (uint32_t)i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int v = v0 + c * 32 + lane;
          if (v < nv) {
            double xv[VEC];
            VT::get(cur[c], xv);
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[c * VEC + e] = __dsub_rn(acc[c * VEC + e], xv[e]);
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int v = v0 + c * 32 + lane;
          if (v < nv) {
            double xv[VEC];
            VT::get(cur[c], xv);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              if (!isfinite(xv[e])) bad = true;
              acc[c * VEC + e] = __dadd_rn(acc[c * VEC + e], __dmul_rn(deg, xv[e]));
            }
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int v = v0 + c * 32 + lane;
      if (v < nv) {
        double* o = out + (size_t)v * VEC;
#pragma unroll
        for (int e = 0; e < VEC; e += 2)
          *reinterpret_cast<double2*>(o + e) = make_double2(acc[c * VEC + e], acc[c * VEC + e + 1]);
      }
    }
  }
  if (bad) atomicOr(flags, 1 << a);
}

// validate_sequence's finiteness check for the variants without K1 (v2v),
// which otherwise rides on k_delta.
template <typename T>
__global__ void k_check_finite(long nF, const T* __restrict__ x0, const T* __restrict__ x1,
                               const T* __restrict__ x2, int* flags) {
  const int a = blockIdx.y;
  const T* X = a == 0 ? x0 : (a == 1 ? x1 : x2);
  bool bad = false;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < nF; t += (long)gridDim.x * blockDim.x)
    bad |= !isfinite((double)X[t]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, 1 << a);
}

// Gram reduction: S = sum of split-K partials in split order, then
// R = 0.5 * (S + S^T) exactly as spectral.cpp:38 symmetrises.
// lower_only: the partials are bitwise symmetric and only their lower
// triangle (f >= g) was computed (Ozaki Gram, ozaki.cu): both sums read it,
// and 0.5 (s + s) == s exactly, the value the full product gives.
__global__ void k_reduce_sym(int F, int splits, int nbatch, const double* __restrict__ part,
                             double* __restrict__ R, int lower_only) {
  const long FF = (long)F * F;
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (t >= FF) return;
  const int f = (int)(t / F), g = (int)(t % F);
  double s1 = 0.0, s2 = 0.0;
  if (lower_only) {
    const long lo = (long)max(f, g) * F + min(f, g);
    for (int sp = 0; sp < splits; ++sp)
      s1 = __dadd_rn(s1, part[((long)sp * nbatch + b) * FF + lo]);
    s2 = s1;
  } else {
    for (int sp = 0; sp < splits; ++sp) {
      const double* P = part + ((long)sp * nbatch + b) * FF;
      s1 = __dadd_rn(s1, P[(long)f * F + g]);
      s2 = __dadd_rn(s2, P[(long)g * F + f]);
    }
  }
  R[b * FF + (long)g * F + f] = __dmul_rn(0.5, __dadd_rn(s1, s2));
}

// Split-K partials (row-major M x N per split and batch) summed in split
// order into column-major out[b][n M + m] (the implicit OI's Z = X^T P).
__global__ void k_reduce_sum(int M, int N, int splits, int nbatch, const double* __restrict__ part,
                             double* __restrict__ out) {
  const long MN = (long)M * N;
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (t >= MN) return;
  const int n = (int)(t / M), m = (int)(t % M);
  double s = 0.0;
  for (int sp = 0; sp < splits; ++sp) s += part[((long)sp * nbatch + b) * MN + (long)m * N + n];
  out[b * MN + t] = s;
}

// pack_matrix with UniformQuantizer(-1.0f, 1.0f, dict_bits) (codec.cpp:122-129).
__global__ void k_quant_dict(long count, int bits, const double* __restrict__ U,
                             uint16_t* __restrict__ q) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= count) return;
  const QParams qp = make_qparams(-1.0f, 1.0f, bits);
  q[t] = (uint16_t)quantize_level(qp.min_, qp.width, qp.levels, false, U[t]);
}

__global__ void k_init_keys(long rows, unsigned long long* keys) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= rows) return;
  keys[2 * t] = ~0ull;  // running min
  keys[2 * t + 1] = 0ull;  // running max
}

// quantize_rows (codec.cpp:244-265): row r of axis a over its own widened
// float range; one CTA per (row, axis).
__global__ void k_quant_rows(int k, int n, const unsigned long long* __restrict__ keys,
                             const uint8_t* __restrict__ bits_in, const double* __restrict__ C,
                             float* rmin, float* rmax, uint8_t* rbits, uint16_t* __restrict__ q,
                             int a0) {
  const int r = blockIdx.x, a = blockIdx.y + a0;
  const long row = (long)a * k + r;
  const double lo = key_to_double(keys[2 * row]);
  const double hi = key_to_double(keys[2 * row + 1]);
  float flo, fhi;
  widened_range(lo, hi, &flo, &fhi);
  const int bits = bits_in[r];
  const QParams qp = make_qparams(flo, fhi, bits);
  if (threadIdx.x == 0) {
    rmin[row] = flo;
    rmax[row] = fhi;
    rbits[row] = (uint8_t)bits;
  }
  const double* c = C + row * n;
  uint16_t* o = q + row * n;
  if ((n & 3) == 0 && (((uintptr_t)c | (uintptr_t)o) & 15) == 0) {
    // four coefficients per thread: two 16-byte loads, one 8-byte store
    for (int i = threadIdx.x * 4; i < n; i += blockDim.x * 4) {
      const double2 v0 = *reinterpret_cast<const double2*>(c + i);
      const double2 v1 = *reinterpret_cast<const double2*>(c + i + 2);
      const uint32_t l0 = quantize_level(qp.min_, qp.width, qp.levels, qp.degenerate, v0.x);
      const uint32_t l1 = quantize_level(qp.min_, qp.width, qp.levels, qp.degenerate, v0.y);
      const uint32_t l2 = quantize_level(qp.min_, qp.width, qp.levels, qp.degenerate, v1.x);
      const uint32_t l3 = quantize_level(qp.min_, qp.width, qp.levels, qp.degenerate, v1.y);
      *reinterpret_cast<uint2*>(o + i) = make_uint2(l0 | (l1 << 16), l2 | (l3 << 16));
    }
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    o[i] = (uint16_t)quantize_level(qp.min_, qp.width, qp.levels, qp.degenerate, c[i]);
}

// Anchor payload (codec.cpp:444-471): global min/max over the anchor
// trajectories of one axis, widened, then quantised anchor-major.
// ---- vertex-row shards: the anchor payload split in two ------
// The global anchor range is a min/max over every anchor trajectory, so a
// shard first reduces its own anchors into ordered keys (combined across
// ranks by one MAX allreduce with the min half complemented), then quantises
// its anchors with the global widened range.  min/max are exact, so the
// levels equal the single-GPU k_anchors bits.
template <typename T>
__global__ void __launch_bounds__(256)
    k_anchor_keys(int na, int F, const uint32_t* __restrict__ rows, const T* __restrict__ x0,
                  const T* __restrict__ x1, const T* __restrict__ x2,
                  unsigned long long* keys) {
  // grid (chunks, 3): axis = blockIdx.y, element range split over blockIdx.x
  const int a = blockIdx.y;
  const T* X = a == 0 ? x0 : (a == 1 ? x1 : x2);
  const long total = (long)na * F;
  double lo = INFINITY, hi = -INFINITY;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const double v = (double)X[(size_t)rows[t / F] * F + t % F];
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0 && lo <= hi) {
    atomicMin(&keys[2 * a], ordered_key(lo));
    atomicMax(&keys[2 * a + 1], ordered_key(hi));
  }
}

// Anchor quantisation (codec.cpp:444-471) from the exact range keys: every
// CTA derives the same widened float range (min / max are order-free, so the
// levels are those of a single-pass reduction).
template <typename T>
__global__ void __launch_bounds__(256)
    k_anchor_quant(int na, int F, const uint32_t* __restrict__ rows, const T* __restrict__ x0,
                   const T* __restrict__ x1, const T* __restrict__ x2, int bits,
                   const unsigned long long* __restrict__ keys, float* rng,
                   uint16_t* __restrict__ q) {
  const int a = blockIdx.y;
  const T* X = a == 0 ? x0 : (a == 1 ? x1 : x2);
  float flo, fhi;
  widened_range(key_to_double(keys[2 * a]), key_to_double(keys[2 * a + 1]), &flo, &fhi);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rng[2 * a] = flo;
    rng[2 * a + 1] = fhi;
  }
  const QParams qp = make_qparams(flo, fhi, bits);
  const long total = (long)na * F;
  uint16_t* o = q + (size_t)a * total;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const double v = (double)X[(size_t)rows[t / F] * F + t % F];
    o[t] = (uint16_t)quantize_level(qp.min_, qp.width, qp.levels, qp.degenerate, v);
  }
}

// keys[2 r] <- ~keys[2 r]: turns the running-min half into a max-reducible key
// (and back), so one NCCL MAX allreduce combines both halves.
__global__ void k_flip_min_keys(long rows, unsigned long long* keys) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t < rows) keys[2 * t] = ~keys[2 * t];
}

}  // namespace

// axis < 0: all three axes in one launch; else that axis alone (the drop-in
// encode runs an axis as soon as its input has arrived).
cudaError_t launch_delta(cudaStream_t s, int n, int F, const uint32_t* lap_rp,
                         const uint32_t* lap_ci, const void* const x[3], bool f32, double* delta,
                         int* flags, int axis) {
  const int a0 = axis < 0 ? 0 : axis;
  dim3 grid((n + kDeltaWarps - 1) / kDeltaWarps, axis < 0 ? 3 : 1);
  const size_t esz = f32 ? 4 : 8;
  bool vec = (F * esz) % 16 == 0;  // every row 16-byte aligned
  for (int a = 0; a < 3; ++a)
    if (axis < 0 || a == axis) vec = vec && ((uintptr_t)x[a] % 16 == 0);
  static const bool scalar = getenv("DMCG_DELTA_SCALAR") != nullptr;  // tests
  if (vec && !scalar) {
    if (f32)
      k_delta_vec<float><<<grid, kDeltaWarps * 32, 0, s>>>(n, F, lap_rp, lap_ci, (const float*)x[0],
                                                           (const float*)x[1], (const float*)x[2],
                                                           delta, flags, a0);
    else
      k_delta_vec<double><<<grid, kDeltaWarps * 32, 0, s>>>(n, F, lap_rp, lap_ci, (const double*)x[0],
                                                            (const double*)x[1], (const double*)x[2],
                                                            delta, flags, a0);
    return cudaGetLastError();
  }
  if (f32)
    k_delta<float><<<grid, kDeltaWarps * 32, 0, s>>>(n, F, lap_rp, lap_ci, (const float*)x[0],
                                                     (const float*)x[1], (const float*)x[2],
                                                     delta, flags, a0);
  else
    k_delta<double><<<grid, kDeltaWarps * 32, 0, s>>>(n, F, lap_rp, lap_ci, (const double*)x[0],
                                                      (const double*)x[1], (const double*)x[2],
                                                      delta, flags, a0);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(cudaStream_t s, int n, int F, const void* const x[3], bool f32,
                                int* flags) {
  const long nF = (long)n * F;
  const dim3 grid((unsigned)std::min<long>((nF + 255) / 256, 1024), 3);
  if (f32)
    k_check_finite<float><<<grid, 256, 0, s>>>(nF, (const float*)x[0], (const float*)x[1],
                                               (const float*)x[2], flags);
  else
    k_check_finite<double><<<grid, 256, 0, s>>>(nF, (const double*)x[0], (const double*)x[1],
                                                (const double*)x[2], flags);
  return cudaGetLastError();
}

cudaError_t launch_reduce_sym(cudaStream_t s, int F, int splits, int nbatch, const double* part,
                              double* R, bool lower_only) {
  const long FF = (long)F * F;
  dim3 grid((unsigned)((FF + 255) / 256), nbatch);
  k_reduce_sym<<<grid, 256, 0, s>>>(F, splits, nbatch, part, R, lower_only ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_reduce_sum(cudaStream_t s, int M, int N, int splits, int nbatch,
                              const double* part, double* out) {
  const long MN = (long)M * N;
  dim3 grid((unsigned)((MN + 255) / 256), nbatch);
  k_reduce_sum<<<grid, 256, 0, s>>>(M, N, splits, nbatch, part, out);
  return cudaGetLastError();
}

cudaError_t launch_quant_dict(cudaStream_t s, long count, int bits, const double* U, uint16_t* q) {
  k_quant_dict<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(count, bits, U, q);
  return cudaGetLastError();
}

cudaError_t launch_init_keys(cudaStream_t s, long rows, unsigned long long* keys) {
  if (rows <= 0) return cudaSuccess;
  k_init_keys<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(rows, keys);
  return cudaGetLastError();
}

cudaError_t launch_quant_rows(cudaStream_t s, int k, int n, const unsigned long long* keys,
                              const uint8_t* bits_in, const double* C, float* rmin, float* rmax,
                              uint8_t* rbits, uint16_t* q, int axis) {
  if (k <= 0) return cudaSuccess;
  k_quant_rows<<<dim3(k, axis < 0 ? 3 : 1), 256, 0, s>>>(k, n, keys, bits_in, C, rmin, rmax, rbits, q,
                                                       axis < 0 ? 0 : axis);
  return cudaGetLastError();
}

static unsigned anchor_chunks(long total) {
  const long c = (total + 4 * 256 - 1) / (4 * 256);  // ~4 elements per thread
  return (unsigned)(c < 1 ? 1 : (c > 296 ? 296 : c));
}

cudaError_t launch_anchor_keys(cudaStream_t s, int na, int F, const uint32_t* rows,
                               const void* const x[3], bool f32, unsigned long long* keys) {
  if (na <= 0) return cudaSuccess;
  const dim3 grid(anchor_chunks((long)na * F), 3);
  if (f32)
    k_anchor_keys<float><<<grid, 256, 0, s>>>(na, F, rows, (const float*)x[0], (const float*)x[1],
                                              (const float*)x[2], keys);
  else
    k_anchor_keys<double><<<grid, 256, 0, s>>>(na, F, rows, (const double*)x[0],
                                               (const double*)x[1], (const double*)x[2], keys);
  return cudaGetLastError();
}

cudaError_t launch_anchor_quant(cudaStream_t s, int na, int F, const uint32_t* rows,
                                const void* const x[3], bool f32, int bits,
                                const unsigned long long* keys, float* rng, uint16_t* q) {
  const dim3 grid(anchor_chunks((long)na * F), 3);
  if (f32)
    k_anchor_quant<float><<<grid, 256, 0, s>>>(na, F, rows, (const float*)x[0], (const float*)x[1],
                                               (const float*)x[2], bits, keys, rng, q);
  else
    k_anchor_quant<double><<<grid, 256, 0, s>>>(na, F, rows, (const double*)x[0],
                                                (const double*)x[1], (const double*)x[2], bits, keys,
                                                rng, q);
  return cudaGetLastError();
}

// Single-GPU anchors: range keys over many CTAs, then the quantisation
// (the former one-CTA-per-axis kernel ran on 3 SMs).  keys: 3 pairs.
cudaError_t launch_anchors(cudaStream_t s, int n_c, int F, const uint32_t* idx,
                           const void* const x[3], bool f32, int bits, float* rng, uint16_t* q,
                           unsigned long long* keys) {
  if (n_c <= 0) return cudaSuccess;
  cudaError_t e = launch_init_keys(s, 3, keys);
  if (e == cudaSuccess) e = launch_anchor_keys(s, n_c, F, idx, x, f32, keys);
  if (e == cudaSuccess) e = launch_anchor_quant(s, n_c, F, idx, x, f32, bits, keys, rng, q);
  return e;
}

cudaError_t launch_flip_min_keys(cudaStream_t s, long rows, unsigned long long* keys) {
  if (rows <= 0) return cudaSuccess;
  k_flip_min_keys<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(rows, keys);
  return cudaGetLastError();
}

}  // namespace dmcg

// ---- f1: DMC1 payload bit packing on the device (stream.cpp BitWriter) ------
namespace dmcg {
namespace {

// ORs symbol v (b bits, MSB first) into the stream at bit position P; bytes
// are little-endian inside the 32-bit words of `out` (byte B at word B/4).
__device__ __forceinline__ void put_bits(uint32_t* out, unsigned long long P, uint32_t v, int b) {
  const unsigned long long end = P + (unsigned)b;
  for (unsigned long long B = P >> 3; B <= (end - 1) >> 3; ++B) {
    const unsigned long long lo = P > B * 8 ? P : B * 8;
    const unsigned long long hi = end < B * 8 + 8 ? end : B * 8 + 8;
    const int nb = (int)(hi - lo);
    const uint32_t part = (v >> (unsigned)(end - hi)) & ((1u << nb) - 1u);
    const uint32_t byte = part << (unsigned)(B * 8 + 8 - hi);
    atomicOr(&out[B >> 2], byte << (8 * (unsigned)(B & 3)));
  }
}

__global__ void k_pack_uniform(const uint16_t* __restrict__ sym, long count, int bits,
                               unsigned long long base_bit, uint32_t* out) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= count) return;
  put_bits(out, base_bit + (unsigned long long)t * bits, sym[t], bits);
}

// Rows of n symbols; row r starts at row_bitoff[r] (~0: row carries no payload).
__global__ void k_pack_rows(const uint16_t* __restrict__ sym, long n, int rows,
                            const uint8_t* __restrict__ row_bits,
                            const unsigned long long* __restrict__ row_bitoff,
                            unsigned long long base_bit, uint32_t* out) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= n * rows) return;
  const int r = (int)(t / n);
  const long i = t % n;
  const unsigned long long off = row_bitoff[r];
  if (off == ~0ull) return;
  const int b = row_bits[r];
  put_bits(out, base_bit + off + (unsigned long long)i * b, sym[t], b);
}

}  // namespace

cudaError_t launch_pack_uniform(cudaStream_t s, const uint16_t* sym, long count, int bits,
                                unsigned long long base_byte, uint32_t* out) {
  if (count <= 0) return cudaSuccess;
  k_pack_uniform<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(sym, count, bits, base_byte * 8,
                                                                 out);
  return cudaGetLastError();
}

cudaError_t launch_pack_rows(cudaStream_t s, const uint16_t* sym, long n, int rows,
                             const uint8_t* row_bits, const unsigned long long* row_bitoff,
                             unsigned long long base_byte, uint32_t* out) {
  if (n <= 0 || rows <= 0) return cudaSuccess;
  const long tot = n * rows;
  k_pack_rows<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(sym, n, rows, row_bits, row_bitoff,
                                                            base_byte * 8, out);
  return cudaGetLastError();
}

}  // namespace dmcg
