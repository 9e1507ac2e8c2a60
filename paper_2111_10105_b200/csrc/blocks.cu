// Blocks variant (n_b > 1) kernels: frame padding, the per-axis chain of
// warm-started orthogonal iterations with its eigenbasis fallback and sign
// alignment (block_dictionaries, src/codec.cpp:149-172), and the closed-loop
// dictionary difference coder / decoder (encode_dictionaries /
// decode_dictionaries, src/codec.cpp:290-349).
//
// The chain is sequential over blocks (block b starts from block b-1's
// dictionary) and each step is a k_f x k_f problem, so it runs as one CTA
// per axis; the per-block autocorrelations, eigenbases, projections and the
// decode-side reconstruction are batched GEMM / Jacobi launches over all
// 3 n_b blocks (pipeline.cu enqueue_encode_blocks).  Compiled with
// --fmad=false like encode.cu: the quantiser and the difference chain
// follow the reference's arithmetic operation by operation.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace dmcg {
namespace {

constexpr int kChainThreads = 1024;
constexpr int kWarps = kChainThreads / 32;

template <typename T>
__global__ void k_pad_frames(int n, int F, int Fp, const T* __restrict__ x0,
                             const T* __restrict__ x1, const T* __restrict__ x2,
                             T* __restrict__ out) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long nFp = (long)n * Fp;
  if (t >= 3 * nFp) return;
  const int a = (int)(t / nFp);
  const long rem = t % nFp;
  const long i = rem / Fp;
  const int f = (int)(rem % Fp);
  const T* x = a == 0 ? x0 : (a == 1 ? x1 : x2);
  out[t] = x[i * F + (f < F ? f : F - 1)];
}

__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < kWarps ? red[lane] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// Householder QR of the m x m column-major Z in place (Eigen HouseholderQR /
// makeHouseholder, restated in oracle householder_factor): essential parts
// below the diagonal, R diagonal in beta, tau per reflector.
__device__ void qr_factor(int m, double* Z, double* tau, double* beta, double* sc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = 0; j < m; ++j) {
    double* x = Z + (long)j * m;
    if (w == 0) {
      double tail = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) tail = __dadd_rn(tail, __dmul_rn(x[i], x[i]));
      tail = warp_sum(tail);
      if (lane == 0) {
        const double c0 = x[j];
        if (tail <= DBL_MIN) {
          tau[j] = 0.0;
          beta[j] = c0;
          sc[0] = 0.0;  // zero the tail, no update
        } else {
          double b = sqrt(__dadd_rn(__dmul_rn(c0, c0), tail));
          if (c0 >= 0.0) b = -b;
          tau[j] = __ddiv_rn(__dsub_rn(b, c0), b);
          beta[j] = b;
          sc[0] = __dsub_rn(c0, b);  // denominator of v
        }
      }
    }
    __syncthreads();
    // v = x / denom is formed on the fly by the column updates (the same
    // __ddiv_rn as the stored essential part) and written back to column j
    // after the barrier below: one barrier per column instead of two.
    const double denom = sc[0];
    const double tj = tau[j];
    if (tj != 0.0)
      for (int c = j + 1 + w; c < m; c += kWarps) {
        double* y = Z + (long)c * m;
        double d = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32)
          d = __dadd_rn(d, __dmul_rn(__ddiv_rn(x[i], denom), y[i]));
        d = __dadd_rn(warp_sum(d), y[j]);
        d = __dmul_rn(tj, d);
        if (lane == 0) y[j] = __dsub_rn(y[j], d);
        for (int i = j + 1 + lane; i < m; i += 32)
          y[i] = __dsub_rn(y[i], __dmul_rn(d, __ddiv_rn(x[i], denom)));
      }
    __syncthreads();
    for (int i = j + 1 + (int)threadIdx.x; i < m; i += kChainThreads)
      x[i] = denom == 0.0 ? 0.0 : __ddiv_rn(x[i], denom);
    if (threadIdx.x == 0 && denom != 0.0) x[j] = beta[j];
    // (column j is not read again in this factorisation: the next step's
    // warp-0 reduction reads column j + 1, after the barrier at its end)
  }
}

// B (m x m) = H_0 ... H_{m-1} B with B = I on entry (Q = householderQ * I);
// columns c < j are untouched by H_j (they are e_c there).
__device__ void qr_form_q(int m, const double* Z, const double* tau, double* B) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long e = threadIdx.x; e < (long)m * m; e += kChainThreads)
    B[e] = (e % m) == (e / m) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = m - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj == 0.0) continue;
    const double* v = Z + (long)j * m;
    for (int c = j + w; c < m; c += kWarps) {
      double* y = B + (long)c * m;
      double d = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) d = __dadd_rn(d, __dmul_rn(v[i], y[i]));
      d = __dadd_rn(warp_sum(d), y[j]);
      d = __dmul_rn(tj, d);
      if (lane == 0) y[j] = __dsub_rn(y[j], d);
      for (int i = j + 1 + lane; i < m; i += 32) y[i] = __dsub_rn(y[i], __dmul_rn(d, v[i]));
    }
    __syncthreads();
  }
}

// canonicalize_signs (spectral.cpp:41-47): warp per column, first index of
// the largest |u| wins ties.
__device__ void canon_columns(int m, double* U) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = w; c < m; c += kWarps) {
    double* u = U + (long)c * m;
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = lane; i < m; i += 32) {
      const double v = fabs(u[i]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (bi >= m) bi = 0;  // an all-NaN column (non-finite input, flagged by K1)
    const bool neg = u[bi] < 0.0;
    __syncwarp();
    if (neg)
      for (int i = lane; i < m; i += 32) u[i] = -u[i];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kChainThreads)
    k_block_chain(int nb, int kf, int t_max, double tol, const double* __restrict__ R,
                  const double* __restrict__ Ueig, double* U, double* work, int* flags,
                  int use_smem) {
  __shared__ double tau[512], beta[512], red[kWarps], sc[2];
  __shared__ int s_def;
  extern __shared__ double dsm[];  // use_smem: Z, N and the working dictionary
  const int a = blockIdx.x, m = kf, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long kk = (long)m * m;
  const double* Ra = R + (long)a * nb * kk;
  const double* Ea = Ueig + (long)a * nb * kk;
  double* Ua = U + (long)a * nb * kk;
  // Every QR phase reads what other warps wrote in the previous one: with
  // the k_f x k_f operands in shared memory (k_f <= 93) those round trips
  // cost ~30 cycles instead of an L2 round trip.
  double* Z = use_smem ? dsm : work + (long)a * 2 * kk;
  double* N = use_smem ? dsm + kk : Z + kk;
  for (long e = threadIdx.x; e < kk; e += kChainThreads) Ua[e] = Ea[e];  // full_eigenbasis
  __syncthreads();
  for (int b = 1; b < nb; ++b) {
    const double* Rb = Ra + b * kk;
    const double* prev = Ua + (b - 1) * kk;
    double* const out = Ua + b * kk;
    double* cur = use_smem ? dsm + 2 * kk : out;
    for (long e = threadIdx.x; e < kk; e += kChainThreads) cur[e] = prev[e];
    if (threadIdx.x == 0) s_def = 0;
    __syncthreads();
    for (int it = 2; it <= t_max; ++it) {
      // Z = R_b U (ascending inner index, as the oracle's gemm_nn)
      for (long e = threadIdx.x; e < kk; e += kChainThreads) {
        const int i = (int)(e % m);
        const double* uc = cur + (e / m) * m;
        double s = 0.0;
        for (int q = 0; q < m; ++q) s = __dadd_rn(s, __dmul_rn(Rb[(long)q * m + i], uc[q]));
        Z[e] = s;
      }
      __syncthreads();
      qr_factor(m, Z, tau, beta, sc);
      // RankDeficiency: |R_jj| <= m eps max |R_jj| (spectral.cpp:80-88)
      double mx = 0.0;
      for (int j = threadIdx.x; j < m; j += kChainThreads) mx = fmax(mx, fabs(beta[j]));
      mx = block_max(mx, red);
      const double rtol = (double)m * DBL_EPSILON * mx;
      for (int j = threadIdx.x; j < m; j += kChainThreads)
        if (fabs(beta[j]) <= rtol) s_def = 1;
      __syncthreads();
      if (s_def) break;
      qr_form_q(m, Z, tau, N);
      double moved = 0.0;
      if (tol >= 0.0) {  // principal-angle stop (spectral.cpp:90-97)
        for (int c = w; c < m; c += kWarps) {
          double d = 0.0;
          for (int i = lane; i < m; i += 32) d += cur[(long)c * m + i] * N[(long)c * m + i];
          d = warp_sum(d);
          moved = fmax(moved, acos(fmin(fabs(d), 1.0)));
        }
        moved = block_max(moved, red);
      }
      for (long e = threadIdx.x; e < kk; e += kChainThreads) cur[e] = N[e];
      __syncthreads();
      if (tol >= 0.0 && moved < tol) break;
    }
    if (s_def) {  // catch (RankDeficiency): full_eigenbasis(r)
      for (long e = threadIdx.x; e < kk; e += kChainThreads) cur[e] = Ea[b * kk + e];
      if (threadIdx.x == 0) atomicAdd(flags, 1);
      __syncthreads();
    } else {
      canon_columns(m, cur);
    }
    // align_signs(prev, cur)
    for (int c = w; c < m; c += kWarps) {
      double d = 0.0;
      for (int i = lane; i < m; i += 32) d += prev[(long)c * m + i] * cur[(long)c * m + i];
      d = warp_sum(d);
      if (d < 0.0)
        for (int i = lane; i < m; i += 32) cur[(long)c * m + i] = -cur[(long)c * m + i];
    }
    __syncthreads();
    if (use_smem) {
      for (long e = threadIdx.x; e < kk; e += kChainThreads) out[e] = cur[e];
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kChainThreads)
    k_dict_encode_blocks(int nb, int kf, int dict_bits, int diff_bits, const double* __restrict__ U,
                         double* work, uint16_t* __restrict__ q, float* __restrict__ rng) {
  __shared__ double red[kWarps];
  __shared__ unsigned char flip[512];
  const int a = blockIdx.x, m = kf, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long kk = (long)m * m;
  const double* Ua = U + (long)a * nb * kk;
  uint16_t* qa = q + (long)a * nb * kk;
  double* Dec = work + (long)a * 2 * kk;  // payload.decoded.back()
  double* diff = Dec + kk;
  const QParams q0 = make_qparams(-1.0f, 1.0f, dict_bits);
  for (long e = threadIdx.x; e < kk; e += kChainThreads) {
    const uint32_t lv = quantize_level(q0.min_, q0.width, q0.levels, false, Ua[e]);
    qa[e] = (uint16_t)lv;
    Dec[e] = dequantize_level(q0.min_, q0.width, false, lv);
  }
  __syncthreads();
  for (int b = 1; b < nb; ++b) {
    const double* cur = Ua + b * kk;
    // auto_realign: a column closer to the negated predecessor is flipped
    for (int c = w; c < m; c += kWarps) {
      double st = 0.0, fl = 0.0;
      for (int i = lane; i < m; i += 32) {
        const double x = cur[(long)c * m + i], p = Dec[(long)c * m + i];
        const double d = __dsub_rn(x, p), e = __dsub_rn(-x, p);
        st = __dadd_rn(st, __dmul_rn(d, d));
        fl = __dadd_rn(fl, __dmul_rn(e, e));
      }
      st = warp_sum(st);
      fl = warp_sum(fl);
      if (lane == 0) flip[c] = (st > 2.0 && fl < st) ? 1 : 0;
    }
    __syncthreads();
    double lo = INFINITY, hi = -INFINITY;
    for (long e = threadIdx.x; e < kk; e += kChainThreads) {
      const double x = flip[e / m] ? -cur[e] : cur[e];
      const double d = __dsub_rn(x, Dec[e]);  // diff = cur - prev
      diff[e] = d;
      lo = fmin(lo, d);
      hi = fmax(hi, d);
    }
    hi = block_max(hi, red);
    lo = -block_max(-lo, red);
    float flo, fhi;
    widened_range(lo, hi, &flo, &fhi);
    if (threadIdx.x == 0) {
      rng[((long)a * (nb - 1) + b - 1) * 2] = flo;
      rng[((long)a * (nb - 1) + b - 1) * 2 + 1] = fhi;
    }
    const QParams qd = make_qparams(flo, fhi, diff_bits);
    uint16_t* qb = qa + b * kk;
    for (long e = threadIdx.x; e < kk; e += kChainThreads) {
      const uint32_t lv = quantize_level(qd.min_, qd.width, qd.levels, qd.degenerate, diff[e]);
      qb[e] = (uint16_t)lv;
      Dec[e] = __dadd_rn(Dec[e], dequantize_level(qd.min_, qd.width, qd.degenerate, lv));
    }
    __syncthreads();
  }
}

// One thread per dictionary entry: the closed-loop sum over blocks is a
// sequential chain per entry only.
__global__ void k_dict_decode_blocks(int nb, int kf, int dict_bits, int diff_bits,
                                     const uint16_t* __restrict__ q, const float* __restrict__ rng,
                                     int* flags, double* __restrict__ Ud) {
  const long kk = (long)kf * kf;
  const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const int a = blockIdx.y;
  if (e >= kk) return;
  const uint16_t* qa = q + (long)a * nb * kk;
  double* oa = Ud + (long)a * nb * kk;
  const QParams q0 = make_qparams(-1.0f, 1.0f, dict_bits);
  uint32_t lv = qa[e];
  if (lv >= q0.levels) atomicOr(flags, 1);
  double v = dequantize_level(q0.min_, q0.width, false, lv);
  oa[e] = v;
  for (int b = 1; b < nb; ++b) {
    const long r = ((long)a * (nb - 1) + b - 1) * 2;
    const QParams qd = make_qparams(rng[r], rng[r + 1], diff_bits);
    lv = qa[b * kk + e];
    if (lv >= qd.levels) atomicOr(flags, 1);
    v = __dadd_rn(v, dequantize_level(qd.min_, qd.width, qd.degenerate, lv));
    oa[b * kk + e] = v;
  }
}

__global__ void k_pad_anchor_levels(int n_c, int F, int Fp, uint16_t* q) {
  const int P = Fp - F;
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= 3L * n_c * P) return;
  const long row = t / P;  // (axis, anchor)
  const int p = (int)(t % P);
  q[row * Fp + F + p] = q[row * Fp + F - 1];
}

}  // namespace

size_t block_work_doubles(int kf) { return 2 * (size_t)kf * kf; }

cudaError_t launch_pad_frames(cudaStream_t s, int n, int F, int Fp, const void* const x[3],
                              bool f32, void* out) {
  const long total = 3L * n * Fp;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (f32)
    k_pad_frames<float><<<grid, 256, 0, s>>>(n, F, Fp, (const float*)x[0], (const float*)x[1],
                                             (const float*)x[2], (float*)out);
  else
    k_pad_frames<double><<<grid, 256, 0, s>>>(n, F, Fp, (const double*)x[0], (const double*)x[1],
                                              (const double*)x[2], (double*)out);
  return cudaGetLastError();
}

cudaError_t launch_block_chain(cudaStream_t s, int nb, int kf, int t_max, double tol,
                               const double* R, const double* Ueig, double* U, double* work,
                               int* flags) {
  if (kf > 512) return cudaErrorInvalidValue;
  const size_t smem = 3 * (size_t)kf * kf * sizeof(double);
  const bool use_smem = smem <= 200 * 1024;
  if (use_smem) {
    cudaError_t e = cudaFuncSetAttribute((const void*)k_block_chain,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_block_chain<<<3, kChainThreads, use_smem ? smem : 0, s>>>(nb, kf, t_max, tol, R, Ueig, U, work,
                                                              flags, use_smem ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_dict_encode_blocks(cudaStream_t s, int nb, int kf, int dict_bits,
                                      int diff_bits, const double* U, double* work, uint16_t* q,
                                      float* rng) {
  if (kf > 512) return cudaErrorInvalidValue;
  k_dict_encode_blocks<<<3, kChainThreads, 0, s>>>(nb, kf, dict_bits, diff_bits, U, work, q, rng);
  return cudaGetLastError();
}

cudaError_t launch_dict_decode_blocks(cudaStream_t s, int nb, int kf, int dict_bits,
                                      int diff_bits, const uint16_t* q, const float* rng,
                                      int* flags, double* Ud) {
  const long kk = (long)kf * kf;
  k_dict_decode_blocks<<<dim3((unsigned)((kk + 255) / 256), 3), 256, 0, s>>>(
      nb, kf, dict_bits, diff_bits, q, rng, flags, Ud);
  return cudaGetLastError();
}

cudaError_t launch_pad_anchor_levels(cudaStream_t s, int n_c, int F, int Fp, uint16_t* q) {
  if (Fp <= F || n_c <= 0) return cudaSuccess;
  const long total = 3L * n_c * (Fp - F);
  k_pad_anchor_levels<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(n_c, F, Fp, q);
  return cudaGetLastError();
}

}  // namespace dmcg
