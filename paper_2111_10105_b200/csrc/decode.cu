// Decode-side kernels: dequantiser parameters, the anchored right-hand side
// and K7, the column-block conjugate-gradient solve of the anchored normal
// equations (reference: SimplicialLDLT + one refinement, src/solver.cpp:
// 62-90).
//
// CG layout.  The 3F right-hand sides (all axes, all frames) are solved
// together.  Vectors are stored column-block-major: block c/kCB holds rows
// 0..n-1, each a 32-byte group of kCB = 4 columns, so one CTA owns complete
// columns.  Every CTA therefore runs an independent CG on its 4 columns:
// dot products are CTA-local (deterministic, no grid-wide sync), converged
// columns freeze, and each neighbour gather is exactly one 32 B sector.
#include <cfloat>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace dmcg {

namespace {

__global__ void k_row_params(int rows, const float* rmin, const float* rmax, const uint8_t* rbits,
                             double* rowp) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows) return;
  const QParams q = make_qparams(rmin[t], rmax[t], rbits[t]);
  rowp[2 * t] = q.min_;
  rowp[2 * t + 1] = q.degenerate ? 0.0 : q.width;
}

// Column sums of a row-major rows x cols block (leading dimension ld,
// batch z via blockIdx.z), deterministic: CTA (x, y) sums rows y, y + R, ...
// of 32 columns with a fixed 8-way split, partial[z][y][c]; the finalisers
// below add the R partials in order.
template <typename T>
__global__ void __launch_bounds__(256)
    k_colsum_partial(int rows, int cols, long ld, const T* __restrict__ X0,
                     const T* __restrict__ X1, const T* __restrict__ X2, double* partial) {
  __shared__ double red[8][33];
  const int z = blockIdx.z;
  const T* X = z == 0 ? X0 : (z == 1 ? X1 : X2);
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int R = gridDim.y;
  double s = 0.0;
  if (c < cols)
    for (int i = blockIdx.y * 8 + threadIdx.y; i < rows; i += R * 8) s += (double)X[(size_t)i * ld + c];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    double t = 0.0;
#pragma unroll
    for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
    partial[((size_t)z * R + blockIdx.y) * cols + c] = t;
  }
}

// traj.row(f).mean() as float (codec.cpp:432-441): means[z][f].
__global__ void k_means_final(int rows, int cols, int R, const double* __restrict__ partial,
                              float* means) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x, z = blockIdx.y;
  if (c >= cols) return;
  double s = 0.0;
  for (int y = 0; y < R; ++y) s += partial[((size_t)z * R + y) * cols + c];
  means[(size_t)z * cols + c] = (float)(s / (double)rows);
}

// solve_mean_constrained's shift (solver.cpp:129-131): column c = a Fw + f of
// the n x 3Fw solution moves to the stored mean of frame f0 + f of axis a.
__global__ void k_shift_final(int rows, int Fw, int F_all, int f0, int R,
                              const double* __restrict__ partial, const float* __restrict__ means,
                              double* shift) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x, W = 3 * Fw;
  if (c >= W) return;
  double s = 0.0;
  for (int y = 0; y < R; ++y) s += partial[(size_t)y * W + c];
  const int a = c / Fw, f = c % Fw;
  shift[c] = (double)means[(size_t)a * F_all + f0 + f] - s / (double)rows;
}

// dequantize_rows (codec.cpp:267-288) of all 3 k retained rows into f64
// (row r of axis a at out[(a k + r) n]); a level beyond 2^bits flags a
// corrupt payload.  Memory-bound pre-pass of the reconstruction GEMM, which
// then streams plain f64 tiles through its cp.async ring.
__global__ void k_dequant_rows(int n, const uint16_t* __restrict__ q, const double* __restrict__ rowp,
                               const uint8_t* __restrict__ rbits, int* flags,
                               double* __restrict__ out) {
  const long row = blockIdx.y;
  const double min_ = rowp[2 * row], width = rowp[2 * row + 1];
  const uint32_t levels = 1u << rbits[row];
  const uint16_t* qr = q + row * n;
  double* o = out + row * n;
  bool bad = false;
  if ((n & 7) == 0 && (((uintptr_t)q | (uintptr_t)out) & 15) == 0) {
    // eight symbols per thread: one 16-byte load, four 16-byte stores (the
    // one-symbol loop keeps 2 bytes in flight per thread and ran at 0.75 TB/s)
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n;
         i += gridDim.x * blockDim.x * 8) {
      const uint4 pk = *reinterpret_cast<const uint4*>(qr + i);
      const uint32_t w4[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const uint32_t l0 = w4[h] & 0xffffu, l1 = w4[h] >> 16;
        bad |= width != 0.0 && (l0 >= levels || l1 >= levels);
        const double v0 = width == 0.0 ? min_ : dequantize_level(min_, width, false, l0);
        const double v1 = width == 0.0 ? min_ : dequantize_level(min_, width, false, l1);
        *reinterpret_cast<double2*>(o + i + 2 * h) = make_double2(v0, v1);
      }
    }
  } else {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const uint32_t lv = qr[i];
      bad |= width != 0.0 && lv >= levels;
      o[i] = width == 0.0 ? min_ : dequantize_level(min_, width, false, lv);
    }
  }
  if (bad) atomicOr(flags, 1);
}

// decode_dictionaries (codec.cpp:330-349): columns r < k of U~ over the
// frame window [f0, f0 + Fw) -> out[(a k + r) Fw + f].
__global__ void k_dequant_dict(int F, int k, int f0, int Fw, const uint16_t* __restrict__ q,
                               double width, uint32_t levels, int* flags, double* __restrict__ out) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long total = 3L * k * Fw;
  if (t >= total) return;
  const int f = (int)(t % Fw);
  const long ar = t / Fw;  // a k + r
  const int a = (int)(ar / k), r = (int)(ar % k);
  const uint32_t lv = q[((long)a * F + r) * F + f0 + f];
  if (lv >= levels) atomicOr(flags, 1);
  out[t] = dequantize_level(-1.0, width, false, lv);
}

// rhs = L^T delta~ + S^T a  (solver.cpp:77-80).  One thread per (row,
// column block); Laplacian values implicit; anchors dequantised on the fly
// (anchor_matrix, codec.cpp:174-195).
__global__ void k_rhs(int n, int F, int W, int nblk, const uint32_t* __restrict__ rp,
                      const uint32_t* __restrict__ ci, const int32_t* __restrict__ apos, int n_c,
                      const uint16_t* __restrict__ aq, const float* __restrict__ arng, int abits,
                      const double* __restrict__ D, double* __restrict__ B, int* flags) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= (long)n * nblk) return;
  const int blk = (int)(t / n), i = (int)(t % n);
  const uint32_t pb = rp[i], pe = rp[i + 1];
  const double deg = (double)(pe - pb - 1);
  const double* Db = D + (size_t)blk * n * kCB;
  double acc[kCB] = {0.0, 0.0, 0.0, 0.0};
  for (uint32_t p = pb; p < pe; ++p) {
    const uint32_t j = ci[p];
    const double v = (j == (uint32_t)i) ? deg : -1.0;
    const double2* dj = reinterpret_cast<const double2*>(Db + (size_t)j * kCB);
    const double2 d0 = dj[0], d1 = dj[1];
    acc[0] = __dadd_rn(acc[0], __dmul_rn(v, d0.x));
    acc[1] = __dadd_rn(acc[1], __dmul_rn(v, d0.y));
    acc[2] = __dadd_rn(acc[2], __dmul_rn(v, d1.x));
    acc[3] = __dadd_rn(acc[3], __dmul_rn(v, d1.y));
  }
  const int slot = apos[i];
  if (slot >= 0) {
    const uint32_t levels = 1u << abits;
#pragma unroll
    for (int c = 0; c < kCB; ++c) {
      const int col = blk * kCB + c;
      if (col >= W) continue;
      const int a = col / F, f = col % F;
      const QParams q = make_qparams(arng[2 * a], arng[2 * a + 1], abits);
      const uint32_t lv = aq[((size_t)a * n_c + slot) * F + f];
      if (lv >= levels) atomicOr(flags, 1);
      acc[c] = __dadd_rn(acc[c], dequantize_level(q.min_, q.width, q.degenerate, lv));
    }
  }
  double2* o = reinterpret_cast<double2*>(B + ((size_t)blk * n + i) * kCB);
  o[0] = make_double2(acc[0], acc[1]);
  o[1] = make_double2(acc[2], acc[3]);
}

constexpr int kCgThreads = 512;

__device__ __forceinline__ void load4(const double* p, double (&v)[kCB]) {
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const double2 b = reinterpret_cast<const double2*>(p)[1];
  v[0] = a.x;
  v[1] = a.y;
  v[2] = b.x;
  v[3] = b.y;
}
__device__ __forceinline__ void store4(double* p, const double (&v)[kCB]) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
}

// Sums 4 per-thread partials over the CTA; result in out[0..3] (smem).
__device__ __forceinline__ void block_sum4(double (&v)[kCB], double* red, double* out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < kCB; ++c) v[c] = warp_sum(v[c]);
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < kCB; ++c) red[w * kCB + c] = v[c];
  __syncthreads();
  if (threadIdx.x < kCB) {
    double s = 0.0;
    for (int i = 0; i < kCgThreads / 32; ++i) s += red[i * kCB + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// K7: CG on M = L^T L + S^T S for the 4 columns of block blockIdx.x.
// x0 = 0, r0 = b (stored in R on entry).  Per iteration: q = M p (gather),
// alpha = rho / p.q; x += alpha p; r -= alpha q; beta = rho'/rho;
// p = r + beta p.  A column stops when ||r|| <= rtol ||b||.
__global__ void __launch_bounds__(kCgThreads)
    k_cg(int n, int W, const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
         const float* __restrict__ val, double* X, double* R, double* P, double* Q, double rtol,
         int maxit, int* iters_out, double* res_out) {
  __shared__ double red[(kCgThreads / 32) * kCB];
  __shared__ double s_dot[kCB];
  __shared__ double s_rho[kCB], s_bn[kCB], s_alpha[kCB], s_beta[kCB];
  __shared__ int s_done[kCB], s_it[kCB];
  const int blk = blockIdx.x;
  const size_t off = (size_t)blk * n * kCB;
  double* x = X + off;
  double* r = R + off;
  double* p = P + off;
  double* q = Q + off;
  const int tid = threadIdx.x;

  double acc[kCB] = {0.0, 0.0, 0.0, 0.0};
  for (int i = tid; i < n; i += kCgThreads) {
    double v[kCB];
    load4(r + (size_t)i * kCB, v);
    store4(p + (size_t)i * kCB, v);
    const double z[kCB] = {0.0, 0.0, 0.0, 0.0};
    store4(x + (size_t)i * kCB, z);
#pragma unroll
    for (int c = 0; c < kCB; ++c) acc[c] += v[c] * v[c];
  }
  block_sum4(acc, red, s_dot);
  if (tid < kCB) {
    const int col = blk * kCB + tid;
    s_rho[tid] = s_dot[tid];
    s_bn[tid] = s_dot[tid];
    s_done[tid] = (col >= W) || !(s_dot[tid] > 0.0);
    s_it[tid] = 0;
  }
  __syncthreads();

  for (int it = 0; it < maxit; ++it) {
    if (s_done[0] && s_done[1] && s_done[2] && s_done[3]) break;
    // q = M p ; p.q
#pragma unroll
    for (int c = 0; c < kCB; ++c) acc[c] = 0.0;
    for (int i = tid; i < n; i += kCgThreads) {
      double qi[kCB] = {0.0, 0.0, 0.0, 0.0};
      const uint32_t pb = rp[i], pe = rp[i + 1];
      for (uint32_t e = pb; e < pe; ++e) {
        const double mv = (double)val[e];
        double pj[kCB];
        load4(p + (size_t)ci[e] * kCB, pj);
#pragma unroll
        for (int c = 0; c < kCB; ++c) qi[c] += mv * pj[c];
      }
      store4(q + (size_t)i * kCB, qi);
      double pi[kCB];
      load4(p + (size_t)i * kCB, pi);
#pragma unroll
      for (int c = 0; c < kCB; ++c) acc[c] += pi[c] * qi[c];
    }
    block_sum4(acc, red, s_dot);
    if (tid < kCB) {
      const double pq = s_dot[tid];
      if (s_done[tid] || !(pq > 0.0)) {
        s_alpha[tid] = 0.0;
        if (!s_done[tid]) s_done[tid] = 1;
      } else {
        s_alpha[tid] = s_rho[tid] / pq;
      }
    }
    __syncthreads();
    double al[kCB];
#pragma unroll
    for (int c = 0; c < kCB; ++c) {
      al[c] = s_alpha[c];
      acc[c] = 0.0;
    }
    for (int i = tid; i < n; i += kCgThreads) {
      double xi[kCB], ri[kCB], pi[kCB], qi[kCB];
      load4(x + (size_t)i * kCB, xi);
      load4(r + (size_t)i * kCB, ri);
      load4(p + (size_t)i * kCB, pi);
      load4(q + (size_t)i * kCB, qi);
#pragma unroll
      for (int c = 0; c < kCB; ++c) {
        xi[c] += al[c] * pi[c];
        ri[c] -= al[c] * qi[c];
        acc[c] += ri[c] * ri[c];
      }
      store4(x + (size_t)i * kCB, xi);
      store4(r + (size_t)i * kCB, ri);
    }
    block_sum4(acc, red, s_dot);
    if (tid < kCB) {
      if (!s_done[tid]) {
        const double rr = s_dot[tid];
        s_beta[tid] = rr / s_rho[tid];
        s_rho[tid] = rr;
        s_it[tid] = it + 1;
        if (rr <= rtol * rtol * s_bn[tid]) s_done[tid] = 1;
      } else {
        s_beta[tid] = 0.0;
      }
    }
    __syncthreads();
    double be[kCB];
#pragma unroll
    for (int c = 0; c < kCB; ++c) be[c] = s_beta[c];
    for (int i = tid; i < n; i += kCgThreads) {
      double ri[kCB], pi[kCB];
      load4(r + (size_t)i * kCB, ri);
      load4(p + (size_t)i * kCB, pi);
#pragma unroll
      for (int c = 0; c < kCB; ++c) pi[c] = ri[c] + be[c] * pi[c];
      store4(p + (size_t)i * kCB, pi);
    }
    __syncthreads();
  }
  if (tid < kCB) {
    const int col = blk * kCB + tid;
    if (col < W) {
      iters_out[col] = s_it[tid];
      res_out[col] = s_bn[tid] > 0.0 ? sqrt(s_rho[tid] / s_bn[tid]) : 0.0;
    }
  }
}

// Row-major variants for the direct solver: vectors are n x W, row i =
// [x frames | y frames | z frames] of vertex i.
// rhs = L^T delta~ + S^T a (row-major n x W, W = 3F): one warp per (row,
// 256-column chunk), lane = four column pairs (double2), the row's CSR
// entries broadcast by shuffles, each entry's loads issued before the
// previous entry's adds; the additions run in CSR order with _rn
// intrinsics (same arithmetic as the reference's sparse product order).
constexpr int kRhsCols = 256;
__global__ void __launch_bounds__(256)
    k_rhs_rm(int n, int F, int W, int F_all, int f_off, const uint32_t* __restrict__ rp,
             const uint32_t* __restrict__ ci, const int32_t* __restrict__ apos, int n_c,
             const uint16_t* __restrict__ aq, const float* __restrict__ arng, int abits,
             const double* __restrict__ D, double* __restrict__ B, int* flags) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= n) return;
  const int c0 = blockIdx.y * kRhsCols;
  const uint32_t pb = rp[i], pe = rp[i + 1];
  const int cnt = (int)(pe - pb);
  const double deg = (double)(cnt - 1);
  const bool vec = !(W & 1);
  const uint32_t my_c = lane < cnt ? ci[pb + lane] : 0u;
  auto col = [&](int e) -> uint32_t {
    return e < 32 ? __shfl_sync(0xffffffffu, my_c, e) : ci[pb + e];
  };
  auto load = [&](uint32_t j, double2 (&t)[4]) {
    const double* xr = D + (size_t)j * W;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + 64 * q + 2 * lane;
      t[q] = make_double2(0.0, 0.0);
      if (c + 1 < W && vec) {
        t[q] = *reinterpret_cast<const double2*>(xr + c);
      } else if (c < W) {
        t[q].x = xr[c];
        if (c + 1 < W) t[q].y = xr[c + 1];
      }
    }
  };
  double acc[4][2];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
  double2 nxt[4];
  uint32_t jn = cnt > 0 ? col(0) : 0u;
  if (cnt > 0) load(jn, nxt);
  for (int e = 0; e < cnt; ++e) {
    double2 cur[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
    const uint32_t j = jn;
    if (e + 1 < cnt) {
      jn = col(e + 1);
      load(jn, nxt);
    }
    const double v = (j == (uint32_t)i) ? deg : -1.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      acc[q][0] = __dadd_rn(acc[q][0], __dmul_rn(v, cur[q].x));
      acc[q][1] = __dadd_rn(acc[q][1], __dmul_rn(v, cur[q].y));
    }
  }
  const int slot = apos[i];
  bool bad = false;
  if (slot >= 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = c0 + 64 * q + 2 * lane + h;
        if (c < W) {
          const int a = c / F, f = c - a * F;
          const QParams qp = make_qparams(arng[2 * a], arng[2 * a + 1], abits);
          const uint32_t lv = aq[((size_t)a * n_c + slot) * F_all + f_off + f];
          if (lv >= qp.levels) bad = true;
          acc[q][h] = __dadd_rn(acc[q][h], dequantize_level(qp.min_, qp.width, qp.degenerate, lv));
        }
      }
  }
  if (bad) atomicOr(flags, 1);
  double* br = B + (size_t)i * W;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + 64 * q + 2 * lane;
    if (c + 1 < W && vec) {
      *reinterpret_cast<double2*>(br + c) = make_double2(acc[q][0], acc[q][1]);
    } else if (c < W) {
      br[c] = acc[q][0];
      if (c + 1 < W) br[c + 1] = acc[q][1];
    }
  }
}

// out_a(i, f_off + f) = X(i, a F + f) (+ shift): one CTA per vertex row (or
// several rows per CTA), consecutive threads on consecutive frames, so both
// the row-major read and the vertex-major writes are contiguous.
template <typename T>
__global__ void __launch_bounds__(256)
    k_output_rm(int n, int F, int F_all, int f_off, const double* __restrict__ X, T* o0, T* o1,
                T* o2, const double* __restrict__ shift, int F_out) {
  const int per = 3 * F_out;
  for (int i = blockIdx.x; i < n; i += gridDim.x)
    for (int r = threadIdx.x; r < per; r += blockDim.x) {
      const int a = r / F_out, f = r - a * F_out;
      T* o = a == 0 ? o0 : (a == 1 ? o1 : o2);
      const double v = __ldcs(X + (size_t)i * 3 * F + (size_t)a * F + f);
      o[(size_t)i * F_all + f_off + f] = (T)(shift ? v + shift[a * F + f] : v);
    }
}

template <typename T>
__global__ void k_output(int n, int F, const double* __restrict__ X, T* o0, T* o1, T* o2) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long total = 3L * n * F;
  if (t >= total) return;
  const int a = (int)(t / ((long)n * F));
  const long rem = t % ((long)n * F);
  const int i = (int)(rem / F), f = (int)(rem % F);
  const int col = a * F + f;
  const double v = X[((size_t)(col / kCB) * n + i) * kCB + col % kCB];
  T* o = a == 0 ? o0 : (a == 1 ? o1 : o2);
  o[rem] = (T)v;
}

}  // namespace

cudaError_t launch_row_params(cudaStream_t s, int rows, const float* rmin, const float* rmax,
                              const uint8_t* rbits, double* rowp) {
  if (rows <= 0) return cudaSuccess;
  k_row_params<<<(rows + 255) / 256, 256, 0, s>>>(rows, rmin, rmax, rbits, rowp);
  return cudaGetLastError();
}

static int colsum_split(int rows) {
  const int r = (rows + 8191) / 8192;
  return r < 1 ? 1 : (r > 64 ? 64 : r);
}

cudaError_t launch_frame_means(cudaStream_t s, int n, int F, const void* const x[3], bool f32,
                               double* partial, float* means) {
  const int R = colsum_split(n);
  const dim3 grid((F + 31) / 32, R, 3), block(32, 8);
  if (f32)
    k_colsum_partial<float><<<grid, block, 0, s>>>(n, F, F, (const float*)x[0], (const float*)x[1],
                                                   (const float*)x[2], partial);
  else
    k_colsum_partial<double><<<grid, block, 0, s>>>(n, F, F, (const double*)x[0],
                                                    (const double*)x[1], (const double*)x[2],
                                                    partial);
  k_means_final<<<dim3((F + 127) / 128, 3), 128, 0, s>>>(n, F, R, partial, means);
  return cudaGetLastError();
}

cudaError_t launch_mean_shift(cudaStream_t s, int n, int Fw, int F_all, int f0, const double* X,
                              const float* means, double* partial, double* shift) {
  const int W = 3 * Fw, R = colsum_split(n);
  k_colsum_partial<double><<<dim3((W + 31) / 32, R, 1), dim3(32, 8), 0, s>>>(n, W, W, X, X, X,
                                                                             partial);
  k_shift_final<<<(W + 127) / 128, 128, 0, s>>>(n, Fw, F_all, f0, R, partial, means, shift);
  return cudaGetLastError();
}

cudaError_t launch_dequant_rows(cudaStream_t s, int rows, int n, const uint16_t* q,
                                const double* rowp, const uint8_t* rbits, int* flags, double* out) {
  if (rows <= 0 || n <= 0) return cudaSuccess;
  const int per = (n & 7) == 0 ? 2048 : 256;  // symbols per CTA pass
  const int bx = (n + per - 1) / per < 64 ? (n + per - 1) / per : 64;
  k_dequant_rows<<<dim3(bx, rows), 256, 0, s>>>(n, q, rowp, rbits, flags, out);
  return cudaGetLastError();
}

cudaError_t launch_dequant_dict(cudaStream_t s, int F, int k, int f0, int Fw, const uint16_t* q,
                                int bits, int* flags, double* out) {
  const long total = 3L * k * Fw;
  if (total <= 0) return cudaSuccess;
  const uint32_t levels = 1u << bits;
  k_dequant_dict<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(F, k, f0, Fw, q, 2.0 / (double)levels,
                                                               levels, flags, out);
  return cudaGetLastError();
}

cudaError_t launch_rhs(cudaStream_t s, int n, int F, int W, int nblk, const uint32_t* lap_rp,
                       const uint32_t* lap_ci, const int32_t* anchor_pos, int n_c,
                       const uint16_t* anchor_q, const float* anchor_rng, int anchor_bits,
                       const double* D, double* B, int* flags) {
  const long total = (long)n * nblk;
  k_rhs<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(n, F, W, nblk, lap_rp, lap_ci, anchor_pos,
                                                        n_c, anchor_q, anchor_rng, anchor_bits, D,
                                                        B, flags);
  return cudaGetLastError();
}

cudaError_t launch_cg(cudaStream_t s, int n, int W, int nblk, const uint32_t* m_rp,
                      const uint32_t* m_ci, const float* m_val, double* X, double* R, double* P,
                      double* Q, double rtol, int maxit, int* iters, double* res) {
  k_cg<<<nblk, kCgThreads, 0, s>>>(n, W, m_rp, m_ci, m_val, X, R, P, Q, rtol, maxit, iters, res);
  return cudaGetLastError();
}

cudaError_t launch_rhs_rm(cudaStream_t s, int n, int F, int F_all, int f_off,
                          const uint32_t* lap_rp, const uint32_t* lap_ci, const int32_t* anchor_pos,
                          int n_c, const uint16_t* anchor_q, const float* anchor_rng,
                          int anchor_bits, const double* D, double* B, int* flags) {
  if (n <= 0 || F <= 0) return cudaSuccess;
  const int W = 3 * F;
  const dim3 grid((unsigned)((n + 7) / 8), (unsigned)((W + kRhsCols - 1) / kRhsCols));
  k_rhs_rm<<<grid, 256, 0, s>>>(n, F, W, F_all, f_off, lap_rp, lap_ci, anchor_pos, n_c, anchor_q,
                                anchor_rng, anchor_bits, D, B, flags);
  return cudaGetLastError();
}

cudaError_t launch_output_rm(cudaStream_t s, int n, int F, int F_all, int f_off, const double* X,
                             void* const out[3], bool f32, const double* shift, int F_out) {
  if (F_out < 0) F_out = F;
  const unsigned grid = (unsigned)std::min<long>(n, 148L * 32);
  if (f32)
    k_output_rm<float><<<grid, 256, 0, s>>>(n, F, F_all, f_off, X, (float*)out[0], (float*)out[1],
                                            (float*)out[2], shift, F_out);
  else
    k_output_rm<double><<<grid, 256, 0, s>>>(n, F, F_all, f_off, X, (double*)out[0],
                                             (double*)out[1], (double*)out[2], shift, F_out);
  return cudaGetLastError();
}

cudaError_t launch_output(cudaStream_t s, int n, int F, const double* X, void* const out[3],
                          bool f32) {
  const long total = 3L * n * F;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (f32)
    k_output<float><<<grid, 256, 0, s>>>(n, F, X, (float*)out[0], (float*)out[1], (float*)out[2]);
  else
    k_output<double><<<grid, 256, 0, s>>>(n, F, X, (double*)out[0], (double*)out[1],
                                          (double*)out[2]);
  return cudaGetLastError();
}

}  // namespace dmcg

// ---- f3: distortion metrics on the device (src/metrics.cpp:67-129) --------
namespace dmcg {
namespace {

template <typename T>
__global__ void k_distortion_terms(int n, int F, const uint32_t* __restrict__ lap_rp,
                                   const uint32_t* __restrict__ lap_ci, const T* __restrict__ a0,
                                   const T* __restrict__ a1, const T* __restrict__ a2,
                                   const T* __restrict__ b0, const T* __restrict__ b1,
                                   const T* __restrict__ b2, double* err2, double* enorm,
                                   double* gnorm) {
  // per (vertex i, frame f): |d|^2, |d|, |(L_norm d)_i| with d = orig - recon
  // and L_norm = I - D^{-1} A (LaplacianKind::Normalized, laplacian.cpp:21-37)
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= (long)n * F) return;
  const int i = (int)(t / F), f = (int)(t % F);
  const size_t o = (size_t)i * F + f;
  const double d0 = (double)a0[o] - (double)b0[o], d1 = (double)a1[o] - (double)b1[o],
               d2 = (double)a2[o] - (double)b2[o];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  const uint32_t p0 = lap_rp[i], p1 = lap_rp[i + 1];
  for (uint32_t p = p0; p < p1; ++p) {
    const uint32_t j = lap_ci[p];
    if ((int)j == i) continue;
    const size_t oj = (size_t)j * F + f;
    s0 += (double)a0[oj] - (double)b0[oj];
    s1 += (double)a1[oj] - (double)b1[oj];
    s2 += (double)a2[oj] - (double)b2[oj];
  }
  const double inv = 1.0 / (double)(p1 - p0 - 1);
  const double g0 = d0 - inv * s0, g1 = d1 - inv * s1, g2 = d2 - inv * s2;
  const double q = d0 * d0 + d1 * d1 + d2 * d2;
  err2[o] = q;
  enorm[o] = sqrt(q);
  gnorm[o] = sqrt(g0 * g0 + g1 * g1 + g2 * g2);
}

// column sums over the vertices (thread = frame, ascending i: deterministic)
__global__ void k_frame_sums(int n, int F, const double* __restrict__ err2,
                             const double* __restrict__ enorm, const double* __restrict__ gnorm,
                             double* rms, double* nmsve) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  double s2 = 0.0, se = 0.0, sg = 0.0;
  for (int i = 0; i < n; ++i) {
    const size_t o = (size_t)i * F + f;
    s2 += err2[o];
    se += enorm[o];
    sg += gnorm[o];
  }
  rms[f] = sqrt(s2 / n);
  nmsve[f] = (se + sg) / (2.0 * n);
}

// vertex_mean_error(i) = mean over frames of |d|
__global__ void k_vertex_means(int n, int F, const double* __restrict__ enorm, double* vme) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int f = 0; f < F; ++f) s += enorm[(size_t)i * F + f];
  vme[i] = s / F;
}

}  // namespace

cudaError_t launch_distortion(cudaStream_t s, int n, int F, const uint32_t* lap_rp,
                              const uint32_t* lap_ci, const void* const a[3],
                              const void* const b[3], bool f32, double* work, double* rms,
                              double* nmsve, double* vme) {
  const long tot = (long)n * F;
  double* err2 = work;
  double* en = work + tot;
  double* gn = work + 2 * tot;
  const unsigned g = (unsigned)((tot + 255) / 256);
  if (f32)
    k_distortion_terms<float><<<g, 256, 0, s>>>(
        n, F, lap_rp, lap_ci, (const float*)a[0], (const float*)a[1], (const float*)a[2],
        (const float*)b[0], (const float*)b[1], (const float*)b[2], err2, en, gn);
  else
    k_distortion_terms<double><<<g, 256, 0, s>>>(
        n, F, lap_rp, lap_ci, (const double*)a[0], (const double*)a[1], (const double*)a[2],
        (const double*)b[0], (const double*)b[1], (const double*)b[2], err2, en, gn);
  k_frame_sums<<<(F + 127) / 128, 128, 0, s>>>(n, F, err2, en, gn, rms, nmsve);
  if (vme) k_vertex_means<<<(n + 255) / 256, 256, 0, s>>>(n, F, en, vme);
  return cudaGetLastError();
}

}  // namespace dmcg
