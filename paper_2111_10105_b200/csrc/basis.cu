// K3 — small dense kernels of the temporal basis: Householder QR (rank
// safe), round-robin Jacobi eigensolver, descending sort, canonical signs.
// One CTA per axis; matrices are F x k / k x k (F <= 512) and live in L2 /
// shared memory.  Compiled with --fmad=false so the arithmetic mirrors the
// oracle restatement (oracle/dmc_oracle.c) operation for operation.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace dmcg {

namespace {

constexpr int kBasisThreads = 1024;

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// Householder QR (Eigen::HouseholderQR / makeHouseholder semantics, see
// oracle householder_factor): beta = -sign(c0)||x||, tau = (beta-c0)/beta,
// v = [1; tail/(c0-beta)]; a vanishing tail gives tau = 0, so rank-deficient
// inputs (the normal case) never divide by zero and Q
// stays orthonormal.
__global__ void __launch_bounds__(kBasisThreads)
    k_householder(int m, int p, int c0, int ncols, double* Zall, double* tauall, double* Qall) {
  __shared__ double red[33];
  __shared__ double s_tau, s_den;
  const int b = blockIdx.x;
  double* Z = Zall + (size_t)b * m * p;
  double* tau = tauall + (size_t)b * p;
  double* Q = Qall + (size_t)b * m * ncols;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int pe = p < m ? p : m;
  for (int j = 0; j < pe; ++j) {
    double* x = Z + (size_t)j * m;
    double part = 0.0;
    for (int i = j + 1 + tid; i < m; i += blockDim.x) part = __dadd_rn(part, __dmul_rn(x[i], x[i]));
    const double tail = block_sum(part, red);
    if (tid == 0) {
      const double c = x[j];
      if (tail <= DBL_MIN) {
        s_tau = 0.0;
        s_den = 0.0;
      } else {
        double bb = sqrt(c * c + tail);
        if (c >= 0.0) bb = -bb;
        s_den = c - bb;
        s_tau = (bb - c) / bb;
        x[j] = bb;
      }
      tau[j] = s_tau;
    }
    __syncthreads();
    const double tj = s_tau, den = s_den;
    if (tj == 0.0) {
      for (int i = j + 1 + tid; i < m; i += blockDim.x) x[i] = 0.0;
      __syncthreads();
      continue;
    }
    for (int i = j + 1 + tid; i < m; i += blockDim.x) x[i] = x[i] / den;
    __syncthreads();
    for (int c = j + 1 + warp; c < p; c += nw) {
      double* y = Z + (size_t)c * m;
      double d = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) d += x[i] * y[i];
      d = warp_sum(d);
      d = tj * (y[j] + d);
      __syncwarp();
      if (lane == 0) y[j] = y[j] - d;
      for (int i = j + 1 + lane; i < m; i += 32) y[i] = y[i] - d * x[i];
    }
    __syncthreads();
  }
  // Q = H_0 ... H_{p-1} [e_c0 ... e_{c0+ncols-1}], backward accumulation.
  for (long t = tid; t < (long)m * ncols; t += blockDim.x) Q[t] = 0.0;
  __syncthreads();
  for (int c = tid; c < ncols; c += blockDim.x)
    if (c0 + c < m) Q[(size_t)c * m + c0 + c] = 1.0;
  __syncthreads();
  for (int j = pe - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj == 0.0) continue;
    const double* v = Z + (size_t)j * m;
    // columns whose identity seed sits above row j are untouched by H_j
    // only if their current rows >= j are zero: true for c0 + c < j when
    // c0 == 0 (thin Q); the completion (c0 >= p) touches every column.
    const int cstart = (c0 == 0) ? (j < ncols ? j : ncols) : 0;
    for (int c = cstart + warp; c < ncols; c += nw) {
      double* y = Q + (size_t)c * m;
      double d = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) d += v[i] * y[i];
      d = warp_sum(d);
      d = tj * (y[j] + d);
      __syncwarp();
      if (lane == 0) y[j] = y[j] - d;
      for (int i = j + 1 + lane; i < m; i += 32) y[i] = y[i] - d * v[i];
    }
    __syncthreads();
  }
}

// Round-robin pairing (identical to oracle rr_pair).
__device__ __forceinline__ void rr_pair(int m2, int s, int i, int* p, int* q) {
  const int r = m2 - 1;
  int a, bb;
  if (i == 0) {
    a = 0;
    bb = (s + r - 1) % r + 1;
  } else {
    a = (i + s - 1) % r + 1;
    bb = (r - i + s - 1) % r + 1;
  }
  *p = a < bb ? a : bb;
  *q = a < bb ? bb : a;
}

// Parallel (round-robin) cyclic Jacobi.  Every step applies m2/2 disjoint
// rotations at once; each 2x2 block of A is transformed independently, so
// the arithmetic per element equals the sequential oracle's.
__global__ void __launch_bounds__(kBasisThreads)
    k_jacobi(int m, const double* __restrict__ Aall, double* work, double* Vall, double* wall,
             int* flags, int use_smem) {
  extern __shared__ double dyn[];
  __shared__ double cs[256], sn[256], tn[256];
  __shared__ int P[256], Qi[256];
  __shared__ unsigned char act[256];
  __shared__ int s_rot;
  __shared__ double red[33];
  const int b = blockIdx.x;
  const int m2 = m + (m & 1), h = m2 / 2;
  double* A = use_smem ? dyn : work + (size_t)b * 2 * m2 * m2;
  double* V = A + (size_t)m2 * m2;
  const double* Ain = Aall + (size_t)b * m * m;
  const int tid = threadIdx.x;
  double part = 0.0;
  for (long t = tid; t < (long)m2 * m2; t += blockDim.x) {
    const int c = (int)(t / m2), r = (int)(t % m2);
    const double v = (r < m && c < m) ? Ain[(size_t)c * m + r] : 0.0;
    A[t] = v;
    V[t] = (r == c) ? 1.0 : 0.0;
    part += v * v;
  }
  const double fro = sqrt(block_sum(part, red));
  const double abs_thresh = fro * 1e-22 + DBL_MIN;
  bool converged = (m2 <= 1);
  for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int s = 0; s + 1 < m2; ++s) {
      for (int i = tid; i < h; i += blockDim.x) {
        int p, q;
        rr_pair(m2, s, i, &p, &q);
        P[i] = p;
        Qi[i] = q;
        const double app = A[(size_t)p * m2 + p], aqq = A[(size_t)q * m2 + q];
        const double apq = A[(size_t)q * m2 + p];
        const double rel = 1e-17 * sqrt(fabs(app) * fabs(aqq));
        const double thresh = rel > abs_thresh ? rel : abs_thresh;
        unsigned char on = 0;
        double c = 1.0, sv = 0.0, tt = 0.0;
        if (fabs(apq) > thresh) {
          const double theta = (aqq - app) / (2.0 * apq);
          if (fabs(theta) > 1e150)
            tt = 0.5 / theta;
          else
            tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(tt * tt + 1.0);
          sv = tt * c;
          on = 1;
          atomicAdd(&s_rot, 1);
        }
        cs[i] = c;
        sn[i] = sv;
        tn[i] = tt;
        act[i] = on;
      }
      __syncthreads();
      for (int t = tid; t < h * h; t += blockDim.x) {
        const int a = t / h, bb = t % h;
        if (bb < a) continue;
        const int p1 = P[a], q1 = Qi[a], p2 = P[bb], q2 = Qi[bb];
        if (a == bb) {
          if (act[a]) {
            const double apq = A[(size_t)q1 * m2 + p1];
            A[(size_t)p1 * m2 + p1] = A[(size_t)p1 * m2 + p1] - tn[a] * apq;
            A[(size_t)q1 * m2 + q1] = A[(size_t)q1 * m2 + q1] + tn[a] * apq;
            A[(size_t)q1 * m2 + p1] = 0.0;
            A[(size_t)p1 * m2 + q1] = 0.0;
          }
          continue;
        }
        if (!act[a] && !act[bb]) continue;
        const double ca = cs[a], sa = sn[a], cb = cs[bb], sb = sn[bb];
        const double b00 = A[(size_t)p2 * m2 + p1], b01 = A[(size_t)q2 * m2 + p1];
        const double b10 = A[(size_t)p2 * m2 + q1], b11 = A[(size_t)q2 * m2 + q1];
        const double r00 = ca * b00 - sa * b10, r01 = ca * b01 - sa * b11;
        const double r10 = sa * b00 + ca * b10, r11 = sa * b01 + ca * b11;
        const double n00 = cb * r00 - sb * r01, n01 = sb * r00 + cb * r01;
        const double n10 = cb * r10 - sb * r11, n11 = sb * r10 + cb * r11;
        A[(size_t)p2 * m2 + p1] = n00;
        A[(size_t)p1 * m2 + p2] = n00;
        A[(size_t)q2 * m2 + p1] = n01;
        A[(size_t)p1 * m2 + q2] = n01;
        A[(size_t)p2 * m2 + q1] = n10;
        A[(size_t)q1 * m2 + p2] = n10;
        A[(size_t)q2 * m2 + q1] = n11;
        A[(size_t)q1 * m2 + q2] = n11;
      }
      for (int t = tid; t < h * m2; t += blockDim.x) {
        const int a = t / m2, r = t % m2;
        if (!act[a]) continue;
        double* vp = V + (size_t)P[a] * m2;
        double* vq = V + (size_t)Qi[a] * m2;
        const double x = vp[r], y = vq[r];
        vp[r] = cs[a] * x - sn[a] * y;
        vq[r] = sn[a] * x + cs[a] * y;
      }
      __syncthreads();
    }
    converged = (s_rot == 0);
    __syncthreads();
  }
  double* Vo = Vall + (size_t)b * m * m;
  double* wo = wall + (size_t)b * m;
  for (long t = tid; t < (long)m * m; t += blockDim.x) {
    const int c = (int)(t / m), r = (int)(t % m);
    Vo[t] = V[(size_t)c * m2 + r];
  }
  for (int j = tid; j < m; j += blockDim.x) wo[j] = A[(size_t)j * m2 + j];
  if (!converged && tid == 0) atomicOr(flags, 1);
}

// Stable descending order by rank counting; Vs[:, j] = V[:, idx[j]].
__global__ void k_sort_basis(int m, int ncols_store, const double* __restrict__ Vall,
                             const double* __restrict__ wall, double* Vs, long vs_bs, double* ws,
                             long ws_bs) {
  extern __shared__ double sw[];
  int* idx = (int*)(sw + m);
  const int b = blockIdx.x;
  const double* V = Vall + (size_t)b * m * m;
  const double* w = wall + (size_t)b * m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) sw[i] = w[i];
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double wi = sw[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) rank += (sw[j] > wi) || (sw[j] == wi && j < i);
    idx[rank] = i;
  }
  __syncthreads();
  double* out = Vs + b * vs_bs;
  for (long t = threadIdx.x; t < (long)m * ncols_store; t += blockDim.x) {
    const int j = (int)(t / m), r = (int)(t % m);
    out[t] = V[(size_t)idx[j] * m + r];
  }
  for (int j = threadIdx.x; j < ncols_store; j += blockDim.x) ws[b * ws_bs + j] = sw[idx[j]];
}

// canonicalize_signs (spectral.cpp:41-47): first index of the largest |u|.
__global__ void k_canon_signs(int m, int c0, int ncols, double* Uall, long bs) {
  const int b = blockIdx.y;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= ncols) return;
  double* u = Uall + b * bs + (size_t)(c0 + warp) * m;
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
  const bool flip = u[bi] < 0.0;
  if (flip)
    for (int i = lane; i < m; i += 32) u[i] = -u[i];
}

// H <- 0.5 (H + H^T) (Rayleigh-Ritz matrix).
__global__ void k_symmetrize(int m, double* Hall) {
  double* H = Hall + (size_t)blockIdx.y * m * m;
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= (long)m * m) return;
  const int j = (int)(t / m), i = (int)(t % m);
  if (i >= j) return;
  const double s = 0.5 * (H[(size_t)j * m + i] + H[(size_t)i * m + j]);
  H[(size_t)j * m + i] = s;
  H[(size_t)i * m + j] = s;
}

__global__ void k_fill_zero(double* p, long count) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t < count) p[t] = 0.0;
}

}  // namespace

cudaError_t launch_householder(cudaStream_t s, int nbatch, int m, int p, int c0, int ncols,
                               double* Z, double* tau, double* Qout) {
  k_householder<<<nbatch, kBasisThreads, 0, s>>>(m, p, c0, ncols, Z, tau, Qout);
  return cudaGetLastError();
}

cudaError_t launch_jacobi(cudaStream_t s, int nbatch, int m, const double* A, double* work,
                          double* V, double* w, int* flags) {
  if (m > 512) return cudaErrorInvalidValue;
  const int m2 = m + (m & 1);
  const size_t smem = (size_t)2 * m2 * m2 * sizeof(double);
  int use_smem = smem <= 200 * 1024;
  if (use_smem) {
    cudaError_t e = cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_jacobi<<<nbatch, kBasisThreads, use_smem ? smem : 0, s>>>(m, A, work, V, w, flags, use_smem);
  return cudaGetLastError();
}

cudaError_t launch_sort_basis(cudaStream_t s, int nbatch, int m, int ncols_store, const double* V,
                              const double* w, double* Vs, long vs_bs, double* ws, long ws_bs) {
  const size_t smem = (size_t)m * sizeof(double) + (size_t)m * sizeof(int);
  k_sort_basis<<<nbatch, 512, smem, s>>>(m, ncols_store, V, w, Vs, vs_bs, ws, ws_bs);
  return cudaGetLastError();
}

cudaError_t launch_canon_signs(cudaStream_t s, int nbatch, int m, int c0, int ncols, double* U,
                               long bs) {
  if (ncols <= 0) return cudaSuccess;
  const int warps_per_block = 8;
  dim3 grid((ncols + warps_per_block - 1) / warps_per_block, nbatch);
  k_canon_signs<<<grid, warps_per_block * 32, 0, s>>>(m, c0, ncols, U, bs);
  return cudaGetLastError();
}

cudaError_t launch_symmetrize(cudaStream_t s, int nbatch, int m, double* H) {
  dim3 grid((unsigned)(((long)m * m + 255) / 256), nbatch);
  k_symmetrize<<<grid, 256, 0, s>>>(m, H);
  return cudaGetLastError();
}

cudaError_t launch_fill_zero(cudaStream_t s, double* p, long count) {
  if (count <= 0) return cudaSuccess;
  k_fill_zero<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(p, count);
  return cudaGetLastError();
}

}  // namespace dmcg
