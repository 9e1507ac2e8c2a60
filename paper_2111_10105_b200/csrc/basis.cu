// K3 — small dense kernels of the temporal basis: Householder QR (rank
// safe), round-robin Jacobi eigensolver, descending sort, canonical signs.
// One CTA per axis; matrices are F x k / k x k (F <= 512) and live in L2 /
// shared memory.  Same algorithms and formulas as the oracle restatement
// (oracle/dmc_oracle.c: householder_factor, orc_jacobi_eig, orc_basis);
// reductions run in parallel order and use FMA, so results agree with the
// oracle to rounding, not bit for bit (P3).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace dmcg {

namespace {

constexpr int kBasisThreads = 1024;
constexpr int kOiThreads = 512;  // fused OI kernels: 128 registers per thread

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

// Parallel (round-robin) cyclic Jacobi.  Every step applies m2/2 disjoint
// rotations at once; each 2x2 block of A is transformed independently.  A
// lives in shared memory with an odd leading dimension (m2 + 1: the 2x2
// block gathers of a warp hit distinct banks).  The eigenvector rows are
// split over gridDim.y CTAs per matrix: each CTA repeats the (cheap,
// deterministic) A updates and rotates only its slice of V rows, so no
// inter-CTA traffic is needed.  a_smem = 0 keeps A and V in `work`
// (gridDim.y must then be 1).
constexpr int kJacThreads = 512;

__global__ void __launch_bounds__(kJacThreads)
    k_jacobi(int m, const double* __restrict__ Aall, double* work, double* Vall, double* wall,
             int* flags, int a_smem, int vrows) {
  extern __shared__ double dyn[];
  __shared__ double cs[256], sn[256], tn[256];
  __shared__ int P[256], Qi[256];
  __shared__ double red[33];
  const int b = blockIdx.x, sp = blockIdx.y;
  const int m2 = m + (m & 1), h = m2 / 2, ld = m2 + 1, rr = m2 - 1;
  const int r0 = sp * vrows, r1 = min(m2, r0 + vrows), nr = r1 - r0;
  const int tid = threadIdx.x, NT = blockDim.x;
  double* A;
  double* V;  // V(c, r) = V[c * ldv + r - r0]
  int ldv;
  if (a_smem) {
    A = dyn;
    V = dyn + (size_t)m2 * ld;
    ldv = nr;
  } else {
    A = work + (size_t)b * 2 * m2 * ld;
    V = A + (size_t)m2 * ld;
    ldv = m2;
  }
  const double* Ain = Aall + (size_t)b * m * m;
  double part = 0.0;
  for (int c = 0; c < m2; ++c)
    for (int r = tid; r < m2; r += NT) {
      const double v = (r < m && c < m) ? Ain[(size_t)c * m + r] : 0.0;
      A[c * ld + r] = v;
      part += v * v;
    }
  for (int c = 0; c < m2; ++c)
    for (int r = r0 + tid; r < r1; r += NT) V[c * ldv + r - r0] = (r == c) ? 1.0 : 0.0;
  const double fro = sqrt(block_sum(part, red));
  const double abs_thresh = fro * 1e-22 + DBL_MIN;
  // per-thread task cursors (square h x h for A blocks, h x nr for V rows)
  const int da = NT / h, db = NT % h;
  const int dva = nr > 0 ? NT / nr : 0, dvr = nr > 0 ? NT % nr : 0;
  bool converged = (m2 <= 1);
  for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
    int any = 0;
    for (int s = 0; s + 1 < m2; ++s) {
      int on = 0;
      for (int i = tid; i < h; i += NT) {
        int x, y;
        if (i == 0) {
          x = 0;
          y = s + rr - 1;
          if (y >= rr) y -= rr;
          ++y;
        } else {
          x = i + s - 1;
          if (x >= rr) x -= rr;
          ++x;
          y = rr - i + s - 1;
          if (y >= rr) y -= rr;
          ++y;
        }
        const int p = x < y ? x : y, q = x < y ? y : x;
        P[i] = p;
        Qi[i] = q;
        const double app = A[p * ld + p], aqq = A[q * ld + q];
        const double apq = A[q * ld + p];
        const double rel = 1e-17 * sqrt(fabs(app) * fabs(aqq));
        const double thresh = rel > abs_thresh ? rel : abs_thresh;
        double c = 1.0, sv = 0.0, tt = 0.0;
        if (fabs(apq) > thresh) {
          const double theta = (aqq - app) / (2.0 * apq);
          if (fabs(theta) > 1e150)
            tt = 0.5 / theta;
          else
            tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = rsqrt(tt * tt + 1.0);
          sv = tt * c;
          on = 1;
        }
        cs[i] = c;
        sn[i] = sv;
        tn[i] = tt;
      }
      if (!__syncthreads_or(on)) continue;  // nothing to rotate at this step
      any = 1;
      {
        int a = tid / h, bb = tid % h;
        for (; a < h; a += da, bb += db) {
          if (bb >= h) {
            bb -= h;
            ++a;
            if (a >= h) break;
          }
          if (bb < a) continue;
          const int p1 = P[a], q1 = Qi[a];
          if (a == bb) {
            const double t = tn[a];
            if (t != 0.0) {
              const double apq = A[q1 * ld + p1];
              A[p1 * ld + p1] = A[p1 * ld + p1] - t * apq;
              A[q1 * ld + q1] = A[q1 * ld + q1] + t * apq;
              A[q1 * ld + p1] = 0.0;
              A[p1 * ld + q1] = 0.0;
            }
            continue;
          }
          const double sa = sn[a], sb = sn[bb];
          if (sa == 0.0 && sb == 0.0) continue;
          const int p2 = P[bb], q2 = Qi[bb];
          const double ca = cs[a], cb = cs[bb];
          const double b00 = A[p2 * ld + p1], b01 = A[q2 * ld + p1];
          const double b10 = A[p2 * ld + q1], b11 = A[q2 * ld + q1];
          const double r00 = ca * b00 - sa * b10, r01 = ca * b01 - sa * b11;
          const double r10 = sa * b00 + ca * b10, r11 = sa * b01 + ca * b11;
          const double n00 = cb * r00 - sb * r01, n01 = sb * r00 + cb * r01;
          const double n10 = cb * r10 - sb * r11, n11 = sb * r10 + cb * r11;
          A[p2 * ld + p1] = n00;
          A[p1 * ld + p2] = n00;
          A[q2 * ld + p1] = n01;
          A[p1 * ld + q2] = n01;
          A[p2 * ld + q1] = n10;
          A[q1 * ld + p2] = n10;
          A[q2 * ld + q1] = n11;
          A[q1 * ld + q2] = n11;
        }
      }
      if (nr > 0) {
        int a = tid / nr, r = tid % nr;
        for (; a < h; a += dva, r += dvr) {
          if (r >= nr) {
            r -= nr;
            ++a;
            if (a >= h) break;
          }
          const double sa = sn[a];
          if (sa == 0.0) continue;
          const double ca = cs[a];
          double* vp = V + P[a] * ldv;
          double* vq = V + Qi[a] * ldv;
          const double x = vp[r], y = vq[r];
          vp[r] = ca * x - sa * y;
          vq[r] = sa * x + ca * y;
        }
      }
      __syncthreads();
    }
    converged = !any;
  }
  double* Vo = Vall + (size_t)b * m * m;
  for (int c = 0; c < m; ++c)
    for (int r = r0 + tid; r < min(r1, m); r += NT) Vo[(size_t)c * m + r] = V[c * ldv + r - r0];
  if (sp == 0) {
    double* wo = wall + (size_t)b * m;
    for (int j = tid; j < m; j += NT) wo[j] = A[j * ld + j];
    if (!converged && tid == 0) atomicOr(flags, 1);
  }
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

// ---------------------------------------------------------------------------
// Fused orthogonal iterations: one CTA per axis runs every round
//   Z = R Q  (SIMT, R from L2, Q in smem);  Q = thin Householder Q of Z
// and the Rayleigh-Ritz matrix H = Q^T R Q, with Z and Q in shared memory
// when 2 F k doubles fit (else in a global work area, L1/L2 resident).
// The Householder QR needs one CTA barrier per column: the warp that
// updates column j+1 in step j also computes column j+1's reflector, and
// the scaling of reflector j is deferred to step j+1 (column j is read
// unscaled, divided on the fly, during step j).
// ---------------------------------------------------------------------------
struct QrShared {
  double tau[512], rinv[512];
};

// Register-blocked warp primitives: a lane owns rows j+1+lane+32t,
// t < MAXR (MAXR = ceil(F/32) <= 16), so all its loads issue back to back.

// Reflector of column c (rows >= c) by one warp: tau and 1/(c0 - beta), the
// diagonal set to beta (the oracle's householder_factor formulas; the GPU
// scales by the reciprocal instead of dividing element by element, a
// 1-ulp difference inside the P3 tolerance).
template <int MAXR, typename P>
__device__ __forceinline__ void qr_reflector(P Z, int m, int c, QrShared& q, int lane) {
  P x = Z + c * m;
  double p0 = 0.0, p1 = 0.0;
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    const int i = c + 1 + lane + 32 * t;
    const double xi = i < m ? x[i] : 0.0;
    if (t & 1)
      p1 += xi * xi;
    else
      p0 += xi * xi;
  }
  const double tail = warp_sum(p0 + p1);
  const double c0 = x[c];
  double rinv = 0.0, tau = 0.0;
  if (tail > DBL_MIN) {
    const double s2 = c0 * c0 + tail;
    const double r = rsqrt(s2);
    const double nrm = s2 * r;
    const double bb = c0 >= 0.0 ? -nrm : nrm;
    const double ibb = c0 >= 0.0 ? -r : r;
    rinv = __drcp_rn(c0 - bb);
    tau = (bb - c0) * ibb;
    __syncwarp();
    if (lane == 0) x[c] = bb;
  }
  if (lane == 0) {
    q.tau[c] = tau;
    q.rinv[c] = rinv;
  }
  __syncwarp();
}

// y_c -= tau v (v^T y_c) for columns c = c0, c0 + stride, ... < cend (rows > j
// of v are vs * v[i]; v[j] = 1 implicit), two columns per pass so their
// warp reductions overlap.
template <int MAXR, typename PY, typename PV>
__device__ __forceinline__ void apply_reflector_cols(PY Y, int ld, int j, PV v, double vs,
                                                     double tau, int c0, int cend, int stride,
                                                     int lane, int m) {
  if (c0 >= cend) return;
  double vr[MAXR];
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    const int i = j + 1 + lane + 32 * t;
    vr[t] = i < m ? v[i] * vs : 0.0;
  }
  for (int c = c0; c < cend; c += 2 * stride) {
    const bool two = c + stride < cend;
    PY ya = Y + c * ld;
    PY yb = Y + (two ? c + stride : c) * ld;
    double ra[MAXR], rb[MAXR];
#pragma unroll
    for (int t = 0; t < MAXR; ++t) {
      const int i = j + 1 + lane + 32 * t;
      ra[t] = i < m ? ya[i] : 0.0;
      rb[t] = (two && i < m) ? yb[i] : 0.0;
    }
    double da0 = 0.0, da1 = 0.0, db0 = 0.0, db1 = 0.0;
#pragma unroll
    for (int t = 0; t < MAXR; ++t) {
      if (t & 1) {
        da1 += vr[t] * ra[t];
        db1 += vr[t] * rb[t];
      } else {
        da0 += vr[t] * ra[t];
        db0 += vr[t] * rb[t];
      }
    }
    double da = da0 + da1, db = db0 + db1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      da += __shfl_xor_sync(0xffffffffu, da, o);
      db += __shfl_xor_sync(0xffffffffu, db, o);
    }
    const double yja = ya[j], yjb = two ? yb[j] : 0.0;
    da = tau * (yja + da);
    db = tau * (yjb + db);
    __syncwarp();
    if (lane == 0) {
      ya[j] = yja - da;
      if (two) yb[j] = yjb - db;
    }
#pragma unroll
    for (int t = 0; t < MAXR; ++t) {
      const int i = j + 1 + lane + 32 * t;
      if (i < m) {
        ya[i] = ra[t] - da * vr[t];
        if (two) yb[i] = rb[t] - db * vr[t];
      }
    }
    __syncwarp();
  }
}

template <typename P>
__device__ __forceinline__ void qr_scale(P Z, int m, int j, const QrShared& q) {
  P x = Z + j * m;
  const double r = q.rinv[j];
  const bool zero = q.tau[j] == 0.0;
  for (int i = j + 1 + (int)threadIdx.x; i < m; i += blockDim.x) x[i] = zero ? 0.0 : x[i] * r;
}

// In-place Householder factorisation of the m x p column-major Z; on exit
// column j below the diagonal holds the scaled reflector (Eigen layout).
// One CTA barrier per column: reflector j+1 is computed by warp 0 right
// after it updates column j+1, and the scaling of column j is deferred to
// step j+1 (during step j the raw column is read and scaled on the fly).
template <int MAXR, typename P>
__device__ void qr_factor(P Z, int m, int p, QrShared& q) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int pe = p < m ? p : m;
  if (pe <= 0) return;
  if (warp == 0) qr_reflector<MAXR>(Z, m, 0, q, lane);
  __syncthreads();
  for (int j = 0; j < pe; ++j) {
    const double tj = q.tau[j], rj = q.rinv[j];
    if (j > 0) qr_scale(Z, m, j - 1, q);
    // warp 0: column j+1 alone, then reflector j+1, then its share of the
    // rest; columns j+2.. are spread over all warps.
    if (warp == 0 && j + 1 < p) {
      if (tj != 0.0) apply_reflector_cols<MAXR>(Z, m, j, Z + j * m, rj, tj, j + 1, j + 2, 1, lane, m);
      if (j + 1 < pe) qr_reflector<MAXR>(Z, m, j + 1, q, lane);
    }
    if (tj != 0.0) apply_reflector_cols<MAXR>(Z, m, j, Z + j * m, rj, tj, j + 2 + warp, p, nw, lane, m);
    __syncthreads();
  }
  qr_scale(Z, m, pe - 1, q);
  __syncthreads();
}

// Qout (m x ncols, leading dimension ldq) = H_0 ... H_{pe-1} [e_c0 ...].
template <int MAXR, typename PZ, typename PQ>
__device__ void qr_form(PZ Z, int m, int p, int c0, int ncols, PQ Qo, int ldq, const QrShared& q) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int pe = p < m ? p : m;
  for (int t = threadIdx.x; t < m * ncols; t += blockDim.x) {
    const int c = t / m, r = t % m;
    Qo[c * ldq + r] = (r == c0 + c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = pe - 1; j >= 0; --j) {
    const double tj = q.tau[j];
    if (tj == 0.0) continue;
    PZ v = Z + j * m;
    const int cstart = (c0 == 0) ? (j < ncols ? j : ncols) : 0;
    apply_reflector_cols<MAXR>(Qo, ldq, j, v, 1.0, tj, cstart + warp, ncols, nw, lane, m);
    __syncthreads();
  }
}

// Z (F x k) = R (F x F, symmetric, global) * Q (F x k) on the FP64 tensor
// pipe: each warp owns an 8-row block and up to 64 columns (8 DMMA tiles of
// 8x8, K = F in steps of 4).  A fragments stream from L2, B from Q.
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename PA, typename PB, typename PC>
__device__ void warp_gemm_tn(int M, int N, int K, PA A, int lda, PB B, int ldb, PC C, int ldc) {
  // C (M x N, col-major ldc) = A^T B with A (K x M, col-major lda: A(k,i) =
  // A[i*lda + k]) ... general form: C(i, j) = sum_k A[i*lda + k] * B[j*ldb + k]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mb = (M + 7) / 8, nbk = (N + 63) / 64;
  for (int t = warp; t < mb * nbk; t += nw) {
    const int i0 = (t % mb) * 8, j00 = (t / mb) * 64;
    double acc[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u][0] = acc[u][1] = 0.0;
    const int ia = i0 + (lane >> 2);
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int ka = k0 + (lane & 3);
      const double a = (ia < M && ka < K) ? A[ia * lda + ka] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int jb = j00 + u * 8 + (lane >> 2);
        const double b = (jb < N && ka < K) ? B[jb * ldb + ka] : 0.0;
        dmma884(acc[u], a, b);
      }
    }
    const int ir = i0 + (lane >> 2);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jc = j00 + u * 8 + (lane & 3) * 2 + e;
        if (ir < M && jc < N) C[jc * ldc + ir] = acc[u][e];
      }
  }
}

// Z = R Q: Z(g, j) = sum_f R(g, f) Q(f, j) = sum_f R[g*F + f] Q[j*F + f]
// (R symmetric, so its column g is its row g).
template <typename P>
__device__ void oi_apply(const double* __restrict__ R, int F, int k, P Q, P Z) {
  warp_gemm_tn(F, k, F, R, F, Q, F, Z, F);
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Blocked (compact-WY) Householder QR.  Columns are factored in panels of
// QNB: only the panel sees per-column steps (one barrier each); the rest of
// the matrix and the formation of Q are updated with small DMMA GEMMs,
//   Y <- (I - V T V^T)^T Y,   Q <- (I - V T V^T) Q,
// T being the LAPACK dlarft forward/columnwise triangular factor.  Scratch
// (global, L1-resident): T of every panel, W (QNB x ncols), G (QNB x QNB).
// ---------------------------------------------------------------------------
constexpr int QNB = 16;

// CTA GEMM on the FP64 tensor pipe with functor operands:
//   for m < M, n < N:  st(m, n, sum_k la(m, k) * lb(k, n))
template <class LA, class LB, class ST>
__device__ void cta_gemm(int M, int N, int K, const LA& la, const LB& lb, const ST& st) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mt = (M + 7) / 8, nt = (N + 31) / 32;
  for (int t = warp; t < mt * nt; t += nw) {
    const int m0 = (t % mt) * 8, n0 = (t / mt) * 32;
    double acc[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u][0] = acc[u][1] = 0.0;
    const int ma = m0 + (lane >> 2);
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int ka = k0 + (lane & 3);
      const double a = (ma < M && ka < K) ? la(ma, ka) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int nb = n0 + u * 8 + (lane >> 2);
        const double b = (nb < N && ka < K) ? lb(ka, nb) : 0.0;
        dmma884(acc[u], a, b);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int nc = n0 + u * 8 + (lane & 3) * 2 + e;
        if (ma < M && nc < N) st(ma, nc, acc[u][e]);
      }
  }
  __syncthreads();
}

// V(g, i) of the panel starting at column c0, g counted from row c0: unit
// diagonal, zero above it, the stored (scaled) reflector below.
template <typename P>
struct PanelV {
  P Z;
  int m, c0;
  __device__ __forceinline__ double operator()(int g, int i) const {
    return g < i ? 0.0 : (g == i ? 1.0 : Z[(c0 + i) * m + c0 + g]);
  }
};

// Unblocked factorisation of the panel columns [c0, ce), one barrier per column.
template <int MAXR, typename P>
__device__ void panel_factor(P Z, int m, int c0, int ce, QrShared& q) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (warp == 0) qr_reflector<MAXR>(Z, m, c0, q, lane);
  __syncthreads();
  for (int j = c0; j < ce; ++j) {
    const double tj = q.tau[j], rj = q.rinv[j];
    if (j > c0) qr_scale(Z, m, j - 1, q);
    if (warp == 0 && j + 1 < ce) {
      if (tj != 0.0) apply_reflector_cols<MAXR>(Z, m, j, Z + j * m, rj, tj, j + 1, j + 2, 1, lane, m);
      qr_reflector<MAXR>(Z, m, j + 1, q, lane);
    }
    if (tj != 0.0) apply_reflector_cols<MAXR>(Z, m, j, Z + j * m, rj, tj, j + 2 + warp, ce, nw, lane, m);
    __syncthreads();
  }
  qr_scale(Z, m, ce - 1, q);
  __syncthreads();
}

// T (row-major QNB x QNB, upper) of the panel [c0, c0+pb): T(i,i) = tau_i,
// T(0:i, i) = -tau_i T(0:i, 0:i) (V(:, 0:i)^T v_i).
template <typename P>
__device__ void panel_T(P Z, int m, int c0, int pb, const QrShared& q, double* T, double* G) {
  PanelV<P> V{Z, m, c0};
  cta_gemm(pb, pb, m - c0, [&](int a, int g) { return V(g, a); }, V,
           [&](int a, int b, double v) { G[a * QNB + b] = v; });
  if (threadIdx.x < 32) {
    const int j = threadIdx.x;
    for (int i = 0; i < pb; ++i) {
      const double ti = q.tau[c0 + i];
      if (j < i) {
        double acc = 0.0;
        for (int l = j; l < i; ++l) acc += T[j * QNB + l] * G[l * QNB + i];
        T[j * QNB + i] = -ti * acc;
      }
      if (j == i) T[i * QNB + i] = ti;
      if (j > i && j < QNB) T[j * QNB + i] = 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
}

template <int MAXR, typename P>
__device__ void bqr_factor(P Z, int m, int p, QrShared& q, double* scr, int wcols) {
  const int pe = p < m ? p : m;
  double* G = scr;                 // QNB x QNB
  double* W = G + QNB * QNB;       // QNB x wcols (wcols >= p)
  double* Ts = W + QNB * wcols;    // T of every panel
  for (int c0 = 0; c0 < pe; c0 += QNB) {
    const int pb = min(QNB, pe - c0);
    panel_factor<MAXR>(Z, m, c0, c0 + pb, q);
    double* T = Ts + (c0 / QNB) * QNB * QNB;
    panel_T(Z, m, c0, pb, q, T, G);
    const int rem = p - (c0 + pb);
    if (rem <= 0) continue;
    PanelV<P> V{Z, m, c0};
    P Y = Z + (c0 + pb) * m + c0;  // rows c0.., columns c0+pb..
    // W = V^T Y
    cta_gemm(pb, rem, m - c0, [&](int i, int g) { return V(g, i); },
             [&](int g, int c) { return Y[c * m + g]; }, [&](int i, int c, double v) { W[i * rem + c] = v; });
    // W <- T^T W  (row i needs rows l <= i: descending in place)
    for (int c = threadIdx.x; c < rem; c += blockDim.x)
      for (int i = pb - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int l = 0; l <= i; ++l) acc += T[l * QNB + i] * W[l * rem + c];
        W[i * rem + c] = acc;
      }
    __syncthreads();
    // Y -= V W
    cta_gemm(m - c0, rem, pb, V, [&](int i, int c) { return W[i * rem + c]; },
             [&](int g, int c, double v) { Y[c * m + g] -= v; });
  }
}

// Qout (m x ncols, leading dimension ldq) = H_0 ... H_{pe-1} [e_cid ...].
template <typename PZ, typename PQ>
__device__ void bqr_form(PZ Z, int m, int p, int cid, int ncols, PQ Qo, int ldq, double* scr,
                         int wcols) {
  const int pe = p < m ? p : m;
  double* W = scr + QNB * QNB;     // QNB x wcols (wcols >= ncols)
  const double* Ts = W + QNB * wcols;
  for (int t = threadIdx.x; t < m * ncols; t += blockDim.x) {
    const int c = t / m, r = t % m;
    Qo[c * ldq + r] = (r == cid + c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int npan = (pe + QNB - 1) / QNB;
  for (int pi = npan - 1; pi >= 0; --pi) {
    const int c0 = pi * QNB, pb = min(QNB, pe - c0);
    const double* T = Ts + pi * QNB * QNB;
    PanelV<PZ> V{Z, m, c0};
    // columns whose rows >= c0 are still zero are untouched (thin Q: c < c0)
    const int cs = (cid == 0) ? (c0 < ncols ? c0 : ncols) : 0;
    const int nc = ncols - cs;
    if (nc <= 0) continue;
    PQ Y = Qo + cs * ldq + c0;
    cta_gemm(pb, nc, m - c0, [&](int i, int g) { return V(g, i); },
             [&](int g, int c) { return Y[c * ldq + g]; }, [&](int i, int c, double v) { W[i * nc + c] = v; });
    // W <- T W  (row i needs rows l >= i: ascending in place)
    for (int c = threadIdx.x; c < nc; c += blockDim.x)
      for (int i = 0; i < pb; ++i) {
        double acc = 0.0;
        for (int l = i; l < pb; ++l) acc += T[i * QNB + l] * W[l * nc + c];
        W[i * nc + c] = acc;
      }
    __syncthreads();
    cta_gemm(m - c0, nc, pb, V, [&](int i, int c) { return W[i * nc + c]; },
             [&](int g, int c, double v) { Y[c * ldq + g] -= v; });
  }
}

template <int MAXR, typename P>
__device__ void oi_body(int F, int k, int rounds, const double* __restrict__ R,
                        const double* __restrict__ start, P Z, P Q, double* Qo, double* H,
                        QrShared& q, double* scr) {
  const int Fk = F * k;
  for (int t = threadIdx.x; t < Fk; t += blockDim.x) Z[t] = start[t];
  __syncthreads();
  bqr_factor<MAXR>(Z, F, k, q, scr, k);
  bqr_form(Z, F, k, 0, k, Q, F, scr, k);
  for (int r = 0; r < rounds; ++r) {
    oi_apply(R, F, k, Q, Z);
    bqr_factor<MAXR>(Z, F, k, q, scr, k);
    bqr_form(Z, F, k, 0, k, Q, F, scr, k);
  }
  // Rayleigh-Ritz: H = Q^T (R Q), symmetrised; Q out.
  oi_apply(R, F, k, Q, Z);
  // H(i, j) = sum_g Q(g, i) Z(g, j), then symmetrised like the oracle
  warp_gemm_tn(k, k, F, Q, F, Z, F, H, k);
  __syncthreads();
  for (int t = threadIdx.x; t < k * k; t += blockDim.x) {
    const int i = t % k, j = t / k;
    if (i >= j) continue;
    const double sv = 0.5 * (H[j * k + i] + H[i * k + j]);
    H[j * k + i] = sv;
    H[i * k + j] = sv;
  }
  for (int t = threadIdx.x; t < Fk; t += blockDim.x) Qo[t] = Q[t];
}

template <bool SMEM, int MAXR>
__global__ void __launch_bounds__(kOiThreads)
    k_oi_fused(int F, int k, int rounds, const double* __restrict__ Rall,
               const double* __restrict__ start, double* Qall, double* Hall, double* work,
               double* scr_all, size_t scr_stride, int scr_smem) {
  extern __shared__ double dyn[];
  __shared__ QrShared q;
  const int b = blockIdx.x;
  const size_t Fk = (size_t)F * k;
  const double* R = Rall + (size_t)b * F * F;
  double* scr = scr_smem ? dyn + (SMEM ? 2 * Fk : 0) : scr_all + b * scr_stride;
  if (SMEM)
    oi_body<MAXR>(F, k, rounds, R, start + b * Fk, dyn, dyn + Fk, Qall + b * Fk,
                  Hall + (size_t)b * k * k, q, scr);
  else
    oi_body<MAXR>(F, k, rounds, R, start + b * Fk, work + b * 2 * Fk, work + b * 2 * Fk + Fk,
                  Qall + b * Fk, Hall + (size_t)b * k * k, q, scr);
}

// Completion: columns k..F-1 of the full Householder Q of U_k (F x k, the
// first k columns of U), written straight into U.
template <bool SMEM, int MAXR>
__global__ void __launch_bounds__(kOiThreads)
    k_complete(int F, int k, double* Uall, double* work, double* scr_all, size_t scr_stride,
               int scr_smem) {
  extern __shared__ double dyn[];
  __shared__ QrShared q;
  const int b = blockIdx.x;
  const int Fk = F * k;
  double* Z = SMEM ? dyn : work + (size_t)b * Fk;
  double* U = Uall + (size_t)b * F * F;
  double* scr = scr_smem ? dyn + (SMEM ? Fk : 0) : scr_all + b * scr_stride;
  const int wc = k > F - k ? k : F - k;
  for (int t = threadIdx.x; t < Fk; t += blockDim.x) Z[t] = U[t];
  __syncthreads();
  if (SMEM) {
    bqr_factor<MAXR>(dyn, F, k, q, scr, wc);
    bqr_form(dyn, F, k, k, F - k, U + Fk, F, scr, wc);
  } else {
    bqr_factor<MAXR>(Z, F, k, q, scr, wc);
    bqr_form(Z, F, k, k, F - k, U + Fk, F, scr, wc);
  }
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

static cudaError_t set_smem_attr(const void* fn, size_t bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

constexpr size_t kBasisSmemMax = 200 * 1024;  // + ~17 KB static QrShared <= 227 KB

// Blocked-QR scratch: G (QNB^2) | W (QNB x wcols) | T of every panel.
static size_t qr_scratch(int wcols, int k) {
  const int npan = (k + QNB - 1) / QNB;
  return (size_t)QNB * QNB + (size_t)QNB * wcols + (size_t)npan * QNB * QNB;
}

size_t qr_scratch_doubles(int F, int k) { return qr_scratch(F > k ? F : k, k); }

// Dynamic shared memory left for `fn` next to its static shared memory.
static size_t smem_room(const void* fn) {
  static int optin = -1;
  if (optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      optin = 227 * 1024;
  }
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return 0;
  return (size_t)optin > fa.sharedSizeBytes + 256 ? optin - fa.sharedSizeBytes - 256 : 0;
}

cudaError_t launch_jacobi(cudaStream_t s, int nbatch, int m, const double* A, double* work,
                          double* V, double* w, int* flags) {
  if (m > 512) return cudaErrorInvalidValue;
  const int m2 = m + (m & 1);
  const size_t abytes = (size_t)m2 * (m2 + 1) * sizeof(double);
  const size_t room = smem_room((const void*)k_jacobi);
  int nsplit = 0;
  for (int sp = 1; sp <= 8 && abytes < room; sp *= 2) {
    const int vr = (m2 + sp - 1) / sp;
    if (abytes + (size_t)m2 * vr * sizeof(double) <= room) {
      nsplit = sp;
      break;
    }
  }
  if (nsplit > 0) {
    const int vr = (m2 + nsplit - 1) / nsplit;
    const size_t smem = abytes + (size_t)m2 * vr * sizeof(double);
    cudaError_t e = set_smem_attr((const void*)k_jacobi, smem);
    if (e != cudaSuccess) return e;
    k_jacobi<<<dim3(nbatch, nsplit), kJacThreads, smem, s>>>(m, A, work, V, w, flags, 1, vr);
  } else {
    k_jacobi<<<dim3(nbatch, 1), kJacThreads, 0, s>>>(m, A, work, V, w, flags, 0, m2);
  }
  return cudaGetLastError();
}

template <int MAXR>
static cudaError_t oi_fused_impl(cudaStream_t s, int nbatch, int F, int k, int rounds,
                                 const double* R, const double* start, double* Q, double* H,
                                 double* work, double* scr) {
  const size_t pair = (size_t)2 * F * k * sizeof(double);
  const size_t sbytes = qr_scratch(k, k) * sizeof(double);
  const size_t ss = qr_scratch_doubles(F, k);
  if (pair <= kBasisSmemMax) {
    const void* fn = (const void*)k_oi_fused<true, MAXR>;
    const int in_smem = pair + sbytes <= smem_room(fn);
    const size_t smem = pair + (in_smem ? sbytes : 0);
    cudaError_t e = set_smem_attr(fn, smem);
    if (e != cudaSuccess) return e;
    k_oi_fused<true, MAXR><<<nbatch, kOiThreads, smem, s>>>(F, k, rounds, R, start, Q, H, work,
                                                            scr, ss, in_smem);
  } else {
    const void* fn = (const void*)k_oi_fused<false, MAXR>;
    const int in_smem = sbytes <= smem_room(fn);
    const size_t smem = in_smem ? sbytes : 0;
    cudaError_t e = set_smem_attr(fn, smem);
    if (e != cudaSuccess) return e;
    k_oi_fused<false, MAXR><<<nbatch, kOiThreads, smem, s>>>(F, k, rounds, R, start, Q, H, work,
                                                             scr, ss, in_smem);
  }
  return cudaGetLastError();
}

cudaError_t launch_oi_fused(cudaStream_t s, int nbatch, int F, int k, int rounds, const double* R,
                            const double* start, double* Q, double* H, double* work, double* scr) {
  if (F > 512) return cudaErrorInvalidValue;
  if (F <= 64) return oi_fused_impl<2>(s, nbatch, F, k, rounds, R, start, Q, H, work, scr);
  if (F <= 128) return oi_fused_impl<4>(s, nbatch, F, k, rounds, R, start, Q, H, work, scr);
  if (F <= 256) return oi_fused_impl<8>(s, nbatch, F, k, rounds, R, start, Q, H, work, scr);
  return oi_fused_impl<16>(s, nbatch, F, k, rounds, R, start, Q, H, work, scr);
}

template <int MAXR>
static cudaError_t complete_impl(cudaStream_t s, int nbatch, int F, int k, double* U, double* work,
                                 double* scr) {
  const size_t zb = (size_t)F * k * sizeof(double);
  const size_t sbytes = qr_scratch(k > F - k ? k : F - k, k) * sizeof(double);
  const size_t ss = qr_scratch_doubles(F, k);
  if (zb <= kBasisSmemMax) {
    const void* fn = (const void*)k_complete<true, MAXR>;
    const int in_smem = zb + sbytes <= smem_room(fn);
    const size_t smem = zb + (in_smem ? sbytes : 0);
    cudaError_t e = set_smem_attr(fn, smem);
    if (e != cudaSuccess) return e;
    k_complete<true, MAXR><<<nbatch, kOiThreads, smem, s>>>(F, k, U, work, scr, ss, in_smem);
  } else {
    const void* fn = (const void*)k_complete<false, MAXR>;
    const int in_smem = sbytes <= smem_room(fn);
    const size_t smem = in_smem ? sbytes : 0;
    cudaError_t e = set_smem_attr(fn, smem);
    if (e != cudaSuccess) return e;
    k_complete<false, MAXR><<<nbatch, kOiThreads, smem, s>>>(F, k, U, work, scr, ss, in_smem);
  }
  return cudaGetLastError();
}

cudaError_t launch_complete(cudaStream_t s, int nbatch, int F, int k, double* U, double* work,
                            double* scr) {
  if (F > 512) return cudaErrorInvalidValue;
  if (F <= 64) return complete_impl<2>(s, nbatch, F, k, U, work, scr);
  if (F <= 128) return complete_impl<4>(s, nbatch, F, k, U, work, scr);
  if (F <= 256) return complete_impl<8>(s, nbatch, F, k, U, work, scr);
  return complete_impl<16>(s, nbatch, F, k, U, work, scr);
}

cudaError_t launch_fill_zero(cudaStream_t s, double* p, long count) {
  if (count <= 0) return cudaSuccess;
  k_fill_zero<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(p, count);
  return cudaGetLastError();
}

}  // namespace dmcg
