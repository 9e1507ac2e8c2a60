// K3 — small dense kernels of the temporal basis: fused orthogonal
// iterations with a blocked Householder QR (rank safe), round-robin Jacobi
// eigensolver, descending sort, canonical signs, orthogonal completion.
// One CTA per axis; matrices are F x k / k x k (F <= 512) and live in L2 /
// shared memory.  Same algorithms and formulas as the oracle restatement
// (oracle/dmc_oracle.c: householder_factor, orc_jacobi_eig, orc_basis);
// reductions run in parallel order and use FMA, so results agree with the
// oracle to rounding, not bit for bit (P3).
#include <mutex>
#include <string>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace dmcg {

namespace {

constexpr int kOiThreads = 256;  // fused OI kernels: register-resident QR panels

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

// Parallel (round-robin) cyclic Jacobi.  Every step applies m2/2 disjoint
// rotations at once; each 2x2 block of A is transformed independently.  A
// lives in shared memory with an odd leading dimension (m2 + 1: the 2x2
// block gathers of a warp hit distinct banks).  The eigenvector rows are
// split over gridDim.y CTAs per matrix: each CTA repeats the (cheap,
// deterministic) A updates and rotates only its slice of V rows, so no
// inter-CTA traffic is needed.  a_smem = 0 keeps A and V in `work`
// (gridDim.y must then be 1).
constexpr int kJacThreads = 1024;
// Relative rotation threshold |a_pq| > rel sqrt(|a_pp a_qq|) (the oracle's
// orc_jacobi_eig uses 1e-17; DMCG_JAC_REL overrides it for experiments).
__constant__ double c_jac_rel = 1e-17, c_jac_rel2 = 1e-34;
__device__ int g_jacobi_sweeps[8];  // sweeps of the last k_jacobi per matrix (DMCG_DEBUG)
__device__ long long g_jacobi_cyc[64];  // cycles per sweep of matrix 0 (DMCG_DEBUG)

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
  // Fast path: the tasks of a thread are the same every round, so their
  // (pair, pair) / (pair, row) indices are computed once here (upper
  // triangle of the h x h block grid incl. its diagonal; h x nr V rows).
  constexpr int kTA = 4, kTV = 8;
  const int ntri = h * (h + 1) / 2, nvt = h * nr;
  const bool fast = ntri <= kTA * NT && nvt <= kTV * NT;
  int ta[kTA], tb[kTA], va[kTV], vr[kTV];
#pragma unroll
  for (int k = 0; k < kTA; ++k) {
    const int t = tid + k * NT;
    int a = 0, off = 0;
    if (t < ntri)
      while (off + (h - a) <= t) {
        off += h - a;
        ++a;
      }
    ta[k] = t < ntri ? a : -1;
    tb[k] = t < ntri ? a + (t - off) : 0;
  }
#pragma unroll
  for (int k = 0; k < kTV; ++k) {
    const int t = tid + k * NT;
    va[k] = (nr > 0 && t < nvt) ? t / nr : -1;
    vr[k] = (nr > 0 && t < nvt) ? t % nr : 0;
  }
  bool converged = (m2 <= 1);
  for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
    const long long sw_t0 = clock64();
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
        // |apq| > max(rel sqrt(|app aqq|), abs_thresh), compared in squares
        const double rel2 = c_jac_rel2 * fabs(app) * fabs(aqq);
        const double apq2 = apq * apq;
        double c = 1.0, sv = 0.0, tt = 0.0;
        if (apq2 > rel2 && fabs(apq) > abs_thresh) {
          // reciprocal forms of the oracle's divisions (last-ulp differences)
          const double theta = (aqq - app) * (0.5 * __drcp_rn(apq));
          const double at = fabs(theta);
          if (at > 1e150)
            tt = 0.5 * __drcp_rn(theta);
          else
            tt = (theta >= 0.0 ? 1.0 : -1.0) * __drcp_rn(at + sqrt(fma(theta, theta, 1.0)));
          c = rsqrt(fma(tt, tt, 1.0));
          sv = tt * c;
          on = 1;
        }
        cs[i] = c;
        sn[i] = sv;
        tn[i] = tt;
      }
      if (!__syncthreads_or(on)) continue;  // nothing to rotate at this step
      any = 1;
      if (fast) {
#pragma unroll
        for (int k = 0; k < kTA; ++k) {
          const int a = ta[k], bb = tb[k];
          if (a < 0) continue;
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
#pragma unroll
        for (int k = 0; k < kTV; ++k) {
          const int a = va[k], r = vr[k];
          if (a < 0) continue;
          const double sa = sn[a];
          if (sa == 0.0) continue;
          const double ca = cs[a];
          double* vp = V + P[a] * ldv;
          double* vq = V + Qi[a] * ldv;
          const double x = vp[r], y = vq[r];
          vp[r] = ca * x - sa * y;
          vq[r] = sa * x + ca * y;
        }
        __syncthreads();
        continue;
      }
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
    if (!converged) {
      // A sweep that rotated is followed by a rotation-free one only if no
      // pair is above its threshold now (A does not change during a sweep
      // without rotations, and a sweep visits every pair): test that
      // directly instead of running the empty sweep.
      int hot = 0;
      for (int t = tid; t < m2 * m2; t += NT) {
        const int p = t % m2, q = t / m2;
        if (p >= q) continue;
        const double app = A[p * ld + p], aqq = A[q * ld + q], apq = A[q * ld + p];
        const double rel = c_jac_rel * sqrt(fabs(app) * fabs(aqq));
        if (fabs(apq) > (rel > abs_thresh ? rel : abs_thresh)) hot = 1;
      }
      converged = !__syncthreads_or(hot);
    }
    if (threadIdx.x == 0 && sp == 0 && b < 8) g_jacobi_sweeps[b] = sweep + 1;
    if (threadIdx.x == 0 && sp == 0 && b == 0 && sweep < 64) g_jacobi_cyc[sweep] = clock64() - sw_t0;
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
    // NaN (a non-finite input flagged by K1) ranks last, so idx stays a
    // permutation and the gathers below stay in bounds
    const bool ni = isnan(wi);
    for (int j = 0; j < m; ++j) {
      const double wj = sw[j];
      const bool nj = isnan(wj);
      rank += (wj > wi) || (ni && !nj) || ((wj == wi || (ni && nj)) && j < i);
    }
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
  if (bi >= m) bi = 0;  // an all-NaN column (non-finite input, flagged by K1)
  const bool flip = u[bi] < 0.0;
  if (flip)
    for (int i = lane; i < m; i += 32) u[i] = -u[i];
}


// ---------------------------------------------------------------------------
// Fused orthogonal iterations: one CTA per axis runs every round
//   Z = R Q  (DMMA, R from L2, Q in smem);  Q = thin Householder Q of Z
// and the Rayleigh-Ritz matrix H = Q^T R Q, with Z and Q in shared memory
// when 2 F k doubles fit (else in a global work area, L1/L2 resident).
// ---------------------------------------------------------------------------
struct QrShared {
  double tau[512];
};

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
    for (int k0 = 0; k0 < K; k0 += 16) {
      // the loads of four k-steps issue before their DMMAs (A may stream from L2)
      double av[4], bv[4][8];
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const int ka = k0 + 4 * s4 + (lane & 3);
        av[s4] = (ia < M && ka < K) ? A[ia * lda + ka] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int jb = j00 + u * 8 + (lane >> 2);
          bv[s4][u] = (jb < N && ka < K) ? B[jb * ldb + ka] : 0.0;
        }
      }
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
        for (int u = 0; u < 8; ++u) dmma884(acc[u], av[s4], bv[s4][u]);
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


// ---------------------------------------------------------------------------
// Blocked (compact-WY) Householder QR with register-resident panels.
// A panel of PW columns (rows >= its first column) is factored by warp 0
// entirely in registers — a lane owns rows lane + 32 t — so a column step is
// a handful of interleaved warp reductions with no CTA barrier.  The warp
// also forms the panel's dlarft triangle T.  The trailing columns and the
// thin Q are then updated by all warps with DMMA (mma.sync.m8n8k4.f64):
//   W = V^T Y,  W = T^T W (factor) / T W (formation),  Y -= V W.
// Scratch (shared memory when it fits): W (PW x wcols), T of every panel.
// Reflector formulas are the oracle's householder_factor (tau, beta,
// v = x / (x0 - beta)); the GPU multiplies by the reciprocal, a 1-ulp
// difference inside the P3 tolerance.
// ---------------------------------------------------------------------------
__device__ long long g_pan_prof[8];
__device__ long long g_pan_last;
#ifndef PANEL_STAMP
#define PANEL_STAMP(i)                                            \
  do {                                                            \
    if (lane == 0 && blockIdx.x == 32) {                          \
      const long long _t = clock64();                             \
      if ((i) > 0) g_pan_prof[(i)] += _t - g_pan_last;            \
      g_pan_last = _t;                                            \
    }                                                             \
  } while (0)
#endif
#ifndef FACT_STAMP
#define FACT_STAMP(i)
#endif

template <int MAXR>
struct QrPanel {
  static constexpr int PW = MAXR <= 8 ? 8 : 4;  // a[MAXR][PW] stays in registers
};

// V(g, i) of the panel whose first column is c0 (g relative to row c0):
// zero above the unit diagonal, the stored reflector below.
template <typename P>
struct PanelV {
  P Z;
  int ld, c0;  // leading dimension of Z, first column of the panel
  __device__ __forceinline__ double operator()(int g, int i) const {
    return g < i ? 0.0 : (g == i ? 1.0 : Z[(c0 + i) * ld + c0 + g]);
  }
};

// Leading dimension of F-row matrices in shared memory: odd, so the 8 rows
// x 4 columns of a DMMA fragment fall on distinct banks.
__host__ __device__ __forceinline__ int odd_ld(int F) { return F | 1; }

template <int MAXR, int PW, typename P>
__device__ __noinline__ void warp_panel_qr(P Z, int m, int ld, int c0, int pb, double* tau,
                                           int lane) {
  const unsigned FULL = 0xffffffffu;
  const int M = m - c0;
  P base = Z + c0 * ld + c0;
  PANEL_STAMP(0);
  double a[MAXR][PW];
#pragma unroll
  for (int t = 0; t < MAXR; ++t)
#pragma unroll
    for (int c = 0; c < PW; ++c) {
      const int g = lane + 32 * t;
      a[t][c] = (c < pb && g < M) ? base[c * ld + g] : 0.0;
    }
  PANEL_STAMP(1);
  double tv[PW];
#pragma unroll
  for (int j = 0; j < PW; ++j) {
    // Columns j >= pb are zero: their reflector is the identity (tail 0,
    // tau 0), so no branch on pb is needed around the shuffles below.
    // One reduction round per column: the norm of the tail of column j and
    // the raw products x^T y_l with the later columns are summed together;
    // v = x / (x0 - beta) only rescales them (d_l = tau (y_l[j] + rinv x^T y_l)).
    double r[PW + 1];
#pragma unroll
    for (int l = 0; l <= PW; ++l) r[l] = 0.0;
#pragma unroll
    for (int t = 0; t < MAXR; ++t) {
      const int g = lane + 32 * t;
      const double x = g > j ? a[t][j] : 0.0;
      r[PW] = fma(x, x, r[PW]);
#pragma unroll
      for (int l = 0; l < PW; ++l)
        if (l > j) r[l] = fma(x, a[t][l], r[l]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r[PW] += __shfl_xor_sync(FULL, r[PW], o);
#pragma unroll
      for (int l = 0; l < PW; ++l)
        if (l > j) r[l] += __shfl_xor_sync(FULL, r[l], o);
    }
    const double tail = r[PW];
    const double x0 = __shfl_sync(FULL, a[0][j], j);
    double yj[PW];
#pragma unroll
    for (int l = 0; l < PW; ++l) yj[l] = l > j ? __shfl_sync(FULL, a[0][l], j) : 0.0;
    double rinv = 0.0, tj = 0.0, beta = x0;
    if (tail > DBL_MIN) {
      const double s2 = x0 * x0 + tail;
      const double rs = rsqrt(s2);
      const double nrm = s2 * rs;
      beta = x0 >= 0.0 ? -nrm : nrm;
      const double ibb = x0 >= 0.0 ? -rs : rs;
      rinv = __drcp_rn(x0 - beta);
      tj = (beta - x0) * ibb;
    }
#pragma unroll
    for (int t = 0; t < MAXR; ++t) {
      const int g = lane + 32 * t;
      if (g > j) a[t][j] *= rinv;
    }
    if (lane == j) a[0][j] = beta;
    tv[j] = tj;
    // H_j applied to the panel columns l > j
#pragma unroll
    for (int l = 0; l < PW; ++l) {
      if (l <= j) continue;
      const double sl = tj * fma(rinv, r[l], yj[l]);
#pragma unroll
      for (int t = 0; t < MAXR; ++t) {
        const int g = lane + 32 * t;
        if (g > j) a[t][l] = fma(-sl, a[t][j], a[t][l]);
      }
      if (lane == j) a[0][l] -= sl;
    }
  }
  PANEL_STAMP(2);
  PANEL_STAMP(3);
  // write the factored panel back
#pragma unroll
  for (int t = 0; t < MAXR; ++t)
#pragma unroll
    for (int c = 0; c < PW; ++c) {
      const int g = lane + 32 * t;
      if (c < pb && g < M) base[c * ld + g] = a[t][c];
    }
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < PW; ++j)
      if (j < pb) tau[c0 + j] = tv[j];
  PANEL_STAMP(4);
}

// warp_panel_qr + dlarft in the same reduction rounds (panel = the whole
// block, B == PW): at column j the round that sums the tail norm and x^T y_l
// (l > j) also sums x^T v_l for the earlier reflectors l < j, which gives
// G(l, j) = v_l^T v_j = v_l(j) + rinv x^T v_l; lane l then extends row l of T:
//   T(l, j) = -tau_j sum_{m=l}^{j-1} T(l, m) G(m, j),  T(j, j) = tau_j.
// Z points at the block's diagonal row; T row-major PW x PW.
template <int MAXR, int PW, typename P>
__device__ __noinline__ void warp_panel_qr_T(P Z, int m, int ld, int pb, double* tau, double* T,
                                             int lane) {
  const unsigned FULL = 0xffffffffu;
  const int M = m;
  double a[MAXR][PW];
#pragma unroll
  for (int t = 0; t < MAXR; ++t)
#pragma unroll
    for (int c = 0; c < PW; ++c) {
      const int g = lane + 32 * t;
      a[t][c] = (c < pb && g < M) ? Z[c * ld + g] : 0.0;
    }
  double tv[PW], tr[PW];
#pragma unroll
  for (int i = 0; i < PW; ++i) tr[i] = 0.0;
#pragma unroll
  for (int j = 0; j < PW; ++j) {
    double r[PW + 1];
#pragma unroll
    for (int l = 0; l <= PW; ++l) r[l] = 0.0;
#pragma unroll
    for (int t = 0; t < MAXR; ++t) {
      const int g = lane + 32 * t;
      const double x = g > j ? a[t][j] : 0.0;
      r[PW] = fma(x, x, r[PW]);
#pragma unroll
      for (int l = 0; l < PW; ++l)
        if (l != j) r[l] = fma(x, a[t][l], r[l]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r[PW] += __shfl_xor_sync(FULL, r[PW], o);
#pragma unroll
      for (int l = 0; l < PW; ++l)
        if (l != j) r[l] += __shfl_xor_sync(FULL, r[l], o);
    }
    const double tail = r[PW];
    const double x0 = __shfl_sync(FULL, a[0][j], j);
    double yj[PW];
#pragma unroll
    for (int l = 0; l < PW; ++l) yj[l] = l != j ? __shfl_sync(FULL, a[0][l], j) : 0.0;
    double rinv = 0.0, tj = 0.0, beta = x0;
    if (tail > DBL_MIN) {
      const double s2 = x0 * x0 + tail;
      const double rs = rsqrt(s2);
      const double nrm = s2 * rs;
      beta = x0 >= 0.0 ? -nrm : nrm;
      const double ibb = x0 >= 0.0 ? -rs : rs;
      rinv = __drcp_rn(x0 - beta);
      tj = (beta - x0) * ibb;
    }
    // G(l, j) for l < j (yj[l] = v_l(j), the stored reflector entry in row j)
    double gcol[PW];
#pragma unroll
    for (int l = 0; l < PW; ++l) gcol[l] = l < j ? fma(rinv, r[l], yj[l]) : 0.0;
    {
      double acc = 0.0;
#pragma unroll
      for (int mm = 0; mm < PW; ++mm)
        if (mm < j && mm >= lane) acc = fma(tr[mm], gcol[mm], acc);
      const double tl = lane < j ? -tj * acc : (lane == j ? tj : 0.0);
#pragma unroll
      for (int i = 0; i < PW; ++i)
        if (i == j) tr[i] = j < pb ? tl : 0.0;
    }
#pragma unroll
    for (int t = 0; t < MAXR; ++t) {
      const int g = lane + 32 * t;
      if (g > j) a[t][j] *= rinv;
    }
    if (lane == j) a[0][j] = beta;
    tv[j] = tj;
#pragma unroll
    for (int l = 0; l < PW; ++l) {
      if (l <= j) continue;
      const double sl = tj * fma(rinv, r[l], yj[l]);
#pragma unroll
      for (int t = 0; t < MAXR; ++t) {
        const int g = lane + 32 * t;
        if (g > j) a[t][l] = fma(-sl, a[t][j], a[t][l]);
      }
      if (lane == j) a[0][l] -= sl;
    }
  }
#pragma unroll
  for (int t = 0; t < MAXR; ++t)
#pragma unroll
    for (int c = 0; c < PW; ++c) {
      const int g = lane + 32 * t;
      if (c < pb && g < M) Z[c * ld + g] = a[t][c];
    }
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < PW; ++j)
      if (j < pb) tau[j] = tv[j];
  if (lane < PW)
#pragma unroll
    for (int i = 0; i < PW; ++i) T[lane * PW + i] = lane < pb ? tr[i] : 0.0;
}

// dlarft: T (PW x PW row-major, upper) from G(l, i) = v_l^T v_i (row-major,
// ld ldg) and tau; lane j of warp 0 forms row j:
//   T(j, j) = tau_j,  T(j, i) = -tau_i sum_{l=j}^{i-1} T(j, l) G(l, i).
template <int PW>
__device__ void panel_T(const double* G, int ldg, const double* tau, int pb, double* T,
                        int lane) {
  if (lane >= PW) return;
  const int j = lane;
  double tr[PW];
#pragma unroll
  for (int i = 0; i < PW; ++i) {
    double v = 0.0;
    if (i < pb && i == j) v = tau[i];
    if (i < pb && i > j) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < PW; ++l)
        if (l < i && l >= j) acc = fma(tr[l], G[l * ldg + i], acc);
      v = -tau[i] * acc;
    }
    tr[i] = j < pb ? v : 0.0;
  }
#pragma unroll
  for (int i = 0; i < PW; ++i) T[j * PW + i] = tr[i];
}

// Branch-free operand fetch: element g of column `col` (pointer to its row
// c0) masked to V's shape — zero above the unit diagonal at `diag` (diag < 0:
// a plain column) and zero past the M rows / outside the tile.
__device__ __forceinline__ double vfetch(const double* col, int g, int M, int diag, bool valid) {
  const double x = col[g < M ? g : M - 1];
  const double v = diag < 0 ? x : (g > diag ? x : (g == diag ? 1.0 : 0.0));
  return (valid && g < M) ? v : 0.0;
}

// W (PW x nc, row-major) = V^T [V_nv | Y] over the rows g < M of the panel:
// the first nv right-hand columns are V's own (G = V^T V), the rest Y.  One
// warp per 8-column tile; K = M in steps of 16 with the next step's
// operands loaded before the current step's DMMAs (four accumulators).
template <int PW, typename PZ, typename PY>
__device__ void wy_vty(const PanelV<PZ>& V, int M, int pb, int nv, PY Y, int ldy, int nc,
                       double* W) {
  // one 8-column tile of W per warp group, the M rows split over the warps
  // left (ks groups), partial tiles summed in split order (deterministic)
  __shared__ double vty_part[kOiThreads / 32][64];  // callers run kOiThreads threads
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int i = lane >> 2, q = lane & 3;
  const int ic = i < pb ? i : pb - 1;
  const double* acol = V.Z + (V.c0 + ic) * V.ld + V.c0;
  const bool avalid = i < pb;
  const int nct = (nc + 7) / 8;
  const int ks = nct >= nw ? 1 : nw / nct;
  const int nch = (M + 15) / 16;
  for (int wt = warp; wt < nct * ks; wt += nw) {
    const int ct = wt % nct, kc = wt / nct;
    const int ch0 = (int)((long)nch * kc / ks), ch1 = (int)((long)nch * (kc + 1) / ks);
    const int c = ct * 8 + i;
    const bool bvalid = c < nc;
    const int cc = bvalid ? c : nc - 1;
    const double* bcol = cc < nv ? V.Z + (V.c0 + cc) * V.ld + V.c0 : Y + (cc - nv) * ldy;
    const int bdiag = cc < nv ? cc : -1;
    double acc[4][2] = {};
    if (ch0 < ch1) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = vfetch(acol, 16 * ch0 + 4 * u + q, M, ic, avalid);
        bv[u] = vfetch(bcol, 16 * ch0 + 4 * u + q, M, bdiag, bvalid);
      }
      for (int ch = ch0 + 1; ch <= ch1; ++ch) {
        const int k0 = 16 * ch;
        double an[4], bn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          an[u] = vfetch(acol, k0 + 4 * u + q, M, ic, avalid);
          bn[u] = vfetch(bcol, k0 + 4 * u + q, M, bdiag, bvalid);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma884(acc[u], av[u], bv[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          av[u] = an[u];
          bv[u] = bn[u];
        }
      }
    }
    if (ks == 1) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int co = ct * 8 + q * 2 + e;
        if (i < PW && co < nc) W[i * nc + co] = (acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 2; ++e)
        vty_part[wt][i * 8 + q * 2 + e] = (acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e]);
    }
  }
  if (ks > 1) {
    __syncthreads();
    for (int t = threadIdx.x; t < PW * nc; t += blockDim.x) {
      const int r = t / nc, co = t % nc, ct = co / 8;
      double sum = 0.0;
      for (int kc = 0; kc < ks; ++kc) sum += vty_part[ct + kc * nct][r * 8 + co % 8];
      W[r * nc + co] = sum;
    }
  }
}

template <int PW>
__device__ void wy_tw(const double* T, int pb, double* W, int ldw, int nc, bool trans) {
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    double w[PW], o[PW];
#pragma unroll
    for (int i = 0; i < PW; ++i) w[i] = i < pb ? W[i * ldw + c] : 0.0;
#pragma unroll
    for (int i = 0; i < PW; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < PW; ++l) {
        if (trans ? (l <= i) : (l >= i)) acc = fma(trans ? T[l * PW + i] : T[i * PW + l], w[l], acc);
      }
      o[i] = acc;
    }
#pragma unroll
    for (int i = 0; i < PW; ++i)
      if (i < pb) W[i * ldw + c] = o[i];
  }
}

// Y (rows g < M, nc columns) -= V W; one warp per 8-row tile with the V
// fragment in registers, the column tiles in groups of four whose W and Y
// fragments are all loaded before their DMMAs.
template <int PW, typename PZ, typename PY>
__device__ void wy_update(const PanelV<PZ>& V, int M, int pb, PY Y, int ldy, int nc,
                          const double* W, int ldw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int nct = (nc + 7) / 8;
  for (int mt = warp; mt * 8 < M; mt += nw) {
    const int g = mt * 8 + r;
    double av[PW / 4];
#pragma unroll
    for (int u = 0; u < PW / 4; ++u) {
      const int i = 4 * u + q;
      const int icl = i < pb ? i : pb - 1;
      av[u] = vfetch(V.Z + (V.c0 + icl) * V.ld + V.c0, g, M, icl, i < pb);
    }
    const int gc = g < M ? g : M - 1;
    for (int ct0 = 0; ct0 < nct; ct0 += 4) {
      double bw[4][PW / 4], yv[4][2], acc[4][2];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
#pragma unroll
        for (int u = 0; u < PW / 4; ++u) {
          const int i = 4 * u + q, c = (ct0 + t) * 8 + r;
          const bool ok = i < pb && c < nc;
          bw[t][u] = ok ? W[(i < pb ? i : 0) * ldw + (c < nc ? c : 0)] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = (ct0 + t) * 8 + 2 * q + e;
          yv[t][e] = Y[(c < nc ? c : nc - 1) * ldy + gc];
          acc[t][e] = 0.0;
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < PW / 4; ++u) dmma884(acc[t], av[u], bw[t][u]);
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = (ct0 + t) * 8 + 2 * q + e;
          if (g < M && c < nc) Y[c * ldy + g] = yv[t][e] - acc[t][e];
        }
    }
  }
}

// Householder factor of the p columns of Z (m x p, in place): R on and
// above the diagonal, V below, tau[j]; T of panel b at Ts + b PW^2.
template <int MAXR, typename P>
__device__ void wqr_factor(P Z, int m, int ld, int p, double* tau, double* scr, int wcols) {
  constexpr int PW = QrPanel<MAXR>::PW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pe = p < m ? p : m;
  double* W = scr;                   // PW x (pb + rem): [G | V^T Y]
  double* Ts = scr + PW * (wcols + PW);
  for (int c0 = 0; c0 < pe; c0 += PW) {
    const int pb = min(PW, pe - c0);
    double* T = Ts + (c0 / PW) * PW * PW;
    FACT_STAMP(0);
    if (warp == 0) warp_panel_qr<MAXR, PW>(Z, m, ld, c0, pb, tau, lane);
    __syncthreads();
    FACT_STAMP(1);
    const int rem = p - (c0 + pb), ncw = pb + max(rem, 0);
    const PanelV<P> V{Z, ld, c0};
    P Y = Z + (c0 + pb) * ld + c0;
    wy_vty<PW>(V, m - c0, pb, pb, Y, ld, ncw, W);   // one pass: G = V^T V and V^T Y
    __syncthreads();
    FACT_STAMP(2);
    if (warp == 0) panel_T<PW>(W, ncw, tau + c0, pb, T, lane);
    __syncthreads();
    FACT_STAMP(3);
    if (rem <= 0) continue;
    wy_tw<PW>(T, pb, W + pb, ncw, rem, true);
    __syncthreads();
    FACT_STAMP(4);
    wy_update<PW>(V, m - c0, pb, Y, ld, rem, W + pb, ncw);
    __syncthreads();
    FACT_STAMP(5);
  }
}

// Qout (m x ncols, leading dimension ldq) = H_0 ... H_{pe-1} [e_cid ...]
// from the factor of wqr_factor (same scratch).
template <int MAXR, typename PZ, typename PQ>
__device__ void wqr_form(PZ Z, int m, int ldz, int p, int cid, int ncols, PQ Qo, int ldq,
                         double* scr, int wcols) {
  constexpr int PW = QrPanel<MAXR>::PW;
  const int pe = p < m ? p : m;
  double* W = scr;
  const double* Ts = scr + PW * (wcols + PW);
  for (int t = threadIdx.x; t < m * ncols; t += blockDim.x) {
    const int c = t / m, r = t % m;
    Qo[c * ldq + r] = (r == cid + c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int npan = (pe + PW - 1) / PW;
  for (int pi = npan - 1; pi >= 0; --pi) {
    const int c0 = pi * PW, pb = min(PW, pe - c0);
    // thin Q: columns c < c0 are still e_c, zero on the rows this panel touches
    const int cs = (cid == 0) ? (c0 < ncols ? c0 : ncols) : 0;
    const int nc = ncols - cs;
    if (nc <= 0) continue;
    const PanelV<PZ> V{Z, ldz, c0};
    PQ Y = Qo + cs * ldq + c0;
    wy_vty<PW>(V, m - c0, pb, 0, Y, ldq, nc, W);
    __syncthreads();
    wy_tw<PW>(Ts + pi * PW * PW, pb, W, nc, nc, false);
    __syncthreads();
    wy_update<PW>(V, m - c0, pb, Y, ldq, nc, W, nc);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Z = R Q spread over a thread-block cluster of `cs` CTAs per axis.  The QR
// is sequential and stays on the cluster's rank-0 CTA; the product (63 % of
// an OI round's flops) is split by row blocks over the cluster.  Q goes out
// through L2 (qbuf, written by rank 0), the Z blocks come back through
// distributed shared memory; two cluster barriers per round (release /
// acquire at cluster scope).
// ---------------------------------------------------------------------------
__device__ long long g_oi_prof[256];  // per-CTA cycle split of the last k_oi_fused (DMCG_DEBUG)

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Rows [8 mt0, 8 mt1) of Z = R Q: 8-row x 16-column DMMA tasks over the
// warps of this CTA; A = rows 8 mt0.. of R (shared memory when staged, else
// L2; loaded two 16-deep k-batches ahead of the DMMAs), B = Q.
template <typename PQ, typename PZ>
__device__ void rq_tasks(const double* R, int ldr, int F, int k, PQ Qb, int ldq, PZ Zo, int ldz,
                         int mt0, int mt1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nt = (k + 15) / 16, ntask = (mt1 - mt0) * nt;
  const int r = lane >> 2, q = lane & 3;
  for (int t = warp; t < ntask; t += nw) {
    const int m0 = (mt0 + t % (mt1 - mt0)) * 8, n0 = (t / (mt1 - mt0)) * 16;
    const int g = m0 + r, gc = g < F ? g : F - 1;
    const int c0 = n0 + r, c1 = n0 + 8 + r;
    const int cc0 = c0 < k ? c0 : k - 1, cc1 = c1 < k ? c1 : k - 1;
    // row g of R (= column g, R symmetric); R holds rows from 8 mt0 on
    const double* Ar = R + (size_t)(gc - 8 * mt0) * ldr;
    double acc[2][2][2] = {};
    double a0[4], a1[4];
    auto fetch_a = [&](int k0, double* a) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = k0 + 4 * u + q;
        a[u] = kk < F ? Ar[kk] : 0.0;
      }
    };
    fetch_a(0, a0);
    fetch_a(16, a1);
    for (int k0 = 0; k0 < F; k0 += 16) {
      double an[4];
      fetch_a(k0 + 32, an);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = k0 + 4 * u + q, kc = kk < F ? kk : F - 1;
        const double y0 = kk < F ? Qb[cc0 * ldq + kc] : 0.0;
        const double y1 = kk < F ? Qb[cc1 * ldq + kc] : 0.0;
        dmma884(acc[u & 1][0], a0[u], y0);
        dmma884(acc[u & 1][1], a0[u], y1);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0[u] = a1[u];
        a1[u] = an[u];
      }
    }
    if (g < F)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = n0 + 8 * h + 2 * q + e;
          if (c < k) Zo[c * ldz + g] = acc[0][h][e] + acc[1][h][e];
        }
  }
}

// Row block of the Z = R Q tasks owned by cluster rank `rank`: ranks 1..cs-1
// split the 8-row tiles (rank 0 runs the QR); cs == 1: everything.
__device__ __forceinline__ void rq_rows(int F, int rank, int cs, int* mt0, int* mt1) {
  const int mt = (F + 7) / 8;
  if (cs == 1) {
    *mt0 = 0;
    *mt1 = mt;
    return;
  }
  *mt0 = (int)((long)mt * (rank - 1) / (cs - 1));
  *mt1 = (int)((long)mt * rank / (cs - 1));
}

// All CTAs of the cluster call this (same arguments except rank).  Rank 0
// publishes Q to L2 (qbuf); ranks > 0 copy it into their own shared memory
// and compute their rows of Z from their resident rows of R (Rs, staged once
// per kernel, leading dimension ldr), storing them straight into rank 0's Z
// (distributed shared memory, or the global work area when Z does not fit
// on chip).
template <bool SMEM, int MAXR, typename P>
__device__ void oi_apply_cluster(const double* R, int ldr, int F, int k, P Q, int ld, P Z,
                                 double* qbuf, int rank, int cs) {
  int mt0, mt1;
  rq_rows(F, rank, cs, &mt0, &mt1);
  if (cs == 1) {
    rq_tasks(R, ldr, F, k, Q, ld, Z, ld, mt0, mt1);
    __syncthreads();
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (rank == 0) {
    for (int c = warp; c < k; c += nw) {
      double v[MAXR];
#pragma unroll
      for (int u = 0; u < MAXR; ++u) {
        const int r = lane + 32 * u;
        v[u] = r < F ? Q[c * ld + r] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < MAXR; ++u) {
        const int r = lane + 32 * u;
        if (r < F) qbuf[c * F + r] = v[u];
      }
    }
    __threadfence();
  }
  cluster_sync_all();
  if (rank != 0) {
    const double* Qsrc = qbuf;
    int ldqs = F;
    if (SMEM) {
      // this CTA's copy of Q (its own Q area is free): four columns in flight per warp
      for (int c0 = warp * 4; c0 < k; c0 += nw * 4) {
        double v[4][MAXR];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int u = 0; u < MAXR; ++u) {
            const int r = lane + 32 * u, c = c0 + j;
            v[j][u] = (r < F && c < k) ? __ldcg(qbuf + c * F + r) : 0.0;
          }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int u = 0; u < MAXR; ++u) {
            const int r = lane + 32 * u, c = c0 + j;
            if (r < F && c < k) Q[c * ld + r] = v[j][u];
          }
      }
      __syncthreads();
      Qsrc = Q;
      ldqs = ld;
    }
    // (global path: Z, Q in the work area; read Q from L2, the barrier invalidated L1)
    P Zdst = SMEM ? cg::this_cluster().map_shared_rank(Z, 0) : Z;
    if (mt1 > mt0) rq_tasks(R, ldr, F, k, Qsrc, ldqs, Zdst, ld, mt0, mt1);
  }
  cluster_sync_all();
}

template <bool SMEM, int MAXR, typename P>
__device__ void oi_body(int F, int k, int rounds, const double* __restrict__ R,
                        const double* __restrict__ start, P Z, P Q, double* Qo, double* H,
                        QrShared& q, double* scr, double* qbuf, int rank, int cs) {
  const int ld = odd_ld(F);  // Z and Q: F x k, leading dimension ld
  const bool lead = rank == 0;
  if (lead) {
    for (int t = threadIdx.x; t < F * k; t += blockDim.x) Z[(t / F) * ld + t % F] = start[t];
    __syncthreads();
    wqr_factor<MAXR>(Z, F, ld, k, q.tau, scr, k);
    wqr_form<MAXR>(Z, F, ld, k, 0, k, Q, ld, scr, k);
  }
  // ranks > 0 keep their rows of R resident (their Z area is free)
  const double* Rr = R;
  int ldr = F;
  if (SMEM && !lead) {
    int mt0, mt1;
    rq_rows(F, rank, cs, &mt0, &mt1);
    const int r0 = 8 * mt0, nr = min(F, 8 * mt1) - r0;
    if (nr > 0 && (size_t)nr * ld <= (size_t)ld * k) {
      for (int t = threadIdx.x; t < nr * F; t += blockDim.x) Z[(t / F) * ld + t % F] = R[(size_t)r0 * F + t];
      __syncthreads();
      Rr = Z;
      ldr = ld;
    } else {
      Rr = R + (size_t)r0 * F;
    }
  } else if (!lead) {
    int mt0, mt1;
    rq_rows(F, rank, cs, &mt0, &mt1);
    Rr = R + (size_t)8 * mt0 * F;
  }
  long long t_rq = 0, t_f = 0, t_q = 0;
  for (int r = 0; r <= rounds; ++r) {
    const long long t0 = clock64();
    oi_apply_cluster<SMEM, MAXR>(Rr, ldr, F, k, Q, ld, Z, qbuf, rank, cs);
    const long long t1 = clock64();
    t_rq += t1 - t0;
    if (lead && r < rounds) {
      wqr_factor<MAXR>(Z, F, ld, k, q.tau, scr, k);
      const long long t2 = clock64();
      wqr_form<MAXR>(Z, F, ld, k, 0, k, Q, ld, scr, k);
      t_f += t2 - t1;
      t_q += clock64() - t2;
    }
  }
  if (threadIdx.x == 0 && blockIdx.x < 64) {
    g_oi_prof[blockIdx.x * 4 + 0] = t_rq;
    g_oi_prof[blockIdx.x * 4 + 1] = t_f;
    g_oi_prof[blockIdx.x * 4 + 2] = t_q;
  }
  if (!lead) return;
  // Rayleigh-Ritz: H = Q^T (R Q), symmetrised like the oracle; Q out.
  warp_gemm_tn(k, k, F, Q, ld, Z, ld, H, k);
  __syncthreads();
  for (int t = threadIdx.x; t < k * k; t += blockDim.x) {
    const int i = t % k, j = t / k;
    if (i >= j) continue;
    const double sv = 0.5 * (H[j * k + i] + H[i * k + j]);
    H[j * k + i] = sv;
    H[i * k + j] = sv;
  }
  for (int t = threadIdx.x; t < F * k; t += blockDim.x) Qo[t] = Q[(t / F) * ld + t % F];
}

template <bool SMEM, int MAXR>
__global__ void __launch_bounds__(kOiThreads)
    k_oi_fused(int F, int k, int rounds, const double* __restrict__ Rall,
               const double* __restrict__ start, double* Qall, double* Hall, double* work,
               double* scr_all, size_t scr_stride, int scr_smem, int cs) {
  extern __shared__ double dyn[];
  __shared__ QrShared q;
  const int b = blockIdx.x / cs, rank = blockIdx.x % cs;
  const size_t Fk = (size_t)F * k, Lk = (size_t)odd_ld(F) * k;
  const double* R = Rall + (size_t)b * F * F;
  double* scr = scr_smem ? dyn + (SMEM ? 2 * Lk : 0) : scr_all + b * scr_stride;
  // Qo doubles as the L2 staging buffer of Q during the rounds
  double* qbuf = Qall + b * Fk;
  if (SMEM) {
    oi_body<true, MAXR>(F, k, rounds, R, start + b * Fk, dyn, dyn + Lk, Qall + b * Fk,
                        Hall + (size_t)b * k * k, q, scr, qbuf, rank, cs);
  } else {
    oi_body<false, MAXR>(F, k, rounds, R, start + b * Fk, work + b * 2 * Lk,
                         work + b * 2 * Lk + Lk, Qall + b * Fk, Hall + (size_t)b * k * k, q, scr,
                         qbuf, rank, cs);
  }
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
  const int ld = odd_ld(F), Lk = ld * k;
  double* Z = SMEM ? dyn : work + (size_t)b * Lk;
  double* U = Uall + (size_t)b * F * F;
  double* scr = scr_smem ? dyn + (SMEM ? Lk : 0) : scr_all + b * scr_stride;
  const int wc = k > F - k ? k : F - k;
  for (int t = threadIdx.x; t < F * k; t += blockDim.x) Z[(t / F) * ld + t % F] = U[t];
  __syncthreads();
  wqr_factor<MAXR>(Z, F, ld, k, q.tau, scr, wc);
  wqr_form<MAXR>(Z, F, ld, k, k, F - k, U + (size_t)F * k, F, scr, wc);
}

__global__ void k_fill_zero(double* p, long count) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t < count) p[t] = 0.0;
}

// Householder factor of a whole PW-column block by all kOiThreads threads
// of the CTA (the rows split R per thread: g = tid + 256 t), with its dlarft
// triangle T formed in the same reductions as warp_panel_qr_T: at column j
// one block reduction sums the tail norm, x^T y_l for the later columns and
// x^T v_l for the earlier reflectors (G(l, j) = v_l(j) + rinv x^T v_l).  Two
// barriers per column instead of the blocked panel sequence (4-column
// register panels + V^T Y + T + T W + update per panel).  Same reflector
// formulas as warp_panel_qr_T / the oracle's householder_factor; the
// reductions sum in a different order (rounding-level differences, P3).
template <int R, int PW, int NT = kOiThreads>
__device__ void cta_panel_qr_T(double* Z, int m, int ld, int pb, double* tau, double* T) {
  __shared__ double red[kOiThreads / 32][PW + 1];
  __shared__ double tot[2 * PW + 1];  // [0, PW]: sums, [PW + 1, 2 PW]: row j of the block
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = NT >> 5;
  const bool act = tid < NT;  // threads >= NT only join the barriers
  double a[R][PW];
#pragma unroll
  for (int t = 0; t < R; ++t)
#pragma unroll
    for (int c = 0; c < PW; ++c) {
      const int g = tid + NT * t;
      a[t][c] = (act && c < pb && g < m) ? Z[c * ld + g] : 0.0;
    }
  double tv[PW], tr[PW];
#pragma unroll
  for (int i = 0; i < PW; ++i) tr[i] = tv[i] = 0.0;
#pragma unroll
  for (int j = 0; j < PW; ++j) {
    // 32 partial sums per thread (PW + 1 used), reduced over the warp by
    // recursive halving: each round every lane sends the half it gives up
    // and keeps the other, so lane L ends with the total of value L after
    // 16 + 8 + 4 + 2 + 1 exchanges (not 5 (PW + 1): SHFL / DADD throughput)
    static_assert(PW + 1 <= 32, "one value per lane");
    double r[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) r[l] = 0.0;
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int g = tid + NT * t;
      const double x = g > j ? a[t][j] : 0.0;
      r[PW] = fma(x, x, r[PW]);
#pragma unroll
      for (int l = 0; l < PW; ++l)
        if (l != j) r[l] = fma(x, a[t][l], r[l]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const bool hi = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < o; ++i) {
        const double send = hi ? r[i] : r[i + o];
        const double keep = hi ? r[i + o] : r[i];
        r[i] = keep + __shfl_xor_sync(FULL, send, o);
      }
    }
    if (act && lane <= PW) red[warp][lane] = r[0];
    if (tid == j)  // row j (j < PW <= 256: thread j, t = 0)
#pragma unroll
      for (int l = 0; l < PW; ++l) tot[PW + 1 + l] = a[0][l];
    __syncthreads();
    if (tid <= PW) {
      double sum = 0.0;
      for (int w = 0; w < nw; ++w) sum += red[w][tid];
      tot[tid] = sum;
    }
    __syncthreads();
    const double tail = tot[PW];
    const double x0 = tot[PW + 1 + j];
    double rinv = 0.0, tj = 0.0, beta = x0;
    if (tail > DBL_MIN) {
      const double s2 = x0 * x0 + tail;
      const double rs = rsqrt(s2);
      const double nrm = s2 * rs;
      beta = x0 >= 0.0 ? -nrm : nrm;
      const double ibb = x0 >= 0.0 ? -rs : rs;
      rinv = __drcp_rn(x0 - beta);
      tj = (beta - x0) * ibb;
    }
    if (tid < PW) {  // thread l extends row l of T
      double acc = 0.0;
#pragma unroll
      for (int mm = 0; mm < PW; ++mm)
        if (mm < j && mm >= tid) acc = fma(tr[mm], fma(rinv, tot[mm], tot[PW + 1 + mm]), acc);
      const double tl = tid < j ? -tj * acc : (tid == j ? tj : 0.0);
      tr[j] = j < pb ? tl : 0.0;
    }
    double sl[PW];
#pragma unroll
    for (int l = 0; l < PW; ++l) sl[l] = l > j ? tj * fma(rinv, tot[l], tot[PW + 1 + l]) : 0.0;
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int g = tid + NT * t;
      if (act && g > j) a[t][j] *= rinv;
    }
    if (tid == j) a[0][j] = beta;
    tv[j] = tj;
#pragma unroll
    for (int l = 0; l < PW; ++l) {
      if (l <= j) continue;
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int g = tid + NT * t;
        if (act && g > j) a[t][l] = fma(-sl[l], a[t][j], a[t][l]);
      }
      if (tid == j) a[0][l] -= sl[l];
    }
  }
#pragma unroll
  for (int t = 0; t < R; ++t)
#pragma unroll
    for (int c = 0; c < PW; ++c) {
      const int g = tid + NT * t;
      if (act && c < pb && g < m) Z[c * ld + g] = a[t][c];
    }
  if (tid == 0)
#pragma unroll
    for (int j = 0; j < PW; ++j)
      if (j < pb) tau[j] = tv[j];
  if (tid < PW)
#pragma unroll
    for (int i = 0; i < PW; ++i) T[tid * PW + i] = tid < pb ? tr[i] : 0.0;
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Column-distributed orthogonal iterations (k_oi_cluster): the cluster's cs
// CTAs of one axis each own a block of B columns of Z and Q (F x B in
// shared memory), so both the QR and Z = R Q spread over the cluster:
//   * Z_c = R Q_c needs only the CTA's own Q block (R streams from L2);
//   * the Householder QR is a wavefront over the blocks: CTA c applies the
//     block reflectors H_p (p < c) of the earlier CTAs to its block as soon
//     as each is published (V_p read over distributed shared memory), then
//     factors its own block, forms T_c (dlarft) and publishes it with a
//     release flag — no cluster-wide barrier per panel;
//   * the thin Q block Q_c = H_0 ... H_c E_c needs only the published
//     reflectors, so every CTA forms its block independently;
//   * one cluster barrier per round (all remote reads of V done before the
//     next R Q overwrites Z).
// Same reflector formulas as the single-CTA path (warp_panel_qr /
// wqr_factor), so the result agrees with the oracle's householder_factor to
// rounding (P3).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire_cluster(const int* p) {
  int v;
  asm volatile("ld.acquire.cluster.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cluster(int* p, int v) {
  asm volatile("st.release.cluster.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Masked element of a unit-lower-trapezoidal block V (M x nb, column i at
// Vb + i ldv, row 0 = the block's diagonal row).
__device__ __forceinline__ double vmask(const double* Vb, int ldv, int g, int i, int M, int nb) {
  const int gc = g < M ? g : M - 1, ic = i < nb ? i : nb - 1;
  const double x = Vb[ic * ldv + gc];
  const double v = g > i ? x : (g == i ? 1.0 : 0.0);
  return (g < M && i < nb) ? v : 0.0;
}

// W (nb x nc, row-major ld B) = V^T Y over M rows (Y: column j at Yb + j ldy;
// y_is_v: Y is V itself, masked the same way -> G = V^T V).  8 x 8 DMMA
// tiles; K split over the warps left after one warp per tile, partial tiles
// summed in `part` (nw x 64 doubles).
template <int B>
__device__ void blk_vty(const double* Vb, int ldv, int nb, const double* Yb, int ldy, int nc,
                        bool y_is_v, int M, double* W, double* part, const double* T = nullptr,
                        bool trans = false) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  constexpr int TR = B / 8;
  const int tc = (nc + 7) / 8, ntile = TR * tc;
  const int nk = nw / ntile > 0 ? nw / ntile : 1;
  const int i = lane >> 2, q = lane & 3;
  if (warp < ntile * nk) {
    const int tile = warp % ntile, kc = warp / ntile;
    const int ti = tile % TR, tj = tile / TR;
    const int ksteps = (M + 3) / 4;
    const int k0 = (int)((long)ksteps * kc / nk) * 4, k1 = (int)((long)ksteps * (kc + 1) / nk) * 4;
    double acc[2][2] = {};
    const int ia = ti * 8 + i, jb = tj * 8 + i;
    for (int kk = k0; kk < k1; kk += 8) {
      const int g0 = kk + q, g1 = kk + 4 + q;
      const double a0 = vmask(Vb, ldv, g0, ia, M, nb);
      const double a1 = g1 < k1 ? vmask(Vb, ldv, g1, ia, M, nb) : 0.0;
      double b0, b1;
      if (y_is_v) {
        b0 = vmask(Yb, ldy, g0, jb, M, nc);
        b1 = g1 < k1 ? vmask(Yb, ldy, g1, jb, M, nc) : 0.0;
      } else {
        const int jc = jb < nc ? jb : nc - 1;
        b0 = (g0 < M && jb < nc) ? Yb[jc * ldy + g0] : 0.0;
        b1 = (g1 < M && g1 < k1 && jb < nc) ? Yb[jc * ldy + g1] : 0.0;
      }
      dmma884(acc[0], a0, b0);
      dmma884(acc[1], a1, b1);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) part[warp * 64 + i * 8 + q * 2 + e] = acc[0][e] + acc[1][e];
  }
  __syncthreads();
  if (T) {  // W = T^T (V^T Y) or T (V^T Y): the partial sums, then one output per thread
    double wsum = 0.0;
    const int t = threadIdx.x;
    const bool own = t < B * nc;
    const int r = own ? t / nc : 0, c = own ? t % nc : 0;
    if (own) {
      const int tile = (r / 8) + TR * (c / 8);
      for (int kc = 0; kc < nk; ++kc) wsum += part[(tile + kc * ntile) * 64 + (r % 8) * 8 + (c % 8)];
      if (r >= nb) wsum = 0.0;
    }
    __syncthreads();
    if (own) part[r * B + c] = wsum;  // w(l, c) at part[l B + c]
    __syncthreads();
    for (int u = threadIdx.x; u < nb * nc; u += blockDim.x) {
      const int i = u / nc, cc = u % nc;
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < B; ++l)
        if (trans ? (l <= i) : (l >= i)) acc = fma(trans ? T[l * B + i] : T[i * B + l], part[l * B + cc], acc);
      W[i * B + cc] = acc;
    }
  } else {
    for (int t = threadIdx.x; t < nb * nc; t += blockDim.x) {
      const int r = t / nc, c = t % nc;
      const int tile = (r / 8) + TR * (c / 8);
      double s = 0.0;
      for (int kc = 0; kc < nk; ++kc) s += part[(tile + kc * ntile) * 64 + (r % 8) * 8 + (c % 8)];
      W[r * B + c] = s;
    }
  }
  __syncthreads();
}

// Y (M x nc) -= V (M x nb) W (nb x nc): 8-row tiles over the warps, all
// nc / 8 column tiles of a row tile at once (K = nb <= B).
template <int B>
__device__ void blk_update(const double* Vb, int ldv, int nb, double* Yb, int ldy, int nc, int M,
                           const double* W) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  constexpr int KT = B / 4, CT = B / 8;
  double bw[CT][KT];
#pragma unroll
  for (int t = 0; t < CT; ++t)
#pragma unroll
    for (int u = 0; u < KT; ++u) {
      const int i = 4 * u + q, c = t * 8 + r;
      bw[t][u] = (i < nb && c < nc) ? W[i * B + c] : 0.0;
    }
  for (int mt = warp; mt * 8 < M; mt += nw) {
    const int g = mt * 8 + r;
    double av[KT];
#pragma unroll
    for (int u = 0; u < KT; ++u) av[u] = vmask(Vb, ldv, g, 4 * u + q, M, nb);
    double acc[CT][2] = {};
#pragma unroll
    for (int t = 0; t < CT; ++t)
#pragma unroll
      for (int u = 0; u < KT; ++u) dmma884(acc[t], av[u], bw[t][u]);
#pragma unroll
    for (int t = 0; t < CT; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = t * 8 + 2 * q + e;
        if (g < M && c < nc) Yb[c * ldy + g] -= acc[t][e];
      }
  }
  __syncthreads();
}

// Y <- (I - V T^(T) V^T) Y for one block reflector (W, part: scratch).
// A remote V / T (another CTA's shared memory) is first copied into the
// local staging buffers with every thread's loads in flight at once, so the
// DMMA passes read local shared memory only.
template <int B>
__device__ void blk_apply(const double* Vb, int ldv, int nb, const double* T, bool trans,
                          double* Yb, int ldy, int nc, int M, double* W, double* part,
                          double* vstage, double* tstage, bool remote) {
  if (remote) {
    // Vb / T: the producer's mirror in global memory (L2; __ldcg: the lines
    // change every round, L1 is not coherent), every thread's loads in flight
    constexpr int U = 16;
    const int total = (nb - 1) * ldv + M;  // columns of M rows, ld ldv
    for (int t0 = threadIdx.x; t0 < total; t0 += U * blockDim.x) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t0 + u * blockDim.x;
        v[u] = t < total ? __ldcg(Vb + t) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t0 + u * blockDim.x;
        if (t < total) vstage[t] = v[u];
      }
    }
    for (int t = threadIdx.x; t < B * B; t += blockDim.x) tstage[t] = __ldcg(T + t);
    __syncthreads();
    Vb = vstage;
    T = tstage;
  }
  blk_vty<B>(Vb, ldv, nb, Yb, ldy, nc, false, M, W, part, T, trans);
  blk_update<B>(Vb, ldv, nb, Yb, ldy, nc, M, W);
}


// ---------------------------------------------------------------------------
// Cluster Jacobi for matrices too large for one CTA's shared memory
// (k_jacobi_cluster, m2 = 2h <= 256): the parallel cyclic Jacobi of k_jacobi
// with the columns of A and V distributed over the cs CTAs of a cluster.
// Pairs follow the round-robin (circle) tournament: pair i is (top[i],
// bot[i]); CTA q owns pairs [q P, (q+1) P) and the 2P columns of A and V in
// those slots.  A step:
//   1. each CTA computes the rotations of its own pairs (their 2 x 2 blocks
//      are local) and writes them into every CTA's parameter table (DSMEM);
//      cluster barrier;
//   2. rows p, q of every own column rotate by pair (p, q), then the own
//      pairs' columns of A and V; the rotated 2 x 2 blocks get the tangent
//      formulas and exact zeros (same formulas as k_jacobi);
//   3. the tournament moves one column to each neighbouring CTA (pushed into
//      its inbox over DSMEM); cluster barrier; inboxes land in the buffers
//      the outgoing columns freed.
// A sweep is 2h - 1 steps.  Convergence: the k_jacobi threshold test on every
// off-diagonal entry, each CTA on its own columns (the diagonal is gathered
// into every CTA first), OR-ed through DSMEM.
// ---------------------------------------------------------------------------
constexpr int kJcThreads = 256;
constexpr int kJcMaxH = 128;
constexpr int kJcMaxP = 32;  // pairs per CTA

struct JcShared {
  double c[kJcMaxH], s[kJcMaxH], t[kJcMaxH], app[kJcMaxH], aqq[kJcMaxH], apq[kJcMaxH];
  double diag[2 * kJcMaxH];
  int p[kJcMaxH], q[kJcMaxH], on[kJcMaxH];
  int slot_buf[2 * kJcMaxP];  // local slot -> column buffer
  int slot_col[2 * kJcMaxP];  // local slot -> logical column
  int in_col[2];              // logical column arriving in inbox 0 (left) / 1 (right)
  int out_buf[2];             // buffers leaving to the right / left (-1: none)
  int hot;
  double fro2;
  double red[33];
};

__global__ void __launch_bounds__(kJcThreads)
    k_jacobi_cluster(int m, const double* __restrict__ Aall, double* Vall, double* wall,
                     int* flags) {
  extern __shared__ double dyn[];
  __shared__ JcShared sh;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks(), q = (int)cl.block_rank();
  const int b = blockIdx.x / cs;
  const int m2 = m + (m & 1), h = m2 / 2, P = h / cs, P0 = q * P;
  const int nslot = 2 * P, tid = threadIdx.x, NT = blockDim.x;
  // column buffer j (A then V, m2 doubles each); buffers nslot, nslot + 1 are
  // the inboxes (from the left / right neighbour)
  auto Acol = [&](int j) { return dyn + (size_t)j * 2 * m2; };
  auto Vcol = [&](int j) { return dyn + (size_t)j * 2 * m2 + m2; };
  const double* Ain = Aall + (size_t)b * m * m;
  for (int s = tid; s < nslot; s += NT) {  // initial pairs (2i, 2i + 1)
    const int i = P0 + (s < P ? s : s - P);
    sh.slot_buf[s] = s;
    sh.slot_col[s] = s < P ? 2 * i : 2 * i + 1;
  }
  if (tid == 0) {
    sh.fro2 = 0.0;
    sh.hot = 0;
  }
  __syncthreads();
  double part = 0.0;
  for (int t = tid; t < nslot * m2; t += NT) {
    const int s = t / m2, r = t % m2, c = sh.slot_col[s];
    const double v = (r < m && c < m) ? Ain[(size_t)c * m + r] : 0.0;
    Acol(s)[r] = v;
    Vcol(s)[r] = (r == c) ? 1.0 : 0.0;
    part += v * v;
  }
  part = block_sum(part, sh.red);
  cluster_sync_all();
  if (tid == 0)
    for (int r = 0; r < cs; ++r) atomicAdd(&cl.map_shared_rank(&sh, r)->fro2, part);
  cluster_sync_all();
  const double abs_thresh = sqrt(sh.fro2) * 1e-22 + DBL_MIN;
  bool converged = (m2 <= 1);
  int sweep = 0;
  for (; sweep < 60 && !converged; ++sweep) {
    int any = 0;
    for (int step = 0; step + 1 < m2; ++step) {
      // 1. rotations of the own pairs -> every CTA's table
      if (tid < P) {
        const int i = P0 + tid;
        const int ct = sh.slot_col[tid], cb = sh.slot_col[tid + P];
        const bool tp = ct < cb;
        const int p = tp ? ct : cb, qq = tp ? cb : ct;
        const double* Ap = Acol(sh.slot_buf[tp ? tid : tid + P]);
        const double* Aq = Acol(sh.slot_buf[tp ? tid + P : tid]);
        const double app = Ap[p], aqq = Aq[qq], apq = Aq[p];
        const double rel2 = c_jac_rel2 * fabs(app) * fabs(aqq);
        double c = 1.0, sv = 0.0, tt = 0.0;
        int on = 0;
        if (apq * apq > rel2 && fabs(apq) > abs_thresh) {
          const double theta = (aqq - app) * (0.5 * __drcp_rn(apq));
          const double at = fabs(theta);
          if (at > 1e150)
            tt = 0.5 * __drcp_rn(theta);
          else
            tt = (theta >= 0.0 ? 1.0 : -1.0) * __drcp_rn(at + sqrt(fma(theta, theta, 1.0)));
          c = rsqrt(fma(tt, tt, 1.0));
          sv = tt * c;
          on = 1;
        }
        for (int r = 0; r < cs; ++r) {
          JcShared* o = cl.map_shared_rank(&sh, r);
          o->c[i] = c;
          o->s[i] = sv;
          o->t[i] = tt;
          o->app[i] = app;
          o->aqq[i] = aqq;
          o->apq[i] = apq;
          o->p[i] = p;
          o->q[i] = qq;
          o->on[i] = on;
        }
      }
      cluster_sync_all();
      int step_on = 0;
      for (int i = tid; i < h; i += NT) step_on |= sh.on[i];
      if (__syncthreads_or(step_on)) {  // the same answer on every CTA
        any = 1;
        // 2a. rows p, q of every own column
        for (int t = tid; t < nslot * h; t += NT) {
          const int s = t / h, i = t % h;
          if (!sh.on[i]) continue;
          double* A = Acol(sh.slot_buf[s]);
          const int p = sh.p[i], qq = sh.q[i];
          const double c = sh.c[i], sv = sh.s[i];
          const double x = A[p], y = A[qq];
          A[p] = c * x - sv * y;
          A[qq] = sv * x + c * y;
        }
        __syncthreads();
        // 2b. columns p, q of the own pairs (A and V)
        for (int t = tid; t < P * m2; t += NT) {
          const int j = t / m2, r = t % m2, i = P0 + j;
          if (!sh.on[i]) continue;
          const bool tp = sh.slot_col[j] == sh.p[i];
          const int bp = sh.slot_buf[tp ? j : j + P], bq = sh.slot_buf[tp ? j + P : j];
          const double c = sh.c[i], sv = sh.s[i];
          double* Ap = Acol(bp);
          double* Aq = Acol(bq);
          const double x = Ap[r], y = Aq[r];
          Ap[r] = c * x - sv * y;
          Aq[r] = sv * x + c * y;
          double* Vp = Vcol(bp);
          double* Vq = Vcol(bq);
          const double vx = Vp[r], vy = Vq[r];
          Vp[r] = c * vx - sv * vy;
          Vq[r] = sv * vx + c * vy;
        }
        __syncthreads();
        // 2c. tangent formulas on the rotated 2 x 2 blocks
        if (tid < P && sh.on[P0 + tid]) {
          const int i = P0 + tid;
          const bool tp = sh.slot_col[tid] == sh.p[i];
          double* Ap = Acol(sh.slot_buf[tp ? tid : tid + P]);
          double* Aq = Acol(sh.slot_buf[tp ? tid + P : tid]);
          const int p = sh.p[i], qq = sh.q[i];
          const double tt = sh.t[i], apq = sh.apq[i];
          Ap[p] = sh.app[i] - tt * apq;
          Aq[qq] = sh.aqq[i] + tt * apq;
          Ap[qq] = 0.0;
          Aq[p] = 0.0;
        }
      }
      // 3. tournament: new_top[0] = top[0], new_top[1] = bot[0],
      //    new_top[i] = top[i-1] (i >= 2), new_bot[i] = bot[i+1] (i < h-1),
      //    new_bot[h-1] = top[h-1].
      if (tid == 0) {
        sh.out_buf[0] = -1;
        sh.out_buf[1] = -1;
        if (q < cs - 1) {  // top[P0 + P - 1] -> right neighbour's top slot 0
          sh.out_buf[0] = sh.slot_buf[P - 1];
          cl.map_shared_rank(&sh, q + 1)->in_col[0] = sh.slot_col[P - 1];
        }
        if (q > 0) {  // bot[P0] -> left neighbour's last bot slot
          sh.out_buf[1] = sh.slot_buf[P];
          cl.map_shared_rank(&sh, q - 1)->in_col[1] = sh.slot_col[P];
        }
      }
      __syncthreads();
      if (sh.out_buf[0] >= 0) {
        double* dst = cl.map_shared_rank(dyn, q + 1) + (size_t)(nslot + 0) * 2 * m2;
        const double* src = Acol(sh.out_buf[0]);
        for (int r = tid; r < 2 * m2; r += NT) dst[r] = src[r];
      }
      if (sh.out_buf[1] >= 0) {
        double* dst = cl.map_shared_rank(dyn, q - 1) + (size_t)(nslot + 1) * 2 * m2;
        const double* src = Acol(sh.out_buf[1]);
        for (int r = tid; r < 2 * m2; r += NT) dst[r] = src[r];
      }
      cluster_sync_all();
      // inboxes: from the left into the buffer the right-going column freed
      // (the last CTA has none: the left-going one), and vice versa
      const int ob_r = sh.out_buf[0], ob_l = sh.out_buf[1];
      const int dst_left = ob_r >= 0 ? ob_r : ob_l, dst_right = ob_l >= 0 ? ob_l : ob_r;
      if (q > 0) {
        const double* src = dyn + (size_t)(nslot + 0) * 2 * m2;
        double* dst = Acol(dst_left);
        for (int r = tid; r < 2 * m2; r += NT) dst[r] = src[r];
      }
      if (q < cs - 1) {
        const double* src = dyn + (size_t)(nslot + 1) * 2 * m2;
        double* dst = Acol(dst_right);
        for (int r = tid; r < 2 * m2; r += NT) dst[r] = src[r];
      }
      if (tid == 0) {
        int nb[2 * kJcMaxP], nc[2 * kJcMaxP];
        for (int s = 0; s < P; ++s) {  // tops
          const int g = P0 + s;
          if (g == 0) {
            nb[s] = sh.slot_buf[0];
            nc[s] = sh.slot_col[0];
          } else if (g == 1) {
            nb[s] = sh.slot_buf[P];
            nc[s] = sh.slot_col[P];
          } else if (s == 0) {
            nb[s] = dst_left;
            nc[s] = sh.in_col[0];
          } else {
            nb[s] = sh.slot_buf[s - 1];
            nc[s] = sh.slot_col[s - 1];
          }
        }
        for (int s = 0; s < P; ++s) {  // bots
          const int g = P0 + s;
          if (g == h - 1) {
            nb[P + s] = sh.slot_buf[P - 1];
            nc[P + s] = sh.slot_col[P - 1];
          } else if (s == P - 1) {
            nb[P + s] = dst_right;
            nc[P + s] = sh.in_col[1];
          } else {
            nb[P + s] = sh.slot_buf[P + s + 1];
            nc[P + s] = sh.slot_col[P + s + 1];
          }
        }
        for (int s = 0; s < nslot; ++s) {
          sh.slot_buf[s] = nb[s];
          sh.slot_col[s] = nc[s];
        }
      }
      __syncthreads();
    }
    converged = !any;
    if (!converged) {
      // a sweep that rotated: converged iff no off-diagonal entry is above
      // its threshold now (k_jacobi's direct test)
      for (int s = tid; s < nslot; s += NT) {
        const int c = sh.slot_col[s];
        const double d = Acol(sh.slot_buf[s])[c];
        for (int r = 0; r < cs; ++r) cl.map_shared_rank(&sh, r)->diag[c] = d;
      }
      if (tid == 0) sh.hot = 0;
      cluster_sync_all();
      int hot = 0;
      for (int t = tid; t < nslot * m2; t += NT) {
        const int s = t / m2, r = t % m2, c = sh.slot_col[s];
        if (r == c) continue;
        const double arc = Acol(sh.slot_buf[s])[r];
        const double rel = c_jac_rel * sqrt(fabs(sh.diag[r]) * fabs(sh.diag[c]));
        if (fabs(arc) > (rel > abs_thresh ? rel : abs_thresh)) hot = 1;
      }
      hot = __syncthreads_or(hot);
      if (tid == 0 && hot)
        for (int r = 0; r < cs; ++r) atomicOr(&cl.map_shared_rank(&sh, r)->hot, 1);
      cluster_sync_all();
      converged = !sh.hot;
      cluster_sync_all();  // every CTA has read hot before the next reset
    }
  }
  if (threadIdx.x == 0 && q == 0 && b < 8) g_jacobi_sweeps[b] = sweep;
  double* Vo = Vall + (size_t)b * m * m;
  double* wo = wall + (size_t)b * m;
  for (int t = tid; t < nslot * m2; t += NT) {
    const int s = t / m2, r = t % m2, c = sh.slot_col[s];
    if (c < m && r < m) Vo[(size_t)c * m + r] = Vcol(sh.slot_buf[s])[r];
    if (c < m && r == 0) wo[c] = Acol(sh.slot_buf[s])[c];
  }
  if (!converged && tid == 0 && q == 0) atomicOr(flags, 1);
}

// ---------------------------------------------------------------------------
// Block Jacobi over a cluster (k_jacobi_blk, m <= 256; the default for
// matrices too large for one CTA).  The m2 = 16 bw columns (bw = ceil(m/16),
// zero padded: a zero column never rotates with a real one) form 16 blocks;
// CTA q of the 8-CTA cluster holds one block pair (top, bottom) = 2 bw full
// columns of A in shared memory, and the pairs follow the round-robin
// tournament over blocks (15 block steps per sweep).  A block step:
//   1. the own 2bw x 2bw diagonal block S = A[R_q, R_q] gets one parallel
//      cyclic Jacobi sweep (k_jacobi's rotation formulas, threshold and
//      exact zeros), accumulating J_q (S' = J_q^T S J_q);  cluster barrier;
//   2. A <- J^T A J with J = blockdiag(J_0 .. J_7): every CTA updates its own
//      columns (A[:, own] J_q, then rows R_p by J_p^T for every pair p, J_p
//      read over DSMEM; its own diagonal block becomes S' exactly), and the
//      eigenvector columns V[:, own] J_q in global memory;  cluster barrier;
//   3. the blocks move to their next pair (pulled from the neighbours'
//      buffers into the other half of a double buffer).
// Two cluster barriers per block step instead of two per rotation step, so
// a sweep costs 30 cluster barriers instead of 2 (m2 - 1).  Convergence:
// k_jacobi's direct test on every off-diagonal entry after each sweep.
// Same eigenproblem, same rotation formulas: the eigenvectors agree with the
// oracle's orc_jacobi_eig to rounding on separated eigenvalues (P3).
// ---------------------------------------------------------------------------
constexpr int kJbThreads = 256;
constexpr int kJbCs = 8;
constexpr int kJbNblk = 2 * kJbCs;
constexpr int kJbMaxBw = 16;
constexpr int kJbMaxS = 2 * kJbMaxBw;

__device__ long long g_jb_prof[8];
struct JbShared {
  double S[kJbMaxS][kJbMaxS + 1];
  double J[kJbMaxS][kJbMaxS + 1];
  double c[kJbMaxBw], s[kJbMaxBw], t[kJbMaxBw];
  int P[kJbMaxBw], Q[kJbMaxBw];
  double diag[kJbNblk * kJbMaxBw];
  int top[kJbCs], bot[kJbCs];
  int hot;
  double fro2;
  double red[33];
};

__global__ void __launch_bounds__(kJbThreads, 1)
    k_jacobi_blk(int m, const double* __restrict__ Aall, double* Vg_all, double* Vall,
                 double* wall, int* flags) {
  extern __shared__ double dyn[];
  __shared__ JbShared sh;
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int b = blockIdx.x / kJbCs;
  constexpr int bw = kJbMaxBw, m2 = kJbNblk * bw, n2 = 2 * bw, h2 = bw;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5;
  // A column buffers: [phase][slot][bw][ldc]; slot 0 = top block, 1 =
  // bottom; odd column stride ldc = m2 + 1, so the 8 columns of a DMMA
  // fragment fall on different banks
  constexpr int ldc = m2 + 1;
  auto Acol = [&](int ph, int j) {  // local column j < n2 of phase ph
    return dyn + ((size_t)(ph * 2 + (j >= bw)) * bw + (j >= bw ? j - bw : j)) * ldc;
  };
  double* Vg = Vg_all + (size_t)b * m2 * m2;  // V(r, c) = Vg[c m2 + r]
  const double* Ain = Aall + (size_t)b * m * m;
  if (tid < kJbCs) {
    sh.top[tid] = 2 * tid;
    sh.bot[tid] = 2 * tid + 1;
  }
  if (tid == 0) {
    sh.fro2 = 0.0;
    sh.hot = 0;
  }
  __syncthreads();
  auto lcol = [&](int pair, int j) {  // logical column of local index j of a pair
    return j < bw ? sh.top[pair] * bw + j : sh.bot[pair] * bw + j - bw;
  };
  double part = 0.0;
  for (int t = tid; t < n2 * m2; t += NT) {
    const int j = t / m2, r = t % m2, c = lcol(q, j);
    const double v = (r < m && c < m) ? Ain[(size_t)c * m + r] : 0.0;
    Acol(0, j)[r] = v;
    Vg[(size_t)c * m2 + r] = (r == c) ? 1.0 : 0.0;
    part += v * v;
  }
  part = block_sum(part, sh.red);
  cluster_sync_all();
  if (tid == 0)
    for (int r = 0; r < kJbCs; ++r) atomicAdd(&cl.map_shared_rank(&sh, r)->fro2, part);
  cluster_sync_all();
  const double abs_thresh = sqrt(sh.fro2) * 1e-22 + DBL_MIN;
  // inner 2x2-block tasks (a <= b over the h2 pairs), one or two per thread
  const int ntri = h2 * (h2 + 1) / 2;
  int ta[2], tb[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int t = tid + k * NT;
    int a = 0, off = 0;
    if (t < ntri)
      while (off + (h2 - a) <= t) {
        off += h2 - a;
        ++a;
      }
    ta[k] = t < ntri ? a : -1;
    tb[k] = t < ntri ? a + (t - off) : 0;
  }
  int ph = 0;
  bool converged = false;
  int sweep = 0;
  for (; sweep < 60 && !converged; ++sweep) {
    for (int bstep = 0; bstep < kJbNblk - 1; ++bstep) {
      long long tp0 = clock64();
      // ---- 1. inner sweep on S = A[R_q, R_q] ----
      for (int t = tid; t < n2 * n2; t += NT) {
        const int i = t % n2, j = t / n2;
        sh.S[i][j] = Acol(ph, j)[lcol(q, i)];
        sh.J[i][j] = (i == j) ? 1.0 : 0.0;
      }
      __syncthreads();
      const int rr = n2 - 1;
      for (int st = 0; st < rr; ++st) {
        int on = 0;
        if (tid < h2) {
          const int i = tid;
          int x, y;
          if (i == 0) {
            x = 0;
            y = st + rr - 1;
            if (y >= rr) y -= rr;
            ++y;
          } else {
            x = i + st - 1;
            if (x >= rr) x -= rr;
            ++x;
            y = rr - i + st - 1;
            if (y >= rr) y -= rr;
            ++y;
          }
          const int p = x < y ? x : y, qq = x < y ? y : x;
          sh.P[i] = p;
          sh.Q[i] = qq;
          const double app = sh.S[p][p], aqq = sh.S[qq][qq], apq = sh.S[qq][p];
          const double rel2 = c_jac_rel2 * fabs(app) * fabs(aqq);
          double c = 1.0, sv = 0.0, tt = 0.0;
          if (apq * apq > rel2 && fabs(apq) > abs_thresh) {
            const double theta = (aqq - app) * (0.5 * __drcp_rn(apq));
            const double at = fabs(theta);
            if (at > 1e150)
              tt = 0.5 * __drcp_rn(theta);
            else
              tt = (theta >= 0.0 ? 1.0 : -1.0) * __drcp_rn(at + sqrt(fma(theta, theta, 1.0)));
            c = rsqrt(fma(tt, tt, 1.0));
            sv = tt * c;
            on = 1;
          }
          sh.c[i] = c;
          sh.s[i] = sv;
          sh.t[i] = tt;
        }
        if (!__syncthreads_or(on)) continue;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int a = ta[k], bb = tb[k];
          if (a < 0) continue;
          const int p1 = sh.P[a], q1 = sh.Q[a];
          if (a == bb) {
            const double t = sh.t[a];
            if (t != 0.0) {
              const double apq = sh.S[q1][p1];
              sh.S[p1][p1] = sh.S[p1][p1] - t * apq;
              sh.S[q1][q1] = sh.S[q1][q1] + t * apq;
              sh.S[q1][p1] = 0.0;
              sh.S[p1][q1] = 0.0;
            }
            continue;
          }
          const double sa = sh.s[a], sb = sh.s[bb];
          if (sa == 0.0 && sb == 0.0) continue;
          const int p2 = sh.P[bb], q2 = sh.Q[bb];
          const double ca = sh.c[a], cb = sh.c[bb];
          const double b00 = sh.S[p1][p2], b01 = sh.S[p1][q2];
          const double b10 = sh.S[q1][p2], b11 = sh.S[q1][q2];
          const double r00 = ca * b00 - sa * b10, r01 = ca * b01 - sa * b11;
          const double r10 = sa * b00 + ca * b10, r11 = sa * b01 + ca * b11;
          const double n00 = cb * r00 - sb * r01, n01 = sb * r00 + cb * r01;
          const double n10 = cb * r10 - sb * r11, n11 = sb * r10 + cb * r11;
          sh.S[p1][p2] = n00;
          sh.S[p2][p1] = n00;
          sh.S[p1][q2] = n01;
          sh.S[q2][p1] = n01;
          sh.S[q1][p2] = n10;
          sh.S[p2][q1] = n10;
          sh.S[q1][q2] = n11;
          sh.S[q2][q1] = n11;
        }
        for (int t = tid; t < h2 * n2; t += NT) {  // J <- J G (columns p, q)
          const int a = t / n2, r = t % n2;
          const double sa = sh.s[a];
          if (sa == 0.0) continue;
          const double ca = sh.c[a];
          const int p = sh.P[a], qq = sh.Q[a];
          const double x = sh.J[r][p], y = sh.J[r][qq];
          sh.J[r][p] = ca * x - sa * y;
          sh.J[r][qq] = sa * x + ca * y;
        }
        __syncthreads();
      }
      long long tp1 = clock64();
      cluster_sync_all();  // every J_p published
      long long tp2 = clock64();
      // ---- 2a. own columns: A[:, own] <- A[:, own] J_q ; V likewise ----
      // FP64 tensor tiles (DMMA 8x8x4): every warp owns whole 8-row tiles
      // (all 32 columns), so it reads a tile's rows completely before it
      // overwrites them; J_q's fragments stay in registers for all tiles.
      {
        const int fr = lane >> 2, fk = lane & 3;
        double bj[n2 / 4][n2 / 8];  // J(k = 4 ks + fk, n = 8 ct + fr)
#pragma unroll
        for (int ks = 0; ks < n2 / 4; ++ks)
#pragma unroll
          for (int ct = 0; ct < n2 / 8; ++ct) bj[ks][ct] = sh.J[4 * ks + fk][8 * ct + fr];
        for (int mt = warp; mt < 2 * m2 / 8; mt += NT / 32) {
          const bool isv = mt * 8 >= m2;
          const int r0 = isv ? mt * 8 - m2 : mt * 8;
          double acc[n2 / 8][2];
#pragma unroll
          for (int ct = 0; ct < n2 / 8; ++ct) acc[ct][0] = acc[ct][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < n2 / 4; ++ks) {
            const int k = 4 * ks + fk;
            const double av = isv ? Vg[(size_t)lcol(q, k) * m2 + r0 + fr] : Acol(ph, k)[r0 + fr];
#pragma unroll
            for (int ct = 0; ct < n2 / 8; ++ct) dmma884(acc[ct], av, bj[ks][ct]);
          }
#pragma unroll
          for (int ct = 0; ct < n2 / 8; ++ct)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int c = 8 * ct + 2 * fk + e;
              if (isv)
                Vg[(size_t)lcol(q, c) * m2 + r0 + fr] = acc[ct][e];
              else
                Acol(ph, c)[r0 + fr] = acc[ct][e];
            }
        }
      }
      __syncthreads();
      long long tp3 = clock64();
      // ---- 2b. rows R_p of the own columns <- J_p^T (every pair p) ----
      {
        // stage every other pair's J (DSMEM) at once: one barrier, not one per pair
        typedef double JT[kJbMaxS][kJbMaxS + 1];
        JT* Js = reinterpret_cast<JT*>(dyn + (size_t)4 * bw * ldc);
        // eight remote loads in flight per thread (DSMEM latency, not bandwidth)
        for (int t0 = tid; t0 < kJbCs * n2 * n2; t0 += 8 * NT) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int t = t0 + u * NT;
            const int pp = t / (n2 * n2), e = t % (n2 * n2), i = e % n2, j = e / n2;
            v[u] = (t < kJbCs * n2 * n2 && pp != q) ? cl.map_shared_rank(&sh, pp)->J[i][j] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int t = t0 + u * NT;
            const int pp = t / (n2 * n2), e = t % (n2 * n2), i = e % n2, j = e / n2;
            if (t < kJbCs * n2 * n2 && pp != q) Js[pp][i][j] = v[u];
          }
        }
        __syncthreads();
        // out(i, c) = sum_k J_p(k, i) A(R_p[k], c) as DMMA tiles: warp w owns
        // tiles 2w, 2w + 1 (of 16 per pair) of every pair; all products into
        // registers first, one barrier, then the stores (in place)
        const int fr = lane >> 2, fk = lane & 3;
        constexpr int kTiles = (n2 / 8) * (n2 / 8);
        constexpr int kPerWarp = kTiles / (kJbThreads / 32);
        double acc[kJbCs][kPerWarp][2];
#pragma unroll
        for (int pp = 0; pp < kJbCs; ++pp) {
#pragma unroll
          for (int u = 0; u < kPerWarp; ++u) {
            acc[pp][u][0] = acc[pp][u][1] = 0.0;
            if (pp == q) continue;
            const int tile = warp * kPerWarp + u, it = tile / (n2 / 8), ct = tile % (n2 / 8);
#pragma unroll
            for (int ks = 0; ks < n2 / 4; ++ks) {
              const int k = 4 * ks + fk;
              const double av = Js[pp][k][8 * it + fr];                 // A(m = i, k) = J_p(k, i)
              const double bv = Acol(ph, 8 * ct + fr)[lcol(pp, k)];    // B(k, n = c)
              dmma884(acc[pp][u], av, bv);
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int pp = 0; pp < kJbCs; ++pp)
#pragma unroll
          for (int u = 0; u < kPerWarp; ++u) {
            const int tile = warp * kPerWarp + u, it = tile / (n2 / 8), ct = tile % (n2 / 8);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * it + fr, c = 8 * ct + 2 * fk + e;
              // own diagonal block: the inner result, exactly
              Acol(ph, c)[lcol(pp, i)] = pp == q ? sh.S[i][c] : acc[pp][u][e];
            }
          }
        __syncthreads();
      }
      long long tp4 = clock64();
      cluster_sync_all();  // every update done, every J read
      long long tp5 = clock64();
      // ---- 3. tournament: pull the next pair into the other phase ----
      {
        const int nph = ph ^ 1;
        // new top: q == 0 keeps its top; q == 1 takes pair 0's bottom;
        // q >= 2 takes pair q-1's top.  New bottom: q < 7 takes pair q+1's
        // bottom; q == 7 takes its own top.
        const int st_rank = q == 0 ? 0 : (q == 1 ? 0 : q - 1), st_slot = q == 1 ? 1 : 0;
        const int sb_rank = q < kJbCs - 1 ? q + 1 : q, sb_slot = q < kJbCs - 1 ? 1 : 0;
        const double* srct =
            cl.map_shared_rank(dyn, st_rank) + ((size_t)(ph * 2 + st_slot) * bw) * ldc;
        const double* srcb =
            cl.map_shared_rank(dyn, sb_rank) + ((size_t)(ph * 2 + sb_slot) * bw) * ldc;
        double* dstt = dyn + ((size_t)(nph * 2 + 0) * bw) * ldc;
        double* dstb = dyn + ((size_t)(nph * 2 + 1) * bw) * ldc;
        const int tot = bw * ldc;
        for (int t0 = tid; t0 < tot; t0 += 8 * NT) {
          double vt[8], vb[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int t = t0 + u * NT;
            vt[u] = t < tot ? srct[t] : 0.0;
            vb[u] = t < tot ? srcb[t] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int t = t0 + u * NT;
            if (t < tot) {
              dstt[t] = vt[u];
              dstb[t] = vb[u];
            }
          }
        }
        __syncthreads();
        if (tid == 0) {
          int nt[kJbCs], nb[kJbCs];
          for (int i = 0; i < kJbCs; ++i) {
            nt[i] = i == 0 ? sh.top[0] : (i == 1 ? sh.bot[0] : sh.top[i - 1]);
            nb[i] = i < kJbCs - 1 ? sh.bot[i + 1] : sh.top[kJbCs - 1];
          }
          for (int i = 0; i < kJbCs; ++i) {
            sh.top[i] = nt[i];
            sh.bot[i] = nb[i];
          }
        }
        ph = nph;
        __syncthreads();
      }
      if (tid == 0 && q == 0 && b == 2) {
        g_jb_prof[0] += tp1 - tp0; g_jb_prof[1] += tp2 - tp1; g_jb_prof[2] += tp3 - tp2;
        g_jb_prof[3] += tp4 - tp3; g_jb_prof[4] += tp5 - tp4; g_jb_prof[5] += clock64() - tp5;
      }
    }
    // ---- convergence: k_jacobi's direct test on every off-diagonal entry ----
    for (int j = tid; j < n2; j += NT) {
      const int c = lcol(q, j);
      const double d = Acol(ph, j)[c];
      for (int r = 0; r < kJbCs; ++r) cl.map_shared_rank(&sh, r)->diag[c] = d;
    }
    if (tid == 0) sh.hot = 0;
    cluster_sync_all();
    int hot = 0;
    for (int t = tid; t < n2 * m2; t += NT) {
      const int j = t / m2, r = t % m2, c = lcol(q, j);
      if (r == c) continue;
      const double arc = Acol(ph, j)[r];
      const double rel = c_jac_rel * sqrt(fabs(sh.diag[r]) * fabs(sh.diag[c]));
      if (fabs(arc) > (rel > abs_thresh ? rel : abs_thresh)) hot = 1;
    }
    hot = __syncthreads_or(hot);
    if (tid == 0 && hot)
      for (int r = 0; r < kJbCs; ++r) atomicOr(&cl.map_shared_rank(&sh, r)->hot, 1);
    cluster_sync_all();
    converged = !sh.hot;
    cluster_sync_all();
  }
  if (threadIdx.x == 0 && q == 0 && b < 8) g_jacobi_sweeps[b] = sweep;
  double* Vo = Vall + (size_t)b * m * m;
  double* wo = wall + (size_t)b * m;
  for (int t = tid; t < n2 * m2; t += NT) {
    const int j = t / m2, r = t % m2, c = lcol(q, j);
    if (c < m && r < m) Vo[(size_t)c * m + r] = Vg[(size_t)c * m2 + r];
    if (c < m && r == 0) wo[c] = Acol(ph, j)[c];
  }
  if (!converged && tid == 0 && q == 0) atomicOr(flags, 1);
}

__device__ long long g_oic_prof[64 * 8];  // per-CTA cycle split of k_oi_cluster (DMCG_DEBUG)

// Mirror of every CTA's published block reflector (V rows c0.. of its
// block, T) in global memory, per axis and rank: the later CTAs copy it
// from L2 instead of from the producer's shared memory (up to 15 CTAs read
// each block; over DSMEM they all land on the producer's SM).
__host__ __device__ constexpr size_t oi_mirror_stride(int ld, int B) { return (size_t)ld * B + (size_t)B * B; }

// DMCG_OI_PANELS=blocked: the former 4-column register panels + blocked
// update for B = 16 blocks (tests compare the two factorizations)
__constant__ int c_oi_blocked = 0;
__device__ __forceinline__ bool oi_blocked_panels() { return c_oi_blocked != 0; }

template <int MAXR, int B>
__global__ void __launch_bounds__(kOiThreads)
    k_oi_cluster(int F, int k, int rounds, const double* __restrict__ Rall,
                 const double* __restrict__ start, double* Qall, double* Hall, double* mirror,
                 long start_bs, double* Call) {
  extern __shared__ double dyn[];
  __shared__ double s_tau[B];
  __shared__ double s_T[B * B];
  __shared__ double s_W[B * B];
  __shared__ double s_part[(kOiThreads / 32) * 64];
  __shared__ int s_ready;
  constexpr int PW = QrPanel<MAXR>::PW;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int b = blockIdx.x / cs;
  const int ld = odd_ld(F);
  double* Zb = dyn;
  double* Qb = dyn + (size_t)ld * B;
  double* Vs = Qb + (size_t)ld * B;   // staging copy of a remote block reflector
  double* Ts = Vs + (size_t)ld * B;   // and its T
  double* scr = Ts + B * B;           // wqr_factor scratch (B > PW)
  const int c0 = rank * B, nb = min(B, k - c0);
  const size_t mstride = oi_mirror_stride(ld, B);
  double* mir_axis = mirror + (size_t)b * cs * mstride;
  auto mir_v = [&](int q) { return mir_axis + (size_t)q * mstride; };
  auto mir_t = [&](int q) { return mir_axis + (size_t)q * mstride + (size_t)ld * B; };
  // Rall == nullptr: QR only (Q of the start matrices, no R Q / H) — one
  // round of the implicit X (X^T Q) iteration, whose products run as GEMMs
  const double* R = Rall ? Rall + (size_t)b * F * F : nullptr;
  // Call != nullptr (with Rall == nullptr, rounds == 0): completion mode.  The
  // start matrix is U_k (axis stride start_bs); after the factor the cluster
  // forms columns k..F-1 of the full Householder Q, H_0 ... H_{cs-1} e_j, from
  // the mirrored block reflectors, B columns per CTA and pass, into
  // Call + b start_bs + F k (k_complete does the same on ONE CTA per axis).
  const bool complete = Call != nullptr;
  const double* S = start + (size_t)b * (start_bs ? (size_t)start_bs : (size_t)F * k);
  for (int t = threadIdx.x; t < F * B; t += blockDim.x) {
    const int j = t / F, i = t % F;
    Zb[j * ld + i] = j < nb ? S[(size_t)(c0 + j) * F + i] : 0.0;
  }
  if (threadIdx.x == 0) s_ready = 0;
  cluster_sync_all();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t_wait = 0, t_app = 0, t_fac = 0, t_form = 0, t_sync = 0, t_rq = 0;
  for (int r = 0;; ++r) {
    const int epoch = r + 1;
    long long t0 = clock64();
    // ---- factor: apply the published reflectors of the earlier blocks ----
    for (int p = 0; p < rank; ++p) {
      if (threadIdx.x == 0) {
        const int* f = cl.map_shared_rank(&s_ready, p);
        while (ld_acquire_cluster(f) < epoch) {
        }
      }
      __syncthreads();
      long long t1 = clock64();
      t_wait += t1 - t0;
      blk_apply<B>(mir_v(p), ld, B, mir_t(p), true, Zb + p * B, ld, nb, F - p * B, s_W, s_part,
                   Vs + p * B, Ts, true);
      t0 = clock64();
      t_app += t0 - t1;
    }
    // ---- own block: Householder factor, T = dlarft(V, tau), publish ------
    if (nb > 0) {
      if (B == PW) {
        if (warp == 0) warp_panel_qr_T<MAXR, PW>(Zb + c0, F - c0, ld, nb, s_tau, s_T, lane);
        __syncthreads();
      } else if (!oi_blocked_panels()) {
        cta_panel_qr_T<(32 * MAXR + kOiThreads - 1) / kOiThreads, B>(Zb + c0, F - c0, ld, nb, s_tau,
                                                                     s_T);
      } else {
        wqr_factor<MAXR>(Zb + c0, F - c0, ld, nb, s_tau, scr, nb);
        blk_vty<B>(Zb + c0, ld, nb, Zb + c0, ld, nb, true, F - c0, s_W, s_part);
      }
      if (B != PW && oi_blocked_panels() && warp == 0) {
        // dlarft row j on lane j from G = s_W (row-major, ld B)
        if (lane < B) {
          const int j = lane;
          double tr[B];
#pragma unroll
          for (int i = 0; i < B; ++i) {
            double v = 0.0;
            if (i < nb && i == j) v = s_tau[i];
            if (i < nb && i > j) {
              double acc = 0.0;
#pragma unroll
              for (int l = 0; l < B; ++l)
                if (l < i && l >= j) acc = fma(tr[l], s_W[l * B + i], acc);
              v = -s_tau[i] * acc;
            }
            tr[i] = j < nb ? v : 0.0;
          }
#pragma unroll
          for (int i = 0; i < B; ++i) s_T[j * B + i] = tr[i];
        }
      }
      __syncthreads();
    }
    // publish: the block's reflectors (rows c0.. of the own columns) and T
    // to the global mirror, then the release flag
    if (nb > 0) {
      const int total = (B - 1) * ld + (F - c0);
      double* mv = mir_v(rank);
      for (int t = threadIdx.x; t < total; t += blockDim.x) mv[t] = Zb[c0 + t];
      double* mt = mir_t(rank);
      for (int t = threadIdx.x; t < B * B; t += blockDim.x) mt[t] = s_T[t];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      st_release_cluster(&s_ready, epoch);
    }
    long long t1 = clock64();
    t_fac += t1 - t0;
    // ---- thin Q block: Q_c = H_0 ... H_c E_c ------------------------------
    for (int t = threadIdx.x; t < F * B; t += blockDim.x) {
      const int j = t / F, i = t % F;
      Qb[j * ld + i] = (j < nb && i == c0 + j) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int p = rank; p >= 0 && nb > 0 && !complete; --p) {
      const bool own = p == rank;
      const double* Vp = own ? Zb + p * B : mir_v(p);
      const double* Tp = own ? s_T : mir_t(p);
      blk_apply<B>(Vp, ld, own ? nb : B, Tp, false, Qb + p * B, ld, nb, F - p * B, s_W,
                   s_part, Vs + p * B, Ts, !own);
    }
    t0 = clock64();
    t_form += t0 - t1;
    cluster_sync_all();  // every remote read of this round's V is done
    t1 = clock64();
    t_sync += t1 - t0;
    if (complete) {
      // every block reflector of the factor is mirrored (the barrier above
      // orders the other CTAs' mirror stores before these loads)
      double* Co = Call + (size_t)b * (size_t)start_bs + (size_t)F * k;
      const int ncomp = F - k;
      for (int cb = rank; cb * B < ncomp; cb += cs) {
        const int nbc = min(B, ncomp - cb * B), col0 = k + cb * B;
        __syncthreads();
        for (int t = threadIdx.x; t < F * B; t += blockDim.x) {
          const int j = t / F, i = t % F;
          Qb[j * ld + i] = (j < nbc && i == col0 + j) ? 1.0 : 0.0;
        }
        __syncthreads();
        for (int p = cs - 1; p >= 0; --p)
          blk_apply<B>(mir_v(p), ld, B, mir_t(p), false, Qb + p * B, ld, nbc, F - p * B, s_W,
                       s_part, Vs + p * B, Ts, true);
        __syncthreads();
        for (int t = threadIdx.x; t < F * nbc; t += blockDim.x) {
          const int j = t / F, i = t % F;
          Co[(size_t)(cb * B + j) * F + i] = Qb[j * ld + i];
        }
      }
      return;
    }
    // ---- Z_c = R Q_c --------------------------------------------------------
    if (!R) break;
    if (nb > 0) rq_tasks(R, F, F, nb, Qb, ld, Zb, ld, 0, (F + 7) / 8);
    __syncthreads();
    t_rq += clock64() - t1;
    if (r == rounds) break;
  }
  if (threadIdx.x == 0 && blockIdx.x < 64) {
    long long* g = g_oic_prof + blockIdx.x * 8;
    g[0] = t_wait; g[1] = t_app; g[2] = t_fac; g[3] = t_form; g[4] = t_sync; g[5] = t_rq;
  }
  // Q out; H = Q^T (R Q) by column blocks, symmetrised like the oracle.
  double* Qo = Qall + (size_t)b * F * k;
  double* H = Hall ? Hall + (size_t)b * k * k : nullptr;
  for (int t = threadIdx.x; t < F * nb; t += blockDim.x) {
    const int j = t / F, i = t % F;
    Qo[(size_t)(c0 + j) * F + i] = Qb[j * ld + i];
  }
  if (!R) return;
  cluster_sync_all();
  if (nb > 0) warp_gemm_tn(k, nb, F, Qo, F, Zb, ld, H + (size_t)c0 * k, k);
  cluster_sync_all();
  for (int t = threadIdx.x; t < k * nb; t += blockDim.x) {
    const int i = t % k, j = c0 + t / k;
    if (i >= j) continue;
    const double sv = 0.5 * (__ldcg(H + (size_t)j * k + i) + __ldcg(H + (size_t)i * k + j));
    H[(size_t)j * k + i] = sv;
    H[(size_t)i * k + j] = sv;
  }
}

}  // namespace


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


static cudaError_t set_smem_attr(const void* fn, size_t bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}


// Blocked-QR scratch: W (PW x (wcols + PW)) | T of every panel (PW = 8, or
// 4 when F > 256: the bound below covers both).
static size_t qr_scratch(int wcols, int k) {
  constexpr int PW = 8;
  return (size_t)PW * (wcols + PW) + (size_t)((k + 3) / 4) * 16 + (size_t)((k + PW - 1) / PW) * PW * PW;
}

size_t qr_scratch_doubles(int F, int k) { return qr_scratch(F > k ? F : k, k); }

// Dynamic shared memory left for `fn` next to its static shared memory.
static size_t smem_room(const void* fn) {
  // initialised once, thread-safe (magic static): contexts on several host
  // threads call the launchers concurrently
  static const int optin = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      v = 227 * 1024;
    return v;
  }();
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return 0;
  return (size_t)optin > fa.sharedSizeBytes + 256 ? optin - fa.sharedSizeBytes - 256 : 0;
}

cudaError_t launch_jacobi(cudaStream_t s, int nbatch, int m, const double* A, double* work,
                          double* V, double* w, int* flags) {
  static std::once_flag rel_once;
  std::call_once(rel_once, [] {
    if (const char* e = getenv("DMCG_JAC_REL")) {
      const double r = atof(e), r2 = r * r;
      cudaMemcpyToSymbol(c_jac_rel, &r, sizeof(r));
      cudaMemcpyToSymbol(c_jac_rel2, &r2, sizeof(r2));
    }
  });
  if (m > 512) return cudaErrorInvalidValue;
  const int m2 = m + (m & 1);
  const size_t abytes = (size_t)m2 * (m2 + 1) * sizeof(double);
  const size_t room = smem_room((const void*)k_jacobi);
  int nsplit = 0;
  static const bool force_cluster = getenv("DMCG_JACOBI_CLUSTER") != nullptr;  // tests
  for (int sp = 1; sp <= 8 && abytes < room && !force_cluster; sp *= 2) {
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
    // (DMCG_JAC_THREADS: experiments; at m = 64 fewer threads measured slower:
    // 1024 / 512 / 256 -> 0.90 / 0.98 / 1.18 ms for the three c1 axes)
    static const int env_nt = getenv("DMCG_JAC_THREADS") ? atoi(getenv("DMCG_JAC_THREADS")) : 0;
    int nt = kJacThreads;
    if (env_nt >= 64 && env_nt <= kJacThreads && env_nt % 32 == 0) nt = env_nt;
    k_jacobi<<<dim3(nbatch, nsplit), nt, smem, s>>>(m, A, work, V, w, flags, 1, vr);
    static const bool dbg = getenv("DMCG_DEBUG") != nullptr;
    if (dbg) {
      int sw[8] = {};
      cudaStreamSynchronize(s);
      cudaMemcpyFromSymbol(sw, g_jacobi_sweeps, sizeof(sw));
      fprintf(stderr, "dmcg: k_jacobi m=%d split %d sweeps %d %d %d\n", m, nsplit, sw[0], sw[1], sw[2]);
      long long cy[64];
      cudaMemcpyFromSymbol(cy, g_jacobi_cyc, sizeof(cy));
      for (int i = 0; i < sw[0] && i < 64; ++i) fprintf(stderr, "  sweep %d: %lld cycles\n", i, cy[i]);
    }
  } else {
    // A does not fit one CTA: the cluster kernel (columns of A and V spread
    // over the cluster), else the global-memory fallback.
    static const bool legacy = getenv("DMCG_JACOBI_LEGACY") != nullptr;
    static const bool cols = getenv("DMCG_JACOBI_COLS") != nullptr;  // the rotation-step cluster kernel
    if (!legacy && !cols && m <= kJbNblk * kJbMaxBw) {
      const int bw = kJbMaxBw;  // zero padded to 256 (padding never rotates)
      const int mb2 = kJbNblk * bw;
      const size_t smem =
          ((size_t)4 * bw * (mb2 + 1) + (size_t)kJbCs * kJbMaxS * (kJbMaxS + 1)) * sizeof(double);
      const void* fn = (const void*)k_jacobi_blk;
      if (smem <= smem_room(fn) && set_smem_attr(fn, smem) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kJbCs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(nbatch * kJbCs);
        cfg.blockDim = dim3(kJbThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        // V accumulates in work (nbatch x mb2 x mb2 doubles: the caller's
        // jacobi scratch holds 2 m2 (m2 + 1) per batch)
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_jacobi_blk, m, A, work, V, w, flags);
        static const bool dbg = getenv("DMCG_DEBUG") != nullptr;
        if (dbg && e == cudaSuccess) {
          int sw[8] = {};
          cudaStreamSynchronize(s);
          cudaMemcpyFromSymbol(sw, g_jacobi_sweeps, sizeof(sw));
          fprintf(stderr, "dmcg: k_jacobi_blk m=%d bw %d sweeps %d %d %d\n", m, bw, sw[0], sw[1], sw[2]);
          long long pr[8];
          cudaMemcpyFromSymbol(pr, g_jb_prof, sizeof(pr));
          fprintf(stderr, "  blk prof (cycles, cumulative): inner %lld bar1 %lld 2a %lld 2b %lld bar2 %lld pull %lld\n",
                  pr[0], pr[1], pr[2], pr[3], pr[4], pr[5]);
        }
        return e;
      }
      cudaGetLastError();
    }
    const int h = m2 / 2;
    int cs = 0;
    for (int c = 8; c >= 2 && !legacy; c /= 2)
      if (h % c == 0 && h / c >= 2 && h / c <= kJcMaxP && h <= kJcMaxH) {
        cs = c;
        break;
      }
    if (cs > 0) {
      const size_t smem = (size_t)(2 * (h / cs) + 2) * 2 * m2 * sizeof(double);
      const void* fn = (const void*)k_jacobi_cluster;
      if (smem <= smem_room(fn) && set_smem_attr(fn, smem) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(nbatch * cs);
        cfg.blockDim = dim3(kJcThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_jacobi_cluster, m, A, V, w, flags);
        static const bool dbg = getenv("DMCG_DEBUG") != nullptr;
        if (dbg && e == cudaSuccess) {
          int sw[8] = {};
          cudaStreamSynchronize(s);
          cudaMemcpyFromSymbol(sw, g_jacobi_sweeps, sizeof(sw));
          fprintf(stderr, "dmcg: k_jacobi_cluster m=%d cluster %d sweeps %d %d %d\n", m, cs, sw[0],
                  sw[1], sw[2]);
        }
        return e;
      }
      cudaGetLastError();
    }
    k_jacobi<<<dim3(nbatch, 1), kJacThreads, 0, s>>>(m, A, work, V, w, flags, 0, m2);
  }
  return cudaGetLastError();
}

// CTAs per axis for the distributed R Q (a portable cluster size).
constexpr int kOiCluster = 8;

template <bool SMEM, int MAXR>
static cudaError_t oi_launch(cudaStream_t s, int nbatch, size_t smem, int F, int k, int rounds,
                             const double* R, const double* start, double* Q, double* H,
                             double* work, double* scr, size_t ss, int in_smem) {
  const void* fn = (const void*)k_oi_fused<SMEM, MAXR>;
  cudaError_t e = set_smem_attr(fn, smem);
  if (e != cudaSuccess) return e;
  static const int cs_env = getenv("DMCG_OI_CLUSTER") ? atoi(getenv("DMCG_OI_CLUSTER")) : 0;
  int cs = cs_env >= 1 && cs_env <= 8 ? cs_env : kOiCluster;  // override for tests
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(nbatch * cs);
  cfg.blockDim = dim3(kOiThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cs == 1 ||
      cudaOccupancyMaxActiveClusters(&nclusters, k_oi_fused<SMEM, MAXR>, &cfg) != cudaSuccess ||
      nclusters < 1) {
    cudaGetLastError();
    cs = 1;  // no room for a cluster of this size: one CTA per axis
  }
  static const bool dbg = getenv("DMCG_DEBUG") != nullptr;
  if (dbg) fprintf(stderr, "dmcg: k_oi_fused F=%d k=%d cluster %d (max active clusters %d)\n", F, k, cs, nclusters);
  if (cs == 1) {
    k_oi_fused<SMEM, MAXR><<<nbatch, kOiThreads, smem, s>>>(F, k, rounds, R, start, Q, H, work,
                                                            scr, ss, in_smem, 1);
    return cudaGetLastError();
  }
  e = cudaLaunchKernelEx(&cfg, k_oi_fused<SMEM, MAXR>, F, k, rounds, R, start, Q, H, work, scr,
                         ss, in_smem, cs);
  if (dbg && e == cudaSuccess) {
    long long h[256];
    cudaStreamSynchronize(s);
    (void)0;
    cudaMemcpyFromSymbol(h, g_oi_prof, sizeof(h));
    for (int c = 0; c < nbatch * cs && c < 32; c += 1)
      fprintf(stderr, "  cta %d: rq %lld factor %lld form %lld | publish %lld sync %lld copy %lld tasks %lld\n",
              c, h[4 * c], h[4 * c + 1], h[4 * c + 2], h[128 + 4 * c], h[129 + 4 * c], h[130 + 4 * c],
              h[131 + 4 * c]);
  }
  return e;
}

template <int MAXR>
static cudaError_t oi_fused_impl(cudaStream_t s, int nbatch, int F, int k, int rounds,
                                 const double* R, const double* start, double* Q, double* H,
                                 double* work, double* scr) {
  const size_t pair = (size_t)2 * odd_ld(F) * k * sizeof(double);
  const size_t sbytes = qr_scratch(k, k) * sizeof(double);
  const size_t ss = qr_scratch_doubles(F, k);
  if (pair <= smem_room((const void*)k_oi_fused<true, MAXR>)) {
    const int in_smem = pair + sbytes <= smem_room((const void*)k_oi_fused<true, MAXR>);
    return oi_launch<true, MAXR>(s, nbatch, pair + (in_smem ? sbytes : 0), F, k, rounds, R, start,
                                 Q, H, work, scr, ss, in_smem);
  }
  const int in_smem = sbytes <= smem_room((const void*)k_oi_fused<false, MAXR>);
  return oi_launch<false, MAXR>(s, nbatch, in_smem ? sbytes : 0, F, k, rounds, R, start, Q, H,
                                work, scr, ss, in_smem);
}

// Column-distributed OI (k_oi_cluster): B columns per CTA, cs = ceil(k / B)
// CTAs per axis in one cluster (up to 16, the non-portable maximum).
template <int MAXR, int B>
static cudaError_t oi_cluster_launch(cudaStream_t s, int nbatch, int F, int k, int rounds,
                                     const double* R, const double* start, double* Q, double* H,
                                     double* mirror, bool* launched, long start_bs = 0,
                                     double* complete_out = nullptr) {
  *launched = false;
  const int cs = (k + B - 1) / B;
  constexpr int PW = QrPanel<MAXR>::PW;
  const size_t smem =
      ((size_t)3 * odd_ld(F) * B + B * B + (B > PW ? qr_scratch(B, B) : 0)) * sizeof(double);
  const void* fn = (const void*)k_oi_cluster<MAXR, B>;
  if (smem > smem_room(fn)) return cudaSuccess;
  cudaError_t e = set_smem_attr(fn, smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cudaSuccess;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(nbatch * cs);
  cfg.blockDim = dim3(kOiThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, k_oi_cluster<MAXR, B>, &cfg) != cudaSuccess ||
      nclusters < 1) {
    cudaGetLastError();
    return cudaSuccess;
  }
  {
    // DMCG_OI_PANELS=blocked (experiments, tests): stream-ordered, so it is
    // also legal inside a graph capture of the plan stream
    static const int blocked = [] {
      const char* e = getenv("DMCG_OI_PANELS");
      return (e && std::string(e) == "blocked") ? 1 : 0;
    }();
    if (blocked) {
      cudaError_t e = cudaMemcpyToSymbolAsync(c_oi_blocked, &blocked, sizeof(blocked), 0,
                                              cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return e;
    }
  }
  static const bool dbg = getenv("DMCG_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr, "dmcg: k_oi_cluster F=%d k=%d B=%d cluster %d smem %zu (max active %d)\n", F,
            k, B, cs, smem, nclusters);
  e = cudaLaunchKernelEx(&cfg, k_oi_cluster<MAXR, B>, F, k, rounds, R, start, Q, H, mirror,
                         start_bs, complete_out);
  *launched = e == cudaSuccess;
  if (dbg && e == cudaSuccess) {
    long long h[64 * 8];
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(h, g_oic_prof, sizeof(h));
    for (int c = 0; c < cs && c < 64; ++c) {
      if (c == 0) {
        long long pp[8];
        cudaMemcpyFromSymbol(pp, g_pan_prof, sizeof(pp));
        fprintf(stderr, "  warp_panel_qr (cta 32): load %lld columns %lld store %lld\n", pp[1], pp[2],
                pp[4]);
      }
      fprintf(stderr, "  cta %d: wait %lld apply %lld factor %lld form %lld sync %lld rq %lld\n", c,
              h[8 * c], h[8 * c + 1], h[8 * c + 2], h[8 * c + 3], h[8 * c + 4], h[8 * c + 5]);
    }
  }
  return e;
}

template <int MAXR>
static cudaError_t oi_cluster_dispatch(cudaStream_t s, int nbatch, int F, int k, int rounds,
                                       const double* R, const double* start, double* Q, double* H,
                                       double* mirror, bool* launched, long start_bs = 0,
                                       double* complete_out = nullptr) {
  *launched = false;
  if (k <= 0 || k >= F) return cudaSuccess;
  static const int bsel = getenv("DMCG_OI_B") ? atoi(getenv("DMCG_OI_B")) : 0;  // experiments
  if (bsel == 16 && (k + 15) / 16 <= 16)
    return oi_cluster_launch<MAXR, 16>(s, nbatch, F, k, rounds, R, start, Q, H, mirror, launched,
                                       start_bs, complete_out);
  if ((k + 7) / 8 <= 16)
    return oi_cluster_launch<MAXR, 8>(s, nbatch, F, k, rounds, R, start, Q, H, mirror, launched,
                                      start_bs, complete_out);
  if ((k + 15) / 16 <= 16)
    return oi_cluster_launch<MAXR, 16>(s, nbatch, F, k, rounds, R, start, Q, H, mirror, launched,
                                       start_bs, complete_out);
  return cudaSuccess;
}

size_t oi_mirror_doubles(int F, int nbatch) {
  return (size_t)nbatch * 16 * oi_mirror_stride(odd_ld(F), 16);
}

cudaError_t launch_qr_cluster(cudaStream_t s, int nbatch, int F, int k, const double* Z,
                              double* Q, double* mirror) {
  if (F > 512 || k <= 0 || k >= F) return cudaErrorInvalidValue;
  bool done = false;
  cudaError_t e = cudaSuccess;
  if (F <= 64) e = oi_cluster_dispatch<2>(s, nbatch, F, k, 0, nullptr, Z, Q, nullptr, mirror, &done);
  else if (F <= 128) e = oi_cluster_dispatch<4>(s, nbatch, F, k, 0, nullptr, Z, Q, nullptr, mirror, &done);
  else if (F <= 256) e = oi_cluster_dispatch<8>(s, nbatch, F, k, 0, nullptr, Z, Q, nullptr, mirror, &done);
  else e = oi_cluster_dispatch<16>(s, nbatch, F, k, 0, nullptr, Z, Q, nullptr, mirror, &done);
  if (e == cudaSuccess && !done) e = cudaErrorNotSupported;  // no cluster of this size fits
  return e;
}

cudaError_t launch_oi_fused(cudaStream_t s, int nbatch, int F, int k, int rounds, const double* R,
                            const double* start, double* Q, double* H, double* work, double* scr,
                            double* mirror) {
  if (F > 512) return cudaErrorInvalidValue;
  static const bool legacy = getenv("DMCG_OI_LEGACY") != nullptr;
  if (!legacy) {
    bool done = false;
    cudaError_t e = cudaSuccess;
    if (F <= 64) e = oi_cluster_dispatch<2>(s, nbatch, F, k, rounds, R, start, Q, H, mirror, &done);
    else if (F <= 128) e = oi_cluster_dispatch<4>(s, nbatch, F, k, rounds, R, start, Q, H, mirror, &done);
    else if (F <= 256) e = oi_cluster_dispatch<8>(s, nbatch, F, k, rounds, R, start, Q, H, mirror, &done);
    else e = oi_cluster_dispatch<16>(s, nbatch, F, k, rounds, R, start, Q, H, mirror, &done);
    if (e != cudaSuccess || done) return e;
  }
  if (F <= 64) return oi_fused_impl<2>(s, nbatch, F, k, rounds, R, start, Q, H, work, scr);
  if (F <= 128) return oi_fused_impl<4>(s, nbatch, F, k, rounds, R, start, Q, H, work, scr);
  if (F <= 256) return oi_fused_impl<8>(s, nbatch, F, k, rounds, R, start, Q, H, work, scr);
  return oi_fused_impl<16>(s, nbatch, F, k, rounds, R, start, Q, H, work, scr);
}

template <int MAXR>
static cudaError_t complete_impl(cudaStream_t s, int nbatch, int F, int k, double* U, double* work,
                                 double* scr) {
  const size_t zb = (size_t)odd_ld(F) * k * sizeof(double);
  const size_t sbytes = qr_scratch(k > F - k ? k : F - k, k) * sizeof(double);
  const size_t ss = qr_scratch_doubles(F, k);
  if (zb <= smem_room((const void*)k_complete<true, MAXR>)) {
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
                            double* scr, double* mirror) {
  if (F > 512) return cudaErrorInvalidValue;
  // the OI's cluster (one per axis) factors U_k and forms the completion
  // blocks on all its CTAs; k_complete (one CTA per axis) is the fallback
  static const bool single = getenv("DMCG_COMPLETE_SINGLE") != nullptr;  // tests
  if (mirror && !single && k > 0 && k < F) {
    bool done = false;
    const long FF = (long)F * F;
    cudaError_t e = cudaSuccess;
    if (F <= 64) e = oi_cluster_dispatch<2>(s, nbatch, F, k, 0, nullptr, U, nullptr, nullptr, mirror, &done, FF, U);
    else if (F <= 128) e = oi_cluster_dispatch<4>(s, nbatch, F, k, 0, nullptr, U, nullptr, nullptr, mirror, &done, FF, U);
    else if (F <= 256) e = oi_cluster_dispatch<8>(s, nbatch, F, k, 0, nullptr, U, nullptr, nullptr, mirror, &done, FF, U);
    else e = oi_cluster_dispatch<16>(s, nbatch, F, k, 0, nullptr, U, nullptr, nullptr, mirror, &done, FF, U);
    if (e != cudaSuccess || done) return e;
  }
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
