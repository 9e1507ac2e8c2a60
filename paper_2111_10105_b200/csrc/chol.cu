// K7 (direct) — supernodal multifrontal Cholesky of M = L^T L + S^T S and the
// multi-RHS solve, level by level over the supernodal elimination tree.
//
// Per level (leaves first):
//   assemble  one CTA per front: zero, scatter M, extend-add children
//   panel     one CTA per front: unblocked Cholesky of a 32-column panel
//   trailing  grouped DMMA tiles (64x64, K = 32) over every front's
//             lower-triangular trailing block  (C -= P P^T)
//   inverse   one CTA per front: L11^{-1} (row-major) so the solves are GEMMs
// Solves (forward L y = P b leaves-first, backward L^T x = y roots-first)
// are grouped DMMA GEMMs per level over (front, 64-row tile, 64-column tile).
// Reference semantics: SimplicialLDLT factor + solve + one refinement pass
// (src/solver.cpp:43-58, 82-90); the refinement is done by the caller.
#include <atomic>
#include <cfloat>

#include "chol_dev.h"

#include <cstdio>
#include <cstdlib>
#include <vector>
#include "gemm.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace dmcg {

namespace {

__device__ __forceinline__ uint32_t front_m(const CholDev& d, uint32_t s) {
  return (uint32_t)(d.str_ptr[s + 1] - d.str_ptr[s]);
}
__device__ __forceinline__ uint32_t front_w(const CholDev& d, uint32_t s) {
  return d.first[s + 1] - d.first[s];
}

// Assembly, parallel over 32-column chunks of each front: zero the chunk,
// scatter M's entries, then extend-add every child's update columns that
// land in the chunk (children in order, so the sum order is deterministic).
constexpr int kAsmCols = 32;

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_assemble(CholDev d, const uint32_t* lsup) {
  const uint32_t s = lsup[blockIdx.y];
  const uint32_t m = front_m(d, s);
  const uint32_t cc0 = blockIdx.x * kAsmCols;
  if (cc0 >= m) return;
  const uint32_t cc1 = min(m, cc0 + kAsmCols);
  double* A = d.F + d.front_off[s];
  for (long t = threadIdx.x; t < (long)(cc1 - cc0) * m; t += blockDim.x)
    A[(size_t)cc0 * m + t] = 0.0;
  __syncthreads();
  {
    const uint32_t* pos = d.a_pos + d.a_ptr[s];
    const uint32_t na = (uint32_t)(d.a_ptr[s + 1] - d.a_ptr[s]);
    const uint32_t e0 = lower_bound_u32(pos, na, cc0 * m);
    const uint32_t e1 = lower_bound_u32(pos, na, cc1 * m);
    for (uint32_t e = e0 + threadIdx.x; e < e1; e += blockDim.x)
      A[pos[e]] = (double)d.a_val[d.a_ptr[s] + e];
  }
  __syncthreads();
  for (uint32_t q = d.child_ptr[s]; q < d.child_ptr[s + 1]; ++q) {
    const uint32_t c = d.child_idx[q];
    const uint32_t mc = front_m(d, c), wc = front_w(d, c), uc = mc - wc;
    const double* C = d.F + d.front_off[c];
    const uint32_t* rel = d.rel_idx + d.rel_ptr[c];
    const uint32_t b0 = lower_bound_u32(rel, uc, cc0);
    const uint32_t b1 = lower_bound_u32(rel, uc, cc1);
    // (b, a) over columns b in [b0, b1) x rows a in [b, uc): eight updates
    // per thread are loaded before any is stored (distinct targets)
    const uint32_t nb = b1 - b0;
    const long tot = (long)nb * uc;
    for (long t0 = threadIdx.x; t0 < tot; t0 += 8L * blockDim.x) {
      double sv[8], dv[8];
      double* dp[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long t = t0 + (long)u * blockDim.x;
        const uint32_t b = b0 + (uint32_t)(t / uc), a = (uint32_t)(t % uc);
        const bool ok = t < tot && a >= b;
        dp[u] = ok ? A + (size_t)rel[b] * m + rel[a] : nullptr;
        sv[u] = ok ? C[(size_t)(wc + b) * mc + wc + a] : 0.0;
        dv[u] = ok ? *dp[u] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (dp[u]) *dp[u] = dv[u] + sv[u];
    }
    __syncthreads();
  }
}

// Panel [k0, k0 + pw) of a front: warp 0 factors the pw x pw diagonal block
// in registers (left-looking, lane = row, shuffles instead of barriers),
// then every thread solves rows of the panel below against it (row-wise
// TRSM).  The rows below are split over a cluster of up to 8 CTAs per front
// (grid.y); each refactors the small block, and one cluster barrier keeps
// rank 0's write-back after every rank's read.  Pivots are applied as reciprocal square roots (the CPU
// reference divides by the square root; results agree to rounding).
constexpr int kPanelThreads = 256;  // 32 panel values per thread stay in registers
constexpr int kNB = 32;

__global__ void __launch_bounds__(kPanelThreads)
    k_panel(CholDev d, const uint32_t* lsup, int k0, int nb) {
  __shared__ double D[kNB][kNB + 1];
  __shared__ double dinv[kNB];
  const uint32_t s = lsup[blockIdx.x];
  const int w = (int)front_w(d, s), m = (int)front_m(d, s);
  if (k0 >= w) return;
  const int pw = min(nb, w - k0);
  double* A = d.F + d.front_off[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  cg::cluster_group cl = cg::this_cluster();
  const int ny = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  if (warp == 0) {
    // Right-looking Cholesky of the kNB x kNB diagonal block in registers,
    // redundantly in every CTA of the cluster: lane r holds row r; pivot j's
    // column is broadcast by independent shuffles (no barrier, no chain).
    double a[kNB];
#pragma unroll
    for (int c = 0; c < kNB; ++c)
      a[c] = (lane < pw && c < pw && c <= lane) ? A[(size_t)(k0 + c) * m + k0 + lane] : 0.0;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < kNB; ++j) {
      const double djj = __shfl_sync(0xffffffffu, a[j], j);
      const double ip = rsqrt(fmax(djj, DBL_MIN));
      if (j < pw && !(djj > 0.0)) bad = true;
      const double lj = lane > j ? a[j] * ip : (lane == j ? djj * ip : 0.0);
      a[j] = lj;
      if (lane == 0 && j < pw) dinv[j] = ip;
#pragma unroll
      for (int c = j + 1; c < kNB; ++c) a[c] = fma(-lj, __shfl_sync(0xffffffffu, lj, c), a[c]);
    }
    if (bad && lane == 0 && rank == 0) atomicOr(d.flags, 1);
#pragma unroll
    for (int c = 0; c < kNB; ++c) D[lane][c] = c <= lane ? a[c] : 0.0;
    if (ny > 1) {
      // every CTA of the cluster has read the block before rank 0 rewrites it
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    if (rank == 0 && lane < pw)
#pragma unroll
      for (int c = 0; c < kNB; ++c)
        if (c < pw && c <= lane) A[(size_t)(k0 + c) * m + k0 + lane] = a[c];
  } else if (ny > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  __syncthreads();
  // rows below: x = a L^{-T}; column-oriented substitution so the updates
  // of one pivot are independent (ILP) instead of one long FMA chain.
  for (int i = k0 + pw + rank * kPanelThreads + threadIdx.x; i < m; i += ny * kPanelThreads) {
    double x[kNB];
#pragma unroll
    for (int c = 0; c < kNB; ++c) x[c] = c < pw ? A[(size_t)(k0 + c) * m + i] : 0.0;
#pragma unroll
    for (int j = 0; j < kNB; ++j) {
      if (j < pw) {
        x[j] *= dinv[j];
#pragma unroll
        for (int c = j + 1; c < kNB; ++c) x[c] -= x[j] * D[c][j];
      }
    }
#pragma unroll
    for (int c = 0; c < kNB; ++c)
      if (c < pw) A[(size_t)(k0 + c) * m + i] = x[c];
  }
}

// Trailing update of each front in the level: A22 -= P P^T (lower tiles).
struct LoadPanel {
  static constexpr bool kKContig = false;
  const double* A;
  int m, k0, off;
  __device__ __forceinline__ double operator()(int, int k, int i) const {
    return A[(size_t)(k0 + k) * m + off + i];
  }
  __device__ __forceinline__ const double* addr(int, int k, int i) const {
    return A + (size_t)(k0 + k) * m + off + i;
  }
};
// Epilogues that read the destination load every target first and store
// afterwards: a load -> subtract -> store loop on one pointer issues in
// order and would wait one L2 round trip per element (the compiler cannot
// hoist the next load above a possibly aliasing store).
struct SubLower {
  double* A;
  int m, off;
  __device__ __forceinline__ void operator()(int, int, int mb, int nb, int lane, int M, int N,
                                             const WarpTile& wt) const {
    double v[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, c;
          frag_rc(i, j, e, lane, &r, &c);
          const int mi = mb + r, ni = nb + c;
          v[i][j][e] = (mi < M && ni < N && mi >= ni) ? A[(size_t)(off + ni) * m + off + mi] : 0.0;
        }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, c;
          frag_rc(i, j, e, lane, &r, &c);
          const int mi = mb + r, ni = nb + c;
          if (mi < M && ni < N && mi >= ni)
            A[(size_t)(off + ni) * m + off + mi] = v[i][j][e] - wt.acc[i][j][e];
        }
  }
};

__global__ void __launch_bounds__(kGemmThreads)
    k_trailing(CholDev d, const uint32_t* lsup, int k0, int nb) {
  const uint32_t s = lsup[blockIdx.y];
  const int w = (int)front_w(d, s), m = (int)front_m(d, s);
  if (k0 >= w) return;
  const int pw = min(nb, w - k0);
  const int off = k0 + pw, T = m - off;
  if (T <= 0) return;
  const int nt = (T + kBM - 1) / kBM;
  const int t = blockIdx.x;
  if (t >= nt * (nt + 1) / 2) return;
  int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  const int tj = t - ti * (ti + 1) / 2;
  double* A = d.F + d.front_off[s];
  LoadPanel lp{A, m, k0, off};
  gemm_tile(0, T, T, ti * kBM, tj * kBN, 0, pw, 0, lp, lp, SubLower{A, m, off});
}

// V = L11^{-1} (row-major w x w) in 64-blocks.  Step 1: invert every
// diagonal 64x64 block (one CTA per block, one thread per column, in smem).
constexpr int kIB = 64;

constexpr size_t kInvDiagSmem = 2 * kIB * (kIB + 1) * sizeof(double);

__global__ void __launch_bounds__(kIB) k_inv_diag(CholDev d, const uint32_t* lsup) {
  extern __shared__ double inv_smem[];
  double(*Ls)[kIB + 1] = reinterpret_cast<double(*)[kIB + 1]>(inv_smem);
  double(*Xs)[kIB + 1] = reinterpret_cast<double(*)[kIB + 1]>(inv_smem + kIB * (kIB + 1));
  const uint32_t s = lsup[blockIdx.y];
  const int w = (int)front_w(d, s), m = (int)front_m(d, s);
  const int b0 = blockIdx.x * kIB;
  if (b0 >= w) return;
  const int bs = min(kIB, w - b0);
  const double* A = d.F + d.front_off[s];
  double* V = d.Linv + d.inv_off[s];
  const int c = threadIdx.x;
  __shared__ double rdiag[kIB];
  // thread = row, 16 column loads in flight (column-major front)
  for (int c8 = 0; c8 < kIB; c8 += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int cc = c8 + u;
      v[u] = (c < bs && cc < bs && cc <= c) ? A[(size_t)(b0 + cc) * m + b0 + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) Ls[c][c8 + u] = v[u];
  }
  __syncthreads();
  if (c < bs) rdiag[c] = 1.0 / Ls[c][c];
  __syncthreads();
  if (c < bs) {
    for (int r = 0; r < bs; ++r) {
      if (r < c) {
        Xs[r][c] = 0.0;
        continue;
      }
      // two partial sums so the chain over k is half as long
      double a0 = (r == c) ? 1.0 : 0.0, a1 = 0.0;
      int k = c;
      for (; k + 1 < r; k += 2) {
        a0 -= Ls[r][k] * Xs[k][c];
        a1 -= Ls[r][k + 1] * Xs[k + 1][c];
      }
      if (k < r) a0 -= Ls[r][k] * Xs[k][c];
      Xs[r][c] = (a0 + a1) * rdiag[r];
    }
  }
  __syncthreads();
  for (int r = 0; r < bs; ++r)
    if (c < bs) V[(size_t)(b0 + r) * w + b0 + c] = Xs[r][c];
}

// Step 2: one CTA per block column J walks the row blocks i > J in order:
//   T = sum_{k = J..i-1} L(i, k) X(k, J)      (DMMA, K = 64 (i - J))
//   X(i, J) = -X(i, i) T                       (DMMA, K = 64)
struct LoadLinvRM {  // X(k, c) = V[(r0 + k) * w + c0 + c]
  static constexpr bool kKContig = false;
  const double* V;
  int w, r0, c0;
  __device__ __forceinline__ double operator()(int, int k, int c) const {
    return V[(size_t)(r0 + k) * w + c0 + c];
  }
  __device__ __forceinline__ const double* addr(int, int k, int c) const {
    return V + (size_t)(r0 + k) * w + c0 + c;
  }
};
struct LoadLinvRowsK {  // X(k, r) = V[(r0 + r) * w + c0 + k]   (k contiguous)
  static constexpr bool kKContig = true;
  const double* V;
  int w, r0, c0;
  __device__ __forceinline__ double operator()(int, int k, int r) const {
    return V[(size_t)(r0 + r) * w + c0 + k];
  }
  __device__ __forceinline__ const double* addr(int, int k, int r) const {
    return V + (size_t)(r0 + r) * w + c0 + k;
  }
};
struct LoadFrontCM {  // X(k, r) = A[(c0 + k) * m + r0 + r]
  static constexpr bool kKContig = false;
  const double* A;
  int m, r0, c0;
  __device__ __forceinline__ double operator()(int, int k, int r) const {
    return A[(size_t)(c0 + k) * m + r0 + r];
  }
  __device__ __forceinline__ const double* addr(int, int k, int r) const {
    return A + (size_t)(c0 + k) * m + r0 + r;
  }
};
struct LoadColMajorT {  // X(k, i) = p[k * ld + i]
  static constexpr bool kKContig = false;
  const double* p;
  int ld;
  __device__ __forceinline__ double operator()(int, int k, int i) const {
    return p[(size_t)k * ld + i];
  }
  __device__ __forceinline__ const double* addr(int, int k, int i) const {
    return p + (size_t)k * ld + i;
  }
};
struct StoreTile {  // out[r * ld + c] = sign * v
  double* out;
  int ld;
  double sign;
  __device__ __forceinline__ void operator()(int, int, int mb, int nb, int lane, int M, int N,
                                             const WarpTile& wt) const {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, c;
          frag_rc(i, j, e, lane, &r, &c);
          const int mi = mb + r, ni = nb + c;
          if (mi < M && ni < N) out[(size_t)mi * ld + ni] = sign * wt.acc[i][j][e];
        }
  }
};

__global__ void __launch_bounds__(kGemmThreads) k_inv_offdiag(CholDev d, const uint32_t* lsup,
                                                              double* scratch) {
  const uint32_t s = lsup[blockIdx.y];
  const int w = (int)front_w(d, s), m = (int)front_m(d, s);
  const int J = blockIdx.x, c0 = J * kIB;
  if (c0 >= w) return;
  const int cw = min(kIB, w - c0);
  const double* A = d.F + d.front_off[s];
  double* V = d.Linv + d.inv_off[s];
  double* T = scratch + ((size_t)blockIdx.y * gridDim.x + J) * kIB * kIB;
  for (int r0 = c0 + kIB; r0 < w; r0 += kIB) {
    const int rh = min(kIB, w - r0);
    // T(rh x cw) = L(r0.., c0..r0) X(c0..r0, c0..)
    gemm_tile(0, rh, cw, 0, 0, 0, r0 - c0, 0, LoadFrontCM{A, m, r0, c0},
              LoadLinvRM{V, w, c0, c0}, StoreTile{T, kIB, 1.0});
    __syncthreads();
    // X(r0.., c0..) = -X(r0.., r0..) T
    gemm_tile(0, rh, cw, 0, 0, 0, rh, 0, LoadLinvRowsK{V, w, r0, r0},
              LoadColMajorT{T, kIB}, StoreTile{V + (size_t)r0 * w + c0, w, -1.0});
    __syncthreads();
  }
}

// ---- solve operator -----------------------------------------------------
// P_s = [L11^{-1}; -L21 L11^{-1}] (m x w, column-major, ld = m).  With it one
// supernode's forward step is ONE product and its backward step another:
//   forward   [y_s; U_s] = P_s r_s + [0; pulled child updates]
//             (y_s = L11^{-1} r_s,  U_s = R_s[w:m] - L21 y_s)
//   backward  x_s = P_s^T [y_s; x_below]
//             (= L11^{-T} (y_s - L21^T x_below))
// so no per-front right-hand-side panel is materialised: r_s (own rows) is
// gathered into the x buffer, U_s is written once by the forward epilogue
// and read once by the parent.

// Top block: P[j m + i] = Linv[i w + j] (lower triangle, zeros above).
__global__ void __launch_bounds__(256) k_form_p_top(CholDev d, const uint32_t* lsup) {
  const uint32_t s = lsup[blockIdx.y];
  const int w = (int)front_w(d, s), m = (int)front_m(d, s);
  const double* V = d.Linv + d.inv_off[s];
  double* P = d.P + d.op_off[s];
  // one 32 x 32 tile per CTA through shared memory (coalesced both ways)
  __shared__ double t[32][33];
  const int tiles = (w + 31) / 32;
  for (int tt = blockIdx.x; tt < tiles * tiles; tt += gridDim.x) {
    const int ti = tt / tiles, tj = tt % tiles;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = ty; r < 32; r += 8) {
      const int i = ti * 32 + r, j = tj * 32 + tx;
      t[r][tx] = (i < w && j < w) ? V[(size_t)i * w + j] : 0.0;
    }
    __syncthreads();
    for (int c = ty; c < 32; c += 8) {
      const int j = tj * 32 + c, i = ti * 32 + tx;
      if (i < w && j < w) P[(size_t)j * m + i] = t[tx][c];
    }
    __syncthreads();
  }
}

struct StoreNegCM {  // P[(n) * ld + off + m] = -v
  double* P;
  int ld, off;
  __device__ __forceinline__ void operator()(int, int, int mb, int nb, int lane, int M, int N,
                                             const WarpTile& wt) const {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, c;
          frag_rc(i, j, e, lane, &r, &c);
          const int mi = mb + r, ni = nb + c;
          if (mi < M && ni < N) P[(size_t)ni * ld + off + mi] = -wt.acc[i][j][e];
        }
  }
};

// Bottom block: P[j m + w + i] = -(L21 L11^{-1})(i, j), K restricted to
// k >= j0 (L11^{-1} is lower triangular).
__global__ void __launch_bounds__(kGemmThreads) k_form_p_bot(CholDev d, const uint32_t* lsup,
                                                             int tiles_w) {
  const uint32_t s = lsup[blockIdx.y];
  const int w = (int)front_w(d, s), m = (int)front_m(d, s), u = m - w;
  const int ti = blockIdx.x / tiles_w, tj = blockIdx.x % tiles_w;
  if (ti * kBM >= u || tj * kBN >= w) return;
  const double* A = d.F + d.front_off[s];
  const double* V = d.Linv + d.inv_off[s];
  gemm_tile(0, u, w, ti * kBM, tj * kBN, tj * kBN, w, 0, LoadColMajorT{A + w, m},
            LoadColMajorT{V, w}, StoreNegCM{d.P + d.op_off[s], m, w});
}

// ---- solves -------------------------------------------------------------

// r_s (own rows of front s) = b(perm) + the children's update rows pulled
// into them (CholPlan::pull_*: children in a fixed order, deterministic),
// written to rows first[s] .. of the permuted buffer r.
__global__ void __launch_bounds__(256) k_gather_own(CholDev d, const uint32_t* lsup,
                                                    const double* __restrict__ b,
                                                    double* __restrict__ r) {
  const uint32_t s = lsup[blockIdx.z];
  const int W = (int)d.W;
  const int c0 = blockIdx.y * 128;
  const uint32_t w = front_w(d, s), f0 = d.first[s];
  const uint32_t r0 = blockIdx.x * 8;
  if (r0 >= w) return;
  const uint32_t r1 = min(w, r0 + 8);
  const unsigned long long g0 = d.rhs_off[s];
  const double* __restrict__ R = d.R;
  for (uint32_t rr = r0 + (threadIdx.x >> 5); rr < r1; rr += 8) {
    const size_t g = g0 + rr;
    const uint32_t e0 = d.pull_ptr[g], e1 = d.pull_ptr[g + 1];
    const double* brow = b + (size_t)d.perm[f0 + rr] * W;
    double* out = r + (size_t)(f0 + rr) * W;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + q * 32 + (threadIdx.x & 31);
      if (c < W) {
        double v = brow[c];
        for (uint32_t e = e0; e < e1; ++e) v += R[(size_t)d.pull_src[e] * W + c];
        out[c] = v;
      }
    }
  }
}

struct LoadColMajor {  // X(k, i) = p[k * ld + i]   (i contiguous)
  static constexpr bool kKContig = false;
  const double* p;
  int ld;
  __device__ __forceinline__ double operator()(int, int k, int i) const {
    return p[(size_t)k * ld + i];
  }
  __device__ __forceinline__ const double* addr(int, int k, int i) const {
    return p + (size_t)k * ld + i;
  }
};
struct LoadRowMajor {  // X(k, i) = p[i * ld + k]   (k contiguous)
  static constexpr bool kKContig = true;
  const double* p;
  int ld;
  __device__ __forceinline__ double operator()(int, int k, int i) const {
    return p[(size_t)i * ld + k];
  }
  __device__ __forceinline__ const double* addr(int, int k, int i) const {
    return p + (size_t)i * ld + k;
  }
};
// b(perm[k], c): the own rows of a leaf front straight from the caller's
// right-hand side (leaves have no children to pull from, so r_s = b(own rows)
// and the gather pass is skipped for them)
struct LoadPermRows {
  static constexpr bool kKContig = false;
  const double* b;
  const uint32_t* perm;  // perm + first[s]
  int W;
  __device__ __forceinline__ const double* addr(int, int k, int c) const {
    return b + (size_t)perm[k] * W + c;
  }
};
// [y_s; x_below](k, c): own rows from y, the rows below from x (str_idx lists
// the own columns first, so rows[k] = first[s] + k for k < w)
struct LoadYX {
  static constexpr bool kKContig = false;
  const double* y;
  const double* x;
  const uint32_t* rows;
  int w, W;
  __device__ __forceinline__ double operator()(int, int k, int c) const {
    return (k < w ? y : x)[(size_t)rows[k] * W + c];
  }
  __device__ __forceinline__ const double* addr(int, int k, int c) const {
    return (k < w ? y : x) + (size_t)rows[k] * W + c;
  }
};

// Forward epilogue: rows < w -> y (own rows), rows >= w -> the update rows
// U = pulled child updates + (-L21 L11^{-1} r) in d.R.  All loads of a
// fragment are issued before its stores.
template <bool ROWS>
struct StoreFwd {
  double* y;        // y + first[s] * W
  double* U;        // d.R + rhs_off[s] * W
  const double* R;  // d.R (children's update rows)
  const uint32_t* pull_ptr;  // + rhs_off[s]
  const uint32_t* pull_src;
  int w, W;
  // Row-wise finish over the tile staged in shared memory (gemm.cuh
  // RowEpilogue): warp q of 4 takes the rows q, q + 4, ...; its lanes own CPL
  // consecutive columns each, so y / U rows are written and the children's
  // update rows read in contiguous BN-double pieces.  The pull lists of all
  // of a warp's rows are fetched up front by its lanes (lane l: the l-th row's
  // range and first two sources), so the pull_ptr -> pull_src -> row chain is
  // paid once per warp instead of once per thread and row block.
  static constexpr bool kRowEpilogue = ROWS;  // leaves (no pulls) keep the fragment stores
  template <int BM, int BN>
  __device__ __forceinline__ void rows(int m0, int n0, int M, int N, const double* tile,
                                       int ld) const {
    constexpr int CPL = BN / 32;   // columns per lane (2 or 4)
    constexpr int RPW = BM / 4;    // rows per warp (8 or 16)
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int c = lane * CPL, nc = n0 + c;
    const bool vec = !(W & 1);  // rows 16-byte aligned (nc is even)
    // lane l < RPW: the pull range of the warp's l-th row
    uint32_t pe0 = 0, pe1 = 0, ps0 = 0, ps1 = 0;
    {
      const int mi = m0 + wp + 4 * lane;
      if (lane < RPW && mi < M && mi >= w) {
        pe0 = pull_ptr[mi];
        pe1 = pull_ptr[mi + 1];
        if (pe0 < pe1) ps0 = pull_src[pe0];
        if (pe0 + 1 < pe1) ps1 = pull_src[pe0 + 1];
      }
    }
    auto load_row = [&](const double* src, double (&v)[CPL]) {
      if (vec && nc + CPL <= N) {
#pragma unroll
        for (int q = 0; q < CPL; q += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(src + nc + q);
          v[q] = t2.x;
          v[q + 1] = t2.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < CPL; ++q) v[q] = nc + q < N ? src[nc + q] : 0.0;
      }
    };
    auto store_row = [&](double* dst, const double (&v)[CPL]) {
      if (vec && nc + CPL <= N) {
#pragma unroll
        for (int q = 0; q < CPL; q += 2)
          *reinterpret_cast<double2*>(dst + nc + q) = make_double2(v[q], v[q + 1]);
      } else {
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          if (nc + q < N) dst[nc + q] = v[q];
      }
    };
#pragma unroll 2
    for (int rq = 0; rq < RPW; ++rq) {
      const int r = wp + 4 * rq, mi = m0 + r;
      const uint32_t e0 = __shfl_sync(0xffffffffu, pe0, rq), e1 = __shfl_sync(0xffffffffu, pe1, rq);
      const uint32_t s0 = __shfl_sync(0xffffffffu, ps0, rq), s1 = __shfl_sync(0xffffffffu, ps1, rq);
      if (mi >= M) continue;  // warp-uniform
      double acc[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) acc[q] = tile[r * ld + c + q];
      if (mi < w) {
        store_row(y + (size_t)mi * W, acc);
        continue;
      }
      double v[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) v[q] = 0.0;
      // children in order: ((v + c_e) + c_{e+1}) ..., two rows in flight
      uint32_t e = e0;
      for (; e + 1 < e1; e += 2) {
        double t0[CPL], t1[CPL];
        load_row(R + (size_t)(e == e0 ? s0 : pull_src[e]) * W, t0);
        load_row(R + (size_t)(e == e0 ? s1 : pull_src[e + 1]) * W, t1);
#pragma unroll
        for (int q = 0; q < CPL; ++q) v[q] = (v[q] + t0[q]) + t1[q];
      }
      if (e < e1) {
        double t0[CPL];
        load_row(R + (size_t)(e == e0 ? s0 : pull_src[e]) * W, t0);
#pragma unroll
        for (int q = 0; q < CPL; ++q) v[q] += t0[q];
      }
#pragma unroll
      for (int q = 0; q < CPL; ++q) v[q] += acc[q];
      store_row(U + (size_t)mi * W, v);
    }
  }
  __device__ __forceinline__ void operator()(int, int, int mb, int nb, int lane, int M, int N,
                                             const WarpTile& wt) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int mi = mb + i * 8 + (lane >> 2);
      if (mi >= M) continue;
      if (mi < w) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ni = nb + j * 8 + (lane & 3) * 2;
          if (ni + 1 < N && !(W & 1)) {
            *reinterpret_cast<double2*>(y + (size_t)mi * W + ni) =
                make_double2(wt.acc[i][j][0], wt.acc[i][j][1]);
          } else if (ni < N) {
            y[(size_t)mi * W + ni] = wt.acc[i][j][0];
            if (ni + 1 < N) y[(size_t)mi * W + ni + 1] = wt.acc[i][j][1];
          }
        }
      } else {
        const uint32_t e0 = pull_ptr[mi], e1 = pull_ptr[mi + 1];
        double v[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j][0] = v[j][1] = 0.0;
        // two pulled rows per iteration: all eight loads in flight together
        uint32_t e = e0;
        for (; e + 1 < e1; e += 2) {
          const double* s0 = R + (size_t)pull_src[e] * W;
          const double* s1 = R + (size_t)pull_src[e + 1] * W;
          double2 t0[4], t1[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int ni = nb + j * 8 + (lane & 3) * 2;
            t0[j] = t1[j] = make_double2(0.0, 0.0);
            if (ni + 1 < N && !(W & 1)) {
              t0[j] = *reinterpret_cast<const double2*>(s0 + ni);
              t1[j] = *reinterpret_cast<const double2*>(s1 + ni);
            } else if (ni < N) {
              t0[j].x = s0[ni];
              t1[j].x = s1[ni];
              if (ni + 1 < N) {
                t0[j].y = s0[ni + 1];
                t1[j].y = s1[ni + 1];
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {  // children in order: ((v + c_e) + c_{e+1})
            v[j][0] = (v[j][0] + t0[j].x) + t1[j].x;
            v[j][1] = (v[j][1] + t0[j].y) + t1[j].y;
          }
        }
        if (e < e1) {
          const double* src = R + (size_t)pull_src[e] * W;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int ni = nb + j * 8 + (lane & 3) * 2;
            if (ni + 1 < N && !(W & 1)) {
              const double2 t = *reinterpret_cast<const double2*>(src + ni);
              v[j][0] += t.x;
              v[j][1] += t.y;
            } else if (ni < N) {
              v[j][0] += src[ni];
              if (ni + 1 < N) v[j][1] += src[ni + 1];
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ni = nb + j * 8 + (lane & 3) * 2;
          double* dst = U + (size_t)mi * W + ni;
          if (ni + 1 < N && !(W & 1)) {
            *reinterpret_cast<double2*>(dst) =
                make_double2(v[j][0] + wt.acc[i][j][0], v[j][1] + wt.acc[i][j][1]);
          } else if (ni < N) {
            dst[0] = v[j][0] + wt.acc[i][j][0];
            if (ni + 1 < N) dst[1] = v[j][1] + wt.acc[i][j][1];
          }
        }
      }
    }
  }
};

// Backward epilogue: x (permuted, read by the descendants' backward steps)
// and the caller's output row perm[first + mi] in the original order
// (= or += : the refinement accumulates its correction), replacing a
// separate unpermute pass over n x W.
struct StoreBwd {
  double* x;            // x + first[s] * W; null: leaf fronts (no descendant reads them)
  double* out;          // original-order output (n x W)
  const uint32_t* perm;  // perm + first[s]
  int W, accumulate;
  __device__ __forceinline__ void operator()(int, int, int mb, int nb, int lane, int M, int N,
                                             const WarpTile& wt) const {
    const bool vec = !(W & 1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int mi = mb + i * 8 + (lane >> 2);
      if (mi >= M) continue;
      double* xr = x + (size_t)mi * W;
      double* orow = out + (size_t)perm[mi] * W;
      double prev[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ni = nb + j * 8 + (lane & 3) * 2;
        prev[j][0] = prev[j][1] = 0.0;
        if (accumulate) {
          if (ni + 1 < N && vec) {
            const double2 t = *reinterpret_cast<const double2*>(orow + ni);
            prev[j][0] = t.x;
            prev[j][1] = t.y;
          } else if (ni < N) {
            prev[j][0] = orow[ni];
            if (ni + 1 < N) prev[j][1] = orow[ni + 1];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ni = nb + j * 8 + (lane & 3) * 2;
        const double v0 = wt.acc[i][j][0], v1 = wt.acc[i][j][1];
        if (ni + 1 < N && vec) {
          if (x) *reinterpret_cast<double2*>(xr + ni) = make_double2(v0, v1);
          *reinterpret_cast<double2*>(orow + ni) = make_double2(prev[j][0] + v0, prev[j][1] + v1);
        } else if (ni < N) {
          if (x) xr[ni] = v0;
          orow[ni] = prev[j][0] + v0;
          if (ni + 1 < N) {
            if (x) xr[ni + 1] = v1;
            orow[ni + 1] = prev[j][1] + v1;
          }
        }
      }
    }
  }
};

// Tile shape of the solve GEMMs: 64 x 64 for the levels of wide fronts,
// 32 x 128 (four warps side by side, 32-row granularity) for the levels of
// narrow ones, where most M tiles of a 64-row grid would be half padding
// (c3: 4106 leaf fronts of mean width 33).
// Forward: [y_s; U_s] = P_s r_s (+ pulls), M = m, K = w.
template <int BM, int BN, bool LEAF>
__global__ void __launch_bounds__(kGemmThreads, 4) k_fwd(CholDev d, const uint32_t* lsup,
                                                      const double* r, double* y) {
  const uint32_t s = lsup[blockIdx.z];
  const int w = (int)front_w(d, s), m = (int)front_m(d, s), W = (int)d.W;
  if ((int)blockIdx.x * BM >= m) return;
  const size_t f0 = d.first[s];
  const unsigned long long g0 = d.rhs_off[s];
  // rows i < w of P are L11^{-1} (lower triangular): a tile inside the top
  // block needs k <= i only
  const int m0 = blockIdx.x * BM;
  const int kend = m0 + BM <= w ? m0 + BM : w;
  const StoreFwd<!LEAF> ep{y + f0 * W, d.R + g0 * W, d.R, d.pull_ptr + g0, d.pull_src, w, W};
  if constexpr (LEAF)  // r = the caller's b in the original order
    gemm_tile_async<BM, BN>(0, m, W, m0, blockIdx.y * BN, 0, kend, 0,
                            LoadColMajor{d.P + d.op_off[s], m}, LoadPermRows{r, d.perm + f0, W},
                            ep);
  else
    gemm_tile_async<BM, BN>(0, m, W, m0, blockIdx.y * BN, 0, kend, 0,
                            LoadColMajor{d.P + d.op_off[s], m}, LoadColMajor{r + f0 * W, W}, ep);
}

// Backward: x_s = P_s^T [y_s; x_below], M = w, K = m.
template <int BM, int BN>
__global__ void __launch_bounds__(kGemmThreads, 4) k_bwd(CholDev d, const uint32_t* lsup,
                                                      const double* y, double* x, double* out,
                                                      int accumulate, int leaf) {
  const uint32_t s = lsup[blockIdx.z];
  const int w = (int)front_w(d, s), m = (int)front_m(d, s), W = (int)d.W;
  if ((int)blockIdx.x * BM >= w) return;
  const uint32_t* rows = d.str_idx + d.str_ptr[s];
  // P^T's top block is L11^{-T} (upper triangular): row i needs k >= i
  const int m0 = blockIdx.x * BM;
  gemm_tile_async<BM, BN>(0, w, W, m0, blockIdx.y * BN, m0, m, 0,
                          LoadRowMajor{d.P + d.op_off[s], m}, LoadYX{y, x, rows, w, W},
                          StoreBwd{leaf ? nullptr : x + (size_t)d.first[s] * W, out, d.perm + d.first[s],
                                   W, accumulate});
}

// r = b - M x   (M: CSR with float values, original order, n x W row-major).
// One warp per (row, 256-column chunk): the row's CSR entries are read once
// per warp (lane e holds entry e, broadcast by shuffles), every lane owns
// four column pairs (double2, 512 contiguous bytes per warp access) and two
// entries' loads are in flight per step.
constexpr int kResCols = 256;
__global__ void __launch_bounds__(256) k_residual(int n, int W, const uint32_t* __restrict__ rp,
                                                  const uint32_t* __restrict__ ci,
                                                  const float* __restrict__ val,
                                                  const double* __restrict__ b,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ r) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= n) return;
  const int c0 = blockIdx.y * kResCols;
  const uint32_t pb = rp[i], pe = rp[i + 1];
  const int cnt = (int)(pe - pb);
  const bool vec = !(W & 1);
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
  for (int e0 = 0; e0 < cnt; e0 += 32) {
    const int me = e0 + lane;
    const uint32_t my_c = me < cnt ? ci[pb + me] : 0u;
    const double my_v = me < cnt ? (double)val[pb + me] : 0.0;
    const int ne = min(32, cnt - e0);
    for (int e = 0; e < ne; ++e) {
      const uint32_t col = __shfl_sync(0xffffffffu, my_c, e);
      const double v = __shfl_sync(0xffffffffu, my_v, e);
      const double* xr = x + (size_t)col * W;
      double2 t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + 64 * j + 2 * lane;
        t[j] = make_double2(0.0, 0.0);
        if (c + 1 < W && vec) {
          t[j] = *reinterpret_cast<const double2*>(xr + c);
        } else if (c < W) {
          t[j].x = xr[c];
          if (c + 1 < W) t[j].y = xr[c + 1];
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[j][0] = fma(v, t[j].x, acc[j][0]);
        acc[j][1] = fma(v, t[j].y, acc[j][1]);
      }
    }
  }
  const double* br = b + (size_t)i * W;
  double* rr = r + (size_t)i * W;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = c0 + 64 * j + 2 * lane;
    if (c + 1 < W && vec) {
      const double2 bb = *reinterpret_cast<const double2*>(br + c);
      *reinterpret_cast<double2*>(rr + c) = make_double2(bb.x - acc[j][0], bb.y - acc[j][1]);
    } else if (c < W) {
      rr[c] = br[c] - acc[j][0];
      if (c + 1 < W) rr[c + 1] = br[c + 1] - acc[j][1];
    }
  }
}

}  // namespace

// DMCG_LEVEL_TIMING=1: CUDA events around the phases of every level, printed
// after a stream sync (debugging aid; off by default).
struct LevelTimer {
  cudaStream_t s;
  const char* what;
  bool on;
  std::vector<cudaEvent_t> ev;
  LevelTimer(cudaStream_t st, const char* w, uint32_t nlev) : s(st), what(w) {
    static const bool env = std::getenv("DMCG_LEVEL_TIMING") != nullptr;
    on = env;
    if (on) {
      ev.resize((size_t)nlev * 5);
      for (auto& e : ev) cudaEventCreate(&e);
    }
  }
  void mark(uint32_t l, int k) {
    if (on) cudaEventRecord(ev[(size_t)l * 5 + k], s);
  }
  void report(const CholLevels& lv, const char* a, const char* b, const char* c, bool split = false) {
    if (!on) return;
    cudaStreamSynchronize(s);
    for (uint32_t l = 0; l < lv.nlevels; ++l) {
      float t[3];
      const int a0[3] = {0, 1, split ? 3 : 2}, a1[3] = {1, 2, split ? 4 : 3};
      for (int k = 0; k < 3; ++k) cudaEventElapsedTime(&t[k], ev[l * 5 + a0[k]], ev[l * 5 + a1[k]]);
      std::fprintf(stderr, "  %s level %u: %u fronts, maxw %u maxm %u | %s %.3f %s %.3f %s %.3f ms\n", what,
                   l, lv.count[l], lv.maxw[l], lv.maxm[l], a, t[0], b, t[1], c, t[2]);
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
};

cudaError_t chol_factor_device(cudaStream_t s, const CholDev& d, const CholLevels& lv) {
  const int nb = 32;
  {
    static std::atomic<unsigned long long> attr_set{0};  // one bit per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set.load() & (1ull << dev))) {
      // idempotent: two threads racing here both set the same attribute
      cudaError_t e = cudaFuncSetAttribute(k_inv_diag, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kInvDiagSmem);
      if (e != cudaSuccess) return e;
      attr_set.fetch_or(1ull << dev);
    }
  }
  cudaError_t e = cudaMemsetAsync(d.Linv, 0, d.linv_doubles * sizeof(double), s);
  if (e != cudaSuccess) return e;
  LevelTimer lt(s, "factor", lv.nlevels);
  for (uint32_t l = 0; l < lv.nlevels; ++l) {
    const uint32_t cnt = lv.count[l];
    const uint32_t* ls = d.level_sup + lv.offset[l];
    lt.mark(l, 0);
    k_assemble<<<dim3((lv.maxm[l] + kAsmCols - 1) / kAsmCols, cnt), 256, 0, s>>>(d, ls);
    lt.mark(l, 1);
    static const bool per_launch = std::getenv("DMCG_LEVEL_TIMING") &&
                                   std::getenv("DMCG_LEVEL_TIMING")[0] == '2';
    std::vector<cudaEvent_t> pe;
    const bool pl = per_launch && l + 1 == lv.nlevels;
    for (uint32_t k0 = 0; k0 < lv.maxw[l]; k0 += nb) {
      if (pl) {
        pe.emplace_back();
        cudaEventCreate(&pe.back());
        cudaEventRecord(pe.back(), s);
      }
      const uint32_t below = lv.maxm[l] > k0 ? lv.maxm[l] - k0 : 1;
      const uint32_t ny = std::min<uint32_t>(8, (below + kPanelThreads - 1) / kPanelThreads);
      if (ny == 1) {
        k_panel<<<cnt, kPanelThreads, 0, s>>>(d, ls, (int)k0, nb);
      } else {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = ny;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cnt, ny);
        cfg.blockDim = dim3(kPanelThreads);
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_panel, d, ls, (int)k0, nb);
        if (e != cudaSuccess) return e;
      }
      if (pl) {
        pe.emplace_back();
        cudaEventCreate(&pe.back());
        cudaEventRecord(pe.back(), s);
      }
      // bound over the level: a front whose last panel is partial (pw < nb)
      // has a trailing block of m - k0 - pw rows
      const uint32_t T = lv.maxm[l] > k0 + 1 ? lv.maxm[l] - k0 - 1 : 0;
      if (T > 0) {
        const uint32_t nt = (T + kBM - 1) / kBM;
        k_trailing<<<dim3(nt * (nt + 1) / 2, cnt), kGemmThreads, 0, s>>>(d, ls, (int)k0, nb);
      }
    }
    if (pl) {
      pe.emplace_back();
      cudaEventCreate(&pe.back());
      cudaEventRecord(pe.back(), s);
      cudaStreamSynchronize(s);
      for (size_t i = 0; i + 2 < pe.size(); i += 2) {
        float a, b;
        cudaEventElapsedTime(&a, pe[i], pe[i + 1]);
        cudaEventElapsedTime(&b, pe[i + 1], pe[i + 2]);
        std::fprintf(stderr, "    root panel %zu: k_panel %.1f us, k_trailing %.1f us\n", i / 2, a * 1e3, b * 1e3);
      }
      for (auto e : pe) cudaEventDestroy(e);
    }
    lt.mark(l, 2);
    const uint32_t nbk = (lv.maxw[l] + kIB - 1) / kIB;
    k_inv_diag<<<dim3(nbk, cnt), kIB, kInvDiagSmem, s>>>(d, ls);
    if (nbk > 1) k_inv_offdiag<<<dim3(nbk, cnt), kGemmThreads, 0, s>>>(d, ls, d.scratch);
    {
      const uint32_t tw = (lv.maxw[l] + 31) / 32;
      k_form_p_top<<<dim3(std::min<uint32_t>(tw * tw, 64), cnt), 256, 0, s>>>(d, ls);
      if (lv.maxu[l] > 0) {
        const uint32_t tiles_w = (lv.maxw[l] + kBN - 1) / kBN, tiles_u = (lv.maxu[l] + kBM - 1) / kBM;
        k_form_p_bot<<<dim3(tiles_u * tiles_w, cnt), kGemmThreads, 0, s>>>(d, ls, (int)tiles_w);
      }
    }
    lt.mark(l, 3);
  }
  lt.report(lv, "assemble", "panels", "inverse");
  return cudaGetLastError();
}

size_t chol_scratch_doubles(const CholLevels& lv) {
  size_t mx = 0;
  for (uint32_t l = 0; l < lv.nlevels; ++l) {
    const size_t nbk = (lv.maxw[l] + kIB - 1) / kIB;
    mx = std::max(mx, (size_t)lv.count[l] * nbk * kIB * kIB);
  }
  return mx;
}

cudaError_t chol_solve_device(cudaStream_t s, const CholDev& d, const CholLevels& lv,
                              const double* b, double* y, double* x, double* out, bool accumulate,
                              const SolveEvents* tev) {
  // timing points that stay event records inside a graph capture
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (tev && tev->ev) cudaStreamIsCapturing(s, &cap);
  auto tmark = [&](uint32_t l, int k) {
    if (!tev || !tev->ev) return;
    if (cap == cudaStreamCaptureStatusActive)
      cudaEventRecordWithFlags(tev->ev[4 * l + k], s, cudaEventRecordExternal);
    else
      cudaEventRecord(tev->ev[4 * l + k], s);
  };
  const int W = (int)d.W;
  const unsigned tn = (unsigned)((W + kBN - 1) / kBN);
  // levels whose widest front has <= narrow_w own columns take the 32 x 128 tiles
  static const uint32_t narrow_w = [] {
    const char* e = std::getenv("DMCG_SOLVE_NARROW_W");
    return e ? (uint32_t)std::atoi(e) : 200u;
  }();
  auto narrow = [&](uint32_t l) { return lv.maxw[l] <= narrow_w; };
  LevelTimer lt(s, "solve", lv.nlevels);
  // forward, leaves first: r_s -> x rows (scratch until the backward pass
  // overwrites them), [y_s; U_s] = P_s r_s
  for (uint32_t l = 0; l < lv.nlevels; ++l) {
    const uint32_t cnt = lv.count[l];
    const uint32_t* ls = d.level_sup + lv.offset[l];
    lt.mark(l, 0);
    // level 0 = the leaves: no pulls, k_fwd reads b through perm itself
    if (l > 0)
      k_gather_own<<<dim3((lv.maxw[l] + 7) / 8, (W + 127) / 128, cnt), 256, 0, s>>>(d, ls, b, x);
    lt.mark(l, 1);
    tmark(l, 0);
    const dim3 gn((lv.maxm[l] + 31) / 32, (W + 127) / 128, cnt);
    const dim3 gw((lv.maxm[l] + kBM - 1) / kBM, tn, cnt);
    if (l == 0 && narrow(l))
      k_fwd<32, 128, true><<<gn, kGemmThreads, 0, s>>>(d, ls, b, y);
    else if (l == 0)
      k_fwd<kBM, kBN, true><<<gw, kGemmThreads, 0, s>>>(d, ls, b, y);
    else if (narrow(l))
      k_fwd<32, 128, false><<<gn, kGemmThreads, 0, s>>>(d, ls, x, y);
    else
      k_fwd<kBM, kBN, false><<<gw, kGemmThreads, 0, s>>>(d, ls, x, y);
    tmark(l, 1);
    lt.mark(l, 2);
  }
  // backward, roots first: x_s = P_s^T [y_s; x_below]
  for (int l = (int)lv.nlevels - 1; l >= 0; --l) {
    const uint32_t cnt = lv.count[l];
    const uint32_t* ls = d.level_sup + lv.offset[l];
    lt.mark(l, 3);
    tmark(l, 2);
    // (the leaves' x rows are read by no descendant: not written, see k_bwd)
    if (narrow(l))
      k_bwd<32, 128><<<dim3((lv.maxw[l] + 31) / 32, (W + 127) / 128, cnt), kGemmThreads, 0, s>>>(
          d, ls, y, x, out, accumulate ? 1 : 0, l == 0 ? 1 : 0);
    else
      k_bwd<kBM, kBN><<<dim3((lv.maxw[l] + kBM - 1) / kBM, tn, cnt), kGemmThreads, 0, s>>>(
          d, ls, y, x, out, accumulate ? 1 : 0, l == 0 ? 1 : 0);
    tmark(l, 3);
    lt.mark(l, 4);
  }
  lt.report(lv, "gather", "fwd", "bwd", true);
  return cudaGetLastError();
}

cudaError_t normal_residual(cudaStream_t s, int n, int W, const uint32_t* rp, const uint32_t* ci,
                            const float* val, const double* b, const double* x, double* r) {
  if (n <= 0 || W <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((n + 7) / 8), (unsigned)((W + kResCols - 1) / kResCols));
  k_residual<<<grid, 256, 0, s>>>(n, W, rp, ci, val, b, x, r);
  return cudaGetLastError();
}

}  // namespace dmcg
