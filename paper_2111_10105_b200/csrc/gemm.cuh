// FP64 tensor-core GEMM for the small-k / tall-skinny contractions of the
// codec (Gram A A^T, R Q, Q^T Z, Q W, U^T delta^T, U~ c~).
//
// sm_100a has no tcgen05 kind::f64 (ptxas rejects it),
// so FP64 tensor math is DMMA: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4),
// measured at 37 TFLOP/s on this pool's B200 (tools/peak_fp64.cu,
// profiles/r01_peaks.md).  Tile 64x64x16 per 128-thread CTA, each warp a
// 32x32 sub-tile (4x4 DMMA tiles), register-staged double-buffered smem.
//
// C[b](m, n) = sum_k A[b](k, m) * B[b](k, n).  Operands are read through
// loader functors (so dequantisation / f32 upcast fuse into the tile load)
// and written through epilogue functors (strided store, split-K partial,
// row min/max, CG column-block layout).
#pragma once
#include <type_traits>

#include "common.cuh"

namespace dmcg {

constexpr int kBM = 64, kBN = 64, kBK = 16, kGemmThreads = 128;

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Accumulator fragment of one warp: acc[i][j][e] is element
//   (row = i*8 + lane/4, col = j*8 + (lane%4)*2 + e) of the warp's 32x32 tile.
struct WarpTile {
  double acc[4][4][2];
};

// One 64x64 output tile (rows m0.., cols n0..) over k in [kbeg, kend), by
// the 128 threads of the calling CTA.  Callable from any kernel (the grouped
// per-front kernels of chol.cu build their own loaders / epilogues).
struct GemmSmem {
  double As[2][kBK][kBM + 8];
  double Bs[2][kBK][kBN + 8];
};
// One static shared buffer per kernel, shared by every gemm_tile
// instantiation the kernel calls (a non-template function's __shared__
// variable is a single object).
__device__ __forceinline__ GemmSmem& gemm_smem() {
  __shared__ GemmSmem sm;
  return sm;
}

// Loaders that are plain address maps (`addr(b, k, m)`, no transform) take
// the cp.async path below: a 4-stage shared-memory ring filled straight
// from global memory (no register staging), so three k-slices of loads are
// in flight while one is multiplied.
template <class T, class = void>
struct RawLoader : std::false_type {};
template <class T>
struct RawLoader<T, std::void_t<decltype(&T::addr)>> : std::true_type {};

// One raw ring, carved per tile shape: 64 x 64 (two warps by two) or 32 x 128
// (four warps side by side: the solves' small fronts, chol.cu).
constexpr int kAStages = 4, kABK = 8;
struct GemmSmemAsync {
  double raw[kAStages * kABK * ((32 + 4) + (128 + 4))];
};
__device__ __forceinline__ GemmSmemAsync& gemm_smem_async() {
  __shared__ GemmSmemAsync sm;
  return sm;
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cp_async_el(double* smem, const double* gmem, bool pred) {
  cp_async8(smem, gmem, pred);
}
__device__ __forceinline__ void cp_async_el(float* smem, const float* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// The DMMAs of one k-slice of KS rows for the first MI 8-row blocks of a
// warp's 32x32 sub-tile (MI < 4 on ragged tiles: the padding's DMMAs are
// skipped, which frees the tensor pipe for the other CTAs of the SM).
template <int MI, int KS, typename TA, typename TB, int LDA, int LDB>
__device__ __forceinline__ void warp_mma_slice(WarpTile& wt, const TA (*As)[LDA],
                                               const TB (*Bs)[LDB], int wm, int wn, int lane) {
#pragma unroll
  for (int kk = 0; kk < KS / 4; ++kk) {
    const int kr = kk * 4 + (lane & 3);
    double a[MI > 0 ? MI : 1], bb[4];
#pragma unroll
    for (int i = 0; i < MI; ++i) a[i] = (double)As[kr][wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
    for (int j = 0; j < 4; ++j) bb[j] = (double)Bs[kr][wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(wt.acc[i][j], a[i], bb[j]);
  }
}
template <int KS, typename TA, typename TB, int LDA, int LDB>
__device__ __forceinline__ void warp_mma_slice_n(int mi_cnt, WarpTile& wt, const TA (*As)[LDA],
                                                 const TB (*Bs)[LDB], int wm, int wn, int lane) {
  switch (mi_cnt) {  // warp-uniform
    case 4: warp_mma_slice<4, KS>(wt, As, Bs, wm, wn, lane); break;
    case 3: warp_mma_slice<3, KS>(wt, As, Bs, wm, wn, lane); break;
    case 2: warp_mma_slice<2, KS>(wt, As, Bs, wm, wn, lane); break;
    case 1: warp_mma_slice<1, KS>(wt, As, Bs, wm, wn, lane); break;
    default: break;
  }
}

// Epilogues with `static constexpr bool kRowEpilogue = true` get the CTA's
// whole output tile staged in shared memory (the operand ring, free by then;
// row stride BN + 8 doubles: the fragment stores of a quarter-warp hit 32
// distinct banks) and finish it by rows:
//   ep.template rows<BM, BN>(m0, n0, M, N, tile, BN + 8)
// called by all 128 threads, so every output / gathered row is touched in
// contiguous pieces of BN doubles and per-row index lookups are warp-wide.
template <class EP, class = void>
struct RowEpilogue : std::false_type {};
template <class EP>
struct RowEpilogue<EP, std::enable_if_t<EP::kRowEpilogue>> : std::true_type {};

template <int BM = kBM, int BN = kBN, class LA, class LB, class EP>
__device__ __forceinline__ void gemm_tile_async(int b, int M, int N, int m0, int n0, int kbeg,
                                                int kend, int split, const LA& la, const LB& lb,
                                                const EP& ep) {
  static_assert(BM % 32 == 0 && BN % 32 == 0 && (BM / 32) * (BN / 32) == kGemmThreads / 32,
                "one 32x32 sub-tile per warp");
  static_assert(BM + BN <= 32 + 128, "ring size");
  // operand element types (double, or float upcast when fragments load):
  // the ring is declared for doubles and reinterpreted for narrower types
  using TA = std::remove_cv_t<std::remove_pointer_t<decltype(la.addr(0, 0, 0))>>;
  using TB = std::remove_cv_t<std::remove_pointer_t<decltype(lb.addr(0, 0, 0))>>;
  GemmSmemAsync& smd = gemm_smem_async();
  struct Ring {
    TA (*As)[kABK][BM + 4];
    TB (*Bs)[kABK][BN + 4];
  } sm{reinterpret_cast<TA(*)[kABK][BM + 4]>(smd.raw),
       reinterpret_cast<TB(*)[kABK][BN + 4]>(smd.raw + kAStages * kABK * (BM + 4))};
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  constexpr int WN = BN / 32;
  const int wm = w / WN, wn = w % WN;
  WarpTile wt;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) wt.acc[i][j][0] = wt.acc[i][j][1] = 0.0;
  const int nk = kend > kbeg ? (kend - kbeg + kABK - 1) / kABK : 0;
  // 8-row blocks of this warp's 32x32 sub-tile that hold valid output
  const int mi_cnt = min(4, max(0, (M - (m0 + wm * 32) + 7) >> 3));
  if (nk > 0) {
    const TA* adummy = la.addr(b, kbeg, m0);
    const TB* bdummy = lb.addr(b, kbeg, n0);
    auto issue = [&](int it) {
      const int buf = it % kAStages, kt = kbeg + it * kABK;
#pragma unroll
      for (int q = 0; q < (kABK * BM) / kGemmThreads; ++q) {
        const int e = t + q * kGemmThreads;
        int k, m;
        if (LA::kKContig) {
          k = e % kABK;
          m = e / kABK;
        } else {
          m = e % BM;
          k = e / BM;
        }
        const bool ok = kt + k < kend && m0 + m < M;
        cp_async_el(&sm.As[buf][k][m], ok ? la.addr(b, kt + k, m0 + m) : adummy, ok);
      }
#pragma unroll
      for (int q = 0; q < (kABK * BN) / kGemmThreads; ++q) {
        const int e = t + q * kGemmThreads;
        int kb, nb;
        if (LB::kKContig) {
          kb = e % kABK;
          nb = e / kABK;
        } else {
          nb = e % BN;
          kb = e / BN;
        }
        const bool okb = kt + kb < kend && n0 + nb < N;
        cp_async_el(&sm.Bs[buf][kb][nb], okb ? lb.addr(b, kt + kb, n0 + nb) : bdummy, okb);
      }
    };
#pragma unroll
    for (int s0 = 0; s0 < kAStages - 1; ++s0) {
      if (s0 < nk) issue(s0);
      cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
      cp_async_wait<kAStages - 2>();
      __syncthreads();
      if (it + kAStages - 1 < nk) issue(it + kAStages - 1);
      cp_async_commit();
      const int buf = it % kAStages;
      warp_mma_slice_n<kABK>(mi_cnt, wt, sm.As[buf], sm.Bs[buf], wm, wn, lane);
    }
    cp_async_wait<0>();
    __syncthreads();  // the ring may be refilled by a following tile
  }
  if constexpr (RowEpilogue<EP>::value) {
    constexpr int LD = BN + 8;
    static_assert(BM * LD <= (int)(sizeof(GemmSmemAsync) / sizeof(double)), "tile fits the ring");
    double* tile = smd.raw;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<double2*>(tile + (wm * 32 + i * 8 + (lane >> 2)) * LD + wn * 32 + j * 8 +
                                    (lane & 3) * 2) = make_double2(wt.acc[i][j][0], wt.acc[i][j][1]);
    __syncthreads();
    ep.template rows<BM, BN>(m0, n0, M, N, tile, LD);
    __syncthreads();  // the ring may be refilled by a following tile
  } else {
    ep(b, split, m0 + wm * 32, n0 + wn * 32, lane, M, N, wt);
  }
}

template <class LA, class LB, class EP>
__device__ __forceinline__ void gemm_tile(int b, int M, int N, int m0, int n0, int kbeg, int kend,
                                          int split, const LA& la, const LB& lb, const EP& ep) {
  if constexpr (RawLoader<LA>::value && RawLoader<LB>::value) {
    gemm_tile_async(b, M, N, m0, n0, kbeg, kend, split, la, lb, ep);
    return;
  }
  GemmSmem& sm = gemm_smem();
  auto& As = sm.As;
  auto& Bs = sm.Bs;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wm = w >> 1, wn = w & 1;

  WarpTile wt;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) wt.acc[i][j][0] = wt.acc[i][j][1] = 0.0;

  const int mi_cnt = min(4, max(0, (M - (m0 + wm * 32) + 7) >> 3));  // see gemm_tile_async
  double ra[8], rb[8];
  auto load_tile = [&](int kt) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = t + q * kGemmThreads;
      int k, m;
      if (LA::kKContig) {
        k = e % kBK;
        m = e / kBK;
      } else {
        m = e % kBM;
        k = e / kBM;
      }
      const int gk = kt + k, gm = m0 + m;
      ra[q] = (gk < kend && gm < M) ? la(b, gk, gm) : 0.0;
      int kb, nb;
      if (LB::kKContig) {
        kb = e % kBK;
        nb = e / kBK;
      } else {
        nb = e % kBN;
        kb = e / kBN;
      }
      const int gkb = kt + kb, gn = n0 + nb;
      rb[q] = (gkb < kend && gn < N) ? lb(b, gkb, gn) : 0.0;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = t + q * kGemmThreads;
      if (LA::kKContig)
        As[buf][e % kBK][e / kBK] = ra[q];
      else
        As[buf][e / kBM][e % kBM] = ra[q];
      if (LB::kKContig)
        Bs[buf][e % kBK][e / kBK] = rb[q];
      else
        Bs[buf][e / kBN][e % kBN] = rb[q];
    }
  };

  int buf = 0;
  if (kbeg < kend) {
    load_tile(kbeg);
    store_tile(0);
  }
  __syncthreads();
  for (int kt = kbeg; kt < kend; kt += kBK) {
    const bool more = kt + kBK < kend;
    if (more) load_tile(kt + kBK);
    warp_mma_slice_n<kBK>(mi_cnt, wt, As[buf], Bs[buf], wm, wn, lane);
    if (more) store_tile(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  ep(b, split, m0 + wm * 32, n0 + wn * 32, lane, M, N, wt);
}

template <class LA, class LB, class EP>
__global__ void __launch_bounds__(kGemmThreads)
    gemm_dmma_kernel(int M, int N, int K, int k_chunk, LA la, LB lb, EP ep) {
  const int tiles_n = (N + kBN - 1) / kBN;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int split = blockIdx.y;
  const int kbeg = split * k_chunk;
  const int kend = min(K, kbeg + k_chunk);
  gemm_tile(blockIdx.z, M, N, tm * kBM, tn * kBN, kbeg, kend, split, la, lb, ep);
}

// ---- loaders -------------------------------------------------------------
// Dense operand X(k, idx) = p[b*sb + k*sk + idx*si]; KC = k is contiguous.
template <typename T, bool KC>
struct LoadDense {
  static constexpr bool kKContig = KC;
  const T* p;
  long sb, sk, si;
  __device__ __forceinline__ double operator()(int b, int k, int i) const {
    return (double)p[b * sb + (long)k * sk + (long)i * si];
  }
  __device__ __forceinline__ const T* addr(int b, int k, int i) const {
    return p + b * sb + (long)k * sk + (long)i * si;
  }
};

// Per-batch pointer table variant (independent axis buffers).
template <typename T, bool KC>
struct LoadDense3 {
  static constexpr bool kKContig = KC;
  const T* p0;
  const T* p1;
  const T* p2;
  long sk, si;
  __device__ __forceinline__ double operator()(int b, int k, int i) const {
    const T* p = b == 0 ? p0 : (b == 1 ? p1 : p2);
    return (double)p[(long)k * sk + (long)i * si];
  }
  __device__ __forceinline__ const T* addr(int b, int k, int i) const {
    return (b == 0 ? p0 : (b == 1 ? p1 : p2)) + (long)k * sk + (long)i * si;
  }
};

// ---- epilogues -----------------------------------------------------------
__device__ __forceinline__ void frag_rc(int i, int j, int e, int lane, int* r, int* c) {
  *r = i * 8 + (lane >> 2);
  *c = j * 8 + (lane & 3) * 2 + e;
}

// C[b*sb + m*sm + n*sn] = v
struct StoreStrided {
  double* C;
  long sb, sm, sn;
  __device__ __forceinline__ void operator()(int b, int, int mb, int nb, int lane, int M, int N,
                                             const WarpTile& wt) const {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, c;
          frag_rc(i, j, e, lane, &r, &c);
          const int m = mb + r, n = nb + c;
          if (m < M && n < N) C[b * sb + (long)m * sm + (long)n * sn] = wt.acc[i][j][e];
        }
  }
};

// Split-K partial: P[((split * nbatch + b) * M + m) * N + n]
struct StorePartial {
  double* P;
  int nbatch;
  __device__ __forceinline__ void operator()(int b, int split, int mb, int nb, int lane, int M,
                                             int N, const WarpTile& wt) const {
    double* base = P + ((long)split * nbatch + b) * (long)M * N;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, c;
          frag_rc(i, j, e, lane, &r, &c);
          const int m = mb + r, n = nb + c;
          if (m < M && n < N) base[(long)m * N + n] = wt.acc[i][j][e];
        }
  }
};

// Effective split count (every split gets >= 1 K-tile) and its chunk size.
inline int gemm_splits(int K, int splits, int* k_chunk_out) {
  if (splits < 1) splits = 1;
  int k_chunk = (K + splits - 1) / splits;
  k_chunk = ((k_chunk + kBK - 1) / kBK) * kBK;
  if (k_chunk <= 0) k_chunk = kBK;
  int eff = (K + k_chunk - 1) / k_chunk;
  if (eff < 1) eff = 1;
  if (k_chunk_out) *k_chunk_out = k_chunk;
  return eff;
}

template <class LA, class LB, class EP>
cudaError_t launch_gemm(cudaStream_t s, int nbatch, int M, int N, int K, int splits, LA la, LB lb,
                        EP ep) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  int k_chunk;
  splits = gemm_splits(K, splits, &k_chunk);
  const int tiles = ((M + kBM - 1) / kBM) * ((N + kBN - 1) / kBN);
  dim3 grid(tiles, splits, nbatch);
  gemm_dmma_kernel<LA, LB, EP><<<grid, kGemmThreads, 0, s>>>(M, N, K, k_chunk, la, lb, ep);
  return cudaGetLastError();
}

}  // namespace dmcg
