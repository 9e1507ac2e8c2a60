// k_trailing-like tile GEMM probe: 1..45 CTAs of gemm_tile(64x64xK=32) on a
// 573 x 573 column-major front with the SubLower epilogue, back-to-back
// launches, CUDA events; plus clock64 per CTA.
#include <cstdio>
#include <vector>

#include "../paper_2111_10105_b200/csrc/chol.cu"

using namespace dmcg;

__device__ long long g_cyc[64];
__device__ long long g_ph[8];
struct EpiSum {
  double* out;
  __device__ void operator()(int, int, int, int, int lane, int, int, const WarpTile& wt) const {
    double s = 0;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) s += wt.acc[i][j][0] + wt.acc[i][j][1];
    out[threadIdx.x] = s;
  }
};
template <class LA, class LB>
__device__ void gemm_tile_probe(int M, int N, int m0, int n0, int kend, const LA& la, const LB& lb,
                                double* out) {
  GemmSmem& sm = gemm_smem();
  auto& As = sm.As;
  auto& Bs = sm.Bs;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wm = w >> 1, wn = w & 1;
  long long c0 = clock64();
  WarpTile wt;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) wt.acc[i][j][0] = wt.acc[i][j][1] = 0.0;
  double ra[8], rb[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int e = t + q * kGemmThreads;
    const int m = e % kBM, k = e / kBM;
    ra[q] = (k < kend && m0 + m < M) ? la(0, k, m0 + m) : 0.0;
    rb[q] = (k < kend && n0 + m < N) ? lb(0, k, n0 + m) : 0.0;
  }
  long long c1 = clock64();
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int e = t + q * kGemmThreads;
    As[0][e / kBM][e % kBM] = ra[q];
    Bs[0][e / kBN][e % kBN] = rb[q];
  }
  long long c2 = clock64();
  __syncthreads();
  long long c3 = clock64();
#pragma unroll
  for (int kk = 0; kk < kBK / 4; ++kk) {
    const int kr = kk * 4 + (lane & 3);
    double a[4], bb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = As[0][kr][wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
    for (int j = 0; j < 4; ++j) bb[j] = Bs[0][kr][wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(wt.acc[i][j], a[i], bb[j]);
  }
  long long c4 = clock64();
  double sacc = 0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) sacc += wt.acc[i][j][0] + wt.acc[i][j][1];
  out[t] = sacc;
  long long c5 = clock64();
  if (t == 0) {
    g_ph[0] = c1 - c0; g_ph[1] = c2 - c1; g_ph[2] = c3 - c2; g_ph[3] = c4 - c3; g_ph[4] = c5 - c4;
  }
}


__global__ void __launch_bounds__(kGemmThreads) k_probe(double* A, int m, int k0, int nt, int mode) {
  const long long c0 = clock64();
  const int off = k0 + 32, T = m - off;
  const int t = blockIdx.x;
  int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  const int tj = t - ti * (ti + 1) / 2;
  LoadPanel lp{A, m, k0, off};
  if (mode == 0) {
    gemm_tile(0, T, T, ti * kBM, tj * kBN, 0, 32, 0, lp, lp, SubLower{A, m, off});
  } else if (mode == 1) {  // no epilogue RMW: store to a scratch
    gemm_tile(0, T, T, ti * kBM, tj * kBN, 0, 32, 0, lp, lp, SubLower{A + (size_t)m * m, m, off});
  } else if (mode == 3) {  // K = 16
    gemm_tile(0, T, T, ti * kBM, tj * kBN, 0, 16, 0, lp, lp, SubLower{A + (size_t)m * m, m, off});
  } else if (mode == 4) {  // K = 0: epilogue only
    gemm_tile(0, T, T, ti * kBM, tj * kBN, 0, 0, 0, lp, lp, SubLower{A + (size_t)m * m, m, off});
  } else if (mode == 5) {  // K = 128
    gemm_tile(0, T, T, ti * kBM, tj * kBN, 0, 128, 0, lp, lp, SubLower{A + (size_t)m * m, m, off});
  } else if (mode == 7) {
    gemm_tile(0, T, T, ti * kBM, tj * kBN, 0, 16, 0, lp, lp, EpiSum{A + (size_t)m * m});
  } else if (mode == 6) {
  } else {  // loads only
    double acc = 0.0;
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) acc += lp(0, i / 64, ti * 64 + i % 64);
    if (acc == 12345.0) A[0] = acc;
  }
  if (threadIdx.x == 0 && blockIdx.x < 64) g_cyc[blockIdx.x] = clock64() - c0;
}

int main() {
  const int m = 573;
  std::vector<double> h((size_t)m * m);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1e-3 * (double)(i % 97);
  double* A;
  cudaMalloc(&A, 2 * h.size() * 8);
  cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 8; ++mode)
  for (int k0 : {0, 480}) {
    const int T = m - k0 - 32, nt = (T + 63) / 64, grid = nt * (nt + 1) / 2;
    for (int it = 0; it < 3; ++it) k_probe<<<grid, kGemmThreads>>>(A, m, k0, nt, mode);
    cudaEventRecord(a);
    for (int it = 0; it < 50; ++it) k_probe<<<grid, kGemmThreads>>>(A, m, k0, nt, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long cyc[64];
    cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(cyc));
    long long ph[8];
    cudaMemcpyFromSymbol(ph, g_ph, sizeof(ph));
    if (mode == 6) printf("  probe phases: load %lld sts %lld sync %lld dmma %lld epi %lld\n", ph[0], ph[1], ph[2], ph[3], ph[4]);
    printf("mode %d k0=%d grid %d: %.2f us per launch; CTA0 %lld cycles (%s)\n", mode, k0, grid, ms * 1e3 / 50, cyc[0],
           cudaGetErrorString(cudaGetLastError()));
  }
}
