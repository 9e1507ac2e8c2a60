// Stage latency of the blocked QR inside k_oi_fused (cycles, F=200, k=64):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        tools/oi_bench3.cu -o tools/oi_bench3
#include <cstdio>
#include <vector>

__device__ long long g_stamp[8];
#define PANEL_STAMP_X(i)                                            \
  do {                                                           \
    __syncwarp();                                                \
    if (lane == 0) g_stamp[i] += clock64();                      \
  } while (0)
__device__ long long g_fs[8];
__device__ long long* g_acc;  // generic pointer to the probe kernel's shared accumulators
#define FACT_STAMP_X(i)                                            \
  do {                                                           \
    if (threadIdx.x == 0) {                                      \
      long long* acc_ = g_acc;                                   \
      const long long t_ = clock64();                            \
      if (i > 0) acc_[i] += t_ - acc_[7];                        \
      acc_[7] = t_;                                              \
    }                                                            \
  } while (0)
#include "../paper_2111_10105_b200/csrc/basis.cu"

using namespace dmcg;

__global__ void __launch_bounds__(256) k_probe(int F, int k, const double* R, const double* start,
                                               long long* t) {
  extern __shared__ double dyn[];
  __shared__ QrShared q;
  __shared__ long long s_acc[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) s_acc[i] = 0;
    g_acc = s_acc;
  }
  const int L = odd_ld(F);
  double* Z = dyn;
  double* Q = dyn + L * k;
  double* scr = Q + L * k;
  for (int i = threadIdx.x; i < F * k; i += blockDim.x) Z[i] = start[i];
  __syncthreads();
  long long c0 = clock64();
  wqr_factor<8>(Z, F, L, k, q.tau, scr, k);
  long long c1 = clock64();
  wqr_form<8>(Z, F, L, k, 0, k, Q, L, scr, k);
  long long c2 = clock64();
  oi_apply_cluster<true, 8>(R, F, F, k, Q, L, Z, (double*)nullptr, 0, 1);
  long long c3 = clock64();
  // the register panels alone (warp 0)
  if (threadIdx.x < 32)
    for (int c = 0; c < k; c += 8) warp_panel_qr<8, 8>(Z, F, L, c, 8, q.tau, threadIdx.x);
  __syncthreads();
  long long c4 = clock64();
  long long c5 = c4;
  for (int j = 0; j < 64; ++j) __syncthreads();
  long long c6 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 7; ++i) g_fs[i] = s_acc[i];
    t[0] = c1 - c0;
    t[1] = c2 - c1;
    t[2] = c3 - c2;
    t[3] = c4 - c3;
    t[4] = c5 - c4;
    t[5] = (c6 - c5) / 64;
  }
}

int main() {
  const int F = 200, k = 64;
  std::vector<double> S(F * k), Rh(F * F);
  for (int i = 0; i < F * k; ++i) S[i] = ((i * 7919) % 1000) / 500.0 - 1.0;
  for (int i = 0; i < F; ++i)
    for (int j = 0; j < F; ++j) Rh[i * F + j] = (i == j ? 2.0 : 0.0) + 1.0 / (1 + i + j);
  double *dS, *dR;
  long long* dt;
  cudaMalloc(&dS, F * k * 8);
  cudaMalloc(&dR, F * F * 8);
  cudaMalloc(&dt, 64 * 8);
  cudaMemcpy(dS, S.data(), F * k * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dR, Rh.data(), F * F * 8, cudaMemcpyHostToDevice);
  const size_t smem = 2 * (F | 1) * k * 8 + (8 * (k + 8) + 16 * 16 + 8 * 64) * 8;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int threads : {256}) {
    k_probe<<<1, threads, smem>>>(F, k, dR, dS, dt);
    long long t[6];
    cudaMemcpy(t, dt, sizeof(t), cudaMemcpyDeviceToHost);
    long long st[8];
    cudaMemcpyFromSymbol(st, g_stamp, sizeof(st));
    printf("panel stamps (summed over calls): load %lld loop %lld - %lld store %lld\n", st[1] - st[0],
           st[2] - st[1], st[3] - st[2], st[4] - st[3]);
    long long fs[8];
    cudaMemcpyFromSymbol(fs, g_fs, sizeof(fs));
    printf("factor phases (8 panels): panel %lld vty %lld T %lld tw %lld update %lld\n", fs[1],
           fs[2], fs[3], fs[4], fs[5]);
    printf("threads %d cycles: bqr_factor %lld bqr_form %lld oi_apply %lld | panels %lld T %lld | barrier %lld (%s)\n",
           threads, t[0], t[1], t[2], t[3], t[4], t[5], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
