// Stage latency of the blocked QR inside k_oi_fused (cycles, F=200, k=64):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        tools/oi_bench3.cu -o tools/oi_bench3
#include <cstdio>
#include <vector>

#include "../paper_2111_10105_b200/csrc/basis.cu"

using namespace dmcg;

__global__ void __launch_bounds__(512) k_probe(int F, int k, const double* R, const double* start,
                                               long long* t) {
  extern __shared__ double dyn[];
  __shared__ QrShared q;
  double* Z = dyn;
  double* Q = dyn + F * k;
  double* scr = Q + F * k;
  for (int i = threadIdx.x; i < F * k; i += blockDim.x) Z[i] = start[i];
  __syncthreads();
  long long c0 = clock64();
  bqr_factor<8>(Z, F, k, q, scr, k);
  long long c1 = clock64();
  bqr_form(Z, F, k, 0, k, Q, F, scr, k);
  long long c2 = clock64();
  oi_apply(R, F, k, Q, Z);
  long long c3 = clock64();
  // the panel pieces alone
  for (int c = 0; c < k; c += QNB) panel_factor<8>(Z, F, c, c + QNB, q);
  long long c4 = clock64();
  for (int c = 0; c < k; c += QNB) panel_T(Z, F, c, QNB, q, scr + QNB * QNB + QNB * k, scr);
  long long c5 = clock64();
  for (int j = 0; j < 64; ++j) __syncthreads();
  long long c6 = clock64();
  if (threadIdx.x == 0) {
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
  const size_t smem = 2 * F * k * 8 + (QNB * QNB + QNB * k + 4 * QNB * QNB) * 8;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int threads : {512, 256}) {
    k_probe<<<1, threads, smem>>>(F, k, dR, dS, dt);
    long long t[6];
    cudaMemcpy(t, dt, sizeof(t), cudaMemcpyDeviceToHost);
    printf("threads %d cycles: bqr_factor %lld bqr_form %lld oi_apply %lld | panels %lld T %lld | barrier %lld (%s)\n",
           threads, t[0], t[1], t[2], t[3], t[4], t[5], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
