// wy_vty / wy_update latency probe (F = 200, 64 columns, 8 warps).
#include <cstdio>
#include <vector>

#include "../paper_2111_10105_b200/csrc/basis.cu"

using namespace dmcg;

__global__ void __launch_bounds__(256) k_probe(int F, int k, const double* start, long long* t) {
  extern __shared__ double dyn[];
  const int L = odd_ld(F);
  double* Z = dyn;
  double* W = dyn + L * k;
  for (int i = threadIdx.x; i < F * k; i += blockDim.x) Z[i] = start[i];
  __syncthreads();
  const PanelV<double*> V{Z, L, 0};
  long long c0 = clock64();
  for (int r = 0; r < 8; ++r) {
    wy_vty<8>(V, F, 8, 8, Z + 8 * L, L, 64, W);
    __syncthreads();
  }
  long long c1 = clock64();
  for (int r = 0; r < 8; ++r) {
    wy_update<8>(V, F, 8, Z + 8 * L, L, 56, W + 8, 64);
    __syncthreads();
  }
  long long c2 = clock64();
  for (int r = 0; r < 8; ++r) {
    wy_tw<8>(W, 8, W + 8, 64, 56, true);
    __syncthreads();
  }
  long long c3 = clock64();
  if (threadIdx.x == 0) {
    t[0] = (c1 - c0) / 8;
    t[1] = (c2 - c1) / 8;
    t[2] = (c3 - c2) / 8;
  }
}

int main() {
  const int F = 200, k = 64;
  std::vector<double> S(F * k);
  for (int i = 0; i < F * k; ++i) S[i] = ((i * 7919) % 1000) / 500.0 - 1.0;
  double* dS;
  long long* dt;
  cudaMalloc(&dS, F * k * 8);
  cudaMalloc(&dt, 64 * 8);
  cudaMemcpy(dS, S.data(), F * k * 8, cudaMemcpyHostToDevice);
  const size_t smem = (F | 1) * k * 8 + 8 * 72 * 8;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_probe<<<1, 256, smem>>>(F, k, dS, dt);
  long long t[3];
  cudaMemcpy(t, dt, sizeof(t), cudaMemcpyDeviceToHost);
  printf("cycles per call: vty(64 cols, K=200) %lld update(56 cols) %lld tw %lld (%s)\n", t[0], t[1], t[2],
         cudaGetErrorString(cudaGetLastError()));
}
