// Per-component step latency of qr_factor (cycles per step, F=200, k=64).
#include <cstdio>
#include <vector>

#include "../paper_2111_10105_b200/csrc/basis.cu"

using namespace dmcg;

__global__ void __launch_bounds__(512) k_probe(int F, int k, const double* start, long long* t) {
  extern __shared__ double dyn[];
  __shared__ QrShared q;
  double* Z = dyn;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < F * k; i += blockDim.x) Z[i] = start[i];
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    q.tau[i] = 0.5;
    q.rinv[i] = 0.25;
  }
  __syncthreads();
  long long a = clock64();
  for (int j = 0; j < 64; ++j) __syncthreads();
  long long b = clock64();
  for (int j = 0; j < 64; ++j) {
    qr_scale(Z, F, j, q);
    __syncthreads();
  }
  long long c = clock64();
  for (int j = 0; j < 63; ++j) {
    if (warp == 0) qr_reflector<8>(Z, F, j, q, lane);
    __syncthreads();
  }
  long long d = clock64();
  for (int j = 0; j < 63; ++j) {
    apply_reflector_cols<8>(Z, F, j, Z + j * F, 0.5, 0.25, j + 2 + warp, k, nw, lane, F);
    __syncthreads();
  }
  long long e = clock64();
  for (int j = 0; j < 63; ++j) {
    if (warp == 0) apply_reflector_cols<8>(Z, F, j, Z + j * F, 0.5, 0.25, j + 1, j + 2, 1, lane, F);
    __syncthreads();
  }
  long long f = clock64();
  if (threadIdx.x == 0) {
    t[0] = (b - a) / 64;
    t[1] = (c - b) / 64;
    t[2] = (d - c) / 63;
    t[3] = (e - d) / 63;
    t[4] = (f - e) / 63;
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
  const size_t smem = 2 * F * k * 8;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int threads : {512, 256, 128}) {
    k_probe<<<1, threads, smem>>>(F, k, dS, dt);
    long long t[5];
    cudaMemcpy(t, dt, sizeof(t), cudaMemcpyDeviceToHost);
    printf("threads %d cycles/step: barrier %lld scale %lld reflector %lld apply_all %lld apply_one %lld (%s)\n",
           threads, t[0], t[1], t[2], t[3], t[4], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
