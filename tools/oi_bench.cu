// Phase timing of the fused OI building blocks (qr_factor / qr_form /
// oi_apply) with clock64(), one CTA, F x k in shared memory.
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
  for (int i = threadIdx.x; i < F * k; i += blockDim.x) Z[i] = start[i];
  __syncthreads();
  long long t0 = clock64();
  qr_factor<8>(Z, F, k, q);
  long long t1 = clock64();
  qr_form<8>(Z, F, k, 0, k, Q, F, q);
  long long t2 = clock64();
  oi_apply(R, F, k, Q, Z);
  long long t3 = clock64();
  for (int r = 0; r < 4; ++r) {
    __syncthreads();
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    t[0] = t1 - t0;
    t[1] = t2 - t1;
    t[2] = t3 - t2;
    t[3] = (t4 - t3) / 4;
  }
}

int main() {
  const int F = 200, k = 64;
  std::vector<double> R(F * F), S(F * k);
  for (int i = 0; i < F * F; ++i) R[i] = 1.0 / (1 + (i % 37));
  for (int i = 0; i < F; ++i)
    for (int j = 0; j < F; ++j) R[i * F + j] = R[j * F + i] = 1.0 / (1.0 + i + j);
  for (int i = 0; i < F * k; ++i) S[i] = ((i * 7919) % 1000) / 500.0 - 1.0;
  double *dR, *dS;
  long long* dt;
  cudaMalloc(&dR, F * F * 8);
  cudaMalloc(&dS, F * k * 8);
  cudaMalloc(&dt, 64 * 8);
  cudaMemcpy(dR, R.data(), F * F * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dS, S.data(), F * k * 8, cudaMemcpyHostToDevice);
  const size_t smem = 2 * F * k * 8;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) {
    k_probe<<<1, 512, smem>>>(F, k, dR, dS, dt);
    long long t[4];
    cudaMemcpy(t, dt, sizeof(t), cudaMemcpyDeviceToHost);
    printf("cycles: factor %lld form %lld apply %lld barrier %lld  (%s)\n", t[0], t[1], t[2], t[3],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
