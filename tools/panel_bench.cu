// Phase timing of one register-panel QR (warp_panel_qr<8,8>, F = 200) with
// clock64 stamps stored (not accumulated) by lane 0.
#include <cstdio>
#include <vector>

__device__ long long g_st[8];
#define PANEL_STAMP(i)                           \
  do {                                           \
    if (lane == 0) g_st[i] = clock64();          \
  } while (0)
#include "../paper_2111_10105_b200/csrc/basis.cu"

using namespace dmcg;

__global__ void k(double* Zg, int F) {
  extern __shared__ double dyn[];
  __shared__ double tau[64];
  const int L = F | 1;
  for (int i = threadIdx.x; i < F * 8; i += blockDim.x) dyn[(i / F) * L + i % F] = Zg[i];
  __syncthreads();
  if (threadIdx.x < 32) warp_panel_qr<8, 8>(dyn, F, L, 0, 8, tau, threadIdx.x);
}

int main() {
  const int F = 200;
  std::vector<double> h(F * 8);
  for (int i = 0; i < F * 8; ++i) h[i] = ((i * 7919) % 1000) / 500.0 - 1.0;
  double* d;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  for (int it = 0; it < 3; ++it) {
    k<<<1, 32, (F | 1) * 8 * 8>>>(d, F);
    long long st[8];
    cudaMemcpyFromSymbol(st, g_st, sizeof(st));
    printf("load %lld  columns %lld  store+tau %lld cycles (%s)\n", st[1] - st[0], st[2] - st[1],
           st[4] - st[2], cudaGetErrorString(cudaGetLastError()));
  }
}
