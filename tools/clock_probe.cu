// Effective SM clock: clock64 cycles vs %globaltimer ns over a busy loop.
#include <cstdio>
__global__ void k(long long* out, int n) {
  long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  long long c0 = clock64();
  double x = 1.0;
  for (int i = 0; i < n; ++i) x = x * 1.0000001 + 1e-9;
  long long c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = g1 - g0; out[2] = (long long)x; }
}
int main() {
  long long* d; cudaMalloc(&d, 24);
  for (int n : {1000, 100000, 10000000}) {
    k<<<1, 32>>>(d, n);
    long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("n=%d: %lld cycles in %lld ns -> %.0f MHz\n", n, h[0], h[1], 1e3 * h[0] / (double)h[1]);
  }
}
