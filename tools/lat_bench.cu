// Latency probes (cycles/op, one warp): DMMA m8n8k4 f64 chains, SHFL, DFMA, LDS.
#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void probe(long long* out, double x, int n) {
  __shared__ int chase[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) chase[i] = (i + 33) & 1023;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  double c[2] = {x, x}, d[4][2] = {{x, x}, {x, x}, {x, x}, {x, x}};
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(c, x, x);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(d[u], x, x);
  }
  long long t2 = clock64();
  double s = x;
  for (int i = 0; i < n; ++i) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1.0;
  long long t3 = clock64();
  double f = x;
  for (int i = 0; i < n; ++i) f = fma(f, x, 1.0);
  long long t4 = clock64();
  int p = threadIdx.x;
  for (int i = 0; i < n; ++i) p = chase[p];
  long long t5 = clock64();
  double r = x;
  for (int i = 0; i < n; ++i) r = rsqrt(r + 2.0);
  long long t6 = clock64();
  double q = x;
  for (int i = 0; i < n; ++i) q = __drcp_rn(q + 2.0);
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / n; out[1] = (t2 - t1) / (4 * n); out[2] = (t3 - t2) / n;
    out[3] = (t4 - t3) / n; out[4] = (t5 - t4) / n; out[5] = (t6 - t5) / n; out[6] = (t7 - t6) / n;
    out[7] = (long long)(c[0] + d[0][0] + d[3][1] + s + f + p + r + q);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  probe<<<1, 64>>>(d, 1e-3, 4096);
  long long h[8];
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("cycles/op: dmma-chain %lld dmma-4chains(per op) %lld shfl+dadd %lld dfma %lld lds-chase %lld rsqrt64 %lld drcp_rn %lld (%s)\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], cudaGetErrorString(cudaGetLastError()));
}
