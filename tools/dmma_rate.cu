// DMMA m8n8k4.f64 issue rate: W warps per CTA, 16 independent accumulators per warp.
#include <cstdio>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__global__ void k(double* out, double x, int n, long long* cyc) {
  double acc[16][2];
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = x;
  double a[4], b[4];
  for (int i = 0; i < 4; ++i) { a[i] = x + i; b[i] = x - i; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[i * 4 + j], a[i], b[j]);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {1, 2, 4, 8, 16}) {
    for (int blocks : {1, 148}) {
      const int n = 1000;
      k<<<blocks, 32 * warps>>>(o, 1e-3, n, c);
      cudaEventRecord(e0);
      k<<<blocks, 32 * warps>>>(o, 1e-3, n, c);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
      const double dm = (double)blocks * warps * 16 * n;
      printf("warps/CTA %2d CTAs %3d: %.2f cycles per DMMA per warp, %.1f TFLOP/s\n", warps, blocks,
             (double)cy / (16.0 * n), dm * 512 / (ms * 1e-3) / 1e12);
    }
  }
}
