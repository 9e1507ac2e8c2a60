// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) and DFMA throughput on sm_100a.
// Used to fill the FP64 roofline denominator (not in MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) c[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = fma(a, c[j], b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += c[j];
  if (s == 12345.0) out[0] = s;
}

__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int iters = 20000;
  for (int rep = 0; rep < 3; ++rep) {
    int blocks = sms * 4, threads = 256;
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * threads / 32);
    printf("{\"kernel\":\"dmma_m8n8k4\",\"tflops\":%.3f}\n", flops / ms / 1e9);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * (double)iters * blocks * threads;
    printf("{\"kernel\":\"dfma\",\"tflops\":%.3f}\n", flops / ms / 1e9);
  }
  size_t n = (size_t)1 << 27;  // 4 GiB per buffer as double4? 2^27 * 32 B = 4 GiB
  double4 *a, *b; cudaMalloc(&a, n * 32); cudaMalloc(&b, n * 32);
  cudaMemset(a, 0, n * 32);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy_k<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\":\"copy\",\"gbs\":%.1f}\n", 2.0 * n * 32 / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
