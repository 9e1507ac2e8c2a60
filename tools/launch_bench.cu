// Back-to-back launch cost on this GPU: empty kernels, 128-CTA kernels doing a
// dependent global read-modify-write, stream vs CUDA graph.
#include <cstdio>

__global__ void k_empty() {}
__global__ void k_touch(double* p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  p[i] = p[i] * 1.0000001 + 1.0;
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  double* p;
  cudaMalloc(&p, 128 * 256 * 8);
  cudaMemset(p, 0, 128 * 256 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 200;
  for (int mode = 0; mode < 4; ++mode) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    auto body = [&]() {
      for (int i = 0; i < N; ++i) {
        if (mode & 1) k_touch<<<128, 256, 0, s>>>(p);
        else k_empty<<<1, 32, 0, s>>>();
      }
    };
    if (mode >= 2) {
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      body();
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, s);
    } else {
      body();
    }
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    if (mode >= 2) cudaGraphLaunch(ge, s); else body();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s %s: %.2f us per kernel\n", mode >= 2 ? "graph " : "stream", (mode & 1) ? "touch(128x256)" : "empty", 1e3 * ms / N);
  }
}
