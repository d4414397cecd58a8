// Microbenchmark: issue rate of DADD / DMUL / DFMA / FFMA on this GPU (4 independent chains per thread).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) { x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a); }
    if (OP == 1) { x0 = __dmul_rn(x0, b); x1 = __dmul_rn(x1, b); x2 = __dmul_rn(x2, b); x3 = __dmul_rn(x3, b); }
    if (OP == 2) { x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a); }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void kf(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) { x0 = fmaf(x0, b, a); x1 = fmaf(x1, b, a); x2 = fmaf(x2, b, a); x3 = fmaf(x3, b, a); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
int main() {
  double* d; float* f; cudaMalloc(&d, 148 * 64 * 256 * 8); cudaMalloc(&f, 148 * 64 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096; dim3 g(148 * 16), b(256);
  const char* names[] = {"DADD", "DMUL", "DFMA"};
  for (int rep = 0; rep < 2; ++rep) {
    for (int op = 0; op < 3; ++op) {
      cudaEventRecord(e0);
      if (op == 0) k<0><<<g, b>>>(d, iters, 1e-9, 1.0000001);
      if (op == 1) k<1><<<g, b>>>(d, iters, 1e-9, 1.0000001);
      if (op == 2) k<2><<<g, b>>>(d, iters, 1e-9, 1.0000001);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)g.x * b.x * iters * 4;
      if (rep) printf("%s: %.2f Gop/s (%.1f lanes/clk/SM at 1.9 GHz)\n", names[op], ops / ms / 1e6, ops / ms / 1e6 / 148 / 1.9);
    }
    cudaEventRecord(e0);
    kf<<<g, b>>>(f, iters, 1e-9f, 1.0000001f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)g.x * b.x * iters * 4;
    if (rep) printf("FFMA: %.2f Gop/s (%.1f lanes/clk/SM)\n", ops / ms / 1e6, ops / ms / 1e6 / 148 / 1.9);
  }
  return 0;
}
