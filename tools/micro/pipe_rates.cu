// Issue-rate microbenchmark for the fast-scan inner-loop instructions on sm_100a:
// per SM cycles per warp-instruction of IDP.4A, PRMT, LOP3, IMAD, IADD3 (8 independent
// chains per thread, 16 warps per SM).  nvcc -arch=sm_100a -O3 pipe_rates.cu -o pr
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void bench(unsigned* out, unsigned seed, int iters, long long* cyc) {
  unsigned a[8], b = seed * 2654435761u + threadIdx.x, c = seed ^ 0x9E3779B9u;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * (i + 1) + seed;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = __dp4a(a[i], b, a[i]);
      if (OP == 1) asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
      if (OP == 2) asm volatile("lop3.b32 %0, %0, %1, %2, 0xb8;" : "+r"(a[i]) : "r"(b), "r"(c));
      if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
      if (OP == 4) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
      if (OP == 5) { // 1 prmt + 1 dp4a interleaved
        asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
        a[i] = __dp4a(a[i], b, a[i]);
      }
    }
  }
  long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  const char* names[] = {"IDP.4A", "PRMT", "LOP3", "IMAD", "IADD", "PRMT+IDP"};
  for (int op = 0; op < 6; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: bench<0><<<148, 512>>>(out, 7, iters, cyc); break;
        case 1: bench<1><<<148, 512>>>(out, 7, iters, cyc); break;
        case 2: bench<2><<<148, 512>>>(out, 7, iters, cyc); break;
        case 3: bench<3><<<148, 512>>>(out, 7, iters, cyc); break;
        case 4: bench<4><<<148, 512>>>(out, 7, iters, cyc); break;
        case 5: bench<5><<<148, 512>>>(out, 7, iters, cyc); break;
      }
      cudaDeviceSynchronize();
    }
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double warp_instr = (double)iters * 8 * (op == 5 ? 2 : 1) * 16;  // per SM: 16 warps
    printf("%-10s %.3f warp-instr/cycle/SM  (%.3f per SMSP)\n", names[op], warp_instr / h[0],
           warp_instr / h[0] / 4);
  }
  return 0;
}
