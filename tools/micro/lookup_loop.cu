// Rate of the fast-scan inner loop (lookup8: prmt lookups + sign-replicate masks +
// dp4a accumulation) in isolation: 16 warps/SM, register-resident code words, LUT
// rows from shared memory.  Reports cycles per lookup8 per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
template <int VAR>
__device__ __forceinline__ void lookup8(const uint4& T, uint32_t w, uint32_t (&acc)[8]) {
  const uint32_t x = w & 0x77777777u;
  const uint32_t xh = VAR == 1 ? (x >> 16) : __umulhi(x, 0x10000u);
  const uint32_t w4 = w << 4;
  const uint32_t m0 = prmt(w4, w, 0xD9C8u);
  const uint32_t m1 = prmt(w4, w, 0xFBEAu);
  const uint32_t lo0 = prmt(T.x, T.y, x), hi0 = prmt(T.z, T.w, x);
  const uint32_t lo1 = prmt(T.x, T.y, xh), hi1 = prmt(T.z, T.w, xh);
  const uint32_t r0 = (lo0 & ~m0) | (hi0 & m0);
  const uint32_t r1 = (lo1 & ~m1) | (hi1 & m1);
  if (VAR == 2) {  // u16-pair accumulation instead of dp4a
    acc[0] += r0 & 0x00FF00FFu; acc[1] += (r0 >> 8) & 0x00FF00FFu;
    acc[2] += r1 & 0x00FF00FFu; acc[3] += (r1 >> 8) & 0x00FF00FFu;
    return;
  }
  acc[0] = __dp4a(r0, 0x00000001u, acc[0]);
  acc[1] = __dp4a(r0, 0x00000100u, acc[1]);
  acc[2] = __dp4a(r0, 0x00010000u, acc[2]);
  acc[3] = __dp4a(r0, 0x01000000u, acc[3]);
  acc[4] = __dp4a(r1, 0x00000001u, acc[4]);
  acc[5] = __dp4a(r1, 0x00000100u, acc[5]);
  acc[6] = __dp4a(r1, 0x00010000u, acc[6]);
  acc[7] = __dp4a(r1, 0x01000000u, acc[7]);
}

template <int VAR, int NG>
__global__ void __launch_bounds__(256, 2) loop(uint32_t* out, int iters, long long* cyc) {
  __shared__ uint4 lut[64];
  if (threadIdx.x < 64) lut[threadIdx.x] = make_uint4(threadIdx.x * 0x01010101u, 0x04030201u * threadIdx.x, 7, 9);
  __syncthreads();
  uint32_t acc[NG][8] = {};
  uint4 P[NG], Q[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    P[g] = make_uint4(threadIdx.x * 77 + g, threadIdx.x * 31, threadIdx.x * 13, g);
    Q[g] = make_uint4(threadIdx.x * 7, threadIdx.x * 3 + g, threadIdx.x * 5, threadIdx.x);
  }
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const uint4* L = lut + (it & 15) * 4;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      lookup8<VAR>(L[0], P[g].x, acc[g]);
      lookup8<VAR>(L[1], P[g].y, acc[g]);
      lookup8<VAR>(L[2], P[g].z, acc[g]);
      lookup8<VAR>(L[3], P[g].w, acc[g]);
      lookup8<VAR>(L[0], Q[g].x, acc[g]);
      lookup8<VAR>(L[1], Q[g].y, acc[g]);
      lookup8<VAR>(L[2], Q[g].z, acc[g]);
      lookup8<VAR>(L[3], Q[g].w, acc[g]);
      P[g].x = P[g].x * 1664525u + 1013904223u; P[g].y += P[g].x; P[g].z ^= P[g].y; P[g].w += P[g].z;
      Q[g].x ^= P[g].w; Q[g].y += Q[g].x; Q[g].z ^= Q[g].y; Q[g].w += Q[g].z;
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int g = 0; g < NG; ++g)
#pragma unroll
    for (int v = 0; v < 8; ++v) s += acc[g][v];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int VAR, int NG>
void run(const char* name, uint32_t* out, long long* cyc) {
  const int iters = 2000;
  for (int r = 0; r < 2; ++r) { loop<VAR, NG><<<296, 256>>>(out, iters, cyc); cudaDeviceSynchronize(); }
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  // per SM: 2 CTAs x 8 warps = 16 warps, 4 per SMSP; per warp per iter: 8*NG lookup8
  double l8_per_smsp = (double)iters * 8 * NG * 4;
  printf("%-28s %.2f cycles per lookup8 per SMSP (ideal issue 19 + 1 word update)\n", name, h / l8_per_smsp);
}

int main() {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 296 * 256 * 4); cudaMalloc(&cyc, 296 * 8);
  run<0, 1>("dp4a, umulhi, 1 group", out, cyc);
  run<0, 2>("dp4a, umulhi, 2 groups", out, cyc);
  run<1, 1>("dp4a, shift, 1 group", out, cyc);
  run<2, 1>("u16 pairs, 1 group", out, cyc);
  run<2, 2>("u16 pairs, 2 groups", out, cyc);
  return 0;
}
