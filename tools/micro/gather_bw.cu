// Random-row gather bandwidth on one B200: rows of ROWB bytes at random
// indices of a 3.84 GB array, every warp keeping many rows in flight (the
// refine stage's access pattern: bigK candidate rows of 384 B per query).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 gather_bw.cu -o gather_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int ROWB, int INFL>
__global__ void gather(const uint4* __restrict__ X, int64_t nrows, const uint32_t* __restrict__ idx,
                       int64_t nidx, uint4* __restrict__ sink) {
  constexpr int LPR = ROWB / 16;  // lanes per row
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int64_t base = warp * INFL; base < nidx; base += nw * INFL) {
    uint4 v[INFL];
#pragma unroll
    for (int j = 0; j < INFL; ++j) {
      const int64_t i = base + j;
      v[j] = make_uint4(0, 0, 0, 0);
      if (i < nidx && lane < LPR) v[j] = __ldg(X + (int64_t)idx[i] * LPR + lane);
    }
#pragma unroll
    for (int j = 0; j < INFL; ++j) { acc.x ^= v[j].x; acc.y ^= v[j].y; acc.z ^= v[j].z; acc.w ^= v[j].w; }
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

int main() {
  const int64_t nrows = 10000000;  // 10M x 384 B = 3.84 GB (c4's refine store)
  const int64_t nidx = 1000000;    // one c4 batch: 10k queries x bigK 100
  uint4* X; uint32_t* idx; uint4* sink;
  cudaMalloc(&X, nrows * 384);
  cudaMalloc(&idx, nidx * 4);
  cudaMalloc(&sink, 16);
  cudaMemset(X, 1, nrows * 384);
  uint32_t* h = new uint32_t[nidx];
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < nidx; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)(s % nrows); }
  cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
  char* flush; cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, const char* name, int blocks, int threads) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(flush, r, 256 << 20);
      cudaEventRecord(a);
      kern<<<blocks, threads>>>(X, nrows, idx, nidx, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-28s %4d x %4d: %.1f us  %.0f GB/s\n", name, blocks, threads, best * 1e3, nidx * 384.0 / (best * 1e-3) / 1e9);
  };
  for (int bl : {148 * 4, 148 * 8, 148 * 16}) {
    run(gather<384, 4>, "row 384 B, 4 in flight/warp", bl, 256);
    run(gather<384, 8>, "row 384 B, 8 in flight/warp", bl, 256);
    run(gather<384, 16>, "row 384 B, 16 in flight/warp", bl, 256);
  }
  return 0;
}
