// Microbenchmark: dependent-chain latency (cycles per op) of DADD, DMUL, F2F.F64.F32 + DADD,
// and the refine element step (F2F x2, DSUB, DMUL, DADD) on one warp.
#include <cstdio>
__global__ void lat(double* out, float* fin, long long* cyc, int mode, int n) {
  double acc = out[threadIdx.x];
  float f = fin[threadIdx.x];
  double a = 1.0000001;
  long long t0 = clock64();
  if (mode == 0) for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, a);
  else if (mode == 1) for (int i = 0; i < n; ++i) acc = __dmul_rn(acc, a);
  else if (mode == 2) for (int i = 0; i < n; ++i) { acc = __dadd_rn(acc, (double)f); f = __int_as_float(__float_as_int(f) ^ (i & 1)); }
  else for (int i = 0; i < n; ++i) { double df = __dsub_rn((double)f, (double)(f * 0.5f)); acc = __dadd_rn(acc, __dmul_rn(df, df)); f += 1.0f; }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; float* fi; long long* c;
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&fi, 1024 * 4); cudaMalloc(&c, 8);
  cudaMemset(o, 0, 1024 * 8); cudaMemset(fi, 0, 1024 * 4);
  const char* names[] = {"DADD chain", "DMUL chain", "F2F+DADD chain", "refine element (F2F,DSUB,DMUL,DADD)"};
  for (int m = 0; m < 4; ++m) for (int w : {1, 4, 16}) {
    lat<<<1, 32 * w>>>(o, fi, c, m, 4096);
    lat<<<1, 32 * w>>>(o, fi, c, m, 4096);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-40s warps %2d: %.1f cycles per step\n", names[m], w, h / 4096.0);
  }
  return 0;
}
