// lut_common.cuh -- A3 (ComputeLookupTable; LUT P:711-716) with the
// uint8 quantisation (O2, readings R2/R3): one query's LUT by one warp, lane
// per subquantizer.  Shared by fs_lut_kernel (fastscan_kernels.cu) and the
// coarse certify kernel, which builds each query's LUT in its warp while it
// waits on the candidate rows (coarse_kernels.cu).
#pragma once

#include "common.cuh"

namespace rairs {

struct LutArgs {
  const float* queries;  // [nq][d]
  int d, M, M_pad, dsub;
  const float* cbT;      // codebook transposed [16][dsub][M]
  uint4* luts;           // [nq][M_pad] quantised rows (16 x u8 per subquantizer)
  uint8_t* lut_q;        // debug outputs (parity tests): Qv [nq][M][16], a, b
  float* lut_a;
  float* lut_b;
};

// O2 row T[m][0..15] (fp32 RN, ascending t, no FMA); cb = codebook [16][dsub][M]
__device__ __forceinline__ void lut_row(const float* __restrict__ qv, const float* cb, int m, int M,
                                        int dsub, float (&T)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j) T[j] = 0.0f;
  const int S = dsub * M;  // entry stride (the codebook is < 2^31 floats)
  for (int t = 0; t < dsub; ++t) {
    const float qt = __ldg(qv + m * dsub + t);
    const float* c = cb + t * M + m;  // entry j of (t, m) at c[j * S]
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float diff = __fsub_rn(qt, c[j * S]);
      T[j] = __fadd_rn(T[j], __fmul_rn(diff, diff));
    }
  }
}

// The O2 LUT of query q into lut[0..M_pad) (+ debug outputs).  Lane per
// subquantizer; pass 1 computes T (kept in `scratch` as [16][M] when keepT,
// else recomputed in pass 2), mn_m and the span; pass 2 quantises.  scratch:
// (keepT ? 17 : 1) * M floats per warp.
static __device__ __noinline__ void build_lut(const LutArgs& a, int64_t q, uint4* lut, float* scratch,
                                       const float* cb, bool keepT) {
  const int lane = lane_id();
  const int M = a.M;
  const float* qv = a.queries + q * a.d;
  float* Ts = scratch;                          // [16][M] when keepT
  float* mn = scratch + (keepT ? 16 * M : 0);   // [M]
  float spanmax = 0.0f;
  for (int m = lane; m < M; m += 32) {
    float T[16];
    lut_row(qv, cb, m, M, a.dsub, T);
    float lo = T[0], hi = T[0];
#pragma unroll
    for (int j = 1; j < 16; ++j) { lo = fminf(lo, T[j]); hi = fmaxf(hi, T[j]); }
    if (keepT) {
#pragma unroll
      for (int j = 0; j < 16; ++j) Ts[j * M + m] = T[j];
    }
    mn[m] = lo;
    spanmax = fmaxf(spanmax, __fsub_rn(hi, lo));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) spanmax = fmaxf(spanmax, __shfl_xor_sync(0xffffffffu, spanmax, o));
  const bool pos = spanmax > 0.0f;
  const float qa = pos ? __fdiv_rn(255.0f, spanmax) : 1.0f;
  __syncwarp();
  for (int m = lane; m < a.M_pad; m += 32) {
    uint32_t wd[4] = {0u, 0u, 0u, 0u};
    if (m < M && pos) {
      float T[16];
      if (keepT) {
#pragma unroll
        for (int j = 0; j < 16; ++j) T[j] = Ts[j * M + m];
      } else {
        lut_row(qv, cb, m, M, a.dsub, T);
      }
      const float mnm = mn[m];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t v = (uint32_t)min(255, __float2int_rn(__fmul_rn(__fsub_rn(T[j], mnm), qa)));
        wd[j >> 2] |= v << (8 * (j & 3));
      }
    }
    const uint4 row = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    lut[m] = row;
    if (a.lut_q && m < M) reinterpret_cast<uint4*>(a.lut_q + (q * M + m) * 16)[0] = row;
  }
  if (lane == 0) {
    if (a.lut_a) a.lut_a[q] = qa;
    if (a.lut_b) {
      float b = 0.0f;
      for (int m = 0; m < M; ++m) b = __fadd_rn(b, mn[m]);
      a.lut_b[q] = b;
    }
  }
  __syncwarp();
}

// scratch floats per warp and whether T is kept (fits 16 KB)
inline bool lut_keepT(int M) { return M * 17 <= 16 * 1024 / 4; }
inline int lut_scratch_floats(int M) { return lut_keepT(M) ? 17 * M : M; }

}  // namespace rairs
