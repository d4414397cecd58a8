// coarse_kernels.cu -- K1/K2: the coarse quantizer on sm_100a tensor cores.
//
// K1  G[q][l] = ||c_l||^2 - 2 q.c_l   (FindNearestLists; exhaustive
//     O(nlist*D) per query P:1216; bulk per batch P:1862-1864), as a
//     hand-written tcgen05.mma kind::tf32 GEMM: operands streamed by TMA
//     (cp.async.bulk.tensor, 128B swizzle) into a 3-stage shared-memory ring,
//     one elected thread issues the MMAs, the fp32 accumulator lives in TMEM
//     (128 lanes x 256 columns) and the epilogue reads it with tcgen05.ld.
// K2  per query: the first W = nprobe + delta lists by G, their exact fp64
//     distances D64 (O1), re-rank by (D64, l), and CERTIFY (reading R6): every
//     list outside the candidate set has G >= G_(W+1), and the TF32 error of G
//     is bounded by E, so if G_(W+1) - E exceeds the nprobe-th exact distance
//     (minus ||q||^2) no excluded list can enter the probe set.  Otherwise the
//     query is flagged and recomputed by the exact fp64 kernel.  The probe set
//     is therefore always exactly O1's.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "index.cuh"

namespace rairs {

constexpr int CG_BM = 128, CG_BN = 256, CG_BK = 32, CG_S = 3;
constexpr uint32_t CG_A_BYTES = CG_BM * CG_BK * 4;   // 16 KB
constexpr uint32_t CG_B_BYTES = CG_BN * CG_BK * 4;   // 32 KB
constexpr int CG_THREADS = 128;
constexpr size_t CG_SMEM = 1024 + CG_S * (CG_A_BYTES + CG_B_BYTES) + 256 + CG_BN * 4;

// instruction descriptor: D=F32, A=B=TF32, both K-major, N=256, M=128
constexpr uint32_t CG_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(CG_BN >> 3) << 17) |
                              ((uint32_t)(CG_BM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// K-major operand tile, 128-byte swizzle, 8-row groups 1024 B apart (SBO).
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(CG_THREADS, 1)
    coarse_gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA,
                            const __grid_constant__ CUtensorMap tmB, const float* __restrict__ cnorm,
                            int nq, int nlist, int d, float* __restrict__ G, int ldg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + CG_S * CG_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + CG_S * CG_B_BYTES);
  uint64_t* empty = full + CG_S;
  uint64_t* done = empty + CG_S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* cn = reinterpret_cast<float*>(smem + CG_S * (CG_A_BYTES + CG_B_BYTES) + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * CG_BM, n0 = blockIdx.y * CG_BN;
  const int nk = (d + CG_BK - 1) / CG_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < CG_S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < CG_BN; j += CG_THREADS)
    cn[j] = (n0 + j < nlist) ? cnorm[n0 + j] : 0.0f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(CG_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      auto issue = [&](int kc) {
        const int s = kc % CG_S;
        mbar_expect_tx(&full[s], CG_A_BYTES + CG_B_BYTES);
        tma_load_2d(sA + s * CG_A_BYTES, &tmA, kc * CG_BK, m0, &full[s]);
        tma_load_2d(sB + s * CG_B_BYTES, &tmB, kc * CG_BK, n0, &full[s]);
      };
      for (int kc = 0; kc < nk && kc < CG_S; ++kc) issue(kc);
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % CG_S;
        const uint32_t ph = (uint32_t)(kc / CG_S) & 1u;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(sA + s * CG_A_BYTES);
        const uint64_t bd = umma_desc_sw128(sB + s * CG_B_BYTES);
#pragma unroll
        for (int k = 0; k < CG_BK / 8; ++k)  // K = 8 tf32 per MMA = 32 B = +2 desc units
          umma_tf32(tmem, ad + 2 * k, bd + 2 * k, CG_IDESC, (kc | k) != 0 ? 1u : 0u);
        umma_commit(&empty[s]);
        if (kc + CG_S < nk) {
          mbar_wait(&empty[s], ph);
          issue(kc + CG_S);
        }
      }
      umma_commit(done);
    }
    __syncwarp();
  }
  mbar_wait(done, 0);
  tc_fence_after();

  const int row = warp * 32 + lane;
  const int q = m0 + row;
  for (int c = 0; c < CG_BN / 32; ++c) {
    uint32_t v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c * 32), v);
    if (q < nq) {
      float* out = G + (size_t)q * ldg + n0 + c * 32;
      const int lim = nlist - (n0 + c * 32);
      if (lim >= 32 && (ldg & 3) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o;
          o.x = cn[c * 32 + j + 0] - 2.0f * __uint_as_float(v[j + 0]);
          o.y = cn[c * 32 + j + 1] - 2.0f * __uint_as_float(v[j + 1]);
          o.z = cn[c * 32 + j + 2] - 2.0f * __uint_as_float(v[j + 2]);
          o.w = cn[c * 32 + j + 3] - 2.0f * __uint_as_float(v[j + 3]);
          *reinterpret_cast<float4*>(out + j) = o;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < lim) out[j] = cn[c * 32 + j] - 2.0f * __uint_as_float(v[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CG_BN));
}

// ---------------------------------------------------------------------------
// K2: select W candidates by G, exact fp64 re-rank, certify.
constexpr int SEL_THREADS = 256;
constexpr int SEL_WARPS = SEL_THREADS / 32;

__device__ __forceinline__ uint32_t ord_f32(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ void warp_sort_u64(uint64_t* a, int n) {
  const int lane = lane_id();
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (n >> 1); i += 32) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool asc = ((lo & size) == 0);
        uint64_t x = a[lo], y = a[hi];
        if ((x > y) == asc) { a[lo] = y; a[hi] = x; }
      }
      __syncwarp();
    }
  }
}

__device__ void warp_sort_pairs2(uint64_t* k, uint32_t* id, int n) {
  const int lane = lane_id();
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (n >> 1); i += 32) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool asc = ((lo & size) == 0);
        uint64_t ka = k[lo], kb = k[hi];
        uint32_t ia = id[lo], ib = id[hi];
        bool gt = (ka > kb) || (ka == kb && ia > ib);
        if (gt == asc) { k[lo] = kb; k[hi] = ka; id[lo] = ib; id[hi] = ia; }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ float unord_f32(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

// One warp per query.  The W+1 smallest G values are isolated with a 256-bin
// histogram over [min G, max G] (the bin map is monotone in G, so the bins up
// to the first bin whose cumulative count reaches W+1 hold every one of the
// W+1 smallest), then only those survivors are sorted by (G, l).
__global__ void __launch_bounds__(SEL_THREADS)
    coarse_select_kernel(const float* __restrict__ G, int ldg, const float* __restrict__ Q,
                         const float* __restrict__ C, int64_t nq, int nlist, int d, int nprobe,
                         int W, int npow_l, int npow_w, double cmax, int32_t* __restrict__ probes,
                         int32_t* __restrict__ flags, unsigned* __restrict__ nflag) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = warp_id(), lane = lane_id();
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm) + (size_t)warp * npow_l;
  uint64_t* ck = reinterpret_cast<uint64_t*>(sm) + (size_t)SEL_WARPS * npow_l + (size_t)warp * npow_w;
  uint32_t* ci = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(sm) +
                                             (size_t)SEL_WARPS * (npow_l + npow_w)) +
                 (size_t)warp * npow_w;
  uint32_t* hist = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(sm) +
                                               (size_t)SEL_WARPS * (npow_l + npow_w)) +
                   (size_t)SEL_WARPS * npow_w + (size_t)warp * 256;
  const bool all = W >= nlist;
  const int need = all ? nlist : W + 1;
  for (int64_t q = (int64_t)blockIdx.x * SEL_WARPS + warp; q < nq;
       q += (int64_t)gridDim.x * SEL_WARPS) {
    const float* g = G + (size_t)q * ldg;
    float gmin = __int_as_float(0x7f800000), gmax = -gmin;
    for (int l = lane; l < nlist; l += 32) {
      const float v = g[l];
      gmin = fminf(gmin, v);
      gmax = fmaxf(gmax, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      gmin = fminf(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
      gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    }
    const float scale = (gmax > gmin) ? 255.99f / (gmax - gmin) : 0.0f;
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    for (int l = lane; l < nlist; l += 32)
      atomicAdd(&hist[min(255, (int)((g[l] - gmin) * scale))], 1u);
    __syncwarp();
    // first bin b with cumulative count >= need (8 bins per lane)
    uint32_t h8[8], loc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { h8[i] = hist[lane * 8 + i]; loc += h8[i]; }
    uint32_t inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, inc >= (uint32_t)need);
    const int hl = __ffs(hit) - 1;
    int b = 255;
    if (lane == hl) {
      uint32_t run = inc - loc;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        run += h8[i];
        if (run >= (uint32_t)need) { b = lane * 8 + i; break; }
      }
    }
    b = __shfl_sync(0xffffffffu, b, hl);
    // collect survivors as (ord(G) << 32 | l) keys
    int cnt = 0;
    for (int l0 = 0; l0 < nlist; l0 += 32) {
      const int l = l0 + lane;
      float v = 0.0f;
      bool keep = false;
      if (l < nlist) {
        v = g[l];
        keep = min(255, (int)((v - gmin) * scale)) <= b;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) keys[cnt + __popc(bal & ((1u << lane) - 1u))] = ((uint64_t)ord_f32(v) << 32) | (uint32_t)l;
      cnt += __popc(bal);
    }
    int np = 2;
    while (np < cnt) np <<= 1;
    for (int i = cnt + lane; i < np; i += 32) keys[i] = kKeyInf;
    __syncwarp();
    warp_sort_u64(keys, np);
    const int Wc = all ? nlist : W;
    const float gnext = all ? 0.0f : unord_f32((uint32_t)(keys[W] >> 32));
    // exact D64 of the candidates (O1)
    const float* qv = Q + (size_t)q * d;
    for (int i = lane; i < npow_w; i += 32) {
      if (i < Wc) {
        const uint32_t l = (uint32_t)(keys[i] & 0xFFFFFFFFu);
        const float* c = C + (size_t)l * d;
        double acc = 0.0;
        for (int t = 0; t < d; ++t) acc = __dadd_rn(acc, dsq_diff(qv[t], c[t]));
        ck[i] = dbits(acc);
        ci[i] = l;
      } else {
        ck[i] = kKeyInf;
        ci[i] = 0xFFFFFFFFu;
      }
    }
    __syncwarp();
    warp_sort_pairs2(ck, ci, npow_w);
    bool certified = all;
    if (!all) {
      double qn = 0.0;
      for (int t = lane; t < d; t += 32) qn += (double)qv[t] * (double)qv[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) qn += __shfl_xor_sync(0xffffffffu, qn, o);
      const double qnorm = sqrt(qn);
      const double E = (ldexp(1.0, -8) + d * ldexp(1.0, -22)) * qnorm * cmax +
                       ldexp(1.0, -22) * (cmax * cmax + 2.0 * qnorm * cmax);
      const double dnp = __longlong_as_double((long long)ck[nprobe - 1]);
      certified = ((double)gnext - E) > (dnp - qn) + 1e-10 * (dnp + qn);
    }
    for (int i = lane; i < nprobe; i += 32) probes[q * nprobe + i] = (int32_t)ci[i];
    if (lane == 0) {
      flags[q] = certified ? 0 : 1;
      if (!certified) atomicAdd(nflag, 1u);
    }
    __syncwarp();
  }
}

__global__ void cnorm_kernel(const float* __restrict__ C, int nlist, int d, float* __restrict__ cn,
                             double* __restrict__ cmax_out) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlist; l += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) s += (double)C[(size_t)l * d + t] * (double)C[(size_t)l * d + t];
    cn[l] = (float)s;
    // max of sqrt via atomicMax on the bit pattern of a non-negative double
    atomicMax(reinterpret_cast<unsigned long long*>(cmax_out),
              (unsigned long long)__double_as_longlong(sqrt(s)));
  }
}

// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
            cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

static bool make_tmap(CUtensorMap* tm, const float* ptr, int64_t rows, int d, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 4};
  cuuint32_t box[2] = {(cuuint32_t)CG_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

rairs_status coarse_prepare(rairs_index_s* idx, cudaStream_t s) {
  RAIRS_CUDA_TRY(cudaMalloc(&idx->cnorm, (size_t)idx->nlist * 4));
  double* dmax = nullptr;
  RAIRS_CUDA_TRY(cudaMallocAsync(&dmax, 8, s));
  RAIRS_CUDA_TRY(cudaMemsetAsync(dmax, 0, 8, s));
  cnorm_kernel<<<(idx->nlist + 255) / 256, 256, 0, s>>>(idx->centroids, idx->nlist, idx->d,
                                                        idx->cnorm, dmax);
  RAIRS_CHECK_LAUNCH();
  RAIRS_CUDA_TRY(cudaMemcpyAsync(&idx->cmax, dmax, 8, cudaMemcpyDeviceToHost, s));
  RAIRS_CUDA_TRY(cudaFreeAsync(dmax, s));
  RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  idx->device_bytes += (size_t)idx->nlist * 4;
  return RAIRS_OK;
}

bool coarse_gemm_supported(const rairs_index_s* idx, int nprobe) {
  if (idx->coarse_mode == 1) return false;       // forced exact
  if ((idx->d & 3) != 0 || !get_encode()) return false;
  if (idx->coarse_mode == 2) return true;        // forced tensor-core path
  return idx->nlist >= 64 && nprobe < idx->nlist;
}

rairs_status launch_coarse(const rairs_index_s* idx, const float* queries, int64_t nq, int nprobe,
                           int32_t* probes, unsigned* nflag_dev, cudaStream_t s) {
  const int nlist = idx->nlist, d = idx->d;
  const int ldg = (int)round_up(nlist, 4);
  const int delta = 16 + nprobe / 8;
  const int W = std::min(nlist, nprobe + delta);
  const int npow_l = next_pow2(std::max(nlist, 2));
  const int npow_w = next_pow2(std::max(W, 2));
  const size_t sel_smem = (size_t)SEL_WARPS * (npow_l * 8 + npow_w * 12 + 256 * 4);
  if (sel_smem > 220 * 1024) {
    set_error("coarse select: nlist too large for the materialised path");
    return RAIRS_E_UNSUPPORTED;
  }
  float* G = nullptr;
  int32_t* flags = nullptr;
  RAIRS_CUDA_TRY(cudaMallocAsync(&G, (size_t)nq * ldg * 4, s));
  RAIRS_CUDA_TRY(cudaMallocAsync(&flags, (size_t)nq * 4, s));
  CUtensorMap tmA, tmB;
  if (!make_tmap(&tmA, queries, nq, d, CG_BM) || !make_tmap(&tmB, idx->centroids, nlist, d, CG_BN)) {
    cudaFreeAsync(G, s);
    cudaFreeAsync(flags, s);
    set_error("cuTensorMapEncodeTiled failed");
    return RAIRS_E_CUDA;
  }
  static bool attr_set = false;
  if (!attr_set) {
    RAIRS_CUDA_TRY(cudaFuncSetAttribute(coarse_gemm_tf32_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CG_SMEM));
    attr_set = true;
  }
  dim3 grid((unsigned)ceil_div(nq, CG_BM), (unsigned)ceil_div(nlist, CG_BN));
  coarse_gemm_tf32_kernel<<<grid, CG_THREADS, CG_SMEM, s>>>(tmA, tmB, idx->cnorm, (int)nq, nlist, d,
                                                            G, ldg);
  RAIRS_CHECK_LAUNCH();
  RAIRS_CUDA_TRY(cudaFuncSetAttribute(coarse_select_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel_smem));
  const int sgrid = (int)std::min<int64_t>(ceil_div(nq, SEL_WARPS), 148 * 16);
  coarse_select_kernel<<<sgrid, SEL_THREADS, sel_smem, s>>>(G, ldg, queries, idx->centroids, nq,
                                                            nlist, d, nprobe, W, npow_l, npow_w,
                                                            idx->cmax, probes, flags, nflag_dev);
  RAIRS_CHECK_LAUNCH();
  // exact fp64 recomputation of the (rare) uncertified queries
  ProbeArgs pa{};
  pa.X = queries;
  pa.rows = nq;
  pa.d = d;
  pa.C = idx->centroids;
  pa.nl = nlist;
  pa.L = nprobe;
  pa.mode = 0;
  pa.out_idx = probes;
  pa.only_flagged = flags;
  rairs_status st = launch_probe_exact(pa, s);
  cudaFreeAsync(G, s);
  cudaFreeAsync(flags, s);
  return st;
}

}  // namespace rairs
