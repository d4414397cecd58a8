// common.cuh -- shared device/host helpers for librairs (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/rairs.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "librairs is built for sm_100a (B200) only"
#endif

namespace rairs {

// ---- programmatic dependent launch (PDL) ------------------------------------
// Kernels of one dependency chain on a stream are launched with the
// programmatic-serialization attribute: the next kernel's CTAs are scheduled
// (and run their prologue) while the previous grid drains; pdl_wait() then
// blocks until the previous grid has completed and its writes are visible.
// Every kernel launched with launch_pdl calls pdl_wait() before it reads
// anything its predecessor wrote; pdl_trigger() lets the next grid launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}


constexpr uint32_t kSlotPad = 0xFFFFFFFFu;   // padding slot marker in slot_rows
constexpr int kBlk = 32;                     // items per code block (one warp)
constexpr uint64_t kKeyInf = ~0ull;

// thread-local error message for rairs_last_error()
void set_error(const std::string& msg);

struct Status {
  rairs_status code;
};

#define RAIRS_CUDA_TRY(expr)                                                    \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::rairs::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));   \
      return (_e == cudaErrorMemoryAllocation) ? RAIRS_E_OOM : RAIRS_E_CUDA;    \
    }                                                                           \
  } while (0)

#define RAIRS_CHECK_LAUNCH()                                                    \
  do {                                                                          \
    cudaError_t _e = cudaGetLastError();                                        \
    if (_e != cudaSuccess) {                                                    \
      ::rairs::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
      return RAIRS_E_CUDA;                                                      \
    }                                                                           \
  } while (0)

#define RAIRS_TRY(expr)                                                         \
  do {                                                                          \
    rairs_status _s = (expr);                                                   \
    if (_s != RAIRS_OK) return _s;                                              \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Stream-ordered workspaces come from the library's own memory pool (one per
// device, created on first use), which keeps freed blocks cached: a search's
// multi-GB workspace (list-major score rows of a 100M batch) is reused by the
// next search without a driver round trip, and the caller's default pool is
// left untouched.
cudaError_t ws_malloc(void** p, size_t bytes, cudaStream_t s);
template <typename T>
inline cudaError_t ws_malloc(T** p, size_t bytes, cudaStream_t s) {
  return ws_malloc(reinterpret_cast<void**>(p), bytes, s);
}

// RAIRS_DEBUG_SYNC=1: synchronise after the named launch and report a fault
// there (debugging aid for large builds; off by default, no effect on results)
bool debug_sync_enabled();
rairs_status debug_sync_point(cudaStream_t s, const char* what);
#define RAIRS_DEBUG_POINT(s, what)                                  \
  do {                                                              \
    if (::rairs::debug_sync_enabled()) {                            \
      rairs_status _ds = ::rairs::debug_sync_point((s), (what));    \
      if (_ds != RAIRS_OK) return _ds;                              \
    }                                                               \
  } while (0)
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---------------------------------------------------------------------------
// Exactly-rounded arithmetic (no FMA contraction): the parity contract needs
// the same fp64 ordered sums / fp32 LUT values as the CPU oracle (R2).
__device__ __forceinline__ double dsq_diff(float a, float b) {
  double df = __dsub_rn((double)a, (double)b);
  return __dmul_rn(df, df);
}

// u64 bits of a non-negative double: integer order == numeric order.
// Second-list loss of a redundant assignment (Table 2), fp64,
// every operation rounded to nearest (O4):
//   mode 1 AIR   : ||r'||^2 + lambda * r.r'                (Alg. 3 line 8)
//   mode 3 SOARL2: ||r'||^2 + lambda * (r.r' / ||r||)^2
// ss = ||r'||^2, ip = r.r', rr = ||r||^2 (ordered sums); SOAR's projection term
// is 0 when ||r|| = 0 (x on the first centroid: r = 0, so r.r' = 0).
__device__ __forceinline__ double second_list_loss(int mode, double lambda, double ss, double ip,
                                                   double rr) {
  if (mode == 3) {
    if (rr == 0.0) return ss;
    const double pr = __ddiv_rn(ip, __dsqrt_rn(rr));
    return __dadd_rn(ss, __dmul_rn(lambda, __dmul_rn(pr, pr)));
  }
  return __dadd_rn(ss, __dmul_rn(lambda, ip));
}

__device__ __forceinline__ uint64_t dbits(double v) {
  return (uint64_t)__double_as_longlong(v);
}

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// (bits, id) lexicographic argmin across a warp; returns the winning pair in
// every lane.
__device__ __forceinline__ void warp_min_pair(uint64_t& k, uint32_t& id) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t k2 = __shfl_xor_sync(0xffffffffu, k, o);
    uint32_t i2 = __shfl_xor_sync(0xffffffffu, id, o);
    if (k2 < k || (k2 == k && i2 < id)) {
      k = k2;
      id = i2;
    }
  }
}

// In-place ascending bitonic sort of n = power-of-two u64 keys in shared
// memory by all threads of the CTA (caller syncs before; ends with a sync).
__device__ __forceinline__ void cta_bitonic_sort_u64(uint64_t* a, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool asc = ((lo & size) == 0);
        uint64_t x = a[lo], y = a[hi];
        if ((x > y) == asc) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      __syncthreads();
    }
  }
}

inline int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace rairs
