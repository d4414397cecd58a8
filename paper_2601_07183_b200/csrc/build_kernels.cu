// build_kernels.cu -- exact fp64 list selection (coarse probe, RairAssign,
// ground truth), GPU training (k-means, PQ codebook) and the cell-major SEIL
// layout build.  sm_100a.
//
// Paper passages: FindNearestLists (Alg. 2 line 5),
// RairAssign (Alg. 3; RAIR/SRAIR P:1143-1165), PQ encoding
// (P:705-708), SeilInsert (Alg. 4) in the cell-major reading
// (R10): every vector stored once; list l owns the cells (l, j>=l)
// contiguously, list j references cell (i<j, j) by (owner, slot, count).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <queue>
#include <vector>

#include "index.cuh"
#include "tc_helpers.cuh"

namespace rairs {

// ===========================================================================
// Exact selection kernel.
// For R rows at a time, D64(x, c_l) = sum_t ((double)x_t - (double)c_l,t)^2
// (fp64 ordered, no FMA) against tiles of 256 "lists"; a warp per row keeps
// the running first-L by (D64, l) in shared memory.
// ===========================================================================
constexpr int PT = 256;     // threads
constexpr int PNW = PT / 32;
constexpr int TL = 256;     // lists per tile
constexpr int TD = 32;      // dims per tile chunk

struct ProbeSmem {
  int R, d, bufcap;
  size_t off_x, off_ct, off_dk, off_bk, off_bi, off_cnt, total;
};

static ProbeSmem probe_smem(int R, int d, int L) {
  ProbeSmem s;
  s.R = R;
  s.d = d;
  s.bufcap = next_pow2(L + TL);
  size_t o = 0;
  s.off_x = o;  o += (size_t)R * d * sizeof(double);
  o = round_up(o, 16);
  s.off_ct = o; o += (size_t)TL * (TD + 1) * sizeof(float);
  o = round_up(o, 16);
  s.off_dk = o; o += (size_t)R * TL * sizeof(uint64_t);
  s.off_bk = o; o += (size_t)R * s.bufcap * sizeof(uint64_t);
  s.off_bi = o; o += (size_t)R * s.bufcap * sizeof(uint32_t);
  o = round_up(o, 16);
  s.off_cnt = o; o += (size_t)R * sizeof(int);
  s.total = round_up(o, 16);
  return s;
}

// ascending bitonic sort of n (power of two) (key, id) pairs by one warp
__device__ void warp_sort_pairs(uint64_t* k, uint32_t* id, int n) {
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
        if (gt == asc) {
          k[lo] = kb; k[hi] = ka;
          id[lo] = ib; id[hi] = ia;
        }
      }
      __syncwarp();
    }
  }
}

template <int R>
__global__ void __launch_bounds__(PT) probe_exact_kernel(ProbeArgs a, ProbeSmem ps) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* xs = reinterpret_cast<double*>(sm + ps.off_x);
  float* ct = reinterpret_cast<float*>(sm + ps.off_ct);
  uint64_t* dk = reinterpret_cast<uint64_t*>(sm + ps.off_dk);
  uint64_t* bk = reinterpret_cast<uint64_t*>(sm + ps.off_bk);
  uint32_t* bi = reinterpret_cast<uint32_t*>(sm + ps.off_bi);
  int* bcnt = reinterpret_cast<int*>(sm + ps.off_cnt);
  const int d = a.d, L = a.L, cap = ps.bufcap;
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();

  // fallback mode: only_flagged[rows] holds the number of flagged rows
  if (a.flag_count) pdl_wait();  // launched with launch_pdl after the certify kernel
  if (a.only_flagged && a.flag_count && *(volatile const int32_t*)(a.only_flagged + a.rows) == 0) return;
  for (int64_t g = blockIdx.x; g * R < a.rows; g += gridDim.x) {
    const int64_t r0 = g * R;
    const int nr = (int)((a.rows - r0) < (int64_t)R ? (a.rows - r0) : (int64_t)R);
    if (a.only_flagged) {
      const bool mine = (tid < nr) && a.only_flagged[r0 + tid] != 0;
      if (!__syncthreads_or(mine)) continue;
    }
    for (int e = tid; e < R * d; e += PT) {
      int r = e / d, t = e - r * d;
      xs[e] = (r < nr) ? (double)a.X[(r0 + r) * d + t] : 0.0;
    }
    if (tid < R) bcnt[tid] = 0;
    __syncthreads();

    for (int64_t l0 = 0; l0 < a.nl; l0 += TL) {
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
      const int64_t my_l = l0 + tid;
      const bool lv = my_l < a.nl;
      for (int t0 = 0; t0 < d; t0 += TD) {
        const int td = min(TD, d - t0);
        for (int e = tid; e < TL * TD; e += PT) {
          int li = e / TD, tt = e - li * TD;
          int64_t l = l0 + li;
          ct[li * (TD + 1) + tt] = (l < a.nl && tt < td) ? a.C[l * d + t0 + tt] : 0.0f;
        }
        __syncthreads();
        if (lv) {
          for (int tt = 0; tt < td; ++tt) {
            const double c = (double)ct[tid * (TD + 1) + tt];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              double df = __dsub_rn(xs[r * d + t0 + tt], c);
              acc[r] = __dadd_rn(acc[r], __dmul_rn(df, df));
            }
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int r = 0; r < R; ++r) dk[r * TL + tid] = lv ? dbits(acc[r]) : kKeyInf;
      __syncthreads();

      // merge this tile into each row's running first-L
      for (int r = warp; r < nr; r += PNW) {
        uint64_t* keys = bk + (size_t)r * cap;
        uint32_t* ids = bi + (size_t)r * cap;
        int cnt = bcnt[r];
        uint64_t tk = kKeyInf;
        uint32_t ti = 0xFFFFFFFFu;
        if (cnt == L) { tk = keys[L - 1]; ti = ids[L - 1]; }
        int added = 0;
        for (int i = lane; i < TL; i += 32) {
          uint64_t k = dk[r * TL + i];
          uint32_t id = (uint32_t)(l0 + i);
          bool pass = (l0 + i < a.nl) && (k < tk || (k == tk && id < ti));
          unsigned bal = __ballot_sync(0xffffffffu, pass);
          if (pass) {
            int pos = cnt + added + __popc(bal & ((1u << lane) - 1u));
            keys[pos] = k;
            ids[pos] = id;
          }
          added += __popc(bal);
        }
        __syncwarp();
        if (added > 0) {
          int tot = cnt + added;
          int np = 2;
          while (np < tot) np <<= 1;
          for (int i = tot + lane; i < np; i += 32) { keys[i] = kKeyInf; ids[i] = 0xFFFFFFFFu; }
          __syncwarp();
          warp_sort_pairs(keys, ids, np);
          cnt = min(tot, L);
        }
        if (lane == 0) bcnt[r] = cnt;
        __syncwarp();
      }
      __syncthreads();
    }

    // per-row output
    for (int r = warp; r < nr; r += PNW) {
      const int64_t row = r0 + r;
      const uint64_t* keys = bk + (size_t)r * cap;
      const uint32_t* ids = bi + (size_t)r * cap;
      if (a.mode == 0) {
        for (int j = lane; j < L; j += 32) {
          if (a.out_idx) a.out_idx[row * L + j] = (int32_t)ids[j];
          if (a.out_idx64) a.out_idx64[row * L + j] = (int64_t)ids[j];
          if (a.out_d64) a.out_d64[row * L + j] = __longlong_as_double((long long)keys[j]);
        }
      } else if (a.mode == 2) {
        if (lane == 0) { a.l1[row] = (int32_t)ids[0]; a.l2[row] = (int32_t)ids[0]; }
      } else {
        // Alg. 3 lines 3-11: loss_i = L2sqr(r_i) + lambda * <r_0, r_i>, fp64 ordered
        const int start = a.strict ? 1 : 0;
        double loss = 0.0;
        bool ok = (lane >= start) && (lane < L);
        if (ok) {
          const float* c0 = a.C + (int64_t)ids[0] * d;
          const float* ci = a.C + (int64_t)ids[lane] * d;
          const double* x = xs + r * d;
          double ss = 0.0, ip = 0.0, rr = 0.0;
          for (int t = 0; t < d; ++t) {
            double r0t = __dsub_rn((double)c0[t], x[t]);
            double rit = __dsub_rn((double)ci[t], x[t]);
            ss = __dadd_rn(ss, __dmul_rn(rit, rit));
            ip = __dadd_rn(ip, __dmul_rn(r0t, rit));
            rr = __dadd_rn(rr, __dmul_rn(r0t, r0t));
          }
          loss = second_list_loss(a.mode, a.lambda, ss, ip, rr);
        }
        // first argmin over lanes (loss, lane)
        int best = ok ? lane : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          double l2 = __shfl_xor_sync(0xffffffffu, loss, o);
          int b2 = __shfl_xor_sync(0xffffffffu, best, o);
          bool ok2 = b2 != 0x7fffffff;
          if (ok2 && (best == 0x7fffffff || l2 < loss || (l2 == loss && b2 < best))) {
            loss = l2;
            best = b2;
          }
        }
        if (lane == 0) {
          int c0 = (int)ids[0], cb = (int)ids[best];
          a.l1[row] = min(c0, cb);
          a.l2[row] = max(c0, cb);
        }
      }
    }
    __syncthreads();
  }
}

template <int R>
static rairs_status launch_probe_R(const ProbeArgs& a, cudaStream_t s) {
  ProbeSmem ps = probe_smem(R, a.d, a.L);
  if (ps.total > 220 * 1024) {
    set_error("probe_exact: shared memory budget exceeded (d or L too large)");
    return RAIRS_E_UNSUPPORTED;
  }
  RAIRS_CUDA_TRY(cudaFuncSetAttribute(probe_exact_kernel<R>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps.total));
  int64_t groups = ceil_div(a.rows, R);
  // fallback mode (only_flagged): usually no row is flagged, so a small
  // persistent grid just scans the flags (one resident wave, no launch tail)
  int grid = (int)std::min<int64_t>(groups, a.only_flagged ? 148 * 2 : 148 * 8);
  if (grid < 1) return RAIRS_OK;
  if (a.flag_count) {
    RAIRS_CUDA_TRY(launch_pdl(probe_exact_kernel<R>, dim3(grid), dim3(PT), ps.total, s, a, ps));
  } else {
    probe_exact_kernel<R><<<grid, PT, ps.total, s>>>(a, ps);
    RAIRS_CHECK_LAUNCH();
  }
  return RAIRS_OK;
}

// ---------------------------------------------------------------------------
// Exact fallback for a FEW flagged rows over MANY lists (large nlist): each
// flagged row is split over PX_S centroid ranges handled by different CTAs
// (exact fp64 ordered D64 per (row, list), O1; per-range first L by (D64, l)),
// then one CTA per row merges the PX_S partial lists and writes the same
// outputs as probe_exact_kernel (probes / RAIR pair / single).  Rows beyond
// PX_CAP keep their flag for the tiled exact kernel.
constexpr int PX_S = 64;
constexpr int PX_T = 256;

__device__ void cta_sort_pairs(uint64_t* k, uint32_t* id, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool asc = ((lo & size) == 0);
        const uint64_t ka = k[lo], kb = k[hi];
        const uint32_t ia = id[lo], ib = id[hi];
        const bool gt = (ka > kb) || (ka == kb && ia > ib);
        if (gt == asc) { k[lo] = kb; k[hi] = ka; id[lo] = ib; id[hi] = ia; }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(PX_T) probe_split_kernel(ProbeArgs a,
                                                           const uint32_t* __restrict__ list,
                                                           const uint32_t* __restrict__ count,
                                                           int per, int npow,
                                                           uint64_t* __restrict__ tk,
                                                           uint32_t* __restrict__ ti) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm);
  uint32_t* ids = reinterpret_cast<uint32_t*>(keys + npow);
  double* xs = reinterpret_cast<double*>(ids + npow + (npow & 1));
  float* tile = reinterpret_cast<float*>(xs + a.d);  // [PX_T][33]
  pdl_wait();  // launched with launch_pdl: the flagged-row list and count of the previous kernel
  const int64_t n = min(*count, (uint32_t)PX_CAP);
  for (int64_t w = blockIdx.x; w < n * PX_S; w += gridDim.x) {
    const int64_t i = w / PX_S;
    const int sp = (int)(w - i * PX_S);
    const int64_t r = list[i];
    for (int t = threadIdx.x; t < a.d; t += PX_T) xs[t] = (double)a.X[r * a.d + t];
    __syncthreads();
    const int64_t l0 = (int64_t)sp * per;
    // PX_T centroids per pass; their rows staged 32 dims at a time in a padded
    // shared tile (warp w loads rows 32w.. coalesced, lane = dimension, 32
    // loads in flight), then thread e extends centroid e's ordered fp64 sum
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    for (int e0 = 0; e0 < npow; e0 += PX_T) {
      const int e = e0 + threadIdx.x;
      const int64_t l = l0 + e;
      const bool valid = e < per && l < a.nl;
      double acc = 0.0;
      for (int t0 = 0; t0 < a.d; t0 += 32) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int ee = e0 + wp * 32 + i;
          const int64_t rl = l0 + ee;
          v[i] = (ee < per && rl < a.nl && t0 + lane < a.d) ? __ldg(a.C + rl * a.d + t0 + lane) : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) tile[(wp * 32 + i) * 33 + lane] = v[i];
        __syncthreads();
        if (valid) {
          const int dc = min(32, a.d - t0);
          for (int t = 0; t < dc; ++t) {  // ascending t, fp64 ordered (O1)
            const double df = __dsub_rn(xs[t0 + t], (double)tile[threadIdx.x * 33 + t]);
            acc = __dadd_rn(acc, __dmul_rn(df, df));
          }
        }
        __syncthreads();
      }
      keys[e] = valid ? dbits(acc) : kKeyInf;
      ids[e] = (uint32_t)l;
    }
    __syncthreads();
    cta_sort_pairs(keys, ids, npow);
    for (int j = threadIdx.x; j < a.L; j += PX_T) {
      tk[(i * PX_S + sp) * a.L + j] = j < npow ? keys[j] : kKeyInf;
      ti[(i * PX_S + sp) * a.L + j] = j < npow ? ids[j] : 0xFFFFFFFFu;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(PX_T) probe_merge_kernel(ProbeArgs a,
                                                           const uint32_t* __restrict__ list,
                                                           const uint32_t* __restrict__ count,
                                                           int npow, const uint64_t* __restrict__ tk,
                                                           const uint32_t* __restrict__ ti,
                                                           int32_t* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm);
  uint32_t* ids = reinterpret_cast<uint32_t*>(keys + npow);
  pdl_wait();  // launched with launch_pdl: the flagged-row list and count of the previous kernel
  const int64_t n = min(*count, (uint32_t)PX_CAP);
  const int L = a.L, lane = lane_id(), warp = warp_id();
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t row = list[i];
    for (int e = threadIdx.x; e < npow; e += PX_T) {
      const bool v = e < PX_S * L;
      keys[e] = v ? tk[i * PX_S * L + e] : kKeyInf;
      ids[e] = v ? ti[i * PX_S * L + e] : 0xFFFFFFFFu;
    }
    __syncthreads();
    cta_sort_pairs(keys, ids, npow);
    if (a.mode == 0) {
      for (int j = threadIdx.x; j < L; j += PX_T) {
        if (a.out_idx) a.out_idx[row * L + j] = (int32_t)ids[j];
        if (a.out_idx64) a.out_idx64[row * L + j] = (int64_t)ids[j];
        if (a.out_d64) a.out_d64[row * L + j] = __longlong_as_double((long long)keys[j]);
      }
    } else if (a.mode == 2) {
      if (threadIdx.x == 0) { a.l1[row] = (int32_t)ids[0]; a.l2[row] = (int32_t)ids[0]; }
    } else if (warp == 0) {
      // Alg. 3 lines 3-11 over the first L = N_CANDS exact lists (fp64, O4)
      const int start = a.strict ? 1 : 0;
      double loss = 0.0;
      const bool ok = (lane >= start) && (lane < L);
      if (ok) {
        const float* c0 = a.C + (int64_t)ids[0] * a.d;
        const float* cj = a.C + (int64_t)ids[lane] * a.d;
        const float* xr = a.X + row * a.d;
        double ss = 0.0, ip = 0.0, rr = 0.0;
        for (int t = 0; t < a.d; ++t) {
          const double x = (double)xr[t];
          const double r0t = __dsub_rn((double)c0[t], x);
          const double rjt = __dsub_rn((double)cj[t], x);
          ss = __dadd_rn(ss, __dmul_rn(rjt, rjt));
          ip = __dadd_rn(ip, __dmul_rn(r0t, rjt));
          rr = __dadd_rn(rr, __dmul_rn(r0t, r0t));
        }
        loss = second_list_loss(a.mode, a.lambda, ss, ip, rr);
      }
      int best = ok ? lane : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double l2v = __shfl_xor_sync(0xffffffffu, loss, o);
        const int b2 = __shfl_xor_sync(0xffffffffu, best, o);
        if (b2 != 0x7fffffff && (best == 0x7fffffff || l2v < loss || (l2v == loss && b2 < best))) {
          loss = l2v;
          best = b2;
        }
      }
      if (lane == 0) {
        const int c0 = (int)ids[0], cb = (int)ids[best];
        a.l1[row] = min(c0, cb);
        a.l2[row] = max(c0, cb);
      }
    }
    if (threadIdx.x == 0 && flags) flags[row] = 0;  // done: the tiled kernel skips it
    __syncthreads();
  }
}

// Split-path exact fallback for flagged rows (large nlist); leaves flags set
// only for rows it did not handle.  prepare: the workspace when the shape
// qualifies (b.on), before the certify kernel that fills b.list / *count (no
// separate compaction kernel or memset); launch: probe_split_kernel +
// probe_merge_kernel (with no flagged row both exit at once).
rairs_status probe_split_prepare(const ProbeArgs& a, ProbeSplitBufs& b, cudaStream_t s) {
  b = ProbeSplitBufs{};
  static const bool off = [] {  // RAIRS_COARSE_SPLIT=0: the tiled exact kernel takes every flagged row
    const char* e = std::getenv("RAIRS_COARSE_SPLIT");
    return e && std::atoi(e) == 0;
  }();
  if (a.rows <= 0 || a.nl < 8192 || off) return RAIRS_OK;
  b.per = (int)ceil_div(a.nl, PX_S);
  b.npow_s = next_pow2(std::max(b.per, a.L));
  b.npow_m = next_pow2(PX_S * a.L);
  b.sm_s = (size_t)b.npow_s * 12 + 8 + (size_t)a.d * 8 + (size_t)PX_T * 33 * 4;
  b.sm_m = (size_t)b.npow_m * 12 + 8;
  if (b.sm_s > 200 * 1024 || b.sm_m > 200 * 1024) return RAIRS_OK;
  cudaError_t e = ws_malloc(&b.list, PX_CAP * 4, s);
  if (e == cudaSuccess) e = ws_malloc(&b.tk, (size_t)PX_CAP * PX_S * a.L * 8, s);
  if (e == cudaSuccess) e = ws_malloc(&b.ti, (size_t)PX_CAP * PX_S * a.L * 4, s);
  if (e != cudaSuccess) {
    probe_split_free(b, s);
    set_error(std::string("probe split workspace: ") + cudaGetErrorString(e));
    return RAIRS_E_OOM;
  }
  b.on = true;
  return RAIRS_OK;
}

rairs_status probe_split_launch(const ProbeArgs& a, const ProbeSplitBufs& b, const uint32_t* count,
                                int32_t* flags, cudaStream_t s) {
  if (!b.on) return RAIRS_OK;
  // programmatic dependent launches: both kernels wait (griddepcontrol.wait)
  // before reading the list / count / partial lists of their predecessor (an
  // earlier PDL version without the waits read them too early and faulted)
  RAIRS_CUDA_TRY(cudaFuncSetAttribute(probe_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b.sm_s));
  RAIRS_CUDA_TRY(launch_pdl(probe_split_kernel, dim3(148 * 4), dim3(PX_T), b.sm_s, s, a,
                            (const uint32_t*)b.list, count, b.per, b.npow_s, b.tk, b.ti));
  RAIRS_CUDA_TRY(cudaFuncSetAttribute(probe_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b.sm_m));
  RAIRS_CUDA_TRY(launch_pdl(probe_merge_kernel, dim3(148 * 2), dim3(PX_T), b.sm_m, s, a,
                            (const uint32_t*)b.list, count, b.npow_m, (const uint64_t*)b.tk,
                            (const uint32_t*)b.ti, flags));
  return RAIRS_OK;
}

__global__ void probe_iota_kernel(uint32_t* list, uint32_t* count, uint32_t rows) {
  for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) list[i] = i;
  if (threadIdx.x == 0) *count = rows;
}

// Small batches (rows <= PX_CAP - 1, large nlist): every row through the split
// exact path (O1 for all rows: no TF32 GEMM, no certificate).  *done = false
// when the shape does not qualify (the caller takes the fused path).
rairs_status launch_probe_split_all(const ProbeArgs& a, cudaStream_t s, bool* done) {
  *done = false;
  if (a.rows <= 0 || a.rows >= PX_CAP || a.mode != 0) return RAIRS_OK;
  ProbeSplitBufs b;
  RAIRS_TRY(probe_split_prepare(a, b, s));
  if (!b.on) return RAIRS_OK;
  uint32_t* count = b.list + (PX_CAP - 1);  // past the rows: the row count
  probe_iota_kernel<<<1, 256, 0, s>>>(b.list, count, (uint32_t)a.rows);
  rairs_status st = probe_split_launch(a, b, count, nullptr, s);
  probe_split_free(b, s);
  if (st == RAIRS_OK) *done = true;
  return st;
}

void probe_split_free(ProbeSplitBufs& b, cudaStream_t s) {
  cudaFreeAsync(b.list, s);
  cudaFreeAsync(b.tk, s);
  cudaFreeAsync(b.ti, s);
  b = ProbeSplitBufs{};
}

rairs_status launch_probe_exact(const ProbeArgs& a, cudaStream_t s) {
  if (a.rows <= 0) return RAIRS_OK;
  if (a.L < 1 || a.L > 1024 || a.L > a.nl) {
    set_error("probe_exact: bad L");
    return RAIRS_E_INVALID;
  }
  if ((a.mode == 1 || a.mode == 3) && a.L > 32) {
    set_error("probe_exact: n_cands must be <= 32");
    return RAIRS_E_UNSUPPORTED;
  }
  // rows per CTA: amortise the centroid tile over R rows while fitting smem
  for (int R : {8, 4, 2, 1}) {
    if (probe_smem(R, a.d, a.L).total <= 200 * 1024 || R == 1) {
      switch (R) {
        case 8: return launch_probe_R<8>(a, s);
        case 4: return launch_probe_R<4>(a, s);
        case 2: return launch_probe_R<2>(a, s);
        default: return launch_probe_R<1>(a, s);
      }
    }
  }
  return RAIRS_E_INTERNAL;
}

// ===========================================================================
// Training (not in the bit-exact contract; deterministic for a fixed seed).
// ===========================================================================
static uint64_t splitmix64(uint64_t& st) {
  uint64_t z = (st += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// first `cnt` entries of a seeded partial Fisher-Yates permutation of [0, n)
static std::vector<int64_t> sample_rows(int64_t n, int64_t cnt, uint64_t seed) {
  std::vector<int64_t> perm;
  if (cnt >= n) {
    perm.resize(n);
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    // still shuffle the first entries so init centroids are random rows
    uint64_t st = seed;
    for (int64_t i = 0; i < n - 1 && i < 65536; ++i) {
      int64_t j = i + (int64_t)(splitmix64(st) % (uint64_t)(n - i));
      std::swap(perm[i], perm[j]);
    }
    return perm;
  }
  // Floyd's algorithm for cnt distinct rows, then a seeded shuffle of their order
  uint64_t st = seed;
  std::vector<bool> taken((size_t)n, false);
  std::vector<int64_t> chosen;
  chosen.reserve(cnt);
  for (int64_t j = n - cnt; j < n; ++j) {
    int64_t t = (int64_t)(splitmix64(st) % (uint64_t)(j + 1));
    int64_t v = taken[(size_t)t] ? j : t;
    taken[(size_t)v] = true;
    chosen.push_back(v);
  }
  for (int64_t i = (int64_t)chosen.size() - 1; i > 0; --i) {
    int64_t j = (int64_t)(splitmix64(st) % (uint64_t)(i + 1));
    std::swap(chosen[i], chosen[j]);
  }
  return chosen;
}

__global__ void gather_rows_kernel(const float* __restrict__ X, const int64_t* __restrict__ idx,
                                   int64_t cnt, int d, float* __restrict__ out) {
  int64_t total = cnt * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / d;
    int t = (int)(e - r * d);
    out[e] = X[idx[r] * d + t];
  }
}

__global__ void seg_bounds_i32_kernel(const int32_t* __restrict__ keys, int64_t n,
                                      int32_t* __restrict__ seg_start, int32_t* __restrict__ seg_end) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    int32_t k = keys[p];
    if (p == 0 || keys[p - 1] != k) seg_start[k] = (int32_t)p;
    if (p == n - 1 || keys[p + 1] != k) seg_end[k] = (int32_t)(p + 1);
  }
}

__global__ void iota_i32_kernel(int32_t* v, int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    v[p] = (int32_t)p;
}

// centroid l = mean of its members, summed in sorted (point index) order in fp64
__global__ void kmeans_update_kernel(const float* __restrict__ Xt, int d,
                                     const int32_t* __restrict__ sorted_idx,
                                     const int32_t* __restrict__ seg_start,
                                     const int32_t* __restrict__ seg_end,
                                     float* __restrict__ cent) {
  const int l = blockIdx.x;
  const int s = seg_start[l], e = seg_end[l];
  if (e <= s) return;
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    double acc = 0.0;
    for (int p = s; p < e; ++p) acc += (double)Xt[(int64_t)sorted_idx[p] * d + t];
    cent[(int64_t)l * d + t] = (float)(acc / (double)(e - s));
  }
}

static inline unsigned grid_for(int64_t n, int bs = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, bs), 148 * 32));
}

// RAIRS_DEBUG_SYNC=1: synchronise after every training step and name the
// failing one (debugging aid; off by default, no effect on results)
static bool debug_sync() {
  static const bool on = [] {
    const char* e = getenv("RAIRS_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}
#define KM_DEBUG_STEP(name)                                                           \
  do {                                                                                \
    if (debug_sync()) {                                                               \
      cudaError_t _e = cudaStreamSynchronize(s);                                      \
      if (_e != cudaSuccess) {                                                        \
        set_error(std::string("train_kmeans step ") + (name) + ": " + cudaGetErrorString(_e)); \
        cleanup();                                                                    \
        return RAIRS_E_CUDA;                                                          \
      }                                                                               \
    }                                                                                 \
  } while (0)

rairs_status train_kmeans(const float* X, int64_t n, int d, int k, int iters, uint64_t seed,
                          int64_t max_train, float* cent, cudaStream_t s) {
  const int64_t nt = std::min<int64_t>(n, max_train > 0 ? max_train : (int64_t)256 * k);
  if (nt < k) {
    set_error("train_kmeans: fewer training rows than lists");
    return RAIRS_E_INVALID;
  }
  std::vector<int64_t> rows = sample_rows(n, nt, seed);
  int64_t* d_rows = nullptr;
  float* Xt = nullptr;
  int32_t *asg = nullptr, *asg_sorted = nullptr, *iota = nullptr, *idx_sorted = nullptr;
  int32_t *seg_s = nullptr, *seg_e = nullptr;
  unsigned* nflag = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  rairs_status st = RAIRS_OK;
  auto cleanup = [&]() {
    cudaStreamSynchronize(s);
    cudaFree(d_rows); cudaFree(Xt); cudaFree(asg); cudaFree(asg_sorted); cudaFree(iota);
    cudaFree(idx_sorted); cudaFree(seg_s); cudaFree(seg_e); cudaFree(tmp); cudaFree(nflag);
  };
#define KM_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { set_error(std::string(#x) + ": " + cudaGetErrorString(_e)); cleanup(); return _e == cudaErrorMemoryAllocation ? RAIRS_E_OOM : RAIRS_E_CUDA; } } while (0)
  KM_TRY(cudaMalloc(&d_rows, nt * sizeof(int64_t)));
  KM_TRY(cudaMalloc(&Xt, (size_t)nt * d * sizeof(float)));
  KM_TRY(cudaMalloc(&asg, nt * sizeof(int32_t)));
  KM_TRY(cudaMalloc(&asg_sorted, nt * sizeof(int32_t)));
  KM_TRY(cudaMalloc(&iota, nt * sizeof(int32_t)));
  KM_TRY(cudaMalloc(&idx_sorted, nt * sizeof(int32_t)));
  KM_TRY(cudaMalloc(&seg_s, k * sizeof(int32_t)));
  KM_TRY(cudaMalloc(&seg_e, k * sizeof(int32_t)));
  KM_TRY(cudaMemcpyAsync(d_rows, rows.data(), nt * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  gather_rows_kernel<<<grid_for(nt * d), 256, 0, s>>>(X, d_rows, nt, d, Xt);
  KM_DEBUG_STEP("gather");
  // init: the first k sampled rows (distinct rows of X)
  KM_TRY(cudaMemcpyAsync(cent, Xt, (size_t)k * d * sizeof(float), cudaMemcpyDeviceToDevice, s));
  iota_i32_kernel<<<grid_for(nt), 256, 0, s>>>(iota, nt);
  int end_bit = 1;
  while ((1ll << end_bit) < k) ++end_bit;
  KM_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, asg, asg_sorted, iota, idx_sorted,
                                         (int)nt, 0, end_bit, s));
  KM_TRY(cudaMalloc(&tmp, tmp_bytes));
  std::vector<int32_t> hs(k), he(k);
  std::vector<float> hc;
  // large nlist: assignment on tensor cores (fp64 over k x d per row is too slow)
  const bool use_tc = k >= 1024 && (d & 3) == 0 && tma_available();
  if (use_tc) KM_TRY(cudaMalloc(&nflag, sizeof(unsigned)));
  for (int it = 0; it < iters; ++it) {
    if (use_tc) {
      // nearest centroid through the tensor-core coarse path (TF32 filter +
      // fp64 certification + exact fallback: the same argmin as probe_exact)
      rairs_index_s tmp{};
      tmp.centroids = cent;
      tmp.nlist = k;
      tmp.d = d;
      st = coarse_prepare(&tmp, s);
      if (st == RAIRS_OK)
        st = launch_coarse_fused(&tmp, Xt, nt, 1, 0, 0.0, 0, asg, nullptr, nullptr, nflag, s);
      cudaFreeAsync(tmp.cnorm, s);
      if (st == RAIRS_OK) KM_DEBUG_STEP("coarse_fused");
    } else {
      ProbeArgs pa{};
      pa.X = Xt; pa.rows = nt; pa.d = d; pa.C = cent; pa.nl = k; pa.L = 1; pa.mode = 0;
      pa.out_idx = asg;
      st = launch_probe_exact(pa, s);
    }
    if (st != RAIRS_OK) { cleanup(); return st; }
    KM_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, asg, asg_sorted, iota, idx_sorted,
                                           (int)nt, 0, end_bit, s));
    KM_DEBUG_STEP("sort");
    KM_TRY(cudaMemsetAsync(seg_s, 0, k * sizeof(int32_t), s));
    KM_TRY(cudaMemsetAsync(seg_e, 0, k * sizeof(int32_t), s));
    seg_bounds_i32_kernel<<<grid_for(nt), 256, 0, s>>>(asg_sorted, nt, seg_s, seg_e);
    kmeans_update_kernel<<<k, 128, 0, s>>>(Xt, d, idx_sorted, seg_s, seg_e, cent);
    KM_TRY(cudaGetLastError());
    KM_DEBUG_STEP("update");
    // empty clusters: split the largest (host side, deterministic)
    KM_TRY(cudaMemcpyAsync(hs.data(), seg_s, k * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    KM_TRY(cudaMemcpyAsync(he.data(), seg_e, k * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    KM_TRY(cudaStreamSynchronize(s));
    std::vector<int64_t> cnt(k);
    bool any_empty = false;
    for (int l = 0; l < k; ++l) { cnt[l] = he[l] - hs[l]; any_empty |= (cnt[l] == 0); }
    if (any_empty) {
      hc.resize((size_t)k * d);
      KM_TRY(cudaMemcpyAsync(hc.data(), cent, hc.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
      KM_TRY(cudaStreamSynchronize(s));
      // max-heap on (count, -index): the same choice as a linear scan for the
      // first largest cluster, in O(log k) per empty cluster
      std::priority_queue<std::pair<int64_t, int>> heap;
      for (int j = 0; j < k; ++j) heap.push({cnt[j], -j});
      for (int l = 0; l < k; ++l) {
        if (cnt[l] > 0) continue;
        while (heap.top().first != cnt[-heap.top().second]) heap.pop();  // stale entries
        const int big = -heap.top().second;
        heap.pop();
        for (int t = 0; t < d; ++t) {
          float v = hc[(size_t)big * d + t];
          float eps = (v != 0.0f ? std::fabs(v) : 1.0f) / 1024.0f;
          hc[(size_t)l * d + t] = v + eps;
          hc[(size_t)big * d + t] = v - eps;
        }
        cnt[l] = cnt[big] / 2;
        cnt[big] -= cnt[l];
        heap.push({cnt[big], -big});
        heap.push({cnt[l], -l});
      }
      KM_TRY(cudaMemcpyAsync(cent, hc.data(), hc.size() * sizeof(float), cudaMemcpyHostToDevice, s));
      KM_TRY(cudaStreamSynchronize(s));
    }
  }
  KM_TRY(cudaStreamSynchronize(s));
  cleanup();
  return RAIRS_OK;
#undef KM_TRY
}

// PQ: one CTA per subquantizer, Lloyd iterations in fp64 with deterministic
// serial-per-(j,t) centroid sums.
__global__ void pq_kmeans_kernel(const float* __restrict__ Xt, int64_t nt, int d, int dsub,
                                 int iters, const int64_t* __restrict__ init_rows /*[M][16]*/,
                                 uint8_t* __restrict__ asg_all /*[M][nt]*/,
                                 float* __restrict__ codebook) {
  const int m = blockIdx.x;
  __shared__ double cent[16 * 8];
  __shared__ int64_t cnt[16];
  uint8_t* asg = asg_all + (int64_t)m * nt;
  for (int e = threadIdx.x; e < 16 * dsub; e += blockDim.x) {
    int j = e / dsub, t = e - j * dsub;
    cent[e] = (double)Xt[init_rows[m * 16 + j] * d + (int64_t)m * dsub + t];
  }
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    for (int64_t p = threadIdx.x; p < nt; p += blockDim.x) {
      const float* x = Xt + p * d + (int64_t)m * dsub;
      int bj = 0;
      double bd = 0.0;
      for (int j = 0; j < 16; ++j) {
        double acc = 0.0;
        for (int t = 0; t < dsub; ++t) {
          double df = __dsub_rn((double)x[t], cent[j * dsub + t]);
          acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
        if (j == 0 || acc < bd) { bj = j; bd = acc; }
      }
      asg[p] = (uint8_t)bj;
    }
    __syncthreads();
    double nv = 0.0;
    int64_t c = 0;
    const int e = threadIdx.x;
    if (e < 16 * dsub) {
      int j = e / dsub, t = e - j * dsub;
      for (int64_t p = 0; p < nt; ++p) {
        if (asg[p] == j) { nv += (double)Xt[p * d + (int64_t)m * dsub + t]; ++c; }
      }
    }
    __syncthreads();
    if (e < 16 * dsub) {
      int j = e / dsub;
      if (c > 0) cent[e] = nv / (double)c;
      if (e % dsub == 0) cnt[j] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int j = 0; j < 16; ++j) {
        if (cnt[j] > 0) continue;
        int big = 0;
        for (int i = 1; i < 16; ++i) if (cnt[i] > cnt[big]) big = i;
        for (int t = 0; t < dsub; ++t) {
          double v = cent[big * dsub + t];
          double eps = (v != 0.0 ? fabs(v) : 1.0) / 1024.0;
          cent[j * dsub + t] = v + eps;
          cent[big * dsub + t] = v - eps;
        }
        cnt[j] = cnt[big] / 2;
        cnt[big] -= cnt[j];
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < 16 * dsub; e += blockDim.x)
    codebook[(int64_t)m * 16 * dsub + e] = (float)cent[e];
}

rairs_status train_pq(const float* X, int64_t n, int d, int M, int iters, uint64_t seed,
                      int64_t max_train, float* codebook, cudaStream_t s) {
  const int dsub = d / M;
  if (dsub > 8) {
    set_error("train_pq: d/M > 8 unsupported");
    return RAIRS_E_UNSUPPORTED;
  }
  const int64_t nt = std::min<int64_t>(n, max_train > 0 ? max_train : 65536);
  if (nt < 16) {
    set_error("train_pq: need at least 16 training rows");
    return RAIRS_E_INVALID;
  }
  std::vector<int64_t> rows = sample_rows(n, nt, seed ^ 0x5A5A5A5A12345678ull);
  std::vector<int64_t> init((size_t)M * 16);
  for (int m = 0; m < M; ++m) {
    std::vector<int64_t> pick = sample_rows(nt, 16, seed + 0x1000003ull * (uint64_t)(m + 1));
    for (int j = 0; j < 16; ++j) init[(size_t)m * 16 + j] = pick[j];
  }
  int64_t *d_rows = nullptr, *d_init = nullptr;
  float* Xt = nullptr;
  uint8_t* asg = nullptr;
  auto cleanup = [&]() { cudaFree(d_rows); cudaFree(d_init); cudaFree(Xt); cudaFree(asg); };
#define PQ_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { set_error(std::string(#x) + ": " + cudaGetErrorString(_e)); cleanup(); return _e == cudaErrorMemoryAllocation ? RAIRS_E_OOM : RAIRS_E_CUDA; } } while (0)
  PQ_TRY(cudaMalloc(&d_rows, nt * sizeof(int64_t)));
  PQ_TRY(cudaMalloc(&d_init, init.size() * sizeof(int64_t)));
  PQ_TRY(cudaMalloc(&Xt, (size_t)nt * d * sizeof(float)));
  PQ_TRY(cudaMalloc(&asg, (size_t)M * nt));
  PQ_TRY(cudaMemcpyAsync(d_rows, rows.data(), nt * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  PQ_TRY(cudaMemcpyAsync(d_init, init.data(), init.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  gather_rows_kernel<<<grid_for(nt * d), 256, 0, s>>>(X, d_rows, nt, d, Xt);
  pq_kmeans_kernel<<<M, 256, 0, s>>>(Xt, nt, d, dsub, iters, d_init, asg, codebook);
  PQ_TRY(cudaGetLastError());
  PQ_TRY(cudaStreamSynchronize(s));
  cleanup();
  return RAIRS_OK;
#undef PQ_TRY
}

// ===========================================================================
// Cell-major SEIL layout (Alg. 4 reading R10).
// Sort key (l1:17 | l2:17 | row:30) -> list l's owned region = the sorted run
// with l1 == l (cells (l, j>=l) in ascending j, rows ascending), padded to a
// multiple of 32 slots.  Codes are packed per 32-slot block as
// [unit u = 16 subquantizers][lane][8 B], nibble i of unit u = subquantizer
// 16u+i (bits 4i..4i+3).
// ===========================================================================
// cell-major sort key (l1, l2, row); deleted rows sort last (key ~0)
__global__ void make_keys_kernel(const int32_t* __restrict__ l1, const int32_t* __restrict__ l2,
                                 const uint32_t* __restrict__ live_bits, int64_t n,
                                 uint64_t* __restrict__ keys) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const bool live = live_bits == nullptr || ((live_bits[r >> 5] >> (r & 31)) & 1u);
    keys[r] = live ? (((uint64_t)l1[r] << 47) | ((uint64_t)l2[r] << 30) | (uint64_t)r) : ~0ull;
  }
}

__global__ void list_bounds_kernel(const uint64_t* __restrict__ sk, int64_t n, int shift,
                                   uint32_t mask, uint32_t* __restrict__ s_start,
                                   uint32_t* __restrict__ s_end) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t l = (uint32_t)(sk[p] >> shift) & mask;
    if (p == 0 || (((uint32_t)(sk[p - 1] >> shift) & mask) != l)) s_start[l] = (uint32_t)p;
    if (p == n - 1 || (((uint32_t)(sk[p + 1] >> shift) & mask) != l)) s_end[l] = (uint32_t)(p + 1);
  }
}

// thread per (sorted position p, unit u): slot mapping + PQ encode (O5) + pack
__global__ void fill_slots_kernel(const uint64_t* __restrict__ sk, int64_t n,
                                  const uint32_t* __restrict__ own_off,
                                  const uint32_t* __restrict__ seg_start,
                                  const float* __restrict__ X, int d, int M, int dsub, int NU,
                                  const float* __restrict__ codebook,
                                  uint32_t* __restrict__ slot_rows, uint64_t* __restrict__ codes64) {
  const int64_t total = n * NU;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / NU;
    const int u = (int)(e - p * NU);
    const uint64_t key = sk[p];
    const uint32_t l = (uint32_t)(key >> 47);
    const uint32_t r = (uint32_t)(key & ((1ull << 30) - 1));
    const uint64_t slot = (uint64_t)own_off[l] + (uint64_t)(p - seg_start[l]);
    if (u == 0) slot_rows[slot] = r;
    uint64_t w = 0;
    for (int i = 0; i < 16; ++i) {
      const int m = u * 16 + i;
      if (m >= M) break;
      const float* xs = X + (int64_t)r * d + (int64_t)m * dsub;
      int bj = 0;
      double bd = 0.0;
      for (int j = 0; j < 16; ++j) {
        const float* c = codebook + ((int64_t)m * 16 + j) * dsub;
        double acc = 0.0;
        for (int t = 0; t < dsub; ++t) {
          double df = __dsub_rn((double)xs[t], (double)c[t]);
          acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
        if (j == 0 || acc < bd) { bj = j; bd = acc; }
      }
      w |= (uint64_t)bj << (4 * i);
    }
    const uint64_t blk = slot >> 5, lane = slot & 31;
    codes64[(blk * NU + u) * 32 + lane] = w;
  }
}

// one thread per cell start: emit a reference for cells with l1 < l2
__global__ void cells_kernel(const uint64_t* __restrict__ sk, int64_t n,
                             const uint32_t* __restrict__ own_off,
                             const uint32_t* __restrict__ seg_start,
                             unsigned long long* __restrict__ counters /*0 refs, 1 cells, 2 double*/,
                             uint64_t* __restrict__ ref_key, uint64_t* __restrict__ ref_val) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t ck = sk[p] >> 30;
    if (p > 0 && (sk[p - 1] >> 30) == ck) continue;
    int64_t e = p + 1;
    while (e < n && (sk[e] >> 30) == ck) ++e;
    const uint32_t l1 = (uint32_t)(ck >> 17), l2 = (uint32_t)(ck & 0x1FFFF);
    atomicAdd(&counters[1], 1ull);
    if (l1 < l2) {
      atomicAdd(&counters[2], (unsigned long long)(e - p));
      unsigned long long pos = atomicAdd(&counters[0], 1ull);
      const uint32_t start = own_off[l1] + (uint32_t)(p - seg_start[l1]);
      ref_key[pos] = ((uint64_t)l2 << 17) | l1;
      ref_val[pos] = ((uint64_t)start << 32) | (uint64_t)(uint32_t)(e - p);
    }
  }
}

__global__ void refs_finalize_kernel(const uint64_t* __restrict__ rk_sorted,
                                     const uint64_t* __restrict__ rv_sorted, int64_t nr,
                                     int32_t* __restrict__ ref_owner,
                                     uint32_t* __restrict__ ref_start,
                                     uint32_t* __restrict__ ref_cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr;
       i += (int64_t)gridDim.x * blockDim.x) {
    ref_owner[i] = (int32_t)(rk_sorted[i] & 0x1FFFF);
    ref_start[i] = (uint32_t)(rv_sorted[i] >> 32);
    ref_cnt[i] = (uint32_t)(rv_sorted[i] & 0xFFFFFFFFu);
  }
}

// The previous layout of a rebuild (rairs_add / rairs_remove_ids) is kept until
// the new one is complete: on any failure the index keeps its old layout.
struct LayoutStash {
  rairs_index_s* idx;
  uint32_t *own_off, *own_cnt, *slot_rows, *ref_ptr, *ref_start, *ref_cnt;
  int32_t* ref_owner;
  uint8_t* codes;
  int64_t n_slots, n_refs, n_cells, n_double, layout_bytes;
  int max_refs;
  bool committed = false;
  explicit LayoutStash(rairs_index_s* x)
      : idx(x), own_off(x->own_off), own_cnt(x->own_cnt), slot_rows(x->slot_rows),
        ref_ptr(x->ref_ptr), ref_start(x->ref_start), ref_cnt(x->ref_cnt), ref_owner(x->ref_owner),
        codes(x->codes), n_slots(x->n_slots), n_refs(x->n_refs), n_cells(x->n_cells),
        n_double(x->n_double), layout_bytes(x->layout_bytes), max_refs(x->max_refs) {
    x->own_off = x->own_cnt = x->slot_rows = x->ref_ptr = x->ref_start = x->ref_cnt = nullptr;
    x->ref_owner = nullptr;
    x->codes = nullptr;
    x->layout_bytes = 0;
  }
  ~LayoutStash() {
    if (committed) {  // the new layout is in place: release the old one
      cudaFree(own_off); cudaFree(own_cnt); cudaFree(slot_rows); cudaFree(ref_ptr);
      cudaFree(ref_start); cudaFree(ref_cnt); cudaFree(ref_owner); cudaFree(codes);
      idx->device_bytes -= layout_bytes;
      return;
    }
    // failure: free the partial new layout, restore the old one
    cudaFree(idx->own_off); cudaFree(idx->own_cnt); cudaFree(idx->slot_rows); cudaFree(idx->ref_ptr);
    cudaFree(idx->ref_start); cudaFree(idx->ref_cnt); cudaFree(idx->ref_owner); cudaFree(idx->codes);
    idx->own_off = own_off; idx->own_cnt = own_cnt; idx->slot_rows = slot_rows; idx->ref_ptr = ref_ptr;
    idx->ref_start = ref_start; idx->ref_cnt = ref_cnt; idx->ref_owner = ref_owner; idx->codes = codes;
    idx->n_slots = n_slots; idx->n_refs = n_refs; idx->n_cells = n_cells; idx->n_double = n_double;
    idx->layout_bytes = layout_bytes; idx->max_refs = max_refs;
  }
};

rairs_status build_layout(rairs_index_s* idx, cudaStream_t s) {
  const int64_t n = idx->n;
  const int64_t n_live = idx->n_live;  // live rows: the first n_live sorted keys
  LayoutStash stash(idx);
  const int nlist = idx->nlist;
  const int NU = idx->M_pad / 16;
  uint64_t *keys = nullptr, *skeys = nullptr, *rk = nullptr, *rv = nullptr, *rk_s = nullptr,
           *rv_s = nullptr;
  uint32_t *seg_s = nullptr, *seg_e = nullptr, *rseg_s = nullptr, *rseg_e = nullptr;
  unsigned long long* counters = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, tb2 = 0;
  auto cleanup = [&]() {
    cudaFree(keys); cudaFree(skeys); cudaFree(rk); cudaFree(rv); cudaFree(rk_s); cudaFree(rv_s);
    cudaFree(seg_s); cudaFree(seg_e); cudaFree(rseg_s); cudaFree(rseg_e); cudaFree(counters);
    cudaFree(tmp);
  };
#define LY_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { set_error(std::string(#x) + ": " + cudaGetErrorString(_e)); cleanup(); return _e == cudaErrorMemoryAllocation ? RAIRS_E_OOM : RAIRS_E_CUDA; } } while (0)
  LY_TRY(cudaMalloc(&keys, n * sizeof(uint64_t)));
  LY_TRY(cudaMalloc(&skeys, n * sizeof(uint64_t)));
  LY_TRY(cudaMalloc(&seg_s, nlist * sizeof(uint32_t)));
  LY_TRY(cudaMalloc(&seg_e, nlist * sizeof(uint32_t)));
  LY_TRY(cudaMalloc(&counters, 4 * sizeof(unsigned long long)));
  make_keys_kernel<<<grid_for(n), 256, 0, s>>>(idx->l1, idx->l2, idx->live_bits, n, keys);
  LY_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, skeys, (int64_t)n, 0, 64, s));
  LY_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb2, keys, skeys, keys, skeys, (int64_t)n, 0, 64, s));
  tmp_bytes = std::max(tmp_bytes, tb2);
  LY_TRY(cudaMalloc(&tmp, tmp_bytes));
  LY_TRY(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, skeys, (int64_t)n, 0, 64, s));
  LY_TRY(cudaMemsetAsync(seg_s, 0, nlist * sizeof(uint32_t), s));
  LY_TRY(cudaMemsetAsync(seg_e, 0, nlist * sizeof(uint32_t), s));
  list_bounds_kernel<<<grid_for(n_live), 256, 0, s>>>(skeys, n_live, 47, 0x1FFFFu, seg_s, seg_e);
  std::vector<uint32_t> hs(nlist), he(nlist), hoff(nlist), hcnt(nlist);
  LY_TRY(cudaMemcpyAsync(hs.data(), seg_s, nlist * 4, cudaMemcpyDeviceToHost, s));
  LY_TRY(cudaMemcpyAsync(he.data(), seg_e, nlist * 4, cudaMemcpyDeviceToHost, s));
  LY_TRY(cudaStreamSynchronize(s));
  int64_t off = 0;
  for (int l = 0; l < nlist; ++l) {
    hcnt[l] = he[l] - hs[l];
    hoff[l] = (uint32_t)off;
    off += round_up(hcnt[l], kBlk);
  }
  if (off >= (int64_t)0xFFFFFFFFll) {
    set_error("layout: slot count exceeds 2^32");
    cleanup();
    return RAIRS_E_UNSUPPORTED;
  }
  idx->n_slots = off;
  const size_t code_bytes = (size_t)std::max<int64_t>(off, 32) * idx->M_pad / 2;
  LY_TRY(cudaMalloc(&idx->own_off, nlist * 4));
  LY_TRY(cudaMalloc(&idx->own_cnt, nlist * 4));
  LY_TRY(cudaMalloc(&idx->codes, code_bytes));
  LY_TRY(cudaMalloc(&idx->slot_rows, (size_t)std::max<int64_t>(off, 32) * 4));
  idx->layout_bytes += nlist * 8 + code_bytes + (size_t)std::max<int64_t>(off, 32) * 4;
  LY_TRY(cudaMemcpyAsync(idx->own_off, hoff.data(), nlist * 4, cudaMemcpyHostToDevice, s));
  LY_TRY(cudaMemcpyAsync(idx->own_cnt, hcnt.data(), nlist * 4, cudaMemcpyHostToDevice, s));
  LY_TRY(cudaMemsetAsync(idx->codes, 0, code_bytes, s));
  LY_TRY(cudaMemsetAsync(idx->slot_rows, 0xFF, (size_t)std::max<int64_t>(off, 32) * 4, s));
  fill_slots_kernel<<<grid_for(n_live * NU), 256, 0, s>>>(
      skeys, n_live, idx->own_off, seg_s, idx->X, idx->d, idx->M, idx->dsub, NU, idx->codebook,
      idx->slot_rows, reinterpret_cast<uint64_t*>(idx->codes));
  LY_TRY(cudaGetLastError());

  // cells and references
  LY_TRY(cudaMalloc(&rk, n * sizeof(uint64_t)));
  LY_TRY(cudaMalloc(&rv, n * sizeof(uint64_t)));
  LY_TRY(cudaMalloc(&rk_s, n * sizeof(uint64_t)));
  LY_TRY(cudaMalloc(&rv_s, n * sizeof(uint64_t)));
  LY_TRY(cudaMemsetAsync(counters, 0, 4 * sizeof(unsigned long long), s));
  cells_kernel<<<grid_for(n_live), 256, 0, s>>>(skeys, n_live, idx->own_off, seg_s, counters, rk, rv);
  LY_TRY(cudaGetLastError());
  unsigned long long hcount[4];
  LY_TRY(cudaMemcpyAsync(hcount, counters, sizeof(hcount), cudaMemcpyDeviceToHost, s));
  LY_TRY(cudaStreamSynchronize(s));
  const int64_t nr = (int64_t)hcount[0];
  idx->n_refs = nr;
  idx->n_cells = (int64_t)hcount[1];
  idx->n_double = (int64_t)hcount[2];
  std::vector<uint32_t> hptr(nlist + 1, 0);
  LY_TRY(cudaMalloc(&idx->ref_ptr, (nlist + 1) * 4));
  LY_TRY(cudaMalloc(&idx->ref_owner, std::max<int64_t>(nr, 1) * 4));
  LY_TRY(cudaMalloc(&idx->ref_start, std::max<int64_t>(nr, 1) * 4));
  LY_TRY(cudaMalloc(&idx->ref_cnt, std::max<int64_t>(nr, 1) * 4));
  idx->layout_bytes += (nlist + 1) * 4 + std::max<int64_t>(nr, 1) * 12;
  idx->max_refs = 0;
  if (nr > 0) {
    LY_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, rk, rk_s, rv, rv_s, (int64_t)nr, 0, 34, s));
    refs_finalize_kernel<<<grid_for(nr), 256, 0, s>>>(rk_s, rv_s, nr, idx->ref_owner,
                                                      idx->ref_start, idx->ref_cnt);
    LY_TRY(cudaMalloc(&rseg_s, nlist * 4));
    LY_TRY(cudaMalloc(&rseg_e, nlist * 4));
    LY_TRY(cudaMemsetAsync(rseg_s, 0, nlist * 4, s));
    LY_TRY(cudaMemsetAsync(rseg_e, 0, nlist * 4, s));
    list_bounds_kernel<<<grid_for(nr), 256, 0, s>>>(rk_s, nr, 17, 0x1FFFFu, rseg_s, rseg_e);
    LY_TRY(cudaMemcpyAsync(hs.data(), rseg_s, nlist * 4, cudaMemcpyDeviceToHost, s));
    LY_TRY(cudaMemcpyAsync(he.data(), rseg_e, nlist * 4, cudaMemcpyDeviceToHost, s));
    LY_TRY(cudaStreamSynchronize(s));
    for (int l = 0; l < nlist; ++l) {
      uint32_t c = he[l] - hs[l];
      hptr[l + 1] = hptr[l] + c;
      idx->max_refs = std::max<int>(idx->max_refs, (int)c);
    }
  }
  LY_TRY(cudaMemcpyAsync(idx->ref_ptr, hptr.data(), (nlist + 1) * 4, cudaMemcpyHostToDevice, s));
  LY_TRY(cudaStreamSynchronize(s));
  idx->device_bytes += idx->layout_bytes;
  stash.committed = true;
  cleanup();
  return RAIRS_OK;
#undef LY_TRY
}

// ---- exports ---------------------------------------------------------------
__global__ void export_codes_kernel(const uint64_t* __restrict__ codes64,
                                    const uint32_t* __restrict__ slot_rows, int64_t n_slots,
                                    int M, int NU, uint8_t* __restrict__ out) {
  for (int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; slot < n_slots;
       slot += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r = slot_rows[slot];
    if (r == kSlotPad) continue;
    const uint64_t blk = slot >> 5, lane = slot & 31;
    for (int m = 0; m < M; ++m) {
      uint64_t w = codes64[(blk * NU + (m >> 4)) * 32 + lane];
      out[(int64_t)r * M + m] = (uint8_t)((w >> (4 * (m & 15))) & 0xF);
    }
  }
}

rairs_status export_codes(const rairs_index_s* idx, uint8_t* codes, cudaStream_t s) {
  export_codes_kernel<<<grid_for(idx->n_slots), 256, 0, s>>>(
      reinterpret_cast<const uint64_t*>(idx->codes), idx->slot_rows, idx->n_slots, idx->M,
      idx->M_pad / 16, codes);
  RAIRS_CHECK_LAUNCH();
  return RAIRS_OK;
}

__global__ void widen_u32_kernel(const uint32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)in[i];
}

rairs_status export_layout64(const rairs_index_s* idx, int64_t* own_off, int64_t* own_cnt,
                             int64_t* ref_ptr, int32_t* ref_owner, int64_t* ref_start,
                             int64_t* ref_cnt, uint32_t* slot_rows, cudaStream_t s) {
  const int64_t nl = idx->nlist, nr = idx->n_refs;
  if (own_off) widen_u32_kernel<<<grid_for(nl), 256, 0, s>>>(idx->own_off, nl, own_off);
  if (own_cnt) widen_u32_kernel<<<grid_for(nl), 256, 0, s>>>(idx->own_cnt, nl, own_cnt);
  if (ref_ptr) widen_u32_kernel<<<grid_for(nl + 1), 256, 0, s>>>(idx->ref_ptr, nl + 1, ref_ptr);
  if (nr > 0) {
    if (ref_start) widen_u32_kernel<<<grid_for(nr), 256, 0, s>>>(idx->ref_start, nr, ref_start);
    if (ref_cnt) widen_u32_kernel<<<grid_for(nr), 256, 0, s>>>(idx->ref_cnt, nr, ref_cnt);
    if (ref_owner)
      RAIRS_CUDA_TRY(cudaMemcpyAsync(ref_owner, idx->ref_owner, nr * 4, cudaMemcpyDeviceToDevice, s));
  }
  if (slot_rows && idx->n_slots > 0)
    RAIRS_CUDA_TRY(cudaMemcpyAsync(slot_rows, idx->slot_rows, idx->n_slots * 4,
                                   cudaMemcpyDeviceToDevice, s));
  RAIRS_CHECK_LAUNCH();
  return RAIRS_OK;
}

}  // namespace rairs
