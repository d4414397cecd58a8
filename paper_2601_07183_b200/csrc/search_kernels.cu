// search_kernels.cu -- the RAIRS query hot path on sm_100a.
//
// The scan stage (A3-A6) is fastscan_kernels.cu (query-major, register LUTs)
// or listmajor_kernels.cu (list-major, tensor cores); then
//   K6  refine: exact fp64 distances of the bigK candidates,
//       top-k by (fp32 distance, id), one CTA per query.
//   K7  shard merge (O11).
#include <algorithm>
#include <climits>

#include "index.cuh"
#include "tc_helpers.cuh"

namespace rairs {

// ---------------------------------------------------------------------------
// K6 refine: delta = fp32( sum_t ((double)q_t - (double)x_t)^2 ) in ascending t
// (O10), candidates ordered by the key (bits(delta) << 32 | id).
// The bigK candidate rows are gathered coalesced (one warp per row, 128-B
// segments) into a shared-memory tile of RT rows x RDC dims (odd row stride:
// conflict-free column reads); each thread then extends its own row's serial
// fp64 sum over the tile, so the summation order stays ascending in t.
constexpr int RT = 128;

template <int RDC>  // dims per tile (the row stride RDC + 1 keeps column reads conflict-free)
__global__ void __launch_bounds__(RT) refine_kernel(const uint64_t* __restrict__ keys,
                                                    int64_t nq, int bigK, int npow, int k,
                                                    const float* __restrict__ queries,
                                                    const float* __restrict__ X, int d, int G,
                                                    const uint32_t* __restrict__ labels,
                                                    unsigned long long* __restrict__ refined,
                                                    int64_t* __restrict__ out_ids,
                                                    float* __restrict__ out_dists) {
  constexpr int RSTRIDE = RDC + 1;
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* rk = reinterpret_cast<uint64_t*>(sm);
  double* qs = reinterpret_cast<double*>(sm + (size_t)npow * 8);
  float* tile = reinterpret_cast<float*>(sm + (size_t)npow * 8 + (size_t)d * 8);
  uint32_t* rows = reinterpret_cast<uint32_t*>(tile + RT * RSTRIDE);
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
    for (int t = tid; t < d; t += RT) qs[t] = (double)queries[q * d + t];
    for (int c0 = 0; c0 < npow; c0 += RT) {
      const int c = c0 + tid;
      const uint64_t key = (c < bigK) ? keys[q * bigK + c] : kKeyInf;
      const uint32_t gid = (uint32_t)(key & 0xFFFFFFFFu);
      rows[tid] = (key != kKeyInf) ? gid / (uint32_t)G : 0xFFFFFFFFu;
      __syncthreads();
      double acc = 0.0;
      for (int t0 = 0; t0 < d; t0 += RDC) {
        const int dc = min(RDC, d - t0);
        // warp w gathers rows [32w, 32w+32): 8 rows x 4 coalesced 128-B loads in
        // flight per lane before the shared-memory stores
        constexpr int RB = (32 * 32 / RDC) < 32 ? (32 * 32 / RDC) : 32;  // rows per batch: 32 loads in flight
        for (int rb = 0; rb < 32; rb += RB) {
          float v[RB][RDC / 32];
#pragma unroll
          for (int i = 0; i < RB; ++i) {
            const uint32_t row = rows[warp * 32 + rb + i];
            const float* src = X + (size_t)(row == 0xFFFFFFFFu ? 0u : row) * d + t0;
#pragma unroll
            for (int j = 0; j < RDC / 32; ++j) {
              const int t = lane + 32 * j;
              v[i][j] = (row != 0xFFFFFFFFu && t < dc) ? __ldg(src + t) : 0.0f;
            }
          }
#pragma unroll
          for (int i = 0; i < RB; ++i)
#pragma unroll
            for (int j = 0; j < RDC / 32; ++j)
              tile[(warp * 32 + rb + i) * RSTRIDE + lane + 32 * j] = v[i][j];
        }
        __syncthreads();
        if (key != kKeyInf) {
          const float* myrow = tile + tid * RSTRIDE;
          for (int t = 0; t < dc; ++t) {
            double df = __dsub_rn(qs[t0 + t], (double)myrow[t]);
            acc = __dadd_rn(acc, __dmul_rn(df, df));
          }
        }
        __syncthreads();
      }
      uint64_t out = kKeyInf;
      if (key != kKeyInf) {
        const float dist = __double2float_rn(acc);
        out = ((uint64_t)__float_as_uint(dist) << 32) | (labels ? labels[gid / (uint32_t)G] : gid);
        if (refined) atomicAdd(refined, 1ull);
      }
      if (c < npow) rk[c] = out;
    }
    __syncthreads();
    cta_bitonic_sort_u64(rk, npow);
    for (int i = tid; i < k; i += RT) {
      const uint64_t v = (i < npow) ? rk[i] : kKeyInf;
      if (v != kKeyInf) {
        out_ids[q * k + i] = (int64_t)(uint32_t)(v & 0xFFFFFFFFu);
        out_dists[q * k + i] = __uint_as_float((uint32_t)(v >> 32));
      } else {
        out_ids[q * k + i] = -1;
        out_dists[q * k + i] = __int_as_float(0x7f800000);
      }
    }
    __syncthreads();
  }
}

// K6 refine, staged variant (d = 4*D4 <= 128, bigK <= 512): a persistent CTA
// walks (query, chunk) units -- a query's candidates in chunks of 128 rows.
// Warp w gathers the rows w, w+8, ... of a chunk with one coalesced
// 16-B-per-lane load per row (all of its rows in flight at once) into
// registers; the NEXT unit's rows are loaded while thread c runs candidate
// c's serial fp64 sum (ascending t, O10 -- the same order and rounding as
// refine_kernel) over the current chunk's padded shared tile.  After a
// query's last chunk, the top-k by the unique key (bits(delta) << 32 | id) is
// found by rank counting over its bigK keys.
__device__ __forceinline__ float4 ldg_evict_first(const float4* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

constexpr int RS_THREADS = 256;
constexpr int RS_ROWS = 128;
constexpr int RS_MAXK = 512;

template <int D4>
__global__ void __launch_bounds__(RS_THREADS) refine_stage_kernel(
    const uint64_t* __restrict__ keys, int64_t nq, int bigK, int k,
    const float* __restrict__ queries, const float* __restrict__ X, int G,
    const uint32_t* __restrict__ labels, unsigned long long* __restrict__ refined,
    int64_t* __restrict__ out_ids, float* __restrict__ out_dists) {
  constexpr int D = 4 * D4, RSF = D + 4;  // tile row stride (floats): conflict-free float4 reads
  extern __shared__ __align__(16) float tile[];  // [min(bigK, 128) rounded to 8][RSF]
  __shared__ double qs[D];
  __shared__ uint64_t rk[RS_MAXK];
  __shared__ uint32_t gids[RS_ROWS];
  __shared__ uint32_t nvalid_s[2];
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const int myrow = warp + 8 * lane;  // lane j (< 16) fetches the key of row warp + 8j
  const int nch = (bigK + RS_ROWS - 1) / RS_ROWS;
  // one chunk per query (bigK <= 128): the top-k of query u - 1 (warp 0, from
  // the other half of the double-buffered keys) overlaps the fp64 sums of
  // query u (warps 4-7), so the selection's latency leaves the critical path
  const bool pipe = nch == 1;
  const int ci = pipe ? (warp >= 4 ? tid - 128 : RS_ROWS) : tid;  // candidate this thread sums
  auto select_topk = [&](const uint64_t* kb, int64_t qq, uint32_t nv) {
    // warp 0: lane j holds keys j, j+32, j+64, j+96; k rounds of a warp-wide
    // minimum (high word, then the low word among the lanes holding the high
    // minimum); keys are unique, so exactly one lane drops the winner
    uint64_t kr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) kr[u] = (lane + 32 * u < bigK) ? kb[lane + 32 * u] : kKeyInf;
    uint64_t lm = kr[0];
#pragma unroll
    for (int u = 1; u < 4; ++u) lm = kr[u] < lm ? kr[u] : lm;
    int r = 0;
    for (; r < k; ++r) {
      const uint32_t mh = __reduce_min_sync(0xffffffffu, (uint32_t)(lm >> 32));
      const uint32_t ml = __reduce_min_sync(0xffffffffu, (uint32_t)(lm >> 32) == mh ? (uint32_t)lm : 0xFFFFFFFFu);
      const uint64_t m = ((uint64_t)mh << 32) | ml;
      if (m == kKeyInf) break;
      if (lane == 0) {
        out_ids[qq * k + r] = (int64_t)ml;
        out_dists[qq * k + r] = __uint_as_float(mh);
      }
      if (lm == m) {
#pragma unroll
        for (int u = 0; u < 4; ++u) kr[u] = kr[u] == m ? kKeyInf : kr[u];
        lm = kr[0];
#pragma unroll
        for (int u = 1; u < 4; ++u) lm = kr[u] < lm ? kr[u] : lm;
      }
    }
    for (int i = r + lane; i < k; i += 32) {
      out_ids[qq * k + i] = -1;
      out_dists[qq * k + i] = __int_as_float(0x7f800000);
    }
    if (lane == 0 && refined) atomicAdd(refined, (unsigned long long)nv);
  };
  int par = 0;          // pipe: key buffer of the current query
  int64_t qprev = -1;   // pipe: query whose keys wait in buffer par ^ 1
  // candidate rows are read once: evict them first from L2, so the gather does
  // not push out the score rows the concurrent selection streams
  uint64_t l2pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(l2pol));
  pdl_wait();  // the candidate keys of the preceding selection kernel
  // software pipeline: keys of unit u + 2 and rows of unit u + 1 are in
  // flight while unit u is computed (the row loads never wait on a key load)
  auto load_key = [&](int64_t q, int c) -> uint64_t {
    const int row = c * RS_ROWS + myrow;
    return (q < nq && lane < 16 && row < bigK) ? __ldg(keys + q * bigK + row) : kKeyInf;
  };
  auto advance = [&](int64_t& q, int& c) {
    if (++c == nch) {
      c = 0;
      q += gridDim.x;
    }
  };
  uint32_t gid = 0xFFFFFFFFu;
  float4 v[16];
  auto fetch_rows = [&](uint64_t key) {
    gid = 0xFFFFFFFFu;
    uint32_t rowi = 0;
    if (key != kKeyInf) {
      gid = (uint32_t)(key & 0xFFFFFFFFu);
      rowi = gid / (uint32_t)G;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t g = __shfl_sync(0xffffffffu, gid, j);
      const uint32_t r = __shfl_sync(0xffffffffu, rowi, j);
      v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g != 0xFFFFFFFFu && lane < D4)
        v[j] = ldg_evict_first(reinterpret_cast<const float4*>(X + (size_t)r * D) + lane, l2pol);
    }
  };
  int64_t q = blockIdx.x;
  int c = 0;
  if (q < nq) fetch_rows(load_key(q, 0));
  int64_t qn = q;
  int cn = c;
  advance(qn, cn);                                  // the unit after the current one
  uint64_t key_next = load_key(qn, cn);
  float qv = (q < nq && tid < D) ? __ldg(queries + q * D + tid) : 0.0f;  // next query to start
  while (q < nq) {
    const int crow = min(RS_ROWS, bigK - c * RS_ROWS);  // rows in this chunk
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (warp + 8 * j < crow && lane < D4)
        *reinterpret_cast<float4*>(tile + (warp + 8 * j) * RSF + 4 * lane) = v[j];
    if (lane < 16 && myrow < crow) gids[myrow] = gid;
    if (c == 0) {
      if (tid < D) qs[tid] = (double)qv;
      if (tid == 0) nvalid_s[par] = 0;
    }
    __syncthreads();
    int64_t q2 = qn;
    int c2 = cn;
    advance(q2, c2);
    if (qn < nq) {
      fetch_rows(key_next);                        // rows of the next unit: in flight from here
      key_next = load_key(q2, c2);
      if (cn == 0 && tid < D) qv = __ldg(queries + qn * D + tid);
    }
    if (pipe && warp == 0 && qprev >= 0) select_topk(rk + (par ^ 1) * RS_ROWS, qprev, nvalid_s[par ^ 1]);
    if (ci < crow) {
      const uint32_t g = gids[ci];
      uint64_t out = kKeyInf;
      if (g != 0xFFFFFFFFu) {
        const float4* xr = reinterpret_cast<const float4*>(tile + ci * RSF);
        double acc = 0.0;
#pragma unroll 8
        for (int i = 0; i < D4; ++i) {
          const float4 xv = xr[i];
          double df;
          df = __dsub_rn(qs[4 * i + 0], (double)xv.x); acc = __dadd_rn(acc, __dmul_rn(df, df));
          df = __dsub_rn(qs[4 * i + 1], (double)xv.y); acc = __dadd_rn(acc, __dmul_rn(df, df));
          df = __dsub_rn(qs[4 * i + 2], (double)xv.z); acc = __dadd_rn(acc, __dmul_rn(df, df));
          df = __dsub_rn(qs[4 * i + 3], (double)xv.w); acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
        out = ((uint64_t)__float_as_uint(__double2float_rn(acc)) << 32) |
              (labels ? labels[g / (uint32_t)G] : g);  // results carry the caller's ids
        atomicAdd(&nvalid_s[par], 1u);
      }
      rk[(pipe ? par : c) * RS_ROWS + ci] = out;
    }
    __syncthreads();  // tile / gids free for the next unit; rk complete after the last chunk
    if (pipe) {
      qprev = q;
      par ^= 1;
    } else if (c == nch - 1) {
      const uint32_t nvalid = nvalid_s[0];
      for (int i = tid; i < bigK; i += RS_THREADS) {
        const uint64_t kc = rk[i];
        if (kc != kKeyInf) {
          int rank = 0;
#pragma unroll 8
          for (int j = 0; j < bigK; ++j) rank += (rk[j] < kc) ? 1 : 0;
          if (rank < k) {
            out_ids[q * k + rank] = (int64_t)(uint32_t)(kc & 0xFFFFFFFFu);
            out_dists[q * k + rank] = __uint_as_float((uint32_t)(kc >> 32));
          }
        }
      }
      for (int i = (int)nvalid + tid; i < k; i += RS_THREADS) {
        out_ids[q * k + i] = -1;
        out_dists[q * k + i] = __int_as_float(0x7f800000);
      }
      if (tid == 0 && refined) atomicAdd(refined, (unsigned long long)nvalid);
      __syncthreads();  // rk / nvalid / qs free for the next query
    }
    q = qn;
    c = cn;
    qn = q2;
    cn = c2;
  }
  if (pipe && warp == 0 && qprev >= 0) select_topk(rk + (par ^ 1) * RS_ROWS, qprev, nvalid_s[par ^ 1]);
}

template <int D4>
static rairs_status launch_refine_stage(const rairs_index_s* idx, const SearchArgs& a, int bigK,
                                        cudaStream_t s) {
  const size_t smem = (size_t)round_up(std::min(bigK, RS_ROWS), 8) * (4 * D4 + 4) * 4;
  RAIRS_CUDA_TRY(cudaFuncSetAttribute(refine_stage_kernel<D4>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  RAIRS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, refine_stage_kernel<D4>,
                                                               RS_THREADS, smem));
  const int grid = (int)std::min<int64_t>(a.nq, (int64_t)148 * std::max(occ, 1));
  // programmatic dependent launch: the CTAs are resident while the selection
  // kernel drains; pdl_wait() orders the key reads
  RAIRS_CUDA_TRY(launch_pdl(refine_stage_kernel<D4>, dim3(grid), dim3(RS_THREADS), smem, s,
                            (const uint64_t*)a.cand_keys, (int64_t)a.nq, bigK, (int)a.k,
                            (const float*)a.queries, (const float*)idx->X, (int)idx->nshards,
                            (const uint32_t*)idx->labels,
                            a.counters ? a.counters + 1 : (unsigned long long*)nullptr,
                            (int64_t*)a.out_ids, (float*)a.out_dists));
  return RAIRS_OK;
}

// K6 for long rows (d > 128): the generic kernel's gather/sum alternation,
// double-buffered -- chunk c+1's 32 rows x 32 dims are in flight (32 loads per
// lane) while every thread extends its candidate's ordered fp64 sum over chunk
// c from shared memory (O10: ascending t, one rounding to fp32 at the end).
__global__ void __launch_bounds__(RT) refine_long_kernel(const uint64_t* __restrict__ keys,
                                                         int64_t nq, int bigK, int npow, int k,
                                                         const float* __restrict__ queries,
                                                         const float* __restrict__ X, int d, int G,
                                                         const uint32_t* __restrict__ labels,
                                                         unsigned long long* __restrict__ refined,
                                                         int64_t* __restrict__ out_ids,
                                                         float* __restrict__ out_dists) {
  constexpr int S = 33;  // row stride of a 32-dim tile (conflict-free column reads)
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* rk = reinterpret_cast<uint64_t*>(sm);
  float* qs = reinterpret_cast<float*>(sm + (size_t)npow * 8);
  float* tile = qs + ((d + 3) & ~3);                       // [2][RT][S]
  uint32_t* rows = reinterpret_cast<uint32_t*>(tile + 2 * RT * S);
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const int nch = (d + 31) / 32;
  for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
    for (int t = tid; t < d; t += RT) qs[t] = queries[q * d + t];
    for (int c0 = 0; c0 < npow; c0 += RT) {
      const int c = c0 + tid;
      const uint64_t key = (c < bigK) ? keys[q * bigK + c] : kKeyInf;
      const uint32_t gid = (uint32_t)(key & 0xFFFFFFFFu);
      rows[tid] = (key != kKeyInf) ? gid / (uint32_t)G : 0xFFFFFFFFu;
      __syncthreads();
      float v[32];
      auto gather = [&](int ch) {
        const int t = ch * 32 + lane;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const uint32_t row = rows[warp * 32 + i];
          v[i] = (row != 0xFFFFFFFFu && t < d) ? __ldg(X + (size_t)row * d + t) : 0.0f;
        }
      };
      gather(0);
      double acc = 0.0;
      for (int ch = 0; ch < nch; ++ch) {
        float* tb = tile + (ch & 1) * RT * S;
#pragma unroll
        for (int i = 0; i < 32; ++i) tb[(warp * 32 + i) * S + lane] = v[i];
        __syncthreads();
        if (ch + 1 < nch) gather(ch + 1);
        if (key != kKeyInf) {
          const float* myrow = tb + tid * S;
          const int dc = min(32, d - ch * 32);
          for (int t = 0; t < dc; ++t) {
            const double df = __dsub_rn((double)qs[ch * 32 + t], (double)myrow[t]);
            acc = __dadd_rn(acc, __dmul_rn(df, df));
          }
        }
      }
      uint64_t out = kKeyInf;
      if (key != kKeyInf) {
        const float dist = __double2float_rn(acc);
        out = ((uint64_t)__float_as_uint(dist) << 32) | (labels ? labels[gid / (uint32_t)G] : gid);
        if (refined) atomicAdd(refined, 1ull);
      }
      __syncthreads();  // every thread is done with both tiles and rows[]
      if (c < npow) rk[c] = out;
    }
    __syncthreads();
    cta_bitonic_sort_u64(rk, npow);
    for (int i = tid; i < k; i += RT) {
      const uint64_t v2 = (i < npow) ? rk[i] : kKeyInf;
      out_ids[q * k + i] = v2 != kKeyInf ? (int64_t)(uint32_t)(v2 & 0xFFFFFFFFu) : -1;
      out_dists[q * k + i] = v2 != kKeyInf ? __uint_as_float((uint32_t)(v2 >> 32)) : __int_as_float(0x7f800000);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K6 for long rows (d > 128, d % 4 == 0; c3: 6 KB per row): one THREAD per
// candidate streams its own row with eight 16-B loads in flight (no shared
// tile, so ~64 warps per SM keep the gather busy) and extends the fp64
// ordered sum in ascending t (O10); its key (bits(delta) << 32 | id) goes to
// dk[].  Then a warp per query keeps the first k by key.
constexpr int RL_T = 256;
__global__ void __launch_bounds__(RL_T) refine_rows_kernel(const uint64_t* __restrict__ keys,
                                                           int64_t total, int bigK,
                                                           const float* __restrict__ queries,
                                                           const float* __restrict__ X, int d, int G,
                                                           const uint32_t* __restrict__ labels,
                                                           unsigned long long* __restrict__ refined,
                                                           uint64_t* __restrict__ dk) {
  pdl_wait();
  uint32_t nref = 0;
  for (int64_t i = blockIdx.x * (int64_t)RL_T + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * RL_T) {
    const uint64_t key = keys[i];
    uint64_t out = kKeyInf;
    if (key != kKeyInf) {
      const uint32_t gid = (uint32_t)(key & 0xFFFFFFFFu);
      const float4* xr = reinterpret_cast<const float4*>(X + (size_t)(gid / (uint32_t)G) * d);
      const float4* qr = reinterpret_cast<const float4*>(queries + (i / bigK) * d);
      double acc = 0.0;
      const int n4 = d / 4;
      for (int c0 = 0; c0 < n4; c0 += 8) {
        float4 xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          xv[u] = (c0 + u < n4) ? __ldcs(xr + c0 + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (c0 + u < n4) {
            const float4 qv = __ldg(qr + c0 + u);
            double df = __dsub_rn((double)qv.x, (double)xv[u].x);
            acc = __dadd_rn(acc, __dmul_rn(df, df));
            df = __dsub_rn((double)qv.y, (double)xv[u].y);
            acc = __dadd_rn(acc, __dmul_rn(df, df));
            df = __dsub_rn((double)qv.z, (double)xv[u].z);
            acc = __dadd_rn(acc, __dmul_rn(df, df));
            df = __dsub_rn((double)qv.w, (double)xv[u].w);
            acc = __dadd_rn(acc, __dmul_rn(df, df));
          }
        }
      }
      const float dist = __double2float_rn(acc);
      out = ((uint64_t)__float_as_uint(dist) << 32) | (labels ? labels[gid / (uint32_t)G] : gid);
      ++nref;
    }
    dk[i] = out;
  }
  if (refined) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nref += __shfl_xor_sync(0xffffffffu, nref, o);
    if ((threadIdx.x & 31) == 0 && nref) atomicAdd(refined, (unsigned long long)nref);
  }
  pdl_trigger();
}

__global__ void __launch_bounds__(128) refine_topk_kernel(const uint64_t* __restrict__ dk, int64_t nq,
                                                          int bigK, int npow, int k,
                                                          int64_t* __restrict__ out_ids,
                                                          float* __restrict__ out_dists) {
  extern __shared__ __align__(16) uint64_t rt_sm[];
  const int lane = lane_id(), warp = warp_id();
  uint64_t* buf = rt_sm + (size_t)warp * npow;
  pdl_wait();
  for (int64_t q = (int64_t)blockIdx.x * 4 + warp; q < nq; q += (int64_t)gridDim.x * 4) {
    for (int i = lane; i < npow; i += 32) buf[i] = i < bigK ? dk[q * bigK + i] : kKeyInf;
    __syncwarp();
    for (int size = 2; size <= npow; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = lane; i < (npow >> 1); i += 32) {
          const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
          const bool asc = (lo & size) == 0;
          const uint64_t x = buf[lo], y = buf[hi];
          if ((x > y) == asc) { buf[lo] = y; buf[hi] = x; }
        }
        __syncwarp();
      }
    }
    for (int i = lane; i < k; i += 32) {
      const uint64_t v = i < npow ? buf[i] : kKeyInf;
      out_ids[q * k + i] = v != kKeyInf ? (int64_t)(uint32_t)(v & 0xFFFFFFFFu) : -1;
      out_dists[q * k + i] = v != kKeyInf ? __uint_as_float((uint32_t)(v >> 32)) : __int_as_float(0x7f800000);
    }
    __syncwarp();
  }
}

static rairs_status launch_refine_rows(const rairs_index_s* idx, const SearchArgs& a, int bigK,
                                       cudaStream_t s) {
  const int64_t total = a.nq * bigK;
  uint64_t* dk = nullptr;
  RAIRS_CUDA_TRY(ws_malloc(&dk, (size_t)total * 8, s));
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, RL_T), 148 * 8));
  cudaError_t e = launch_pdl(refine_rows_kernel, dim3(g), dim3(RL_T), 0, s, (const uint64_t*)a.cand_keys,
                             total, bigK, a.queries, (const float*)idx->X, idx->d, idx->nshards,
                             (const uint32_t*)idx->labels,
                             a.counters ? a.counters + 1 : (unsigned long long*)nullptr, dk);
  if (e == cudaSuccess) {
    const int npow = next_pow2(std::max(bigK, 2));
    const size_t smem = (size_t)4 * npow * 8;
    e = cudaFuncSetAttribute(refine_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) {
      const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(a.nq, 4), 148 * 16));
      e = launch_pdl(refine_topk_kernel, dim3(g2), dim3(128), smem, s, (const uint64_t*)dk, a.nq, bigK,
                     npow, a.k, a.out_ids, a.out_dists);
    }
  }
  cudaFreeAsync(dk, s);
  if (e != cudaSuccess) {
    set_error(std::string("refine (long rows): ") + cudaGetErrorString(e));
    return RAIRS_E_CUDA;
  }
  return RAIRS_OK;
}

rairs_status launch_refine(const rairs_index_s* idx, const SearchArgs& a, cudaStream_t s) {
  if (a.nq <= 0) return RAIRS_OK;
  {
    const int bigK = a.k * a.refine_factor;
    if (bigK <= RS_MAXK) {
      switch (idx->d) {
        case 32: return launch_refine_stage<8>(idx, a, bigK, s);
        case 64: return launch_refine_stage<16>(idx, a, bigK, s);
        case 96: return launch_refine_stage<24>(idx, a, bigK, s);
        case 128: return launch_refine_stage<32>(idx, a, bigK, s);
        default: break;
      }
    }
  }
  const int bigK = a.k * a.refine_factor;
  // (thread-per-row streaming, launch_refine_rows, measured 4x slower on c3pl: uncoalesced)
  if (std::getenv("RAIRS_REFINE_ROWS") && (idx->d & 3) == 0 && bigK <= 2048)
    return launch_refine_rows(idx, a, bigK, s);
  const int npow = next_pow2(std::max(bigK, 2));
  // narrower tiles for long rows: ~3x smaller shared footprint, more CTAs per SM
  // overlap one CTA's gather with another's serial fp64 sums
  const int rdc = (idx->d > 128 && !std::getenv("RAIRS_REFINE_RDC128")) ? 32 : 128;
  const size_t smem = (size_t)npow * 8 + (size_t)idx->d * 8 + (size_t)RT * (rdc + 1) * 4 + RT * 4;
  if (smem > 220 * 1024) {
    set_error("refine: shared memory budget exceeded");
    return RAIRS_E_UNSUPPORTED;
  }
  const int grid = (int)std::min<int64_t>(a.nq, 1 << 30);
  if (rdc == 32) {
    const size_t lsm = (size_t)npow * 8 + (size_t)((idx->d + 3) & ~3) * 4 + (size_t)2 * RT * 33 * 4 + RT * 4;
    RAIRS_CUDA_TRY(cudaFuncSetAttribute(refine_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)lsm));
    refine_long_kernel<<<grid, RT, lsm, s>>>(a.cand_keys, a.nq, bigK, npow, a.k, a.queries, idx->X,
                                             idx->d, idx->nshards, idx->labels,
                                             a.counters ? a.counters + 1 : nullptr, a.out_ids, a.out_dists);
  } else {
    RAIRS_CUDA_TRY(cudaFuncSetAttribute(refine_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    refine_kernel<128><<<grid, RT, smem, s>>>(a.cand_keys, a.nq, bigK, npow, a.k, a.queries, idx->X,
                                              idx->d, idx->nshards, idx->labels,
                                              a.counters ? a.counters + 1 : nullptr, a.out_ids, a.out_dists);
  }
  RAIRS_CHECK_LAUNCH();
  return RAIRS_OK;
}

// ---------------------------------------------------------------------------
// K7 merge of G per-shard top-k lists: first k by (dist, id) (O11).
// K7: the first k of the G per-shard lists by (fp32 distance, 64-bit id);
// entries with id < 0 (padding) sort last.  The distance is ordered by its
// bits (squared distances are >= 0, +inf last); ids keep all 64 bits.
__global__ void merge_kernel(const int64_t* __restrict__ ids, const float* __restrict__ dists,
                             int G, int64_t nq, int k, int npow, int64_t* __restrict__ out_ids,
                             float* __restrict__ out_dists) {
  extern __shared__ __align__(16) unsigned char sm[];
  int64_t* kid = reinterpret_cast<int64_t*>(sm);
  uint32_t* kd = reinterpret_cast<uint32_t*>(kid + npow);
  for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
    for (int e = threadIdx.x; e < npow; e += blockDim.x) {
      uint32_t d = 0xFFFFFFFFu;
      int64_t id = INT64_MAX;
      if (e < G * k) {
        const int g = e / k, j = e - g * k;
        const int64_t v = ids[((int64_t)g * nq + q) * k + j];
        if (v >= 0) {
          id = v;
          d = __float_as_uint(dists[((int64_t)g * nq + q) * k + j]);
        }
      }
      kid[e] = id;
      kd[e] = d;
    }
    __syncthreads();
    for (int size = 2; size <= npow; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < (npow >> 1); i += blockDim.x) {
          const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
          const bool asc = (lo & size) == 0;
          const uint32_t da = kd[lo], db = kd[hi];
          const int64_t ia = kid[lo], ib = kid[hi];
          const bool gt = da > db || (da == db && ia > ib);
          if (gt == asc) { kd[lo] = db; kd[hi] = da; kid[lo] = ib; kid[hi] = ia; }
        }
        __syncthreads();
      }
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      const bool ok = kid[i] != INT64_MAX;
      out_ids[q * k + i] = ok ? kid[i] : -1;
      out_dists[q * k + i] = ok ? __uint_as_float(kd[i]) : __int_as_float(0x7f800000);
    }
    __syncthreads();
  }
}

rairs_status launch_merge(const int64_t* ids, const float* dists, int G, int64_t nq, int k,
                          int64_t* out_ids, float* out_dists, cudaStream_t s) {
  if (nq <= 0) return RAIRS_OK;
  const int npow = next_pow2(std::max(G * k, 2));
  const size_t smem = (size_t)npow * 12;
  if (smem > 200 * 1024) {
    set_error("merge: G*k too large");
    return RAIRS_E_UNSUPPORTED;
  }
  RAIRS_CUDA_TRY(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  const int grid = (int)std::min<int64_t>(nq, 1 << 30);
  merge_kernel<<<grid, 128, smem, s>>>(ids, dists, G, nq, k, npow, out_ids, out_dists);
  RAIRS_CHECK_LAUNCH();
  return RAIRS_OK;
}

__global__ void split_keys_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                  uint32_t* __restrict__ ids, uint32_t* __restrict__ scores) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = keys[i];
    if (ids) ids[i] = (uint32_t)(v & 0xFFFFFFFFu);
    if (scores) scores[i] = (uint32_t)(v >> 32);
  }
}

rairs_status launch_split_keys(const uint64_t* keys, int64_t count, uint32_t* ids,
                               uint32_t* scores, cudaStream_t s) {
  if (count <= 0) return RAIRS_OK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 256), 148 * 16));
  split_keys_kernel<<<grid, 256, 0, s>>>(keys, count, ids, scores);
  RAIRS_CHECK_LAUNCH();
  return RAIRS_OK;
}

}  // namespace rairs
