// listmajor_kernels.cu -- NEXT-1: list-major batched fast scan on tensor cores.
//
// The paper's query-batch cache optimisation ("group the tasks by
// lists, and process all the queries for the same list back to back") on B200:
// for a list l probed by the queries Q_l of a batch, the integer scores of all
// (item, query) pairs are ONE exact u8 x u8 -> s32 contraction
//     S[x][q] = sum_m Qv_q[m][code_m(x)] = sum_{m,j} onehot(x)[m*16+j] * Qv_q[m][j]
// (K = 16*M), issued as tcgen05.mma.kind::i8 (M = 128 items, N = |Q_l| padded to
// 16, K = 32 per instruction) with the accumulator in TMEM.  The one-hot A tile
// is expanded in shared memory from the 4-bit codes (each code byte read ONCE
// per list-task instead of once per (list, query)); the B tile is the queries'
// quantised LUT rows.  Integer sums are exact (<= 16*M*255 < 2^31), so the
// scores are bit-identical to the SIMT lookup scan (O8).
//
// Pipeline for a batch (all on the search stream, no host sync):
//   lut_batch_kernel   O2 LUT per query -> global [nq][16*M_pad] u8
//   lm_count / lm_scan / lm_scatter / lm_bitmap   group (query, probe) by list
//   lm_tensor_kernel   persistent; task = (list, 128-item tile, 256-query tile)
//                      -> scores of valid pairs into a per-list score block
//   lm_select_kernel   per query: SEIL ranges (R9 dedup) over its score rows,
//                      histogram-threshold top-bigK (same rule as scan_kernel)
#include <algorithm>

#include "index.cuh"
#include "tc_helpers.cuh"

namespace rairs {

// ---------------------------------------------------------------------------
// O2 LUT, one WARP per query (same arithmetic as scan_kernel's prologue).
constexpr int LW = 8;  // warps (queries) per CTA

__device__ __forceinline__ float lm_lut_T(const float* __restrict__ q,
                                          const float* __restrict__ cb, int m, int j, int dsub) {
  const float* c = cb + ((int64_t)m * 16 + j) * dsub;
  const float* qs = q + (int64_t)m * dsub;
  float acc = 0.0f;
  for (int t = 0; t < dsub; ++t) {
    float diff = __fsub_rn(__ldg(qs + t), __ldg(c + t));
    acc = __fadd_rn(acc, __fmul_rn(diff, diff));
  }
  return acc;
}

__global__ void __launch_bounds__(LW * 32) lut_batch_kernel(const float* __restrict__ queries,
                                                            int64_t nq, int d,
                                                            const float* __restrict__ cb, int M,
                                                            int M_pad, int dsub,
                                                            uint8_t* __restrict__ lut,
                                                            float* __restrict__ a_out,
                                                            float* __restrict__ b_out,
                                                            uint8_t* __restrict__ lut_dbg) {
  const int lane = lane_id();
  const int M16 = M * 16, K = M_pad * 16;
  for (int64_t q = (int64_t)blockIdx.x * LW + warp_id(); q < nq; q += (int64_t)gridDim.x * LW) {
    const float* qv = queries + q * d;
    // pass 1: per-subquantizer min and span (16-lane groups), S = max span
    float S = 0.0f, bsum = 0.0f;
    for (int e0 = 0; e0 < M16; e0 += 32) {
      const int e = e0 + lane;
      const bool act = e < M16;
      const float T = act ? lm_lut_T(qv, cb, e >> 4, e & 15, dsub) : 0.0f;
      float lo = act ? T : __int_as_float(0x7f800000);
      float hi = act ? T : -__int_as_float(0x7f800000);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      const float span = __fsub_rn(hi, lo);
      if (act) S = fmaxf(S, span);
      // b = sum_m mn_m in ascending m (fp32): lanes 0 and 16 hold m = e0/16, e0/16+1
      const float lo0 = __shfl_sync(0xffffffffu, lo, 0), lo1 = __shfl_sync(0xffffffffu, lo, 16);
      if (e0 + 0 < M16) bsum = __fadd_rn(bsum, lo0);
      if (e0 + 16 < M16) bsum = __fadd_rn(bsum, lo1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) S = fmaxf(S, __shfl_xor_sync(0xffffffffu, S, o));
    const float a = (S > 0.0f) ? __fdiv_rn(255.0f, S) : 1.0f;
    // pass 2: quantise (recomputing T: identical fp32 values)
    for (int e0 = 0; e0 < K; e0 += 32) {
      const int e = e0 + lane;
      const int m = e >> 4;
      uint32_t v = 0;
      const bool act = m < M;
      const float T = act ? lm_lut_T(qv, cb, m, e & 15, dsub) : 0.0f;
      float lo = act ? T : __int_as_float(0x7f800000);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      if (act && S > 0.0f) {
        const float t2 = __fmul_rn(__fsub_rn(T, lo), a);
        v = (uint32_t)min(255, __float2int_rn(t2));
      }
      lut[q * K + e] = (uint8_t)v;
      if (lut_dbg && act) lut_dbg[q * M16 + e] = (uint8_t)v;
    }
    if (lane == 0) {
      if (a_out) a_out[q] = a;
      if (b_out) b_out[q] = bsum;
    }
  }
}

// ---------------------------------------------------------------------------
// Grouping of (query, probe) pairs by list.
__global__ void lm_count_kernel(const int32_t* __restrict__ probes, int64_t total,
                                uint32_t* __restrict__ cnt, uint32_t* __restrict__ qslot) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    qslot[e] = atomicAdd(&cnt[probes[e]], 1u);
}

__global__ void lm_scatter_kernel(const int32_t* __restrict__ probes, int64_t total, int nprobe,
                                  const uint32_t* __restrict__ qptr,
                                  const uint32_t* __restrict__ qslot, uint32_t* __restrict__ list_q,
                                  uint32_t* __restrict__ qbits, int qwords) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int l = probes[e];
    const uint32_t q = (uint32_t)(e / nprobe);
    list_q[qptr[l] + qslot[e]] = q;
    atomicOr(&qbits[(size_t)q * qwords + (l >> 5)], 1u << (l & 31));
  }
}

// single CTA: exclusive scans over lists of |Q_l| (qptr), |Q_l|*N_l (score
// block base), and #tasks; totals[0] = #tasks.
constexpr int SCN = 1024;
__global__ void __launch_bounds__(SCN) lm_scan_kernel(const uint32_t* __restrict__ cnt,
                                                      const uint32_t* __restrict__ nitems, int nlist,
                                                      uint32_t* __restrict__ qptr,
                                                      uint64_t* __restrict__ sbase,
                                                      uint32_t* __restrict__ tptr,
                                                      uint32_t* __restrict__ totals, int qtile,
                                                      int itile) {
  __shared__ uint32_t wq[SCN / 32], wt[SCN / 32];
  __shared__ uint64_t ws[SCN / 32];
  __shared__ uint32_t carry_q, carry_t;
  __shared__ uint64_t carry_s;
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  if (tid == 0) { carry_q = 0; carry_t = 0; carry_s = 0; }
  __syncthreads();
  for (int base = 0; base < nlist; base += SCN) {
    const int l = base + tid;
    uint32_t c = 0, t = 0;
    uint64_t s = 0;
    if (l < nlist) {
      c = cnt[l];
      const uint32_t ni = nitems[l];
      s = (uint64_t)c * ni;
      t = (c > 0 && ni > 0) ? (uint32_t)(((c + qtile - 1) / qtile) * ((ni + itile - 1) / itile)) : 0u;
    }
    uint32_t ic = c, it = t;
    uint64_t is = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t x = __shfl_up_sync(0xffffffffu, ic, o);
      uint32_t y = __shfl_up_sync(0xffffffffu, it, o);
      uint64_t z = __shfl_up_sync(0xffffffffu, is, o);
      if (lane >= o) { ic += x; it += y; is += z; }
    }
    if (lane == 31) { wq[warp] = ic; wt[warp] = it; ws[warp] = is; }
    __syncthreads();
    if (warp == 0) {
      uint32_t a = wq[lane], b = wt[lane];
      uint64_t d = ws[lane];
      uint32_t ia = a, ib = b;
      uint64_t id = d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t x = __shfl_up_sync(0xffffffffu, ia, o);
        uint32_t y = __shfl_up_sync(0xffffffffu, ib, o);
        uint64_t z = __shfl_up_sync(0xffffffffu, id, o);
        if (lane >= o) { ia += x; ib += y; id += z; }
      }
      wq[lane] = ia - a;
      wt[lane] = ib - b;
      ws[lane] = id - d;
    }
    __syncthreads();
    if (l < nlist) {
      qptr[l] = carry_q + wq[warp] + ic - c;
      tptr[l] = carry_t + wt[warp] + it - t;
      sbase[l] = carry_s + ws[warp] + is - s;
    }
    __syncthreads();
    if (tid == SCN - 1) {
      carry_q += wq[warp] + ic;
      carry_t += wt[warp] + it;
      carry_s += ws[warp] + is;
    }
    __syncthreads();
  }
  if (tid == 0) {
    qptr[nlist] = carry_q;
    tptr[nlist] = carry_t;
    sbase[nlist] = carry_s;
    totals[0] = carry_t;
  }
}

// ---------------------------------------------------------------------------
// Tensor-core scoring, one list at a time (CTAs claim lists atomically).
constexpr int LM_THREADS = 256;   // 2 threads per item row (4 subquantizers of a chunk each)
constexpr int LM_IT = 128;        // items per tile (MMA M)
constexpr int LM_QT = 64;         // queries per tile (MMA N <= 64, TMEM columns)
constexpr int LM_MAXREF = 128;    // references per list on this path
constexpr uint32_t LM_A_BYTES = LM_IT * 128;   // one 128-B K-chunk per item row
constexpr uint32_t LM_BC_BYTES = LM_QT * 128;  // one K-chunk of the LUT tile
constexpr int LM_BRES_MAX = 64 * 1024;         // LUT tile resident for all K if it fits

struct LMArgs {
  const uint64_t* codes64;
  const uint32_t* own_off;
  const uint32_t* own_cnt;
  const uint32_t* ref_ptr;
  const int32_t* ref_owner;
  const uint32_t* ref_start;
  const uint32_t* ref_item_off;  // item offset of each reference inside its list-task
  const uint32_t* list_items;    // N_l = own_cnt + sum of the list's ref_cnt
  int NU, nchunk;                // code units of 16 subquantizers; K chunks of 8 subq (128 B)
  const uint8_t* lut;            // [nq][K]
  int K, b_resident;
  const int32_t* probes;
  int nprobe;
  const uint32_t* qptr;
  const uint32_t* list_q;
  unsigned* list_counter;
  const uint64_t* sbase;
  void* S;
  int score_u32;
  int nlist;
};

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// (no "memory" clobber: ordinary loads may be hoisted above these stores; the
// fence.proxy.async / barrier asm that publishes the tile does carry one)
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z,
                                             uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z),
               "r"(w));
}

// 16-byte one-hot of a 4-bit code: byte n = 1.  c = 8*(n&7) < 64; (hi:lo) =
// 1 << c as two PTX shl (shift counts >= 32 -- including c-32 wrapped for
// c < 32 -- produce 0); bit 3 of n picks words (0,1) or (2,3).
__device__ __forceinline__ void onehot16(uint32_t n, uint32_t& w0, uint32_t& w1, uint32_t& w2,
                                         uint32_t& w3) {
  const uint32_t c = (n & 7u) << 3;
  uint32_t lo, hi;
  asm("shl.b32 %0, 1, %1;" : "=r"(lo) : "r"(c));
  asm("shl.b32 %0, 1, %1;" : "=r"(hi) : "r"(c - 32u));
  const bool h = (n & 8u) != 0;
  w0 = h ? 0u : lo;
  w1 = h ? 0u : hi;
  w2 = h ? lo : 0u;
  w3 = h ? hi : 0u;
}

// Warp-specialised pipeline (no CTA barrier per chunk):
//   warps 0-3  generators: warp g expands the one-hot rows of items 32g..32g+31
//              for each K-chunk into a 4-stage shared-memory ring, then arrives
//              on full[stage] (4 arrivals);
//   warp 4     MMA issuer: waits full[stage], issues 4 x tcgen05.mma.kind::i8
//              into one of 2 TMEM accumulators, commits empty[stage] and, after
//              the last chunk of a tile, tfull[acc];
//   warps 5-8  epilogue: wait tfull[acc], tcgen05.ld the scores (lane group
//              warp%4), store the valid (item, query) scores, arrive tempty[acc].
// The LUT tile of a 64-query tile is loaded once (all K) at the start of the
// query tile; a CTA barrier separates query tiles (no MMA in flight then).
constexpr int LM_GEN_WARPS = 4, LM_MMA_WARP = 4;
constexpr int LM_WS_THREADS = 9 * 32;
constexpr int LM_STAGES = 2;  // 2 x 16 KB A ring + 64 KB LUT tile -> 2 CTAs per SM

__global__ void __launch_bounds__(LM_WS_THREADS, 2) lm_tensor_kernel(LMArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
  uint8_t* sA = smem;                                    // LM_STAGES x 16 KB
  uint8_t* sB = smem + LM_STAGES * LM_A_BYTES;           // nchunk x 8 KB (resident LUT tile)
  int32_t* owners = reinterpret_cast<int32_t*>(sB + (size_t)a.nchunk * LM_BC_BYTES);  // [LM_MAXREF]
  uint32_t* refoff = reinterpret_cast<uint32_t*>(owners + LM_MAXREF);                // [LM_MAXREF+1]
  uint32_t* skipT = refoff + LM_MAXREF + 1;            // [LM_MAXREF][2]: queries skipping ref j
  uint32_t* qid = skipT + LM_MAXREF * 2;               // [LM_QT]
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(qid + LM_QT) + 7) & ~(uintptr_t)7);  // [LM_STAGES]
  uint64_t* empty = full + LM_STAGES;
  uint64_t* tfull = empty + LM_STAGES;   // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ uint32_t sh_list;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < LM_STAGES; ++s) {
      mbar_init(&full[s], LM_GEN_WARPS);
      mbar_init(&empty[s], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&tfull[k], 1);
      mbar_init(&tempty[k], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == LM_MMA_WARP) tmem_alloc(tslot, 2 * LM_QT);
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  uint32_t chunk_ctr = 0;  // chunks produced/consumed so far (same sequence in every role)
  uint32_t tile_ctr = 0;   // item tiles so far

  for (;;) {
    if (tid == 0) sh_list = atomicAdd(a.list_counter, 1u);
    __syncthreads();
    const uint32_t l = sh_list;
    __syncthreads();  // everyone has read sh_list before thread 0 may overwrite it
    if (l >= (uint32_t)a.nlist) break;
    const uint32_t Ql = a.qptr[l + 1] - a.qptr[l];
    const uint32_t Nl = a.list_items[l];
    if (Ql == 0 || Nl == 0) continue;  // uniform across the CTA
    const uint32_t own = a.own_cnt[l], own0 = a.own_off[l];
    const uint32_t r0 = a.ref_ptr[l], nref = a.ref_ptr[l + 1] - r0;
    for (uint32_t j = tid; j < nref; j += LM_WS_THREADS) {
      owners[j] = a.ref_owner[r0 + j];
      refoff[j] = a.ref_item_off[r0 + j];
    }
    if (tid == 0) refoff[nref] = Nl;
    const uint32_t ntiles = (Nl + LM_IT - 1) / LM_IT;
    for (uint32_t q0 = 0; q0 < Ql; q0 += LM_QT) {
      const int nq_tile = (int)min(Ql - q0, (uint32_t)LM_QT);
      const int Npad = ((nq_tile + 15) / 16) * 16;
      __syncthreads();  // previous query tile fully drained (epilogue waited on its MMAs)
      for (uint32_t j = tid; j < nref * 2; j += LM_WS_THREADS) skipT[j] = 0u;
      if (tid < LM_QT) qid[tid] = (tid < nq_tile) ? a.list_q[a.qptr[l] + q0 + tid] : 0xFFFFFFFFu;
      __syncthreads();
      // ref j (owner o) of this list is NOT scanned for query q iff o is probed by q (R9)
      if (tid < nq_tile) {
        const uint32_t q = qid[tid];
        for (int p = 0; p < a.nprobe; ++p) {
          const int pl = a.probes[(size_t)q * a.nprobe + p];
          int lo = 0, hi = (int)nref;  // owners ascending: binary search
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (owners[mid] < pl) lo = mid + 1; else hi = mid;
          }
          if (lo < (int)nref && owners[lo] == pl) atomicOr(&skipT[lo * 2 + (tid >> 5)], 1u << (tid & 31));
        }
      }
      {  // LUT rows of the tile's queries for every K-chunk (128B-swizzled per chunk)
        const int pieces = a.nchunk * Npad * 8;
#pragma unroll 4
        for (int e = tid; e < pieces; e += LM_WS_THREADS) {
          const int c = e / (Npad * 8), rem = e - c * Npad * 8, jq = rem >> 3, k = rem & 7;
          uint4 v = make_uint4(0, 0, 0, 0);
          const uint32_t q = qid[jq];
          if (q != 0xFFFFFFFFu)
            v = __ldg(reinterpret_cast<const uint4*>(a.lut + (size_t)q * a.K + c * 128) + k);
          st_shared_v4(smem_u32(sB + c * LM_BC_BYTES) + jq * 128 + ((k ^ (jq & 7)) << 4), v.x, v.y,
                       v.z, v.w);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();

      if (warp < LM_GEN_WARPS) {
        // ---------------- generators ----------------
        const int row = warp * 32 + lane;
        uint32_t cc = chunk_ctr;
        for (uint32_t t = 0; t < ntiles; ++t) {
          const uint32_t item = t * LM_IT + row;
          const bool ivalid = item < Nl;
          uint32_t slot = 0;
          if (ivalid) {
            if (item < own) {
              slot = own0 + item;
            } else {
              int j = 0;
              while (refoff[j + 1] <= item) ++j;
              slot = a.ref_start[r0 + j] + (item - refoff[j]);
            }
          }
          const uint64_t* cw = a.codes64 + ((size_t)(slot >> 5) * a.NU) * 32 + (slot & 31);
          uint64_t w64 = ivalid ? __ldg(cw) : 0ull;
          for (int c = 0; c < a.nchunk; ++c, ++cc) {
            const int s = cc % LM_STAGES;
            const uint64_t cur = w64;
            if ((c & 1) == 1 && ivalid && (c >> 1) + 1 < a.NU) w64 = __ldg(cw + ((c >> 1) + 1) * 32);
            if (cc >= LM_STAGES) mbar_wait(&empty[s], ((cc / LM_STAGES) - 1) & 1u);
            const uint32_t w32 = (uint32_t)(cur >> (32 * (c & 1)));
            const uint32_t arow = smem_u32(sA + s * LM_A_BYTES) + row * 128;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              uint32_t x = 0, y = 0, z = 0, w = 0;
              if (ivalid) onehot16((w32 >> (4 * k)) & 15u, x, y, z, w);
              st_shared_v4(arow + ((k ^ (row & 7)) << 4), x, y, z, w);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
          }
        }
      } else if (warp == LM_MMA_WARP) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
          const uint32_t idesc =
              (2u << 4) | ((uint32_t)(Npad >> 3) << 17) | ((uint32_t)(LM_IT >> 4) << 24);
          uint32_t cc = chunk_ctr, tc = tile_ctr;
          for (uint32_t t = 0; t < ntiles; ++t, ++tc) {
            const int acc = tc & 1;
            if (tc >= 2) mbar_wait(&tempty[acc], ((tc >> 1) - 1) & 1u);
            tc_fence_after();
            const uint32_t dt = tmem + (uint32_t)(acc * LM_QT);
            for (int c = 0; c < a.nchunk; ++c, ++cc) {
              const int s = cc % LM_STAGES;
              mbar_wait(&full[s], (cc / LM_STAGES) & 1u);
              tc_fence_after();
              const uint64_t ad = umma_desc_sw128(sA + s * LM_A_BYTES);
              const uint64_t bd = umma_desc_sw128(sB + c * LM_BC_BYTES);
#pragma unroll
              for (int k = 0; k < 4; ++k)  // K = 32 bytes per MMA = +2 desc units
                umma_i8(dt, ad + 2 * k, bd + 2 * k, idesc, (c | k) != 0 ? 1u : 0u);
              umma_commit(&empty[s]);
            }
            umma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
      } else {
        // ---------------- epilogue ----------------
        const int lg = warp & 3;  // TMEM lane group of this warp
        const int row = lg * 32 + lane;
        uint32_t tc = tile_ctr;
        for (uint32_t t = 0; t < ntiles; ++t, ++tc) {
          const int acc = tc & 1;
          const uint32_t item = t * LM_IT + row;
          const bool ivalid = item < Nl;
          int myref = -1;
          if (ivalid && item >= own) {
            int j = 0;
            while (refoff[j + 1] <= item) ++j;
            myref = j;
          }
          uint64_t ok = (nq_tile >= 64) ? ~0ull : ((1ull << nq_tile) - 1ull);
          if (myref >= 0) ok &= ~((uint64_t)skipT[myref * 2] | ((uint64_t)skipT[myref * 2 + 1] << 32));
          if (!ivalid) ok = 0;
          mbar_wait(&tfull[acc], (tc >> 1) & 1u);
          tc_fence_after();
          const uint64_t base = a.sbase[l] + (uint64_t)q0 * Nl + item;
          for (int cb = 0; cb < Npad; cb += 16) {
            uint32_t v[16];
            tmem_ld16(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * LM_QT + cb), v);
            if ((ok >> cb) & 0xFFFFull) {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if ((ok >> (cb + j)) & 1ull) {
                  const uint64_t o = base + (uint64_t)(cb + j) * Nl;
                  if (a.score_u32) reinterpret_cast<uint32_t*>(a.S)[o] = v[j];
                  else reinterpret_cast<uint16_t*>(a.S)[o] = (uint16_t)v[j];
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
      }
      chunk_ctr += ntiles * a.nchunk;
      tile_ctr += ntiles;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == LM_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * LM_QT);
  }
}

// ---------------------------------------------------------------------------
// Per query (one WARP per query): SEIL ranges over its score rows (R9 dedup),
// histogram-threshold top-bigK with warp-private state (no CTA barriers).
constexpr int SW_WARPS = 16;
constexpr int SW_NB = 512;

struct SelArgs {
  const int32_t* probes;
  const uint32_t* qslot;
  const uint32_t* qbits;
  int qwords;
  int64_t nq;
  int nprobe, bigK, cap, hshift;
  const uint32_t* own_off;
  const uint32_t* own_cnt;
  const uint32_t* ref_ptr;
  const int32_t* ref_owner;
  const uint32_t* ref_start;
  const uint32_t* ref_cnt;
  const uint32_t* ref_item_off;
  const uint32_t* list_items;
  const uint32_t* slot_rows;
  const uint64_t* sbase;
  const void* S;
  int score_u32;
  int shard_id, nshards;
  uint64_t* out_keys;
  int64_t* dco;
};

__device__ __forceinline__ uint32_t warp_bthr(const uint32_t* hist, uint32_t bigK) {
  // smallest bin b with cumulative count >= bigK (else the last bin)
  const int lane = lane_id();
  constexpr int PER = SW_NB / 32;
  uint32_t h[PER], loc = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) { h[i] = hist[lane * PER + i]; loc += h[i]; }
  uint32_t inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  const unsigned hit = __ballot_sync(0xffffffffu, inc >= bigK);
  if (!hit) return SW_NB - 1;
  const int hl = __ffs(hit) - 1;
  uint32_t b = SW_NB - 1;
  if (lane == hl) {
    uint32_t run = inc - loc;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      run += h[i];
      if (run >= bigK) { b = lane * PER + i; break; }
    }
  }
  return __shfl_sync(0xffffffffu, b, hl);
}

// keep entries with bin <= bthr and key < tau (warp-level stream compaction)
__device__ __forceinline__ uint32_t warp_filter(uint64_t* cand, uint32_t n, uint32_t bthr,
                                                uint64_t tau, int hshift) {
  const int lane = lane_id();
  uint32_t out = 0;
  for (uint32_t i0 = 0; i0 < n; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint64_t v = (i < n) ? cand[i] : kKeyInf;
    const bool k = i < n && (uint32_t)(v >> (32 + hshift)) <= bthr && v <= tau;
    const unsigned bal = __ballot_sync(0xffffffffu, k);
    __syncwarp();
    if (k) cand[out + __popc(bal & ((1u << lane) - 1u))] = v;
    out += __popc(bal);
    __syncwarp();
  }
  return out;
}

__device__ void warp_sort_keys(uint64_t* a, int n) {
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

__global__ void __launch_bounds__(SW_WARPS * 32) lm_select_kernel(SelArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = warp_id(), lane = lane_id();
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm) + warp * SW_NB;
  uint64_t* cand = reinterpret_cast<uint64_t*>(reinterpret_cast<uint32_t*>(sm) + SW_WARPS * SW_NB) +
                   (size_t)warp * a.cap;
  const uint32_t bigK = (uint32_t)a.bigK;
  for (int64_t q = (int64_t)blockIdx.x * SW_WARPS + warp; q < a.nq;
       q += (int64_t)gridDim.x * SW_WARPS) {
    for (int i = lane; i < SW_NB; i += 32) hist[i] = 0u;
    __syncwarp();
    uint32_t cnt = 0, bthr = SW_NB - 1, since = 0, dco = 0;
    uint64_t tau = kKeyInf;
    const uint32_t* qb = a.qbits + (size_t)q * a.qwords;
    for (int p = 0; p < a.nprobe; ++p) {
      const uint32_t l = (uint32_t)a.probes[q * a.nprobe + p];
      const uint32_t Nl = a.list_items[l];
      const uint64_t row = a.sbase[l] + (uint64_t)a.qslot[q * a.nprobe + p] * Nl;
      const uint32_t r0 = a.ref_ptr[l], nref = a.ref_ptr[l + 1] - r0;
      for (int src = -1; src < (int)nref; ++src) {
        uint32_t n, slot0;
        uint64_t off;
        if (src < 0) {
          n = a.own_cnt[l];
          slot0 = a.own_off[l];
          off = row;
        } else {
          const int o = a.ref_owner[r0 + src];
          if ((qb[o >> 5] >> (o & 31)) & 1u) continue;   // owner probed: scanned there (R9)
          n = a.ref_cnt[r0 + src];
          slot0 = a.ref_start[r0 + src];
          off = row + a.ref_item_off[r0 + src];
        }
        dco += n;
        for (uint32_t i00 = 0; i00 < n; i00 += 128) {
          uint32_t sv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {  // 4 independent loads in flight per lane
            const uint32_t i = i00 + 32 * u + lane;
            sv[u] = 0;
            if (i < n)
              sv[u] = a.score_u32 ? reinterpret_cast<const uint32_t*>(a.S)[off + i]
                                  : (uint32_t)reinterpret_cast<const uint16_t*>(a.S)[off + i];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t i = i00 + 32 * u + lane;
            if (i00 + 32 * u >= n) break;   // warp-uniform
            const bool valid = i < n;
            const uint32_t s = sv[u];
            const uint32_t bin = s >> a.hshift;
            const bool maybe = valid && bin <= bthr;
            if (!__any_sync(0xffffffffu, maybe)) continue;
            uint64_t key = kKeyInf;
            if (maybe) {
              const uint32_t r = a.slot_rows[slot0 + i];
              key = ((uint64_t)s << 32) | (r * (uint32_t)a.nshards + (uint32_t)a.shard_id);
            }
            const bool pass = maybe && key < tau;
            const unsigned bal = __ballot_sync(0xffffffffu, pass);
            if (pass) {
              cand[cnt + __popc(bal & ((1u << lane) - 1u))] = key;
              atomicAdd(&hist[bin], 1u);
            }
            cnt += __popc(bal);
            since += __popc(bal);
            __syncwarp();
            if (since >= 64) {
              since = 0;
              bthr = min(bthr, warp_bthr(hist, bigK));
            }
            if (cnt + 32 > (uint32_t)a.cap) {
              bthr = min(bthr, warp_bthr(hist, bigK));
              cnt = warp_filter(cand, cnt, bthr, tau, a.hshift);
              if (cnt + 32 > (uint32_t)a.cap) {   // pathological ties: sort, keep bigK exactly
                int np = 2;
                while (np < (int)cnt) np <<= 1;
                for (int e = cnt + lane; e < np; e += 32) cand[e] = kKeyInf;
                __syncwarp();
                warp_sort_keys(cand, np);
                cnt = bigK;
                tau = cand[bigK - 1];
              }
            }
          }
        }
      }
    }
    bthr = min(bthr, warp_bthr(hist, bigK));
    cnt = warp_filter(cand, cnt, bthr, tau, a.hshift);
    int np = 2;
    while (np < (int)cnt) np <<= 1;
    for (int e = cnt + lane; e < np; e += 32) cand[e] = kKeyInf;
    __syncwarp();
    warp_sort_keys(cand, np);
    const uint32_t keep = min(cnt, bigK);
    for (int e = lane; e < a.bigK; e += 32) a.out_keys[q * a.bigK + e] = ((uint32_t)e < keep) ? cand[e] : kKeyInf;
    if (lane == 0 && a.dco) a.dco[q] = (int64_t)dco;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
static int sel_cap(int bigK) { return next_pow2(2 * bigK + 64); }

bool listmajor_ok(const rairs_index_s* idx, int nprobe, int bigK) {
  if (idx->scan_mode == 1) return false;            // forced SIMT query-major scan
  if (!idx->list_items || !idx->ref_item_off) return false;
  if (idx->max_refs > LM_MAXREF) return false;
  if ((size_t)(idx->M_pad / 8) * LM_BC_BYTES + 4 * LM_A_BYTES > 200 * 1024) return false;
  if ((size_t)SW_WARPS * (SW_NB * 4 + (size_t)sel_cap(bigK) * 8) > 200 * 1024) return false;
  return true;
}

rairs_status launch_listmajor(const rairs_index_s* idx, const SearchArgs& sa, cudaStream_t s) {
  const int64_t nq = sa.nq;
  if (nq <= 0) return RAIRS_OK;
  const int nprobe = sa.nprobe, nlist = idx->nlist;
  const int bigK = sa.k * sa.refine_factor;
  const int K = idx->M_pad * 16;
  const int qwords = (nlist + 31) / 32;
  const int64_t npairs = nq * nprobe;
  const int score_u32 = ((int64_t)idx->M * 255 > 65535) ? 1 : 0;
  uint8_t* lut = nullptr;
  uint32_t *cnt = nullptr, *qslot = nullptr, *qptr = nullptr, *tptr = nullptr, *list_q = nullptr,
           *qbits = nullptr, *totals = nullptr;
  uint64_t* sbase = nullptr;
  void* S = nullptr;
  // bound on the score buffer: every (query, probe) pair times the largest list-task
  const size_t s_elems = (size_t)npairs * (size_t)std::max<int64_t>(idx->max_list_items, 1);
  const size_t s_bytes = s_elems * (score_u32 ? 4 : 2);
  auto cleanup = [&]() {
    cudaFreeAsync(lut, s); cudaFreeAsync(cnt, s); cudaFreeAsync(qslot, s); cudaFreeAsync(qptr, s);
    cudaFreeAsync(tptr, s); cudaFreeAsync(list_q, s); cudaFreeAsync(qbits, s);
    cudaFreeAsync(totals, s); cudaFreeAsync(sbase, s); cudaFreeAsync(S, s);
  };
#define LM_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { set_error(std::string(#x) + ": " + cudaGetErrorString(_e)); cleanup(); return _e == cudaErrorMemoryAllocation ? RAIRS_E_OOM : RAIRS_E_CUDA; } } while (0)
  LM_TRY(cudaMallocAsync(&lut, (size_t)nq * K, s));
  LM_TRY(cudaMallocAsync(&cnt, (size_t)(nlist + 1) * 4 + 16, s));
  LM_TRY(cudaMallocAsync(&qslot, (size_t)npairs * 4, s));
  LM_TRY(cudaMallocAsync(&qptr, (size_t)(nlist + 1) * 4, s));
  LM_TRY(cudaMallocAsync(&tptr, (size_t)(nlist + 1) * 4, s));
  LM_TRY(cudaMallocAsync(&list_q, (size_t)npairs * 4, s));
  LM_TRY(cudaMallocAsync(&qbits, (size_t)nq * qwords * 4, s));
  LM_TRY(cudaMallocAsync(&totals, 16, s));
  LM_TRY(cudaMallocAsync(&sbase, (size_t)(nlist + 1) * 8, s));
  LM_TRY(cudaMallocAsync(&S, std::max<size_t>(s_bytes, 16), s));
  LM_TRY(cudaMemsetAsync(cnt, 0, (size_t)(nlist + 1) * 4 + 16, s));
  LM_TRY(cudaMemsetAsync(qbits, 0, (size_t)nq * qwords * 4, s));
  unsigned* list_counter = cnt + nlist + 1;  // zeroed tail of cnt
  // 1. quantised LUTs (O2), one warp per query
  lut_batch_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nq, LW), 1 << 30), LW * 32, 0, s>>>(
      sa.queries, nq, idx->d, idx->codebook, idx->M, idx->M_pad, idx->dsub, lut, sa.lut_a, sa.lut_b,
      sa.lut_q);
  LM_TRY(cudaGetLastError());
  // 2. group (query, probe) pairs by list
  const unsigned g1 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(npairs, 256), 148 * 8));
  lm_count_kernel<<<g1, 256, 0, s>>>(sa.probes, npairs, cnt, qslot);
  lm_scan_kernel<<<1, SCN, 0, s>>>(cnt, idx->list_items, nlist, qptr, sbase, tptr, totals, LM_QT,
                                   LM_IT);
  lm_scatter_kernel<<<g1, 256, 0, s>>>(sa.probes, npairs, nprobe, qptr, qslot, list_q, qbits, qwords);
  LM_TRY(cudaGetLastError());
  // 3. tensor-core scores, one list at a time
  LMArgs la{};
  la.codes64 = reinterpret_cast<const uint64_t*>(idx->codes);
  la.own_off = idx->own_off;
  la.own_cnt = idx->own_cnt;
  la.ref_ptr = idx->ref_ptr;
  la.ref_owner = idx->ref_owner;
  la.ref_start = idx->ref_start;
  la.ref_item_off = idx->ref_item_off;
  la.list_items = idx->list_items;
  la.NU = idx->M_pad / 16;
  la.nchunk = idx->M_pad / 8;
  la.lut = lut;
  la.K = K;
  la.b_resident = 1;  // LUT tile (64 queries x K) resident per query tile
  la.probes = sa.probes;
  la.nprobe = nprobe;
  la.qptr = qptr;
  la.list_q = list_q;
  la.list_counter = list_counter;
  la.sbase = sbase;
  la.S = S;
  la.score_u32 = score_u32;
  la.nlist = nlist;
  const size_t tsm = 1024 + LM_STAGES * LM_A_BYTES + (size_t)la.nchunk * LM_BC_BYTES + LM_MAXREF * 8 +
                     8 + LM_MAXREF * 8 + LM_QT * 4 + (2 * LM_STAGES + 4) * 8 + 64;
  LM_TRY(cudaFuncSetAttribute(lm_tensor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
  const int per_sm = (tsm <= 110 * 1024) ? 2 : 1;
  lm_tensor_kernel<<<148 * per_sm, LM_WS_THREADS, tsm, s>>>(la);
  LM_TRY(cudaGetLastError());
  // 4. per-query selection (warp per query)
  SelArgs sl{};
  sl.probes = sa.probes;
  sl.qslot = qslot;
  sl.qbits = qbits;
  sl.qwords = qwords;
  sl.nq = nq;
  sl.nprobe = nprobe;
  sl.bigK = bigK;
  sl.cap = sel_cap(bigK);
  sl.hshift = 0;
  while (((int64_t)idx->M * 255) >> sl.hshift >= SW_NB) ++sl.hshift;
  sl.own_off = idx->own_off;
  sl.own_cnt = idx->own_cnt;
  sl.ref_ptr = idx->ref_ptr;
  sl.ref_owner = idx->ref_owner;
  sl.ref_start = idx->ref_start;
  sl.ref_cnt = idx->ref_cnt;
  sl.ref_item_off = idx->ref_item_off;
  sl.list_items = idx->list_items;
  sl.slot_rows = idx->slot_rows;
  sl.sbase = sbase;
  sl.S = S;
  sl.score_u32 = score_u32;
  sl.shard_id = idx->shard_id;
  sl.nshards = idx->nshards;
  sl.out_keys = sa.cand_keys;
  sl.dco = sa.dco;
  const size_t ssm = (size_t)SW_WARPS * (SW_NB * 4 + (size_t)sl.cap * 8);
  LM_TRY(cudaFuncSetAttribute(lm_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
  lm_select_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nq, SW_WARPS), 1 << 30), SW_WARPS * 32, ssm, s>>>(sl);
  LM_TRY(cudaGetLastError());
  cleanup();
  return RAIRS_OK;
#undef LM_TRY
}

// build-time tables: N_l and the item offset of each reference in its list-task
__global__ void lm_items_kernel(const uint32_t* __restrict__ own_cnt,
                                const uint32_t* __restrict__ ref_ptr,
                                const uint32_t* __restrict__ ref_cnt, int nlist,
                                uint32_t* __restrict__ list_items,
                                uint32_t* __restrict__ ref_item_off) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlist; l += gridDim.x * blockDim.x) {
    uint32_t off = own_cnt[l];
    for (uint32_t j = ref_ptr[l]; j < ref_ptr[l + 1]; ++j) {
      ref_item_off[j] = off;
      off += ref_cnt[j];
    }
    list_items[l] = off;
  }
}

rairs_status listmajor_prepare(rairs_index_s* idx, cudaStream_t s) {
  RAIRS_CUDA_TRY(cudaMalloc(&idx->list_items, (size_t)idx->nlist * 4));
  RAIRS_CUDA_TRY(cudaMalloc(&idx->ref_item_off, (size_t)std::max<int64_t>(idx->n_refs, 1) * 4));
  lm_items_kernel<<<(idx->nlist + 255) / 256, 256, 0, s>>>(idx->own_cnt, idx->ref_ptr, idx->ref_cnt,
                                                          idx->nlist, idx->list_items,
                                                          idx->ref_item_off);
  RAIRS_CHECK_LAUNCH();
  std::vector<uint32_t> h(idx->nlist);
  RAIRS_CUDA_TRY(cudaMemcpyAsync(h.data(), idx->list_items, (size_t)idx->nlist * 4,
                                 cudaMemcpyDeviceToHost, s));
  RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  idx->max_list_items = 0;
  for (uint32_t v : h) idx->max_list_items = std::max<int64_t>(idx->max_list_items, v);
  idx->device_bytes += (size_t)idx->nlist * 4 + (size_t)std::max<int64_t>(idx->n_refs, 1) * 4;
  return RAIRS_OK;
}

}  // namespace rairs
