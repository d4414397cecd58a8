// listmajor_kernels.cu -- list-major batched fast scan on tensor cores (A3-A6).
//
// The paper's query-batch cache optimisation ("group the tasks by
// lists, and process all the queries for the same list back to back") on B200:
// for a list l probed by the queries Q_l of a batch, the integer scores of all
// (item, query) pairs are ONE exact u8 x u8 -> s32 contraction
//     S[x][q] = sum_m Qv_q[m][code_m(x)] = sum_{m,j} onehot(x)[m*16+j] * Qv_q[m][j]
// (K = 16*M), issued as tcgen05.mma.kind::i8 (M = 128 items, N = |Q_l| tile
// padded to 16, K = 32 per instruction) with A (the one-hot rows, expanded from
// the 4-bit codes in registers and written with tcgen05.st) in TMEM, B (the
// queries' quantised LUT rows) in shared memory and the accumulator in TMEM.
// Each code byte is read ONCE per list-task instead of once per (list, query).
// Integer sums are exact (<= 16*M*255 < 2^31): scores are bit-identical to O8.
//
// Pipeline for a batch (all on the search stream, no host sync):
//   lm_count / lm_scan / lm_scatter   group the (query, probe) pairs by list
//   lut_tiles_kernel   O2 LUT per query, written into its list-tasks' B tiles
//   lm_tensor_kernel   persistent; task = (list, query tile) -> u16/u32 score
//                      rows (sentinel for SEIL-skipped references, R9)
//   lm_select_kernel   per query: DCO, two-pass histogram top-bigK by (s, id)
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "index.cuh"
#include "tc_helpers.cuh"

namespace rairs {

// ---------------------------------------------------------------------------
// Grouping of (query, probe) pairs by list.
// zeroes the list counters (a kernel, not a memset, so the chain from the
// coarse stage to the scan stays programmatic-dependent-launch)
__global__ void lm_zero_kernel(uint32_t* __restrict__ a, int64_t n) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = 0u;
  pdl_trigger();
}

__global__ void lm_count_kernel(const int32_t* __restrict__ probes, int64_t total,
                                uint32_t* __restrict__ cnt, uint32_t* __restrict__ qslot,
                                uint32_t* __restrict__ qbits, int64_t nbits_words) {
  pdl_wait();  // zeroed counters (lm_zero_kernel) and the probes of the coarse stage
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    qslot[e] = atomicAdd(&cnt[probes[e]], 1u);
  // the per-query probe bitmaps are zeroed here (lm_scatter, launched next, sets them)
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nbits_words;
       w += (int64_t)gridDim.x * blockDim.x)
    qbits[w] = 0u;
  pdl_trigger();
}

__global__ void lm_scatter_kernel(const int32_t* __restrict__ probes, int64_t total, int nprobe,
                                  const uint32_t* __restrict__ qptr,
                                  const uint32_t* __restrict__ qslot, uint32_t* __restrict__ list_q,
                                  uint32_t* __restrict__ qbits, int qwords) {
  pdl_wait();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int l = probes[e];
    const uint32_t q = (uint32_t)(e / nprobe);
    list_q[qptr[l] + qslot[e]] = q;
    atomicOr(&qbits[(size_t)q * qwords + (l >> 5)], 1u << (l & 31));
  }
  pdl_trigger();
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
  pdl_wait();
  __syncthreads();
  for (int base = 0; base < nlist; base += SCN) {
    const int l = base + tid;
    uint32_t c = 0, t = 0;
    uint64_t s = 0;
    if (l < nlist) {
      c = cnt[l];
      const uint32_t ni = nitems[l];
      s = (uint64_t)c * ((ni + 7u) & ~7u);   // score rows padded to 8 items (16-B aligned)
      t = (c + 15u) & ~15u;  // LUT-tile rows of list l (query tiles padded to 16)
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
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// O2 LUT per query, written straight into the pre-tiled, pre-swizzled LUT
// tiles of every list-task the query belongs to (one row per (query, probe)):
// tile t of list l holds the rows of queries t*QT.. of Q_l as nchunk K-chunks
// of [Npad rows x 128 B] in the 128-B-swizzled K-major layout tcgen05 reads,
// so the tensor kernel fetches a whole B tile with ONE bulk copy.
// One WARP per query, lane = subquantizer m (m = lane, lane+32, ...): the 16
// distances T[m][j] are computed in registers (fp32, ascending t, no FMA --
// R2), the codebook is staged transposed in shared memory ([j][t][m]: lanes
// read consecutive words).  b = sum_m mn_m is summed by lane 0 in ascending m.
constexpr int LW = 8;  // warps (queries) per CTA

template <int DSUB>
__device__ __forceinline__ float lut_T(const float* qs, const float* smc, int m, int j, int M) {
  float acc = 0.0f;
#pragma unroll
  for (int t = 0; t < DSUB; ++t) {
    const float diff = __fsub_rn(qs[t], smc[(j * DSUB + t) * M + m]);
    acc = __fadd_rn(acc, __fmul_rn(diff, diff));
  }
  return acc;
}

template <int DSUB, int MPL>
__global__ void __launch_bounds__(LW * 32, 3) lut_tiles_kernel(
    const float* __restrict__ queries, int64_t nq, int d, const float* __restrict__ cb, int M,
    int M_pad, const int32_t* __restrict__ probes, int nprobe,
    const uint32_t* __restrict__ qslot, const uint32_t* __restrict__ qcnt,
    const uint32_t* __restrict__ lrow, int QT, uint8_t* __restrict__ tiles,
    float* __restrict__ a_out, float* __restrict__ b_out, uint8_t* __restrict__ lut_dbg) {
  extern __shared__ __align__(16) float smc[];  // [16][dsub][M] codebook, then [LW][M] mn
  const int lane = lane_id(), warp = warp_id();
  const int K = M_pad * 16;
  for (int e = threadIdx.x; e < M * 16 * DSUB; e += blockDim.x) {
    const int m = e / (16 * DSUB), j = (e / DSUB) % 16, t = e % DSUB;
    smc[(j * DSUB + t) * M + m] = cb[e];
  }
  pdl_wait();  // the grouping kernels' qslot / cnt / lrow (the codebook above is the index's)
  __syncthreads();
  float* mnw = smc + 16 * DSUB * M + warp * M;
  // MPL: subquantizers per lane (ceil(M_pad / 32) <= 4 on the list-major path)
  // the destination of query q's row in each probed list-task's tile: lane p
  // (< nprobe) resolves probe p; the row loop reads it by shuffle
  auto dst_of = [&](int64_t q, int p, uint64_t& base, uint32_t& npad, uint32_t& jqo) {
    const int l = probes[q * nprobe + p];
    const uint32_t j = qslot[q * nprobe + p], Ql = qcnt[l];
    const uint32_t t = j / (uint32_t)QT;
    jqo = j - t * (uint32_t)QT;
    npad = (t < Ql / (uint32_t)QT) ? (uint32_t)QT : ((Ql - t * QT + 15u) & ~15u);
    base = ((uint64_t)lrow[l] + (uint64_t)t * QT) * K;
  };
  auto load_q = [&](int64_t q, float (&qs)[MPL][DSUB]) {
#pragma unroll
    for (int u = 0; u < MPL; ++u) {
      const int m = lane + 32 * u;
#pragma unroll
      for (int t = 0; t < DSUB; ++t) qs[u][t] = (m < M) ? __ldg(queries + q * d + m * DSUB + t) : 0.0f;
    }
  };
  const int64_t qstride = (int64_t)gridDim.x * LW;
  int64_t q = (int64_t)blockIdx.x * LW + warp;
  // the next query's values and destinations are loaded one query ahead
  float qsn[MPL][DSUB];
  uint64_t dbn = 0;
  uint32_t dnn = 0, djn = 0;
  if (q < nq) {
    load_q(q, qsn);
    if (lane < nprobe) dst_of(q, lane, dbn, dnn, djn);
  }
  for (; q < nq; q += qstride) {
    float qsc[MPL][DSUB];
#pragma unroll
    for (int u = 0; u < MPL; ++u)
#pragma unroll
      for (int t = 0; t < DSUB; ++t) qsc[u][t] = qsn[u][t];
    const uint64_t dst_base = dbn;
    const uint32_t dst_npad = dnn, dst_jq = djn;
    if (q + qstride < nq) {
      load_q(q + qstride, qsn);
      if (lane < nprobe) dst_of(q + qstride, lane, dbn, dnn, djn);
    }
    float T[MPL][16];
    float S = 0.0f;
#pragma unroll
    for (int u = 0; u < MPL; ++u) {  // pass 1: distances, per-subquantizer min and span
      const int m = lane + 32 * u;
      if (m < M) {
        const float* qs = qsc[u];
        float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          T[u][j] = lut_T<DSUB>(qs, smc, m, j, M);
          lo = fminf(lo, T[u][j]);
          hi = fmaxf(hi, T[u][j]);
        }
        mnw[m] = lo;
        S = fmaxf(S, __fsub_rn(hi, lo));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) S = fmaxf(S, __shfl_xor_sync(0xffffffffu, S, o));
    const float a = (S > 0.0f) ? __fdiv_rn(255.0f, S) : 1.0f;
    __syncwarp();
    if (lane == 0 && (a_out || b_out)) {  // parity/debug outputs only
      float bsum = 0.0f;
      for (int m = 0; m < M; ++m) bsum = __fadd_rn(bsum, mnw[m]);  // ascending m (O2 step 5)
      if (a_out) a_out[q] = a;
      if (b_out) b_out[q] = bsum;
    }
#pragma unroll
    for (int u = 0; u < MPL; ++u) {  // pass 2: quantise, write every tile row
      const int m = lane + 32 * u;
      if (32 * u >= M_pad) break;  // warp-uniform
      uint32_t w[4] = {0u, 0u, 0u, 0u};
      if (m < M) {
        const float lo = mnw[m];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          uint32_t v = 0;
          if (S > 0.0f) v = (uint32_t)min(255, __float2int_rn(__fmul_rn(__fsub_rn(T[u][j], lo), a)));
          w[j >> 2] |= v << (8 * (j & 3));
        }
        if (lut_dbg)
          *reinterpret_cast<uint4*>(lut_dbg + (size_t)q * M * 16 + m * 16) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      {  // all lanes take part in the shuffles; lanes m >= M_pad store nothing
        const int c = m >> 3, kk = m & 7;
        for (int p = 0; p < nprobe; ++p) {
          uint64_t base;
          uint32_t npad, jq;
          if (p < 32) {  // warp-uniform
            base = __shfl_sync(0xffffffffu, dst_base, p);
            npad = __shfl_sync(0xffffffffu, dst_npad, p);
            jq = __shfl_sync(0xffffffffu, dst_jq, p);
          } else {
            dst_of(q, p, base, npad, jq);
          }
          if (m >= M_pad) continue;
          *reinterpret_cast<uint4*>(tiles + base + (size_t)c * npad * 128 + jq * 128 +
                                    ((kk ^ (jq & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
    __syncwarp();  // mnw reuse
  }
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// Tensor-core scoring, one list at a time (CTAs claim lists atomically).
constexpr int LM_IT = 128;        // items per tile (MMA M)
constexpr int LM_QT = 64;         // max queries per tile (MMA N <= 64)
constexpr int LM_MAXREF = 2048;   // references per list on this path
constexpr uint32_t LM_B_MAX = 64 * 1024;  // LUT tile bytes (QT x K)

struct LMArgs {
  const uint64_t* codes64;
  const uint32_t* own_off;
  const uint32_t* own_cnt;
  const uint32_t* ref_ptr;
  const int32_t* ref_owner;
  const uint32_t* ref_start;
  const uint32_t* ref_item_off;  // item offset of each reference inside its list-task
  const uint32_t* list_items;    // N_l = own_cnt + sum of the list's ref_cnt
  int K, QT;                     // LUT bytes per query (16 * M_pad); queries per tile
  const uint8_t* tiles;          // pre-tiled LUT (lut_tiles_kernel)
  const uint32_t* lrow;          // [nlist] first LUT-tile row of list l
  const int32_t* probes;
  int nprobe;
  const uint32_t* qptr;
  const uint32_t* list_q;
  unsigned* list_counter;
  const uint64_t* sbase;
  void* S;
  int score_u32;
  int nlist;
  const uint32_t* order;  // claim order: lists by descending N_l (longest first), or NULL
  // fused mode (no score rows): an item joins query q's candidates iff its score
  // is <= tau[q] (an upper bound of q's bigK-th score, fs_scan threshold mode);
  // entries (s << 39 | list << 22 | item) go to fcand[q][0 .. fcap), fcnt[q] counts
  int fused;
  const uint32_t* tau;
  uint64_t* fcand;
  uint32_t* fcnt;
  int fcap;
};

// D[tmem] (+)= A[tmem] x B[smem desc]  (A: 128 item rows x 32 K-bytes, 8 columns)
__device__ __forceinline__ void umma_i8_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

// warp-wide variants: every lane executes them with the same (warp-uniform)
// operands, one elected lane issues -- the operands stay in uniform registers
// (no per-instruction lane waterfall around a lone-lane issue)
__device__ __forceinline__ void umma_i8_ta_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
          smem_u32(bar))
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

// 32 columns x 32 lanes (this warp's lane quarter) of 32-bit words
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

// reference j of a list-task holding item `item` (>= the owned count):
// the largest j with refoff[j] <= item (refoff ascending, refoff[nref] = N_l)
__device__ __forceinline__ int lm_ref_of(const uint32_t* refoff, uint32_t nref, uint32_t item) {
  int lo = 0, hi = (int)nref;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (refoff[mid] <= item) lo = mid; else hi = mid;
  }
  return lo;
}

template <int G>
__device__ __forceinline__ uint32_t gcnt_of(const uint32_t (&gc)[G], int g) {
  uint32_t v = gc[0];
#pragma unroll
  for (int i = 1; i < G; ++i) v = (g == i) ? gc[i] : v;  // no dynamic register indexing
  return v;
}

// Warp-specialised pipeline (no CTA barrier per tile):
//   generators  LM_GROUPS groups of four warps (group g takes item tiles
//               t = g mod LM_GROUPS); warp w owns item rows 32(w%4).. (TMEM lane
//               quarter w%4).  Per K-chunk (8 subquantizers = 128 one-hot bytes
//               per row) it expands the 4-bit codes into 32 words in registers
//               and writes them to one of its group's 4 TMEM A stages with
//               tcgen05.st, then arrives on full[stage].  Codes of the group's
//               next tile are loaded while the current one is expanded.
//   MMA warp    waits full[stage], issues 4 x tcgen05.mma.kind::i8 (A from
//               TMEM, B = LUT tile in shared memory) into one of 2 TMEM
//               accumulators, commits empty[stage] and, after a tile, tfull[acc].
//   epilogue    8 warps, 2 per lane quarter (alternating 16-column blocks):
//               tcgen05.ld the scores, store the (item, query) scores /
//               sentinels, arrive tempty[acc].
// The LUT tile of a query tile arrives by one cp.async.bulk (pre-tiled by
// lut_tiles_kernel); a CTA barrier separates query tiles.  TMEM: the A ring
// (32 columns per stage) then two 64-column accumulators.
// Pipeline shape: G generator groups of 4 warps, GS TMEM A stages per group.
template <int G, int GS>
struct LMShape {
  static constexpr int GEN_WARPS = 4 * G, MMA_WARP = 4 * G, EPI0 = 4 * G + 1, EPI_WARPS = 8;
  static constexpr int THREADS = (EPI0 + EPI_WARPS) * 32;
  static constexpr int STAGES = G * GS;
  static constexpr uint32_t ACC_COL = 32 * STAGES;  // accumulators after the A ring
  static constexpr uint32_t COLS_USED = ACC_COL + 2 * 64;
  static constexpr uint32_t TMEM_COLS = COLS_USED <= 256 ? 256 : 512;
  static constexpr int CTAS_PER_SM = TMEM_COLS == 256 ? 2 : 1;
};

template <int NU, int G, int GS>
__global__ void __launch_bounds__(LMShape<G, GS>::THREADS, LMShape<G, GS>::CTAS_PER_SM)
    lm_tensor_kernel(LMArgs a) {
  using SH = LMShape<G, GS>;
  constexpr int LM_GROUPS = G, LM_STAGES = SH::STAGES;
  constexpr int LM_GPAIRS = GS / 2;  // pair-stages (two chunks each) per group
  static_assert(GS % 2 == 0, "stages come in pairs");
  constexpr int LM_GEN_WARPS = SH::GEN_WARPS, LM_MMA_WARP = SH::MMA_WARP, LM_EPI0 = SH::EPI0;
  constexpr int LM_EPI_WARPS = SH::EPI_WARPS, LM_WS_THREADS = SH::THREADS;
  constexpr uint32_t LM_ACC_COL = SH::ACC_COL, LM_TMEM_COLS = SH::TMEM_COLS;
  constexpr int NCHUNK = 2 * NU;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
  uint8_t* sB = smem;                                                    // <= LM_B_MAX
  int32_t* owners = reinterpret_cast<int32_t*>(sB + LM_B_MAX);          // [LM_MAXREF]
  uint32_t* refoff = reinterpret_cast<uint32_t*>(owners + LM_MAXREF);   // [LM_MAXREF+1]
  uint32_t* skipT = refoff + LM_MAXREF + 1;  // [LM_MAXREF][2]: queries skipping ref j
  uint32_t* qid = skipT + LM_MAXREF * 2;     // [LM_QT]
  uint32_t* qtau = qid + LM_QT;              // [LM_QT] fused mode: tau of the tile's queries
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(qtau + LM_QT) + 7) & ~(uintptr_t)7);  // [LM_STAGES]
  uint64_t* empty = full + LM_STAGES;
  uint64_t* tfull = empty + LM_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint64_t* bfull = tempty + 2;         // LUT tile landed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bfull + 1);
  __shared__ uint32_t sh_list;
  // one-hot rows of the 16 nibble values (16 B each): generation is one
  // shared-memory load per nibble instead of ~9 ALU instructions
  __shared__ __align__(16) uint4 onehot16[16];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 16) {
    const uint32_t b = 1u << (8 * (tid & 3));
    const int w = tid >> 2;
    onehot16[tid] = make_uint4(w == 0 ? b : 0u, w == 1 ? b : 0u, w == 2 ? b : 0u, w == 3 ? b : 0u);
  }
  if (tid == 0) {
    for (int s = 0; s < LM_GROUPS * LM_GPAIRS; ++s) {
      mbar_init(&full[s], 4);  // the 4 lane-quarter warps of the tile's generator group
      mbar_init(&empty[s], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&tfull[k], 1);
      mbar_init(&tempty[k], LM_EPI_WARPS);
    }
    mbar_init(bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == LM_MMA_WARP) tmem_alloc(tslot, LM_TMEM_COLS);
  pdl_wait();  // LUT tiles and grouping of the previous kernels
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // chunks produced / consumed so far per generator group (same values in every
  // role).  Each group owns its own 4-stage half of the A ring, so a group is
  // never more than one phase ahead of the MMA on any of its stages (an
  // mbarrier parity wait cannot tell phase k from phase k+2).
  uint32_t gcnt[G];
#pragma unroll
  for (int g = 0; g < G; ++g) gcnt[g] = 0;
  uint32_t tile_ctr = 0;   // item tiles so far
  uint32_t qt_ctr = 0;     // query tiles so far (bfull phase)

  for (;;) {
    if (tid == 0) {  // longest list-tasks first: the persistent CTAs finish together
      const uint32_t c = atomicAdd(a.list_counter, 1u);
      sh_list = (c < (uint32_t)a.nlist && a.order) ? a.order[c] : c;
    }
    __syncthreads();
    const uint32_t l = sh_list;
    __syncthreads();  // everyone has read sh_list before thread 0 may overwrite it
    if (l >= (uint32_t)a.nlist) break;
    const uint32_t Ql = a.qptr[l + 1] - a.qptr[l];
    const uint32_t Nl = a.list_items[l];
    const uint32_t Nl8 = (Nl + 7u) & ~7u;  // score row stride
    if (Ql == 0 || Nl == 0) continue;      // uniform across the CTA
    const uint32_t own = a.own_cnt[l], own0 = a.own_off[l];
    const uint32_t r0 = a.ref_ptr[l], nref = a.ref_ptr[l + 1] - r0;
    for (uint32_t j = tid; j < nref; j += LM_WS_THREADS) {
      owners[j] = a.ref_owner[r0 + j];
      refoff[j] = a.ref_item_off[r0 + j];
    }
    if (tid == 0) refoff[nref] = Nl;
    const uint32_t ntiles = (Nl + LM_IT - 1) / LM_IT;
    for (uint32_t q0 = 0; q0 < Ql; q0 += a.QT) {
      const int nq_tile = (int)min(Ql - q0, (uint32_t)a.QT);
      const int Npad = ((nq_tile + 15) / 16) * 16;
      __syncthreads();  // previous query tile fully drained (epilogue waited on its MMAs)
      if (tid == 0) {   // the LUT tile: one bulk copy (already in the UMMA layout)
        const uint32_t bytes = (uint32_t)Npad * (uint32_t)a.K;
        mbar_expect_tx(bfull, bytes);
        bulk_g2s(sB, a.tiles + ((size_t)a.lrow[l] + q0) * a.K, bytes, bfull);
      }
      for (uint32_t j = tid; j < nref * 2; j += LM_WS_THREADS) skipT[j] = 0u;
      if (tid < LM_QT) {
        const uint32_t qq = (tid < nq_tile) ? a.list_q[a.qptr[l] + q0 + tid] : 0xFFFFFFFFu;
        qid[tid] = qq;
        if (a.fused) qtau[tid] = (tid < nq_tile) ? a.tau[qq] : 0u;
      }
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
      __syncthreads();

      if (warp < LM_GEN_WARPS) {
        // ---------------- generators (2 groups of 4: even / odd item tiles) ----------------
        const int quarter = warp & 3, grp = warp >> 2;  // grp < LM_GROUPS
        const int row = quarter * 32 + lane;
        const uint32_t tq = tmem + ((uint32_t)(quarter * 32) << 16);
        auto load_codes = [&](uint32_t t, uint64_t* w) {
          const uint32_t item = t * LM_IT + row;
          if (t < ntiles && item < Nl) {
            uint32_t slot;
            if (item < own) {
              slot = own0 + item;
            } else {
              const int j = lm_ref_of(refoff, nref, item);
              slot = a.ref_start[r0 + j] + (item - refoff[j]);
            }
            const uint64_t* cw = a.codes64 + ((size_t)(slot >> 5) * NU) * 32 + (slot & 31);
#pragma unroll
            for (int u = 0; u < NU; ++u) w[u] = __ldg(cw + u * 32);
          } else {
#pragma unroll
            for (int u = 0; u < NU; ++u) w[u] = 0ull;
          }
        };
        uint64_t cur[NU], nxt[NU], nxt2[NU];  // codes of this group's tiles t, t+G, t+2G
        load_codes((uint32_t)grp, cur);
        load_codes((uint32_t)grp + LM_GROUPS, nxt);
        for (uint32_t t = (uint32_t)grp; t < ntiles; t += LM_GROUPS) {
          load_codes(t + 2 * LM_GROUPS, nxt2);  // two of this group's tiles ahead
          uint32_t cc = gcnt_of(gcnt, grp) + (t / LM_GROUPS) * NCHUNK;  // group chunk index
#pragma unroll
          for (int c = 0; c < NCHUNK; c += 2, cc += 2) {
            // one pair-stage (two K-chunks, 64 TMEM columns) per hand-off: the
            // first tcgen05.st overlaps the second chunk's expansion, one
            // wait::st / arrive / MMA commit per pair
            const uint32_t pc = cc >> 1;                       // group pair index
            const int ps = grp * LM_GPAIRS + (int)(pc % LM_GPAIRS);
            if (pc >= (uint32_t)LM_GPAIRS) mbar_wait(&empty[ps], ((pc / LM_GPAIRS) - 1) & 1u);
            tc_fence_after();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t w32 = (uint32_t)(cur[(c + h) >> 1] >> (32 * ((c + h) & 1)));
              uint32_t v[32];
#pragma unroll
              for (int k = 0; k < 8; ++k) {  // one-hot of nibble n: byte n of 16 = 1
                const uint4 o = onehot16[(w32 >> (4 * k)) & 15u];
                v[4 * k + 0] = o.x;
                v[4 * k + 1] = o.y;
                v[4 * k + 2] = o.z;
                v[4 * k + 3] = o.w;
              }
              tmem_st32(tq + (uint32_t)((2 * ps + h) * 32), v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[ps]);
          }
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            cur[u] = nxt[u];
            nxt[u] = nxt2[u];
          }
        }
      } else if (warp == LM_MMA_WARP) {
        // ---------------- MMA issuer (whole warp, one elected lane issues) ----------------
        {
          const uint32_t idesc =
              (2u << 4) | ((uint32_t)(Npad >> 3) << 17) | ((uint32_t)(LM_IT >> 4) << 24);
          mbar_wait(bfull, qt_ctr & 1u);
          tc_fence_after();
          uint32_t tc = tile_ctr;
          for (uint32_t t = 0; t < ntiles; ++t, ++tc) {
            const int grp = (int)(t % LM_GROUPS);
            uint32_t cc = gcnt_of(gcnt, grp) + (t / LM_GROUPS) * NCHUNK;
            const int acc = tc & 1;
            if (tc >= 2) mbar_wait(&tempty[acc], ((tc >> 1) - 1) & 1u);
            tc_fence_after();
            const uint32_t dt = tmem + LM_ACC_COL + (uint32_t)(acc * LM_QT);
            for (int c = 0; c < NCHUNK; c += 2, cc += 2) {
              const uint32_t pc = cc >> 1;
              const int ps = grp * LM_GPAIRS + (int)(pc % LM_GPAIRS);
              mbar_wait(&full[ps], (pc / LM_GPAIRS) & 1u);
              tc_fence_after();
              {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const uint64_t bd = umma_desc_sw128(sB + (size_t)(c + h) * Npad * 128);
#pragma unroll
                  for (int k = 0; k < 4; ++k)  // K = 32 bytes per MMA: 8 TMEM columns, +2 desc units
                    umma_i8_ta_warp(dt, tmem + (uint32_t)((2 * ps + h) * 32 + 8 * k), bd + 2 * k,
                                    idesc, ((c + h) | k) != 0 ? 1u : 0u);
                }
              }
              umma_commit_warp(&empty[ps]);
            }
            umma_commit_warp(&tfull[acc]);
          }
        }
        __syncwarp();
      } else {
        // ---------------- epilogue (8 warps: 2 per TMEM lane quarter) ----------------
        const int lg = warp & 3;               // TMEM lane quarter of this warp
        const int half = (warp - LM_EPI0) >> 2;  // column half: blocks 16*half, +32, ...
        const int row = lg * 32 + lane;
        uint32_t tc = tile_ctr;
        for (uint32_t t = 0; t < ntiles; ++t, ++tc) {
          const int acc = tc & 1;
          const uint32_t item = t * LM_IT + row;
          const bool ivalid = item < Nl;
          int myref = -1;
          if (ivalid && item >= own) {
            myref = lm_ref_of(refoff, nref, item);
          }
          uint64_t ok = (nq_tile >= 64) ? ~0ull : ((1ull << nq_tile) - 1ull);
          if (myref >= 0) ok &= ~((uint64_t)skipT[myref * 2] | ((uint64_t)skipT[myref * 2 + 1] << 32));
          if (!ivalid) ok = 0;
          // every (row item < Nl8, tile query) cell is written: the score, or the
          // sentinel (all ones) for a skipped reference (R9) / row padding, so the
          // selection can stream whole rows with 16-B loads
          const bool inrow = item < Nl8;
          mbar_wait(&tfull[acc], (tc >> 1) & 1u);
          tc_fence_after();
          const uint64_t base = a.fused ? 0ull : a.sbase[l] + (uint64_t)q0 * Nl8 + item;
          for (int cb = 16 * half; cb < Npad; cb += 32) {
            uint32_t v[16];
            tmem_ld16(tmem + ((uint32_t)(lg * 32) << 16) + LM_ACC_COL + (uint32_t)(acc * LM_QT + cb), v);
            if (a.fused) {
              // threshold filter: 16 compares; the (rare) passing (item, query)
              // pairs are appended one atomic each
              const int jn = min(16, nq_tile - cb);
              uint32_t pm = 0;
#pragma unroll
              for (int j = 0; j < 16; ++j) pm |= (v[j] <= qtau[cb + j] ? 1u : 0u) << j;
              pm &= ((uint32_t)(ok >> cb) & 0xFFFFu) & ((1u << jn) - 1u);
              if (__any_sync(0xffffffffu, pm != 0)) {
                const uint64_t key_lo = ((uint64_t)l << 22) | (uint64_t)item;
                while (pm) {
                  const int j = __ffs(pm) - 1;
                  pm &= pm - 1;
                  uint32_t sv = v[0];
#pragma unroll
                  for (int jj = 1; jj < 16; ++jj) sv = (jj == j) ? v[jj] : sv;
                  const uint32_t qq = qid[cb + j];
                  const uint32_t pos = atomicAdd(&a.fcnt[qq], 1u);
                  if (pos < (uint32_t)a.fcap) a.fcand[(size_t)qq * a.fcap + pos] = ((uint64_t)sv << 39) | key_lo;
                }
              }
            } else if (inrow) {
              const int jn = min(16, nq_tile - cb);
              const uint32_t okb = (uint32_t)(ok >> cb) & 0xFFFFu;
              if (a.score_u32) {
                uint32_t* p = reinterpret_cast<uint32_t*>(a.S) + base + (uint64_t)cb * Nl8;
                if (jn == 16) {
#pragma unroll
                  for (int j = 0; j < 16; ++j) p[(size_t)j * Nl8] = ((okb >> j) & 1u) ? v[j] : 0xFFFFFFFFu;
                } else {
#pragma unroll
                  for (int j = 0; j < 16; ++j)
                    if (j < jn) p[(size_t)j * Nl8] = ((okb >> j) & 1u) ? v[j] : 0xFFFFFFFFu;
                }
              } else {
                uint16_t* p = reinterpret_cast<uint16_t*>(a.S) + base + (uint64_t)cb * Nl8;
                if (jn == 16) {
#pragma unroll
                  for (int j = 0; j < 16; ++j)
                    p[(size_t)j * Nl8] = ((okb >> j) & 1u) ? (uint16_t)v[j] : (uint16_t)0xFFFFu;
                } else {
#pragma unroll
                  for (int j = 0; j < 16; ++j)
                    if (j < jn) p[(size_t)j * Nl8] = ((okb >> j) & 1u) ? (uint16_t)v[j] : (uint16_t)0xFFFFu;
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g)  // tiles t = g mod G of this query tile
        gcnt[g] += ((ntiles + (uint32_t)(G - 1 - g)) / (uint32_t)G) * NCHUNK;
      tile_ctr += ntiles;
      ++qt_ctr;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == LM_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, LM_TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// Per query (one WARP per query): SEIL ranges over its score rows (R9 dedup),
// histogram-threshold top-bigK with warp-private state (no CTA barriers).
constexpr int SW_WARPS = 8;
constexpr int SW_NB = 512;
constexpr int SEL_P1 = 8;  // 16-B loads in flight per lane in pass 1
// pass 2: 2 loads in flight when the score rows are L2-resident (c2pl), 8 when
// they stream from DRAM (c5: 2 GB of rows; measured scan 11.2 -> 10.8 ms)
constexpr int SEL_P2_L2 = 2, SEL_P2_DRAM = 8;
constexpr size_t SEL_DRAM_BYTES = 256ull << 20;  // score buffers above this stream from DRAM

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
  const uint64_t* list_base;
  const uint32_t* list_ids;
  const uint64_t* sbase;
  const void* S;
  int score_u32;
  int shard_id, nshards;
  uint64_t* out_keys;
  int64_t* dco;
  int64_t q0;  // first query of this launch (queries [q0, nq))
  int sorted_out;  // 1: write each query's bigK keys in (s, id) order (debug outputs)
  unsigned long long* dco_total;  // += DCO of every query (rairs_get_stats) or NULL
  unsigned* qctr;                 // zeroed counter: warps claim queries q0 + atomicAdd (load balance)
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

// smallest bin b of a 256-bin histogram whose cumulative count reaches K
// (K >= 1 and the total >= K); *below = the count of the bins before b
__device__ __forceinline__ uint32_t warp_bsel256(const uint32_t* hist, uint32_t K, uint32_t* below) {
  const int lane = lane_id();
  uint32_t h[8], loc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { h[i] = hist[lane * 8 + i]; loc += h[i]; }
  uint32_t inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  const unsigned hit = __ballot_sync(0xffffffffu, inc >= K);
  const int hl = hit ? __ffs(hit) - 1 : 31;
  uint32_t b = 255, run = inc - loc, bl = 0;
  if (lane == hl) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (run + h[i] >= K) { b = lane * 8 + i; bl = run; break; }
      run += h[i];
    }
  }
  *below = __shfl_sync(0xffffffffu, bl, hl);
  return __shfl_sync(0xffffffffu, b, hl);
}

// Exact top-K of n > K resolved keys (s << 32 | id), written UNORDERED to out:
// a two-level radix select on s (s <= thr < 2^16): 256 bins of s >> sh, then
// the exact s* inside the chosen bin; every key with s < s* is kept, and the
// ties at s* by smallest id.  scratch: 512 u32 of shared memory.  Returns
// false (nothing written) when more than 256 keys tie at s* -- the caller then
// sorts everything.
__device__ bool warp_select_unordered(const uint64_t* cand, uint32_t n, uint32_t K, uint32_t thr,
                                      uint32_t* scratch, uint64_t* out) {
  const int lane = lane_id();
  const uint32_t sh = thr < 256u ? 0u : (uint32_t)(32 - __clz(thr)) - 8u;
  for (int i = lane; i < 512; i += 32) scratch[i] = 0u;
  __syncwarp();
  for (uint32_t i = lane; i < n; i += 32) atomicAdd(&scratch[(uint32_t)(cand[i] >> 32) >> sh], 1u);
  __syncwarp();
  uint32_t below1;
  const uint32_t b1 = warp_bsel256(scratch, K, &below1);
  const uint32_t lo = b1 << sh, hi = lo + (1u << sh);   // scores of bin b1: [lo, hi)
  for (uint32_t i = lane; i < n; i += 32) {
    const uint32_t sc = (uint32_t)(cand[i] >> 32);
    if (sc >= lo && sc < hi) atomicAdd(&scratch[256 + (sc - lo)], 1u);
  }
  __syncwarp();
  uint32_t below2;
  const uint32_t b2 = warp_bsel256(scratch + 256, K - below1, &below2);
  const uint32_t sstar = lo + b2;
  const uint32_t need = K - below1 - below2;       // ties at s* to keep (>= 1)
  const uint32_t ties = scratch[256 + b2];
  if (ties > 256u) return false;
  __syncwarp();
  // keys with s < s* (exactly K - need of them) + the ties, compacted
  uint64_t* tie = reinterpret_cast<uint64_t*>(scratch);  // reuses the histograms
  uint32_t nk = 0, nt = 0;
  for (uint32_t i0 = 0; i0 < n; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint64_t v = i < n ? cand[i] : kKeyInf;
    const uint32_t sc = (uint32_t)(v >> 32);
    const bool keep = i < n && sc < sstar, tq = i < n && sc == sstar;
    const unsigned bk = __ballot_sync(0xffffffffu, keep), bt = __ballot_sync(0xffffffffu, tq);
    const unsigned below_me = (1u << lane) - 1u;
    __syncwarp();
    if (keep) out[nk + __popc(bk & below_me)] = v;
    if (tq) tie[nt + __popc(bt & below_me)] = v;
    nk += __popc(bk);
    nt += __popc(bt);
  }
  __syncwarp();
  if (nt == need) {
    for (uint32_t j = lane; j < nt; j += 32) out[nk + j] = tie[j];
  } else if (nt <= 32) {                           // rank the ties by id
    const uint64_t v = (uint32_t)lane < nt ? tie[lane] : kKeyInf;
    uint32_t rank = 0;
    for (uint32_t j = 0; j < nt; ++j) rank += tie[j] < v ? 1u : 0u;
    if ((uint32_t)lane < nt && rank < need) out[nk + rank] = v;
  } else {
    uint32_t np = 32;
    while (np < nt) np <<= 1;
    for (uint32_t j = nt + lane; j < np; j += 32) tie[j] = kKeyInf;
    __syncwarp();
    warp_sort_keys(tie, (int)np);
    for (uint32_t j = lane; j < need; j += 32) out[nk + j] = tie[j];
  }
  __syncwarp();
  return true;
}

// One WARP per query: exact top-bigK of the keys (s << 32 | id) over U(q).
// The query's score rows (one per probed list, padded to 8 items; skipped
// references and padding hold the all-ones sentinel, R9) are streamed twice
// with 16-B loads:
//   pass 1  histogram of s >> hshift over the minimum of every 16-B vector
//           (8 or 4 items) -> the smallest bin b* whose cumulative count
//           reaches bigK: the bigK-th score of any subset of U(q) bounds that
//           of U(q), so every item of the top-bigK has bin <= b*; the vector
//           minima hold almost all top items, so few more than bigK pass;
//   pass 2  items with bin <= b* are appended as PRE-keys (s << 32 | p << 22 |
//           item) -- no id load on the streaming path;
//   finish  the ids of the (few) candidates are loaded in one batch, the keys
//           sorted, the first bigK written.
// If more than `cap` items share bins <= b* (massive score ties) the warp
// switches to exact mode: candidates are resolved to (s, id) keys, sorted and
// cut to bigK (tau = the bigK-th key), later items are compared against tau.
// DCO = owned + non-skipped referenced items (R17).
__device__ __forceinline__ uint32_t sel_pos(uint32_t p, uint32_t item) {
  return (p << 22) | item;
}

template <bool U32>
__device__ __forceinline__ void sel_resolve(const SelArgs& a, int64_t q, uint64_t* cand,
                                            uint32_t n) {
  const int lane = lane_id();
  for (uint32_t i = lane; i < n; i += 32) {  // independent loads, all in flight
    const uint64_t v = cand[i];
    const uint32_t pos = (uint32_t)v, p = pos >> 22, item = pos & ((1u << 22) - 1u);
    const uint32_t l = (uint32_t)a.probes[q * a.nprobe + p];
    const uint32_t id = __ldg(a.list_ids + a.list_base[l] + item);
    cand[i] = (v & 0xFFFFFFFF00000000ull) | id;
  }
  __syncwarp();
}

template <bool U32, int SEL_P2>
__global__ void __launch_bounds__(SW_WARPS * 32, 4) lm_select_kernel(SelArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = warp_id(), lane = lane_id();
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm) + warp * SW_NB;
  uint64_t* cand = reinterpret_cast<uint64_t*>(reinterpret_cast<uint32_t*>(sm) + SW_WARPS * SW_NB) +
                   (size_t)warp * a.cap;
  const uint32_t bigK = (uint32_t)a.bigK;
  constexpr uint32_t SENT = U32 ? 0xFFFFFFFFu : 0xFFFFu;
  constexpr int PER = U32 ? 4 : 8;  // scores per 16-B vector
  for (;;) {
    // dynamic scheduling: a warp claims its next query when it is free, so the
    // queries with the longest score rows do not pile up on a few warps
    uint32_t claim = 0;
    if (lane == 0) claim = atomicAdd(a.qctr, 1u);
    const int64_t q = a.q0 + (int64_t)__shfl_sync(0xffffffffu, claim, 0);
    if (q >= a.nq) break;
    (void)warp;
    for (int i = lane; i < SW_NB; i += 32) hist[i] = 0u;
    __syncwarp();
    const uint32_t* qb = a.qbits + (size_t)q * a.qwords;
    // per-probe metadata: for nprobe <= 32 lane p resolves probe p once, all
    // probes' dependent loads in flight together (the loops below shuffle it)
    struct PMeta { uint32_t l, Nl8, r0, nref, own; uint64_t row; };
    auto load_meta = [&](int p) {
      PMeta m;
      m.l = (uint32_t)a.probes[q * a.nprobe + p];
      m.Nl8 = (a.list_items[m.l] + 7u) & ~7u;
      m.r0 = a.ref_ptr[m.l];
      m.nref = a.ref_ptr[m.l + 1] - m.r0;
      m.own = a.own_cnt[m.l];
      m.row = a.sbase[m.l] + (uint64_t)a.qslot[q * a.nprobe + p] * m.Nl8;
      return m;
    };
    const bool lane_meta = a.nprobe <= 32;
    PMeta mine{0, 0, 0, 0, 0, 0};
    if (lane_meta && lane < a.nprobe) mine = load_meta(lane);
    auto meta = [&](int p) {
      if (!lane_meta) return load_meta(p);
      PMeta m;
      m.l = __shfl_sync(0xffffffffu, mine.l, p);
      m.Nl8 = __shfl_sync(0xffffffffu, mine.Nl8, p);
      m.r0 = __shfl_sync(0xffffffffu, mine.r0, p);
      m.nref = __shfl_sync(0xffffffffu, mine.nref, p);
      m.own = __shfl_sync(0xffffffffu, mine.own, p);
      m.row = __shfl_sync(0xffffffffu, mine.row, p);
      return m;
    };
    // ---- pass 1: DCO and the score histogram
    uint32_t dco = 0;
    for (int p = 0; p < a.nprobe; ++p) {
      const PMeta pm_ = meta(p);
      const uint32_t l = pm_.l, Nl8 = pm_.Nl8, r0 = pm_.r0, nref = pm_.nref;
      uint32_t c = 0;
      for (uint32_t j = lane; j < nref; j += 32) {
        const int o = a.ref_owner[r0 + j];
        if (!((qb[o >> 5] >> (o & 31)) & 1u)) c += a.ref_cnt[r0 + j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      dco += pm_.own + c;
      const uint64_t row = pm_.row;
      (void)l;
      const uint4* rv = reinterpret_cast<const uint4*>(
          reinterpret_cast<const unsigned char*>(a.S) + row * (U32 ? 4 : 2));
      const uint32_t nv = Nl8 / PER;
      for (uint32_t v0 = 0; v0 < nv; v0 += 32 * SEL_P1) {
        uint4 x[SEL_P1];
#pragma unroll
        for (int u = 0; u < SEL_P1; ++u) {
          const uint32_t vi = v0 + 32 * u + lane;
          x[u] = (vi < nv) ? __ldg(rv + vi) : make_uint4(~0u, ~0u, ~0u, ~0u);
        }
#pragma unroll
        for (int u = 0; u < SEL_P1; ++u) {
          // histogram of the per-vector minima: a subset of U(q) (so the cut
          // stays valid) that holds almost every top item -- the bigK best
          // items rarely share a vector -- at one atomic per 8 (4) items
          uint32_t mn;
          if (U32) {
            mn = min(min(x[u].x, x[u].y), min(x[u].z, x[u].w));
          } else {
            const uint32_t m2 = __vminu2(__vminu2(x[u].x, x[u].y), __vminu2(x[u].z, x[u].w));
            mn = min(m2 & 0xFFFFu, m2 >> 16);
          }
          if (mn != SENT) atomicAdd(&hist[mn >> a.hshift], 1u);
        }
      }
    }
    __syncwarp();
    const uint32_t bstar = warp_bthr(hist, bigK);
    uint32_t thr = min(SENT - 1u, (uint32_t)(((uint64_t)(bstar + 1) << a.hshift) - 1u));
    // ---- pass 2: collect the items with bin <= b*
    uint32_t cnt = 0;
    bool exact = false;
    uint64_t tau = kKeyInf;
    for (int p = 0; p < a.nprobe; ++p) {
      const PMeta pm_ = meta(p);
      const uint32_t l = pm_.l, Nl8 = pm_.Nl8;
      const uint64_t row = pm_.row;
      const uint32_t* lids = a.list_ids + a.list_base[l];
      const uint4* rv = reinterpret_cast<const uint4*>(
          reinterpret_cast<const unsigned char*>(a.S) + row * (U32 ? 4 : 2));
      const uint32_t nv = Nl8 / PER;
      for (uint32_t v0 = 0; v0 < nv; v0 += 32 * SEL_P2) {
        uint4 x[SEL_P2];
#pragma unroll
        for (int u = 0; u < SEL_P2; ++u) {
          const uint32_t vi = v0 + 32 * u + lane;
          x[u] = (vi < nv) ? __ldcs(rv + vi) : make_uint4(~0u, ~0u, ~0u, ~0u);
        }
#pragma unroll
        for (int u = 0; u < SEL_P2; ++u) {
          const uint32_t w4[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
          uint32_t pm = 0;  // this lane's items with score <= thr (the sentinel never passes)
          if (U32) {
#pragma unroll
            for (int e = 0; e < 4; ++e) pm |= (w4[e] <= thr ? 1u : 0u) << e;
          } else {
            const uint32_t t2 = thr | (thr << 16);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t cm = __vcmpleu2(w4[e], t2);  // 0xFFFF per passing half
              pm |= ((cm & 1u) | ((cm >> 15) & 2u)) << (2 * e);
            }
          }
          const uint32_t item0 = (v0 + 32 * u + lane) * PER;
          // fast append: a warp-wide exclusive scan of the per-lane pass counts
          const uint32_t mine = __popc(pm);
          uint32_t incl = mine;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
          }
          const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
          if (total == 0) continue;
          if (!exact && cnt + total + 32 <= (uint32_t)a.cap) {
            uint32_t pos = cnt + incl - mine;
            while (pm) {
              const int e = __ffs(pm) - 1;
              pm &= pm - 1u;
              uint32_t sc;
              if (U32) {
                sc = e == 0 ? w4[0] : e == 1 ? w4[1] : e == 2 ? w4[2] : w4[3];
              } else {
                const uint32_t ww = (e >> 1) == 0 ? w4[0] : (e >> 1) == 1 ? w4[1]
                                  : (e >> 1) == 2 ? w4[2] : w4[3];
                sc = (ww >> (16 * (e & 1))) & 0xFFFFu;
              }
              cand[pos++] = ((uint64_t)sc << 32) | sel_pos((uint32_t)p, item0 + e);
            }
            cnt += total;
            __syncwarp();
            continue;
          }
          // near the capacity, or in exact mode: item by item
          while (__any_sync(0xffffffffu, pm != 0)) {
            bool pass = pm != 0;
            uint64_t key = kKeyInf;
            if (pass) {
              const int e = __ffs(pm) - 1;
              pm &= pm - 1u;
              uint32_t sc;
              if (U32) {
                sc = e == 0 ? w4[0] : e == 1 ? w4[1] : e == 2 ? w4[2] : w4[3];
              } else {
                const uint32_t ww = (e >> 1) == 0 ? w4[0] : (e >> 1) == 1 ? w4[1]
                                  : (e >> 1) == 2 ? w4[2] : w4[3];
                sc = (ww >> (16 * (e & 1))) & 0xFFFFu;
              }
              if (sc > thr) {
                pass = false;  // thr tightened (exact mode) since pm was formed
              } else if (!exact) {
                key = ((uint64_t)sc << 32) | sel_pos((uint32_t)p, item0 + e);
              } else {
                key = ((uint64_t)sc << 32) | __ldg(lids + item0 + e);
                pass = key < tau;
              }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, pass);
            if (pass) cand[cnt + __popc(bal & ((1u << lane) - 1u))] = key;
            cnt += __popc(bal);
            __syncwarp();
            if (cnt + 32 > (uint32_t)a.cap) {  // massive ties: exact (s, id) keys, keep bigK
              if (!exact) {
                sel_resolve<U32>(a, q, cand, cnt);
                exact = true;
              }
              int np = 2;
              while (np < (int)cnt) np <<= 1;
              for (int f = cnt + lane; f < np; f += 32) cand[f] = kKeyInf;
              __syncwarp();
              warp_sort_keys(cand, np);
              cnt = bigK;
              tau = cand[bigK - 1];
              thr = min(thr, (uint32_t)(tau >> 32));
            }
          }
        }
      }
    }
    if (!exact) {
      sel_resolve<U32>(a, q, cand, cnt);
      if (!a.sorted_out && cnt > bigK && thr < 65536u) {
        // production: the refine needs the top-bigK SET only -- select it
        // exactly without sorting every candidate
        if (warp_select_unordered(cand, cnt, bigK, thr, hist, a.out_keys + q * a.bigK)) {
          if (lane == 0 && a.dco) a.dco[q] = (int64_t)dco;
          if (lane == 0 && a.dco_total) atomicAdd(a.dco_total, (unsigned long long)dco);
          __syncwarp();
          continue;
        }
      }
    }
    cnt = warp_filter(cand, cnt, bstar, tau, a.hshift);
    int np = 2;
    while (np < (int)cnt) np <<= 1;
    for (int e = cnt + lane; e < np; e += 32) cand[e] = kKeyInf;
    __syncwarp();
    warp_sort_keys(cand, np);
    const uint32_t keep = min(cnt, bigK);
    for (int e = lane; e < a.bigK; e += 32) a.out_keys[q * a.bigK + e] = ((uint32_t)e < keep) ? cand[e] : kKeyInf;
    if (lane == 0 && a.dco) a.dco[q] = (int64_t)dco;
    if (lane == 0 && a.dco_total) atomicAdd(a.dco_total, (unsigned long long)dco);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Fused mode, per query (one WARP per query): the candidates the tensor
// epilogue appended (every item of U(q) with s <= tau[q], a superset of the
// top-bigK), their ids resolved and sorted by the unique key (s << 32 | id);
// the first bigK are the query's candidates (O9).  DCO from the layout tables
// and the probe bitmap (R9, R17).  Queries whose buffer overflowed are listed
// for the query-major kernel.
constexpr int FIN_WARPS = 4;
struct FinArgs {
  const int32_t* probes;
  int nprobe;
  const uint32_t* qbits;
  int qwords;
  const uint32_t* own_cnt;
  const uint32_t* ref_ptr;
  const int32_t* ref_owner;
  const uint32_t* ref_cnt;
  const uint64_t* list_base;
  const uint32_t* list_ids;
  const uint64_t* fcand;
  const uint32_t* fcnt;
  int fcap;
  int64_t nq;
  int bigK;
  uint64_t* out_keys;
  int64_t* dco;
  unsigned long long* dco_total;
  uint32_t* ovf;
  uint32_t* novf;
  unsigned* qctr;
};

__global__ void __launch_bounds__(FIN_WARPS * 32) lm_final_kernel(FinArgs a) {
  extern __shared__ __align__(16) uint64_t fin_sm[];
  const int lane = lane_id(), warp = warp_id();
  uint64_t* buf = fin_sm + (size_t)warp * a.fcap;
  pdl_wait();  // the tensor kernel's candidates
  for (;;) {
    uint32_t qi = 0;
    if (lane == 0) qi = atomicAdd(a.qctr, 1u);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi >= (uint64_t)a.nq) break;
    const int64_t q = qi;
    const uint32_t n = a.fcnt[q];
    if (n > (uint32_t)a.fcap) {  // overflow: the query-major kernel redoes this query
      if (lane == 0) a.ovf[atomicAdd(a.novf, 1u)] = (uint32_t)q;
      continue;
    }
    // DCO = owned + non-skipped referenced items (R9: owner probed -> skipped)
    const uint32_t* qb = a.qbits + (size_t)q * a.qwords;
    uint32_t dco = 0;
    for (int p = 0; p < a.nprobe; ++p) {
      const int l = a.probes[q * a.nprobe + p];
      const uint32_t r0 = a.ref_ptr[l], r1 = a.ref_ptr[l + 1];
      uint32_t c = 0;
      for (uint32_t j = r0 + lane; j < r1; j += 32) {
        const int o = a.ref_owner[j];
        if (!((qb[o >> 5] >> (o & 31)) & 1u)) c += a.ref_cnt[j];
      }
      dco += c + (lane == 0 ? a.own_cnt[l] : 0u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dco += __shfl_xor_sync(0xffffffffu, dco, o);
    // resolve (s, list, item) -> (s << 32 | global id)
    const uint64_t* src = a.fcand + (size_t)q * a.fcap;
    for (uint32_t i = lane; i < n; i += 32) {
      const uint64_t v = src[i];
      const uint32_t s = (uint32_t)(v >> 39), l = (uint32_t)(v >> 22) & 0x1FFFFu;
      const uint32_t item = (uint32_t)v & 0x3FFFFFu;
      buf[i] = ((uint64_t)s << 32) | a.list_ids[a.list_base[l] + item];
    }
    int p2 = 2;
    while (p2 < (int)n) p2 <<= 1;
    for (int i = (int)n + lane; i < p2; i += 32) buf[i] = kKeyInf;
    __syncwarp();
    warp_sort_keys(buf, p2);
    const uint32_t keep = min(n, (uint32_t)a.bigK);
    for (int i = lane; i < a.bigK; i += 32) a.out_keys[q * a.bigK + i] = ((uint32_t)i < keep) ? buf[i] : kKeyInf;
    if (lane == 0) {
      if (a.dco) a.dco[q] = (int64_t)dco;
      if (a.dco_total) atomicAdd(a.dco_total, (unsigned long long)dco);
    }
    __syncwarp();
  }
  pdl_trigger();
}

static int sel_cap(int bigK) { return next_pow2(2 * bigK + 64); }

static int lm_qt(int K) {  // queries per LUT tile: QT x K <= LM_B_MAX, multiple of 16, <= 64
  int qt = (int)(LM_B_MAX / (uint32_t)K);
  qt = std::min(qt, LM_QT);
  return qt - (qt % 16);
}

constexpr double LM_MIN_QUERIES_PER_LIST = 3.0;

static bool lm_nu_ok(int NU) { return NU == 1 || NU == 2 || NU == 3 || NU == 4 || NU == 6 || NU == 8; }

bool listmajor_ok(const rairs_index_s* idx, int64_t nq, int nprobe, int bigK) {
  if (idx->scan_mode == 1) return false;            // forced SIMT query-major scan
  if (idx->seil_layout == 1) return false;          // paper-literal SEIL: query-major only
  // auto: the list-major contraction pays once a probed list is shared by
  // several queries of the batch (each list-task expands its codes once)
  if (idx->scan_mode == 0 && (double)nq * nprobe < LM_MIN_QUERIES_PER_LIST * idx->nlist)
    return false;
  if (!idx->list_items || !idx->ref_item_off || !idx->list_ids) return false;
  if (idx->max_refs > LM_MAXREF) return false;
  if (!lm_nu_ok(idx->M_pad / 16) || lm_qt(idx->M_pad * 16) < 16) return false;
  if ((size_t)SW_WARPS * (SW_NB * 4 + (size_t)sel_cap(bigK) * 8) > 200 * 1024) return false;
  if (nprobe > 1024 || idx->max_list_items >= (1 << 22)) return false;  // pre-key packing
  if (!(idx->dsub == 1 || idx->dsub == 2 || idx->dsub == 3 || idx->dsub == 4 || idx->dsub == 8))
    return false;
  return true;
}

template <int NU, int G, int GS>
static cudaError_t launch_lm_tensor(const LMArgs& la, size_t tsm, cudaStream_t s) {
  using SH = LMShape<G, GS>;
  cudaError_t e = cudaFuncSetAttribute(lm_tensor_kernel<NU, G, GS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
  if (e != cudaSuccess) return e;
  e = launch_pdl(lm_tensor_kernel<NU, G, GS>, dim3(148 * SH::CTAS_PER_SM), dim3(SH::THREADS), tsm, s, la);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// pipeline shape: one generator group, 4 A stages (2 pair-stages), 2 CTAs/SM
// (measured best of 1x4, 2x4, 4x2, 2x2 -- profiles/r01/SUMMARY.md)
template <int NU>
static cudaError_t launch_lm_tensor_shape(const LMArgs& la, size_t tsm, cudaStream_t s) {
  // RAIRS_LM_SHAPE=22: two generator groups of 2 stages (16 generator warps per
  // SM) -- an experiment for generator-bound batches (few queries per list)
  static const int shape = [] {
    const char* e = std::getenv("RAIRS_LM_SHAPE");
    return e ? std::atoi(e) : 14;
  }();
  if (shape == 22) return launch_lm_tensor<NU, 2, 2>(la, tsm, s);
  return launch_lm_tensor<NU, 1, 4>(la, tsm, s);
}

rairs_status launch_listmajor(const rairs_index_s* idx, const SearchArgs& sa, cudaStream_t s) {
  const int64_t nq = sa.nq;
  if (nq <= 0) return RAIRS_OK;
  const int nprobe = sa.nprobe, nlist = idx->nlist;
  const int bigK = sa.k * sa.refine_factor;
  const int K = idx->M_pad * 16;
  const int QT = lm_qt(K);
  const int qwords = (nlist + 31) / 32;
  const int64_t npairs = nq * nprobe;
  const int score_u32 = ((int64_t)idx->M * 255 > 65535) ? 1 : 0;
  uint8_t* tiles = nullptr;
  uint32_t *cnt = nullptr, *qslot = nullptr, *qptr = nullptr, *lrow = nullptr, *list_q = nullptr,
           *qbits = nullptr, *totals = nullptr;
  uint64_t* sbase = nullptr;
  void* S = nullptr;
  // bound on the score buffer: every (query, probe) pair times the largest list-task
  const size_t s_elems = (size_t)npairs * (size_t)round_up(std::max<int64_t>(idx->max_list_items, 1), 8);
  const size_t s_bytes = s_elems * (score_u32 ? 4 : 2);
  // LUT tiles: every (query, probe) row, plus <= 15 padding rows per list
  const size_t tile_bytes = ((size_t)npairs + 15 * (size_t)nlist) * K;
  // fused mode (no score rows): large batches whose rows would stream from DRAM
  // (RAIRS_LM_FUSED=0/1 overrides)
  const double exp_rows = (double)npairs * ((double)idx->sum_list_items / nlist) * (score_u32 ? 4 : 2);
  bool fused = exp_rows > (double)SEL_DRAM_BYTES;
  if (const char* e = std::getenv("RAIRS_LM_FUSED")) fused = std::atoi(e) != 0;
  const int fcap = std::max(2048, next_pow2(8 * bigK));
  uint4* luts = nullptr;
  uint32_t *tau = nullptr, *fcnt = nullptr, *ovf = nullptr;
  uint64_t* fcand = nullptr;
  auto cleanup = [&]() {
    cudaFreeAsync(tiles, s); cudaFreeAsync(cnt, s); cudaFreeAsync(qslot, s); cudaFreeAsync(qptr, s);
    cudaFreeAsync(lrow, s); cudaFreeAsync(list_q, s); cudaFreeAsync(qbits, s);
    cudaFreeAsync(totals, s); cudaFreeAsync(sbase, s); cudaFreeAsync(S, s);
    cudaFreeAsync(luts, s); cudaFreeAsync(tau, s); cudaFreeAsync(fcnt, s); cudaFreeAsync(ovf, s);
    cudaFreeAsync(fcand, s);
  };
#define LM_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { set_error(std::string(#x) + ": " + cudaGetErrorString(_e)); cleanup(); return _e == cudaErrorMemoryAllocation ? RAIRS_E_OOM : RAIRS_E_CUDA; } } while (0)
  LM_TRY(ws_malloc(&tiles, tile_bytes, s));
  LM_TRY(ws_malloc(&cnt, (size_t)(nlist + 2 + LM_NCH) * 4, s));
  LM_TRY(ws_malloc(&qslot, (size_t)npairs * 4, s));
  LM_TRY(ws_malloc(&qptr, (size_t)(nlist + 1) * 4, s));
  LM_TRY(ws_malloc(&lrow, (size_t)(nlist + 1) * 4, s));
  LM_TRY(ws_malloc(&list_q, (size_t)npairs * 4, s));
  LM_TRY(ws_malloc(&qbits, (size_t)nq * qwords * 4, s));
  LM_TRY(ws_malloc(&totals, 16, s));
  LM_TRY(ws_malloc(&sbase, (size_t)(nlist + 1) * 8, s));

  LM_TRY(launch_pdl(lm_zero_kernel, dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nlist + 2 + LM_NCH, 256), 148))),
                    dim3(256), 0, s, cnt, (int64_t)(nlist + 2 + LM_NCH)));
  unsigned* list_counter = cnt + nlist + 1;  // zeroed tail of cnt
  // 1. group (query, probe) pairs by list
  const unsigned g1 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(npairs, 256), 148 * 8));
  LM_TRY(launch_pdl(lm_count_kernel, dim3(g1), dim3(256), 0, s, (const int32_t*)sa.probes, npairs,
                    cnt, qslot, qbits, (int64_t)(nq * qwords)));
  LM_TRY(launch_pdl(lm_scan_kernel, dim3(1), dim3(SCN), 0, s, (const uint32_t*)cnt,
                    (const uint32_t*)idx->list_items, nlist, qptr, sbase, lrow, totals, QT, LM_IT));
  LM_TRY(launch_pdl(lm_scatter_kernel, dim3(g1), dim3(256), 0, s, (const int32_t*)sa.probes, npairs,
                    nprobe, (const uint32_t*)qptr, (const uint32_t*)qslot, list_q, qbits, qwords));
  LM_TRY(cudaGetLastError());
  // the score rows: the worst-case bound (every pair x the largest list-task)
  // when it is small, else the exact total sum_l |Q_l| * round8(N_l) read back
  // from the scan (one host synchronisation; multi-GB batches only)
  if (!fused) {
    size_t bytes = s_bytes;
    if (s_bytes > (512ull << 20)) {
      uint64_t tot = 0;
      LM_TRY(cudaMemcpyAsync(&tot, sbase + nlist, 8, cudaMemcpyDeviceToHost, s));
      LM_TRY(cudaStreamSynchronize(s));
      bytes = (size_t)tot * (score_u32 ? 4 : 2);
    }
    LM_TRY(ws_malloc(&S, std::max<size_t>(bytes, 16), s));
  }
  // 2. quantised LUTs (O2), one warp per query, written into the list-task tiles
  {
    const size_t lsm = ((size_t)16 * idx->dsub * idx->M + (size_t)LW * idx->M) * 4;
    const unsigned lgrid = (unsigned)std::min<int64_t>(ceil_div(nq, LW), 148 * 3);  // persistent
#define LUT_LAUNCH(DS, MP)                                                                   \
  LM_TRY(cudaFuncSetAttribute(lut_tiles_kernel<DS, MP>,                                      \
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));       \
  LM_TRY(launch_pdl(lut_tiles_kernel<DS, MP>, dim3(lgrid), dim3(LW * 32), lsm, s, sa.queries,  \
                    nq, idx->d, (const float*)idx->codebook, idx->M, idx->M_pad, sa.probes,     \
                    nprobe, (const uint32_t*)qslot, (const uint32_t*)cnt, (const uint32_t*)lrow, \
                    QT, tiles, sa.lut_a, sa.lut_b, sa.lut_q))
#define LUT_LAUNCH_D(DS)                                  \
  switch ((idx->M_pad + 31) / 32) {                        \
    case 1: LUT_LAUNCH(DS, 1); break;                      \
    case 2: LUT_LAUNCH(DS, 2); break;                      \
    case 3: LUT_LAUNCH(DS, 3); break;                      \
    default: LUT_LAUNCH(DS, 4); break;                     \
  }
    switch (idx->dsub) {
      case 1: LUT_LAUNCH_D(1); break;
      case 2: LUT_LAUNCH_D(2); break;
      case 3: LUT_LAUNCH_D(3); break;
      case 4: LUT_LAUNCH_D(4); break;
      case 8: LUT_LAUNCH_D(8); break;
      default: cleanup(); set_error("list-major: unsupported d/M"); return RAIRS_E_UNSUPPORTED;
    }
#undef LUT_LAUNCH_D
#undef LUT_LAUNCH
    LM_TRY(cudaGetLastError());
  }
  if (fused) {
    // 3f. per-query bound tau[q]: the bigK-th smallest score over the members
    // of q's nearest list (query-major kernel, first probe only) -- a subset of
    // U(q), so no item of the top-bigK scores above it
    LM_TRY(ws_malloc(&luts, (size_t)nq * idx->M_pad * 16, s));
    LM_TRY(ws_malloc(&tau, (size_t)nq * 4, s));
    LM_TRY(ws_malloc(&fcnt, (size_t)(nq + 1) * 4, s));
    LM_TRY(ws_malloc(&ovf, (size_t)nq * 4, s));
    LM_TRY(ws_malloc(&fcand, (size_t)nq * fcap * 8, s));
    SearchArgs ta = sa;
    ta.luts = luts;
    FsExtra ex;
    ex.nprobe_eff = 1;
    ex.tau_out = tau;
    {
      const rairs_status rs = launch_fastscan(const_cast<rairs_index_s*>(idx), ta, s, ex);
      if (rs != RAIRS_OK) { cleanup(); return rs; }
    }
    LM_TRY(launch_pdl(lm_zero_kernel, dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nq + 1, 256), 148))),
                      dim3(256), 0, s, fcnt, (int64_t)(nq + 1)));
  }
  // 3. tensor-core scores, one list at a time
  LMArgs la{};
  la.fused = fused ? 1 : 0;
  la.tau = tau;
  la.fcand = fcand;
  la.fcnt = fcnt;
  la.fcap = fcap;
  la.codes64 = reinterpret_cast<const uint64_t*>(idx->codes);
  la.own_off = idx->own_off;
  la.own_cnt = idx->own_cnt;
  la.ref_ptr = idx->ref_ptr;
  la.ref_owner = idx->ref_owner;
  la.ref_start = idx->ref_start;
  la.ref_item_off = idx->ref_item_off;
  la.list_items = idx->list_items;
  la.K = K;
  la.QT = QT;
  la.tiles = tiles;
  la.lrow = lrow;
  la.probes = sa.probes;
  la.nprobe = nprobe;
  la.qptr = qptr;
  la.list_q = list_q;
  la.list_counter = list_counter;
  la.sbase = sbase;
  la.S = S;
  la.score_u32 = score_u32;
  la.nlist = nlist;
  la.order = idx->lm_order;
  const size_t tsm = 1024 + LM_B_MAX + LM_MAXREF * 4 * 4 + 8 + LM_QT * 8 + (2 * 8 + 5) * 8 + 64;
  const bool kev = sa.kev[0] && sa.kev_used;
  if (kev) LM_TRY(cudaEventRecord(sa.kev[0], s));
  switch (idx->M_pad / 16) {
    case 1: LM_TRY(launch_lm_tensor_shape<1>(la, tsm, s)); break;
    case 2: LM_TRY(launch_lm_tensor_shape<2>(la, tsm, s)); break;
    case 3: LM_TRY(launch_lm_tensor_shape<3>(la, tsm, s)); break;
    case 4: LM_TRY(launch_lm_tensor_shape<4>(la, tsm, s)); break;
    case 6: LM_TRY(launch_lm_tensor_shape<6>(la, tsm, s)); break;
    case 8: LM_TRY(launch_lm_tensor_shape<8>(la, tsm, s)); break;
    default: cleanup(); set_error("list-major: unsupported M"); return RAIRS_E_INTERNAL;
  }
  if (kev) {
    LM_TRY(cudaEventRecord(sa.kev[1], s));
    *sa.kev_used = true;
  }
  if (fused) {
    // 4f. candidates -> exact top-bigK per query; overflowed queries (more than
    // fcap items at or below their bound) are redone by the query-major kernel
    FinArgs fa{};
    fa.probes = sa.probes;
    fa.nprobe = nprobe;
    fa.qbits = qbits;
    fa.qwords = qwords;
    fa.own_cnt = idx->own_cnt;
    fa.ref_ptr = idx->ref_ptr;
    fa.ref_owner = idx->ref_owner;
    fa.ref_cnt = idx->ref_cnt;
    fa.list_base = idx->list_base;
    fa.list_ids = idx->list_ids;
    fa.fcand = fcand;
    fa.fcnt = fcnt;
    fa.fcap = fcap;
    fa.nq = nq;
    fa.bigK = bigK;
    fa.out_keys = sa.cand_keys;
    fa.dco = sa.dco;
    fa.dco_total = sa.counters;
    fa.ovf = ovf;
    fa.novf = fcnt + nq;
    fa.qctr = cnt + nlist + 2;
    const size_t fsm = (size_t)FIN_WARPS * fcap * 8;
    LM_TRY(cudaFuncSetAttribute(lm_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
    const unsigned fg = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nq, FIN_WARPS), 148 * 8));
    LM_TRY(launch_pdl(lm_final_kernel, dim3(fg), dim3(FIN_WARPS * 32), fsm, s, fa));
    SearchArgs fb = sa;
    fb.luts = luts;
    FsExtra ex;
    ex.qlist = ovf;
    ex.qcount = fcnt + nq;
    ex.luts_ready = true;
    {
      const rairs_status rs = launch_fastscan(const_cast<rairs_index_s*>(idx), fb, s, ex);
      if (rs != RAIRS_OK) { cleanup(); return rs; }
    }
    if (sa.ev_selected) LM_TRY(cudaEventRecord(sa.ev_selected, s));
    if (sa.fused_refine) {
      SearchArgs ra = sa;
      const rairs_status rs = launch_refine(idx, ra, s);
      if (rs != RAIRS_OK) { cleanup(); return rs; }
    }
    cleanup();
    return RAIRS_OK;
  }
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
  sl.list_base = idx->list_base;
  sl.list_ids = idx->list_ids;
  sl.sbase = sbase;
  sl.S = S;
  sl.score_u32 = score_u32;
  sl.shard_id = idx->shard_id;
  sl.nshards = idx->nshards;
  sl.out_keys = sa.cand_keys;
  sl.dco = sa.dco;
  sl.sorted_out = sa.sorted_keys ? 1 : 0;
  sl.dco_total = sa.counters;
  const size_t ssm = (size_t)SW_WARPS * (SW_NB * 4 + (size_t)sl.cap * 8);
  LM_TRY(cudaFuncSetAttribute(lm_select_kernel<true, SEL_P2_L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
  LM_TRY(cudaFuncSetAttribute(lm_select_kernel<false, SEL_P2_L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
  LM_TRY(cudaFuncSetAttribute(lm_select_kernel<true, SEL_P2_DRAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
  LM_TRY(cudaFuncSetAttribute(lm_select_kernel<false, SEL_P2_DRAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
  // expected score bytes of this batch: pairs x mean list-task length
  const bool dram_rows = (double)npairs * ((double)idx->sum_list_items / nlist) * (score_u32 ? 4 : 2) >
                         (double)SEL_DRAM_BYTES;
  int n_sel = 0;  // select launches so far: each gets its own zeroed counter in cnt's tail
  auto select_range = [&](int64_t q0, int64_t q1, cudaStream_t st) -> cudaError_t {
    SelArgs sr = sl;
    sr.q0 = q0;
    sr.nq = q1;
    sr.qctr = cnt + nlist + 2 + (n_sel++);
    // persistent: 4 CTAs per SM, warps loop over queries (no partial last wave)
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(q1 - q0, SW_WARPS), 148 * 4));
    if (score_u32 && dram_rows) lm_select_kernel<true, SEL_P2_DRAM><<<g, SW_WARPS * 32, ssm, st>>>(sr);
    else if (score_u32) lm_select_kernel<true, SEL_P2_L2><<<g, SW_WARPS * 32, ssm, st>>>(sr);
    else if (dram_rows) lm_select_kernel<false, SEL_P2_DRAM><<<g, SW_WARPS * 32, ssm, st>>>(sr);
    else lm_select_kernel<false, SEL_P2_L2><<<g, SW_WARPS * 32, ssm, st>>>(sr);
    return cudaGetLastError();
  };
  auto refine_range = [&](int64_t q0, int64_t q1, cudaStream_t st) -> rairs_status {
    SearchArgs ra = sa;
    ra.queries = sa.queries + q0 * idx->d;
    ra.nq = q1 - q0;
    ra.cand_keys = sa.cand_keys + q0 * bigK;
    ra.out_ids = sa.out_ids + q0 * sa.k;
    ra.out_dists = sa.out_dists + q0 * sa.k;
    return launch_refine(idx, ra, st);
  };
  const bool overlap = sa.fused_refine && nq >= LM_NCH * LM_OVERLAP_MIN_Q && idx->aux[0];
  if (!overlap) {
    LM_TRY(select_range(0, nq, s));
    if (sa.ev_selected) LM_TRY(cudaEventRecord(sa.ev_selected, s));
    if (sa.fused_refine) {
      const rairs_status rs = refine_range(0, nq, s);
      if (rs != RAIRS_OK) { cleanup(); return rs; }
    }
  } else {
    // 4. + refine: LM_NCH query chunks, each selected then refined on its own
    // auxiliary stream, so one chunk's selection overlaps another's refine
    // gather (both latency-bound)
    std::lock_guard<std::mutex> lock(*idx->aux_mu);
    cudaEvent_t* ev = const_cast<cudaEvent_t*>(idx->aux_ev);
    int64_t qb[LM_NCH + 1];
    for (int h = 0; h <= LM_NCH; ++h) qb[h] = nq * h / LM_NCH;
    LM_TRY(cudaEventRecord(ev[0], s));  // scores ready
    for (int h = 0; h < LM_NCH; ++h) {
      LM_TRY(cudaStreamWaitEvent(idx->aux[h], ev[0], 0));
      LM_TRY(select_range(qb[h], qb[h + 1], idx->aux[h]));
      LM_TRY(cudaEventRecord(ev[1 + h], idx->aux[h]));  // chunk h selected
    }
    for (int h = 0; h < LM_NCH; ++h) {
      const rairs_status rs = refine_range(qb[h], qb[h + 1], idx->aux[h]);
      if (rs != RAIRS_OK) { cleanup(); return rs; }
      LM_TRY(cudaEventRecord(ev[1 + LM_NCH + h], idx->aux[h]));  // chunk h refined
    }
    for (int h = 0; h < LM_NCH; ++h) LM_TRY(cudaStreamWaitEvent(s, ev[1 + h], 0));
    if (sa.ev_selected) LM_TRY(cudaEventRecord(sa.ev_selected, s));
    for (int h = 0; h < LM_NCH; ++h) LM_TRY(cudaStreamWaitEvent(s, ev[1 + LM_NCH + h], 0));
  }
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

// item -> global id of every list-task (owned region, then references in
// ascending owner order): the selection's slow path needs one load per item
__global__ void lm_ids_kernel(const uint32_t* __restrict__ own_off,
                              const uint32_t* __restrict__ own_cnt,
                              const uint32_t* __restrict__ ref_ptr,
                              const uint32_t* __restrict__ ref_start,
                              const uint32_t* __restrict__ ref_cnt,
                              const uint32_t* __restrict__ slot_rows,
                              const uint64_t* __restrict__ list_base, int nlist, int shard_id,
                              int nshards, uint32_t* __restrict__ list_ids) {
  for (int l = blockIdx.x; l < nlist; l += gridDim.x) {
    uint32_t* out = list_ids + list_base[l];
    const uint32_t own = own_cnt[l], o0 = own_off[l];
    for (uint32_t i = threadIdx.x; i < own; i += blockDim.x)
      out[i] = slot_rows[o0 + i] * (uint32_t)nshards + (uint32_t)shard_id;
    uint32_t off = own;
    for (uint32_t j = ref_ptr[l]; j < ref_ptr[l + 1]; ++j) {
      const uint32_t c = ref_cnt[j], s0 = ref_start[j];
      for (uint32_t i = threadIdx.x; i < c; i += blockDim.x)
        out[off + i] = slot_rows[s0 + i] * (uint32_t)nshards + (uint32_t)shard_id;
      off += c;
    }
  }
}

rairs_status listmajor_prepare(rairs_index_s* idx, cudaStream_t s) {
  // a rebuild (after rairs_add / rairs_remove_ids) replaces the previous tables
  cudaFree(idx->list_items); cudaFree(idx->ref_item_off); cudaFree(idx->list_base); cudaFree(idx->list_ids);
  idx->list_items = idx->ref_item_off = idx->list_ids = nullptr;
  idx->list_base = nullptr;
  idx->device_bytes -= idx->lm_bytes;
  idx->lm_bytes = 0;
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
  {  // claim order of the list-major scan: descending N_l (ties by list id)
    std::vector<uint32_t> ord(idx->nlist);
    for (int l = 0; l < idx->nlist; ++l) ord[l] = (uint32_t)l;
    std::stable_sort(ord.begin(), ord.end(), [&](uint32_t x, uint32_t y) { return h[x] > h[y]; });
    cudaFree(idx->lm_order);
    idx->lm_order = nullptr;
    RAIRS_CUDA_TRY(cudaMalloc(&idx->lm_order, (size_t)idx->nlist * 4));
    RAIRS_CUDA_TRY(cudaMemcpyAsync(idx->lm_order, ord.data(), (size_t)idx->nlist * 4,
                                   cudaMemcpyHostToDevice, s));
    RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  }
  std::vector<uint64_t> base(idx->nlist + 1, 0);
  for (int l = 0; l < idx->nlist; ++l) {
    idx->max_list_items = std::max<int64_t>(idx->max_list_items, h[l]);
    base[l + 1] = base[l] + h[l];
  }
  idx->sum_list_items = (int64_t)base[idx->nlist];
  RAIRS_CUDA_TRY(cudaMalloc(&idx->list_base, (size_t)(idx->nlist + 1) * 8));
  RAIRS_CUDA_TRY(cudaMalloc(&idx->list_ids, (size_t)std::max<uint64_t>(base[idx->nlist], 1) * 4));
  RAIRS_CUDA_TRY(cudaMemcpyAsync(idx->list_base, base.data(), (size_t)(idx->nlist + 1) * 8,
                                 cudaMemcpyHostToDevice, s));
  lm_ids_kernel<<<std::min(idx->nlist, 148 * 8), 256, 0, s>>>(
      idx->own_off, idx->own_cnt, idx->ref_ptr, idx->ref_start, idx->ref_cnt, idx->slot_rows,
      idx->list_base, idx->nlist, idx->shard_id, idx->nshards, idx->list_ids);
  RAIRS_CHECK_LAUNCH();
  RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  if (!idx->aux_mu) {
    for (auto& st : idx->aux) RAIRS_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto& e : idx->aux_ev) RAIRS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    RAIRS_CUDA_TRY(cudaStreamCreateWithFlags(&idx->h2d, cudaStreamNonBlocking));
    for (auto& e : idx->h2d_ev) RAIRS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : idx->hq_ev) RAIRS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    idx->hq_mu = new std::mutex();
    idx->aux_mu = new std::mutex();
  }
  idx->lm_bytes = (size_t)idx->nlist * 4 + (size_t)std::max<int64_t>(idx->n_refs, 1) * 4 +
                  (size_t)(idx->nlist + 1) * 8 + (size_t)base[idx->nlist] * 4;
  idx->device_bytes += idx->lm_bytes;
  return RAIRS_OK;
}

}  // namespace rairs
