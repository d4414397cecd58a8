// coarse_kernels.cu -- K1/K2: the coarse quantizer on sm_100a tensor cores.
//
// K1  g[r][l] = ||c_l||^2 - 2 x_r.c_l  for every row r (a query, or a base
//     vector at build time) and every list l (FindNearestLists, P:942;
//     exhaustive O(nlist*D) P:1216; bulk per batch P:1862-1864), as a
//     hand-written tcgen05.mma kind::tf32 GEMM: operands streamed by TMA
//     (cp.async.bulk.tensor, 128B swizzle) through a shared-memory ring, one
//     elected thread issues the MMAs into a double-buffered fp32 accumulator in
//     TMEM (2 x 128 lanes x 256 columns), and four epilogue warps drain it with
//     tcgen05.ld while keeping each row's W+1 smallest g in shared memory --
//     the [rows x nlist] matrix is never written to HBM.
// K2  per row: merge the split lists, exact fp64 distances D64 (O1) of the W
//     best, re-rank by (D64, l), and CERTIFY (reading R6): every list outside
//     the candidate set has g >= g_(W+1) and |g - (D - ||x||^2)| <= E, so if
//     g_(W+1) - E exceeds the L-th exact distance minus ||x||^2, no excluded
//     list can enter the first L.  Uncertified rows are recomputed by the exact
//     fp64 kernel.  Output: probe sets (search), or the RAIR pair (Alg. 3) /
//     single assignment (build).  Results are always exactly O1 / O4.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <mutex>

#include "index.cuh"
#include "tc_helpers.cuh"

namespace rairs {

constexpr int FT_BM = 128, FT_BN = 256, FT_BK = 32;
constexpr uint32_t FT_A_BYTES = FT_BM * FT_BK * 4;  // 16 KB
constexpr uint32_t FT_B_BYTES = FT_BN * FT_BK * 4;  // 32 KB
constexpr int FT_EPI_WARPS = 8;  // warps 0-7 epilogue: lane group w%4, column half w/4
constexpr int FT_PROD_WARP = FT_EPI_WARPS, FT_MMA_WARP = FT_EPI_WARPS + 1;
constexpr int FT_THREADS = (FT_EPI_WARPS + 2) * 32;
constexpr int FT_HALVES = FT_EPI_WARPS / 4;
constexpr int FT_MAX_WP1 = 112;  // smem: lists + staging + 2-3 operand stages <= 227 KB
// instruction descriptor: D=F32, A=B=TF32, both K-major, N=256, M=128
constexpr uint32_t FT_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(FT_BN >> 3) << 17) |
                              ((uint32_t)(FT_BM >> 4) << 24);

struct TopWArgs {
  int64_t rows;
  int nl, d, Wp1, nsplit, tiles_per_split, ntiles, nstage;
  const float* cnorm;  // [round_up(nl, 256)], +inf padding
  int dbg;             // timing experiments (RAIRS_COARSE_DBG): 1 = no epilogue work
  uint32_t lazy_ns;     // sleep between polls of the producer / MMA single-thread waits
  int a_res;           // the A tile (all K-chunks) stays resident in shared memory
  // balanced schedule (lin = 1): the mtiles x ntiles (row tile, column tile)
  // units in row-major order are cut into gridDim.x equal contiguous ranges,
  // one per CTA; a range may cross row tiles (the row's lists are written at
  // each crossing, as piece b - first CTA of the row).  lin = 0: grid
  // (row tile, column split), tiles_per_split column tiles per CTA.
  int lin;
  int64_t total;       // mtiles * ntiles (lin)
  // output entries per (row, split): 32 on the register path (sorted), Wp1
  // on the shared-memory path (unsorted)
  float* out_v;        // [rows][nsplit][Wout]
  uint32_t* out_i;
};

// Per-row candidate list: W+1 slots, UNSORTED, with the running maximum kept in
// registers.  A value below the maximum replaces it and the maximum is
// recomputed (the same fixed-length scan in every lane of the warp, so a
// replacement costs W+1 steps without divergence -- an insertion sort costs up
// to W+1 divergent shifts per value).  Ties at the boundary may keep either
// entry: the certificate only needs every excluded list to have g >= g_(W+1).
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ void topw_rescan(const float* lv, int Wp1, int r, float& mx, int& mp) {
  mx = -__int_as_float(0x7f800000);
  mp = 0;
  for (int i0 = 0; i0 < Wp1; i0 += 8) {  // 8 independent loads in flight
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = (i0 + k < Wp1) ? lv[(i0 + k) * FT_BM + r] : mx;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (x[k] > mx) { mx = x[k]; mp = i0 + k; }
  }
}

template <int KR>
__global__ void __launch_bounds__(FT_THREADS, 1)
    coarse_topw_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB, TopWArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned; offset from smem_raw so the compiler keeps the shared
  // state space (plain LDS/STS, not generic loads, on the staging buffers)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = a.nstage, Wp1 = a.Wp1;
  const int nk = (a.d + FT_BK - 1) / FT_BK;
  // a_res: the row tile's A (all nk K-chunks) is loaded ONCE and stays resident
  // (every column tile of the CTA reuses it); the ring then carries B only
  uint8_t* sA = smem;
  uint8_t* sB = smem + (a.a_res ? (a.lin ? 2 * nk : nk) : S) * FT_A_BYTES;
  float* lv = reinterpret_cast<float*>(sB + S * FT_B_BYTES);  // smem path only
  uint32_t* li = reinterpret_cast<uint32_t*>(lv + (KR > 0 ? 0 : Wp1 * FT_BM));
  // g staging: [32][128] on the shared-memory path (warps 0-3), [32][256] on the
  // register path (8 epilogue warps: column j of warp w's rows at j*256 + 32w + lane)
  float* gbuf = reinterpret_cast<float*>(li + (KR > 0 ? 0 : Wp1 * FT_BM));
  uint64_t* full = reinterpret_cast<uint64_t*>(gbuf + 32 * FT_BM * (KR > 0 ? FT_HALVES : 1));
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tempty + 2;   // [2]: resident A of segment j in buffer j & 1
  uint64_t* aempty = afull + 2;   // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(aempty + 2);
  // ||c||^2 of the current 32-column chunk, per epilogue warp (32 floats): each
  // lane loads one value a chunk ahead, the warp reads them back broadcast
  float* cbuf_all = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(tslot) +
                                             ((16u - (smem_u32(tslot) & 15u)) & 15u) + 16u);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // this CTA's units [u0, u1): unit u = row tile u / ntiles, column tile u % ntiles
  int64_t u0, u1;
  if (a.lin) {
    u0 = (int64_t)blockIdx.x * a.total / gridDim.x;
    u1 = (int64_t)(blockIdx.x + 1) * a.total / gridDim.x;
  } else {
    const int64_t tb = (int64_t)blockIdx.y * a.tiles_per_split;
    u0 = (int64_t)blockIdx.x * a.ntiles + tb;
    u1 = (int64_t)blockIdx.x * a.ntiles + min((int64_t)a.ntiles, tb + a.tiles_per_split);
  }
  const int ntile = (int)(u1 - u0);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&tfull[k], 1);
      mbar_init(&tempty[k], FT_EPI_WARPS);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&afull[k], 1);
      mbar_init(&aempty[k], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (KR == 0 && warp < 4) {  // smem path: column half 0 only (see launcher)
    for (int i = 0; i < Wp1; ++i) {
      lv[i * FT_BM + tid] = __int_as_float(0x7f800000);
      li[i * FT_BM + tid] = 0xFFFFFFFFu;
    }
  }
  if (warp == FT_MMA_WARP) tmem_alloc(tslot, 512);
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == FT_PROD_WARP) {
    if (lane == 0 && ntile > 0) {  // TMA producer
      int it = 0, seg = -1;
      int64_t cur_r = -1, r = u0 / a.ntiles;
      int ct = (int)(u0 - r * a.ntiles);
      for (int t = 0; t < ntile; ++t, ct = (ct + 1 == a.ntiles) ? (++r, 0) : ct + 1) {
        const int m0 = (int)(r * FT_BM);
        if (r != cur_r) {  // a new row tile: its resident A into buffer seg & 1
          ++seg;
          cur_r = r;
          if (a.a_res) {
            const int ab = seg & 1;
            if (seg >= 2) mbar_wait(&aempty[ab], (uint32_t)((seg - 2) >> 1) & 1u);
            mbar_expect_tx(&afull[ab], (uint32_t)nk * FT_A_BYTES);
            for (int kc = 0; kc < nk; ++kc)
              tma_load_2d(sA + (ab * nk + kc) * FT_A_BYTES, &tmA, kc * FT_BK, m0, &afull[ab]);
          }
        }
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % S;
          const uint32_t ph = (uint32_t)(it / S) & 1u;
          if (it >= S) (a.dbg & 2) ? mbar_wait(&empty[s], ph ^ 1u) : mbar_wait_lazy(&empty[s], ph ^ 1u, a.lazy_ns);
          if (a.a_res) {
            mbar_expect_tx(&full[s], FT_B_BYTES);
          } else {
            mbar_expect_tx(&full[s], FT_A_BYTES + FT_B_BYTES);
            tma_load_2d(sA + s * FT_A_BYTES, &tmA, kc * FT_BK, m0, &full[s]);
          }
          tma_load_2d(sB + s * FT_B_BYTES, &tmB, kc * FT_BK, ct * FT_BN, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == FT_MMA_WARP) {
    if (lane == 0 && ntile > 0) {  // MMA issuer
      int it = 0, seg = -1;
      int64_t cur_r = -1, r = u0 / a.ntiles;
      int ct = (int)(u0 - r * a.ntiles);
      for (int t = 0; t < ntile; ++t, ct = (ct + 1 == a.ntiles) ? (++r, 0) : ct + 1) {
        if (r != cur_r) {
          // the previous row tile's MMAs release its A buffer when they complete
          if (seg >= 0 && a.a_res) umma_commit(&aempty[seg & 1]);
          ++seg;
          cur_r = r;
          if (a.a_res) mbar_wait(&afull[seg & 1], (uint32_t)(seg >> 1) & 1u);
        }
        const int acc = t & 1;
        const uint32_t aph = (uint32_t)(t >> 1) & 1u;
        if (t >= 2) (a.dbg & 2) ? mbar_wait(&tempty[acc], aph ^ 1u) : mbar_wait_lazy(&tempty[acc], aph ^ 1u, a.lazy_ns);
        tc_fence_after();
        const uint32_t dt = tmem + (uint32_t)(acc * FT_BN);
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % S;
          const uint32_t ph = (uint32_t)(it / S) & 1u;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(sA + (a.a_res ? (seg & 1) * nk + kc : s) * FT_A_BYTES);
          const uint64_t bd = umma_desc_sw128(sB + s * FT_B_BYTES);
#pragma unroll
          for (int k = 0; k < FT_BK / 8; ++k)  // K = 8 tf32 per MMA = 32 B = +2 desc units
            umma_tf32(dt, ad + 2 * k, bd + 2 * k, FT_IDESC, (kc | k) != 0 ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (KR > 0) {
    const int lg = warp & 3, half = warp >> 2;   // TMEM lane group, column half
    const int rrow = lg * 32 + lane;             // row within the tile
    // epilogue, register path: each row's KR smallest (g, l) kept SORTED in
    // registers; an insertion computes every slot in parallel from the old
    // values (new[i] = old[i-1] > g ? old[i-1] : min(old[i], g)), so it has no
    // dependency chain and no shared-memory round trip.
    float rv[KR > 0 ? KR : 1];
    uint32_t ri[KR > 0 ? KR : 1];
#pragma unroll
    for (int i = 0; i < KR; ++i) {
      rv[i] = __int_as_float(0x7f800000);
      ri[i] = 0xFFFFFFFFu;
    }
    // the lists of row tile r are written as piece `piece` of each row; the
    // CTA holding the row tile's last column tile pads the later pieces
    int64_t cur_r = -1;
    int piece = 0;
    auto flush = [&](int64_t r, bool row_end) {
      const int64_t row = r * FT_BM + rrow;
      if (row < a.rows) {
        float* ov = a.out_v + ((row * a.nsplit + piece) * FT_HALVES + half) * KR;
        uint32_t* oi = a.out_i + ((row * a.nsplit + piece) * FT_HALVES + half) * KR;
#pragma unroll
        for (int i = 0; i < KR; ++i) {
          ov[i] = rv[i];
          oi[i] = ri[i];
        }
        if (row_end)
          for (int p2 = piece + 1; p2 < a.nsplit; ++p2)
            for (int i = 0; i < KR; ++i) {
              a.out_v[((row * a.nsplit + p2) * FT_HALVES + half) * KR + i] = __int_as_float(0x7f800000);
              a.out_i[((row * a.nsplit + p2) * FT_HALVES + half) * KR + i] = 0xFFFFFFFFu;
            }
      }
#pragma unroll
      for (int i = 0; i < KR; ++i) {
        rv[i] = __int_as_float(0x7f800000);
        ri[i] = 0xFFFFFFFFu;
      }
    };
    int64_t r = u0 / a.ntiles;
    int ct = (int)(u0 - r * a.ntiles);
    constexpr int CPW = FT_BN / 32 / FT_HALVES;  // chunks per warp per tile (4)
    static_assert(CPW % 2 == 0, "chunks come in pairs");
    const int cb = half * CPW;
    float* cbuf = cbuf_all + warp * 32;
    float cnl = ntile > 0 ? __ldg(a.cnorm + ct * FT_BN + cb * 32 + lane) : 0.0f;  // first chunk's
    for (int t = 0; t < ntile; ++t, ct = (ct + 1 == a.ntiles) ? (++r, 0) : ct + 1) {
      const int acc = t & 1;
      const uint32_t aph = (uint32_t)(t >> 1) & 1u;
      if (r != cur_r) {
        if (cur_r >= 0) flush(cur_r, true);
        cur_r = r;
        // first CTA holding a unit of row tile r: the largest b with b*total/G <= r*ntiles
        piece = a.lin ? (int)((int64_t)blockIdx.x -
                              (((r * a.ntiles + 1) * gridDim.x + a.total - 1) / a.total - 1))
                      : (int)blockIdx.y;
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int col0 = ct * FT_BN;
      // TMEM reads are the epilogue's bound (LDTM ~64 B/clk/SM): the next chunk's
      // tcgen05.ld is in flight while this one is processed, and the
      // accumulator is released as soon as the last chunk is in registers
      auto process = [&](uint32_t (&v)[32], int c) {
        if ((a.dbg & 1) && t > 0) return;  // timing experiment: MMA + TMA only after tile 0
        // g = ||c||^2 - 2 q.c; ||c||^2 of the chunk's 32 columns: lane j's value
        // (loaded one chunk ahead) through the warp's shared slot, read back by 8
        // broadcast 16-B loads; the chunk minimum decides (warp-wide) whether
        // any value can enter a list -- the common case after the first tiles
        // costs one FFMA + one FMNMX per value
        __syncwarp();
        cbuf[lane] = cnl;
        __syncwarp();
        {  // the warp's next chunk: c + 1 of this tile, else chunk cb of the next tile
          const int nc = c + 1 < cb + CPW ? c + 1 : cb;
          const int ncol0 = c + 1 < cb + CPW ? col0 : (ct + 1 == a.ntiles ? 0 : ct + 1) * FT_BN;
          cnl = __ldg(a.cnorm + ncol0 + nc * 32 + lane);
        }
        const float4* cn4 = reinterpret_cast<const float4*>(cbuf);
        float g[32];
        float gmin = __int_as_float(0x7f800000);
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const float4 cn = cn4[q4];
          g[4 * q4 + 0] = fmaf(-2.0f, __uint_as_float(v[4 * q4 + 0]), cn.x);
          g[4 * q4 + 1] = fmaf(-2.0f, __uint_as_float(v[4 * q4 + 1]), cn.y);
          g[4 * q4 + 2] = fmaf(-2.0f, __uint_as_float(v[4 * q4 + 2]), cn.z);
          g[4 * q4 + 3] = fmaf(-2.0f, __uint_as_float(v[4 * q4 + 3]), cn.w);
        }
        // three-input minimum tree (FMNMX3): 16 instructions, depth 4
        float m1[11];
#pragma unroll
        for (int j = 0; j < 10; ++j) m1[j] = fmin3f(g[3 * j], g[3 * j + 1], g[3 * j + 2]);
        m1[10] = fminf(g[30], g[31]);
        const float m2a = fmin3f(m1[0], m1[1], m1[2]), m2b = fmin3f(m1[3], m1[4], m1[5]);
        const float m2c = fmin3f(m1[6], m1[7], m1[8]), m2d = fminf(m1[9], m1[10]);
        gmin = fminf(fmin3f(m2a, m2b, m2c), m2d);
        const float thr = rv[KR - 1];
        if (!__any_sync(0xffffffffu, gmin < thr)) return;
        uint32_t pass = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (g[j] < thr) {  // only candidates are staged for the insertion loop
            gbuf[j * (FT_BM * FT_HALVES) + warp * 32 + lane] = g[j];
            pass |= 1u << j;
          }
        }
        while (__any_sync(0xffffffffu, pass != 0)) {
          if (pass != 0) {
            const int j = __ffs(pass) - 1;
            pass &= pass - 1;
            const float g = gbuf[j * (FT_BM * FT_HALVES) + warp * 32 + lane];
            if (g < rv[KR - 1]) {
              const uint32_t l = (uint32_t)(col0 + c * 32 + j);
#pragma unroll
              for (int i = KR - 1; i > 0; --i) {
                const bool sh = rv[i - 1] > g;
                const bool here = !sh && rv[i] > g;
                ri[i] = sh ? ri[i - 1] : (here ? l : ri[i]);
                rv[i] = sh ? rv[i - 1] : (here ? g : rv[i]);
              }
              if (rv[0] > g) { rv[0] = g; ri[0] = l; }
            }
          }
        }
            };
      const uint32_t tbase = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * FT_BN);
      uint32_t va[32], vb[32];
      tmem_ld32_nowait(tbase + (uint32_t)(cb * 32), va);
      tmem_wait_ld();
#pragma unroll 1
      for (int c = cb; c < cb + CPW; c += 2) {
        tmem_ld32_nowait(tbase + (uint32_t)((c + 1) * 32), vb);
        process(va, c);
        tmem_wait_ld();
        if (c + 2 < cb + CPW) {
          tmem_ld32_nowait(tbase + (uint32_t)((c + 2) * 32), va);
          process(vb, c + 1);
          tmem_wait_ld();
        } else {  // every chunk of this tile is in registers: release the accumulator
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
          process(vb, c + 1);
        }
      }
    }
    if (cur_r >= 0) flush(cur_r, a.lin && (u1 % a.ntiles) == 0);
  } else if (warp >= 4) {  // shared-memory path: warps 4-7 only release the accumulators
    for (int t = 0; t < ntile; ++t) {
      mbar_wait(&tfull[t & 1], (uint32_t)(t >> 1) & 1u);
      tc_fence_after();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[t & 1]);
    }
  } else {  // epilogue, shared-memory path (large W): unsorted list + running max
    float thr = __int_as_float(0x7f800000);
    int thr_pos = 0, filled = 0;

    for (int t = 0; t < ntile; ++t) {
      const int acc = t & 1;
      const uint32_t aph = (uint32_t)(t >> 1) & 1u;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int col0 = (int)((u0 + t) % a.ntiles) * FT_BN;
      for (int c = 0; c < FT_BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * FT_BN + c * 32), v);
        uint32_t pass = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float g = __ldg(a.cnorm + col0 + c * 32 + j) - 2.0f * __uint_as_float(v[j]);
          gbuf[j * FT_BM + tid] = g;
          if (g < thr) pass |= 1u << j;
        }
        // each lane walks only its own passing values
        while (__any_sync(0xffffffffu, pass != 0)) {
          if (pass != 0) {
            const int j = __ffs(pass) - 1;
            pass &= pass - 1;
            const float g = gbuf[j * FT_BM + tid];
            if (g < thr) {
              const int pos = (filled < Wp1) ? filled++ : thr_pos;
              lv[pos * FT_BM + tid] = g;
              li[pos * FT_BM + tid] = (uint32_t)(col0 + c * 32 + j);
              if (filled == Wp1) topw_rescan(lv, Wp1, tid, thr, thr_pos);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    const int64_t row = (int64_t)blockIdx.x * FT_BM + tid;  // lin = 0 on this path
    if (row < a.rows) {
      float* ov = a.out_v + (row * a.nsplit + blockIdx.y) * Wp1;
      uint32_t* oi = a.out_i + (row * a.nsplit + blockIdx.y) * Wp1;
      for (int i = 0; i < Wp1; ++i) {
        ov[i] = lv[i * FT_BM + tid];
        oi[i] = li[i * FT_BM + tid];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == FT_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// K2: merge splits, exact fp64 re-rank, certify, emit probes / assignment.
constexpr int CT_THREADS = 256;
constexpr int CT_WARPS = CT_THREADS / 32;
#ifndef CT_MINB
#define CT_MINB 3  // certify CTAs per SM the register budget is sized for (4: 64 registers, rematerialised thread ids and spills; 3: coarse stage -4.5 us on c4)
#endif

__device__ __forceinline__ uint32_t ord_f32(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
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

// a[0, n) holds n / run sorted (ascending) runs of length run (powers of 2):
// merge them with the flip + half-cleaner network (log2(n/run) rounds instead
// of a full bitonic sort)
__device__ void warp_merge_runs(uint64_t* a, int run, int n) {
  const int lane = lane_id();
  for (int size = 2 * run; size <= n; size <<= 1) {
    const int hs = size >> 1;
    for (int i = lane; i < (n >> 1); i += 32) {  // flip: (j, size-1-j) of each block
      const int b = i / hs, j = i - b * hs;
      const int lo = b * size + j, hi = b * size + size - 1 - j;
      const uint64_t x = a[lo], y = a[hi];
      if (x > y) { a[lo] = y; a[hi] = x; }
    }
    __syncwarp();
    for (int stride = size >> 2; stride > 0; stride >>= 1) {
      for (int i = lane; i < (n >> 1); i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const uint64_t x = a[lo], y = a[hi];
        if (x > y) { a[lo] = y; a[hi] = x; }
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

struct CertArgs {
  const float* vals;
  const uint32_t* ids;
  int S, Wp1, Wout;
  const float* X;
  int64_t rows;
  int d;
  const float* C;
  int nl, L, mode;  // mode 0 probes, 1 AIR pair, 2 single
  double lambda;
  int strict;
  double cmax;
  int npow_c, npow_w;
  int capped_kr;       // > 0: capped register lists of this length (see launcher)
  int sorted_kr;       // > 0: the split lists are sorted, of this length (register path)
  int run;             // their padded length in keys[] (power of 2)
  int32_t* out_idx;
  int32_t* l1;
  int32_t* l2;
  int32_t* flags;
  unsigned* nflag;
  uint32_t* split_list;   // split exact fallback (large nlist): flagged rows appended here
  uint32_t* split_count;
  int stage_rows;      // stage the candidate centroid rows in shared memory
  size_t stage_off;    // byte offset of the staging area in dynamic smem
  size_t stage_warp;   // bytes per warp
  __device__ float* stage_base(unsigned char* sm, int warp) const {
    return reinterpret_cast<float*>(sm + stage_off + (size_t)warp * stage_warp);
  }
};

__global__ void __launch_bounds__(CT_THREADS, CT_MINB) coarse_certify_kernel(CertArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = warp_id(), lane = lane_id();
  pdl_wait();  // the top-W lists of coarse_topw_kernel
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm) + (size_t)warp * a.npow_c;
  uint64_t* ck = reinterpret_cast<uint64_t*>(sm) + (size_t)CT_WARPS * a.npow_c + (size_t)warp * a.npow_w;
  uint32_t* ci = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(sm) +
                                             (size_t)CT_WARPS * (a.npow_c + a.npow_w)) +
                 (size_t)warp * a.npow_w;
  const int W = a.Wp1 - 1;
  const bool all = W >= a.nl;
  const int Wc = all ? a.nl : W;
  const int tot = a.S * a.Wout;
  for (int64_t r = (int64_t)blockIdx.x * CT_WARPS + warp; r < a.rows;
       r += (int64_t)gridDim.x * CT_WARPS) {
    if (a.sorted_kr > 0) {
      // register path: every (split, half) list is sorted by (g, l) -- merge
      for (int i = lane; i < a.npow_c; i += 32) {
        const int g = i / a.run, j = i - g * a.run;
        uint64_t k = kKeyInf;
        if (j < a.sorted_kr && g * a.sorted_kr < tot) {
          const int e = g * a.sorted_kr + j;
          const uint32_t id = a.ids[r * tot + e];
          const float v = a.vals[r * tot + e];  // -0 as +0: the lists were built with float compares
          if (id != 0xFFFFFFFFu) k = ((uint64_t)ord_f32(v == 0.0f ? 0.0f : v) << 32) | id;
        }
        keys[i] = k;
      }
      __syncwarp();
      warp_merge_runs(keys, a.run, a.npow_c);
    } else {
      for (int i = lane; i < a.npow_c; i += 32) {
        uint64_t k = kKeyInf;
        if (i < tot) {
          const uint32_t id = a.ids[r * tot + i];
          if (id != 0xFFFFFFFFu) k = ((uint64_t)ord_f32(a.vals[r * tot + i]) << 32) | id;
        }
        keys[i] = k;
      }
      __syncwarp();
      warp_sort_u64(keys, a.npow_c);
    }
    float gnext = all ? 0.0f : unord_f32((uint32_t)(keys[W] >> 32));
    if (!all && a.capped_kr > 0) {
      // bound from the capped lists: min over full lists of their largest kept value
      float gb = __int_as_float(0x7f800000);
      for (int gi = lane; gi < tot / a.capped_kr; gi += 32) {
        const uint32_t id = a.ids[r * tot + gi * a.capped_kr + a.capped_kr - 1];
        if (id != 0xFFFFFFFFu) gb = fminf(gb, a.vals[r * tot + gi * a.capped_kr + a.capped_kr - 1]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gb = fminf(gb, __shfl_xor_sync(0xffffffffu, gb, o));
      gnext = fminf(gnext, gb);
    }
    const float* xr = a.X + (size_t)r * a.d;
    if (a.stage_rows) {
      // stage the Wc candidate centroid rows in shared memory with coalesced
      // 16-B loads (all rows in flight at once), row stride d + 4 floats
      float* cs = a.stage_base(sm, warp);
      const int d4 = a.d >> 2, rs4 = d4 + 1;
      for (int i0 = 0; i0 < Wc; i0 += 8) {  // 8 rows' loads in flight before the stores
        for (int t4 = lane; t4 < d4; t4 += 32) {
          float4 r[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (i0 + u < Wc && keys[i0 + u] != kKeyInf) {  // (a short union: no row)
              const uint32_t l = (uint32_t)(keys[i0 + u] & 0xFFFFFFFFu);
              r[u] = __ldg(reinterpret_cast<const float4*>(a.C + (size_t)l * a.d) + t4);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (i0 + u < Wc) reinterpret_cast<float4*>(cs)[(i0 + u) * rs4 + t4] = r[u];
        }
      }
      // the row, widened to fp64 once (exact), after the staged candidate rows
      double* xd = reinterpret_cast<double*>(cs + (size_t)Wc * rs4 * 4 + 2 * ((Wc * rs4 * 4) & 1));
      for (int t = lane; t < a.d; t += 32) xd[t] = (double)xr[t];
      __syncwarp();
      for (int i = lane; i < a.npow_w; i += 32) {
        if (i < Wc && keys[i] != kKeyInf) {
          const float4* c4 = reinterpret_cast<const float4*>(cs) + i * rs4;
          const double2* x2 = reinterpret_cast<const double2*>(xd);
          double acc = 0.0;
#pragma unroll 4
          for (int t4 = 0; t4 < d4; ++t4) {
            const float4 cv = c4[t4];
            const double2 xa = x2[2 * t4], xb = x2[2 * t4 + 1];
            double df;
            df = __dsub_rn(xa.x, (double)cv.x); acc = __dadd_rn(acc, __dmul_rn(df, df));
            df = __dsub_rn(xa.y, (double)cv.y); acc = __dadd_rn(acc, __dmul_rn(df, df));
            df = __dsub_rn(xb.x, (double)cv.z); acc = __dadd_rn(acc, __dmul_rn(df, df));
            df = __dsub_rn(xb.y, (double)cv.w); acc = __dadd_rn(acc, __dmul_rn(df, df));
          }
          ck[i] = dbits(acc);
          ci[i] = (uint32_t)(keys[i] & 0xFFFFFFFFu);
        } else {
          ck[i] = kKeyInf;
          ci[i] = 0xFFFFFFFFu;
        }
      }
      __syncwarp();
    } else
    for (int i = lane; i < a.npow_w; i += 32) {
      if (i < Wc && keys[i] != kKeyInf) {
        const uint32_t l = (uint32_t)(keys[i] & 0xFFFFFFFFu);
        const float* c = a.C + (size_t)l * a.d;
        double acc = 0.0;
        if ((a.d & 3) == 0) {
          const float4* c4 = reinterpret_cast<const float4*>(c);
          const float4* x4 = reinterpret_cast<const float4*>(xr);
#pragma unroll 4
          for (int t4 = 0; t4 < (a.d >> 2); ++t4) {
            const float4 cv = __ldg(c4 + t4), xv = __ldg(x4 + t4);
            acc = __dadd_rn(acc, dsq_diff(xv.x, cv.x));
            acc = __dadd_rn(acc, dsq_diff(xv.y, cv.y));
            acc = __dadd_rn(acc, dsq_diff(xv.z, cv.z));
            acc = __dadd_rn(acc, dsq_diff(xv.w, cv.w));
          }
        } else {
          for (int t = 0; t < a.d; ++t) acc = __dadd_rn(acc, dsq_diff(xr[t], c[t]));
        }
        ck[i] = dbits(acc);
        ci[i] = l;
      } else {
        ck[i] = kKeyInf;
        ci[i] = 0xFFFFFFFFu;
      }
    }
    __syncwarp();
    warp_sort_pairs2(ck, ci, a.npow_w);
    bool certified = all;
    if (!all) {
      double qn = 0.0;
      for (int t = lane; t < a.d; t += 32) qn += (double)xr[t] * (double)xr[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) qn += __shfl_xor_sync(0xffffffffu, qn, o);
      const double qnorm = sqrt(qn);
      const double E = (ldexp(1.0, -8) + a.d * ldexp(1.0, -22)) * qnorm * a.cmax +
                       ldexp(1.0, -22) * (a.cmax * a.cmax + 2.0 * qnorm * a.cmax);
      const double dL = __longlong_as_double((long long)ck[a.L - 1]);
      certified = ((double)gnext - E) > (dL - qn) + 1e-10 * (dL + qn);
    }
    if (a.mode == 0) {
      for (int i = lane; i < a.L; i += 32) a.out_idx[r * a.L + i] = (int32_t)ci[i];
    } else if (a.mode == 2) {
      if (lane == 0) { a.l1[r] = (int32_t)ci[0]; a.l2[r] = (int32_t)ci[0]; }
    } else {
      // Alg. 3 lines 3-11 over the first L = N_CANDS exact lists (fp64, O4)
      const int start = a.strict ? 1 : 0;
      double loss = 0.0;
      const bool ok = (lane >= start) && (lane < a.L) && ci[0] != 0xFFFFFFFFu && ci[lane] != 0xFFFFFFFFu;
      if (ok) {
        const float* c0 = a.C + (size_t)ci[0] * a.d;
        const float* cj = a.C + (size_t)ci[lane] * a.d;
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
        const int c0 = (int)ci[0], cb = (int)ci[best];
        a.l1[r] = min(c0, cb);
        a.l2[r] = max(c0, cb);
      }
    }
    if (lane == 0) {
      a.flags[r] = certified ? 0 : 1;
      if (!certified) {
        atomicAdd(a.nflag, 1u);
        atomicAdd(a.flags + a.rows, 1);  // per-call count: the fallback exits at once when 0
        if (a.split_list) {
          const uint32_t i = atomicAdd(a.split_count, 1u);
          if (i < (uint32_t)PX_CAP) a.split_list[i] = (uint32_t)r;
        }
      }
    }
    __syncwarp();
  }
  pdl_trigger();
}

__global__ void cnorm_kernel(const float* __restrict__ C, int nlist, int npad, int d,
                             float* __restrict__ cn, double* __restrict__ cmax_out) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < npad; l += gridDim.x * blockDim.x) {
    if (l >= nlist) {
      cn[l] = __int_as_float(0x7f800000);
      continue;
    }
    double s = 0.0;
    for (int t = 0; t < d; ++t) s += (double)C[(size_t)l * d + t] * (double)C[(size_t)l * d + t];
    cn[l] = (float)s;
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

bool tma_available() { return get_encode() != nullptr; }

bool make_tmap_f32(CUtensorMap* tm, const float* ptr, int64_t rows, int d, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 4};
  cuuint32_t box[2] = {(cuuint32_t)FT_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

rairs_status coarse_prepare(rairs_index_s* idx, cudaStream_t s) {
  const int npad = (int)round_up(idx->nlist, FT_BN);
  RAIRS_CUDA_TRY(cudaMalloc(&idx->cnorm, (size_t)npad * 4));
  double* dmax = nullptr;
  RAIRS_CUDA_TRY(ws_malloc(&dmax, 8, s));
  RAIRS_CUDA_TRY(cudaMemsetAsync(dmax, 0, 8, s));
  cnorm_kernel<<<(npad + 255) / 256, 256, 0, s>>>(idx->centroids, idx->nlist, npad, idx->d,
                                                  idx->cnorm, dmax);
  RAIRS_CHECK_LAUNCH();
  RAIRS_CUDA_TRY(cudaMemcpyAsync(&idx->cmax, dmax, 8, cudaMemcpyDeviceToHost, s));
  RAIRS_CUDA_TRY(cudaFreeAsync(dmax, s));
  RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  idx->device_bytes += (size_t)npad * 4;
  return RAIRS_OK;
}

template <int KR>
static cudaError_t launch_topw_kr(dim3 grid, size_t smem, cudaStream_t s, const CUtensorMap& tmA,
                                  const CUtensorMap& tmB, const TopWArgs& ta) {
  static const cudaError_t attr = cudaFuncSetAttribute(
      coarse_topw_kernel<KR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (attr != cudaSuccess) return attr;
  coarse_topw_kernel<KR><<<grid, FT_THREADS, smem, s>>>(tmA, tmB, ta);
  return cudaGetLastError();
}

// KR = 0: the shared-memory path (grid of row tiles x column splits)
static cudaError_t launch_topw(int KR, dim3 grid, dim3 grid_smem, size_t smem, cudaStream_t s,
                               const CUtensorMap& tmA, const CUtensorMap& tmB, const TopWArgs& ta) {
  switch (KR) {
    case 0: return launch_topw_kr<0>(grid_smem, smem, s, tmA, tmB, ta);
    case 6: return launch_topw_kr<6>(grid, smem, s, tmA, tmB, ta);
    case 7: return launch_topw_kr<7>(grid, smem, s, tmA, tmB, ta);
    case 8: return launch_topw_kr<8>(grid, smem, s, tmA, tmB, ta);
    case 9: return launch_topw_kr<9>(grid, smem, s, tmA, tmB, ta);
    case 10: return launch_topw_kr<10>(grid, smem, s, tmA, tmB, ta);
    case 11: return launch_topw_kr<11>(grid, smem, s, tmA, tmB, ta);
    case 12: return launch_topw_kr<12>(grid, smem, s, tmA, tmB, ta);
    case 13: return launch_topw_kr<13>(grid, smem, s, tmA, tmB, ta);
    case 16: return launch_topw_kr<16>(grid, smem, s, tmA, tmB, ta);
    case 20: return launch_topw_kr<20>(grid, smem, s, tmA, tmB, ta);
    case 24: return launch_topw_kr<24>(grid, smem, s, tmA, tmB, ta);
    default: return launch_topw_kr<32>(grid, smem, s, tmA, tmB, ta);
  }
}

static int coarse_width(int nl, int L) { return std::min(nl, L + 8 + L / 8); }

// small search batches: every row through the split exact path (c4 one query:
// coarse 0.105 ms on the tensor-core path, whose cost is mostly fixed)
int coarse_small_rows() {
  static const int v = [] {
    const char* e = std::getenv("RAIRS_COARSE_SMALL");
    return e ? std::atoi(e) : 16;
  }();
  return v;
}

bool coarse_fused_ok(const rairs_index_s* idx, int L) {
  if (idx->coarse_mode == 1) return false;  // forced exact
  if ((idx->d & 3) != 0 || !tma_available()) return false;
  const int wp1 = coarse_width(idx->nlist, L) + 1;
  const bool capped_ok = ceil_div(idx->nlist, FT_BN) >= 8 && wp1 <= 256;  // capped register lists
  if (wp1 > FT_MAX_WP1 && !capped_ok) return false;
  if (idx->coarse_mode == 2) return true;   // forced tensor-core path
  return idx->nlist >= 64 && L < idx->nlist;
}

// Rows X[rows x d] against the index's centroids: the first L lists by
// (D64, l), exactly, via K1 (tensor core) + K2 (certify) + exact fallback.
rairs_status launch_coarse_fused(const rairs_index_s* idx, const float* X, int64_t rows, int L,
                                 int mode, double lambda, int strict, int32_t* out_idx,
                                 int32_t* l1, int32_t* l2, unsigned* nflag, cudaStream_t s) {
  if (rows <= 0) return RAIRS_OK;
  const int nl = idx->nlist, d = idx->d;
  const int W = coarse_width(nl, L);
  const int Wp1 = W + 1;
  if (Wp1 > FT_MAX_WP1 && !(ceil_div(nl, FT_BN) >= 8 && Wp1 <= 256)) {
    set_error("coarse: nprobe too large for the fused tensor-core path");
    return RAIRS_E_UNSUPPORTED;
  }
  const int ntiles = (int)ceil_div(nl, FT_BN);
  // register-resident sorted lists; for W + 1 > 32 the lists are CAPPED at 32
  // per (row, column split, half) and K2 lowers its bound to the smallest
  // 32nd value of any full list (the excluded columns of a group are no
  // smaller than the largest value it kept), so the certificate stays valid
  const int nl_tiles = (int)ceil_div(nl, FT_BN);
  const bool capped = Wp1 > 32 && nl_tiles >= 8;
  const bool reg = Wp1 <= 32 || capped;
  // list length = W + 1 rounded up to an instantiated size: the insertion cost
  // and the pass threshold (the KR-th kept value) both shrink with KR
  // Half lists (>= 8 column tiles): each (row, split, half) list keeps only
  // ceil((W + 1) / 2) + 1 entries and K2 bounds the excluded lists by the
  // union's (W+1)-th value AND every full list's last value (as for capped
  // lists): about the same certificate (the union of two half lists of k holds
  // every value below min(last0, last1), ~the 2k-th overall), at a fraction
  // of the insertion work (fewer insertions, shorter networks).
  static const bool half_env = [] {
    const char* e = std::getenv("RAIRS_COARSE_HALFLISTS");
    return e ? std::atoi(e) != 0 : true;
  }();
  const bool short_lists = half_env && !capped && Wp1 <= 32 && nl_tiles >= 8;
  const int kw = short_lists ? (Wp1 + 1) / 2 + 1 : std::max(Wp1, 10);
  const int KR = kw <= 6 ? 6 : kw <= 7 ? 7 : kw <= 8 ? 8 : kw <= 9 ? 9 : kw <= 10 ? 10 : kw <= 11 ? 11
               : kw <= 12 ? 12 : kw <= 13 ? 13 : kw <= 16 ? 16 : kw <= 20 ? 20 : kw <= 24 ? 24 : 32;
  const int Wout = reg ? KR * FT_HALVES : Wp1;  // entries per (row, split)
  const int lists_bytes = reg ? 32 * FT_BM * FT_HALVES * 4 : Wp1 * FT_BM * 8 + 32 * FT_BM * 4;
  const int nkc = (int)ceil_div(d, FT_BK);
  int nsm = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  static const bool lin_env = [] {
    const char* e = std::getenv("RAIRS_COARSE_LIN");
    return e ? std::atoi(e) != 0 : true;
  }();
  // smem plan for nab resident A buffers (0: A streamed with B per stage)
  auto plan = [&](int nab, int& nstage, size_t& smem) {
    if (nab > 0) {
      nstage = (int)std::min<size_t>(6, (227 * 1024 - 2304 - lists_bytes - (size_t)nab * nkc * FT_A_BYTES) / FT_B_BYTES);
    } else {
      nstage = (lists_bytes <= 80 * 1024) ? 3 : 2;
    }
    const size_t ring_bytes = nab > 0 ? (size_t)nab * nkc * FT_A_BYTES + (size_t)nstage * FT_B_BYTES
                                      : (size_t)nstage * (FT_A_BYTES + FT_B_BYTES);
    smem = 1024 + ring_bytes + lists_bytes + (2 * nstage + 8) * 8 + 16 + 32 + FT_EPI_WARPS * 32 * 4;
  };
  // A resident (loaded once per row tile) when it fits next to >= 3 B stages:
  // the ring then moves 2/3 of the bytes per column tile (the TMA ingest bound)
  const bool a_res = (size_t)nkc * FT_A_BYTES + 3 * FT_B_BYTES + lists_bytes + 2304 <= 227 * 1024;
  const bool a_res2 = (size_t)2 * nkc * FT_A_BYTES + 3 * FT_B_BYTES + lists_bytes + 2304 <= 227 * 1024;
  int nstage = 0;
  size_t smem = 0;
  plan(a_res ? 1 : 0, nstage, smem);
  if (smem > 227 * 1024) {
    set_error("coarse: shared memory budget exceeded");
    return RAIRS_E_UNSUPPORTED;
  }
  const int64_t CH = 1 << 21;  // rows per chunk (bounds the candidate buffers)
  const int npow_w = next_pow2(std::max(W, 2));
  for (int64_t r0 = 0; r0 < rows; r0 += CH) {
    const int64_t nr = std::min<int64_t>(CH, rows - r0);
    const int64_t mtiles = ceil_div(nr, FT_BM);
    // column splits: only when there are too few row tiles to occupy the GPU.
    // A split restarts the top-W insertion (the first column tile pays most of
    // it) and doubles the certify merge; measured on c2pl (4 column tiles) and
    // c4 (64): one split per row tile beats covering every SM (coarse 0.120 ->
    // 0.098 ms and 0.305 -> 0.265 ms for 79 row tiles)
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, ceil_div(64, mtiles)));
    // long rows (d >= 512, c3: 1536): a tile's MMA (K = d) dwarfs the top-W
    // insertion a split restarts, so spread the column tiles over >= 4 CTAs
    // per SM (the grid of row tiles alone leaves SMs idle: 79 of 148 at 10k rows)
    if (d >= 512) nsplit = std::max<int>(nsplit, (int)std::min<int64_t>(ntiles, ceil_div(4 * 148, mtiles)));
    if (const char* e = std::getenv("RAIRS_COARSE_NSPLIT")) nsplit = std::max(1, std::min<int>(ntiles, std::atoi(e)));
    if (capped)  // >= 4 capped lists per needed 32 candidates: a group rarely holds > 32 of them
      nsplit = std::max<int>(nsplit, (int)std::min<int64_t>(ntiles, ceil_div(4 * ceil_div(Wp1, 32), FT_HALVES)));
    nsplit = std::max(1, std::min(nsplit, 1024 / Wout));  // K2 merges nsplit * Wout <= 1024 keys
    const int tps = (int)ceil_div(ntiles, nsplit);
    nsplit = (int)ceil_div(ntiles, tps);
    // balanced schedule: search-sized batches whose row tiles alone leave SMs
    // idle (c4: 79 row tiles x 64 column tiles -> 148 ranges of ~34 units
    // instead of 79 CTAs of 64: coarse 0.258 -> 0.245 ms), register lists, no
    // capped lists, and long rows of column tiles (each piece restarts the
    // top-W insertion: c2pl's 16 column tiles measured 0.095 -> 0.121 ms)
    const int64_t total = mtiles * ntiles;
    int lin = 0, nstage_k = nstage;
    size_t smem_k = smem;
    int64_t G = 0;
    if (lin_env && reg && !capped && d < 512 && ntiles >= 32 && mtiles % nsm != 0 && mtiles < 4 * nsm &&
        total >= 2 * nsm && !std::getenv("RAIRS_COARSE_NSPLIT")) {
      G = nsm;
      const int64_t minper = total / G;
      const int pieces = (int)std::min<int64_t>(ntiles, ceil_div(ntiles, minper) + 1);
      if (pieces * Wout <= 1024) {
        lin = 1;
        nsplit = pieces;
        plan(a_res2 ? 2 : 0, nstage_k, smem_k);
      }
    }
    // register path: nsplit * FT_HALVES sorted lists of KR, each padded to a
    // power-of-2 run, merged in K2; shared-memory path: unsorted, fully sorted
    const int run = next_pow2(KR);
    const int npow_c = reg ? next_pow2(std::max(nsplit * FT_HALVES, 1) * run)
                           : next_pow2(std::max(nsplit * Wout, 2));
    const size_t csmem = (size_t)CT_WARPS * ((size_t)npow_c * 8 + (size_t)npow_w * 12);
    if (csmem > 220 * 1024) {
      set_error("coarse certify: shared memory budget exceeded");
      return RAIRS_E_UNSUPPORTED;
    }
    float* vals = nullptr;
    uint32_t* ids = nullptr;
    int32_t* flags = nullptr;
    RAIRS_CUDA_TRY(ws_malloc(&vals, (size_t)nr * nsplit * Wout * 4, s));
    RAIRS_CUDA_TRY(ws_malloc(&ids, (size_t)nr * nsplit * Wout * 4, s));
    // flags[nr]: flagged-row count of this call; flags[nr + 1]: rows in the split list
    RAIRS_CUDA_TRY(ws_malloc(&flags, (size_t)(nr + 2) * 4, s));
    RAIRS_CUDA_TRY(cudaMemsetAsync(flags + nr, 0, 8, s));
    const float* Xc = X + (size_t)r0 * d;
    CUtensorMap tmA, tmB;
    if (!make_tmap_f32(&tmA, Xc, nr, d, FT_BM) || !make_tmap_f32(&tmB, idx->centroids, nl, d, FT_BN)) {
      cudaFreeAsync(vals, s); cudaFreeAsync(ids, s); cudaFreeAsync(flags, s);
      set_error("cuTensorMapEncodeTiled failed");
      return RAIRS_E_CUDA;
    }
    TopWArgs ta{};
    ta.rows = nr;
    ta.nl = nl;
    ta.d = d;
    ta.Wp1 = Wp1;
    ta.nsplit = nsplit;
    ta.tiles_per_split = tps;
    ta.ntiles = ntiles;
    ta.nstage = nstage_k;
    ta.a_res = (lin ? a_res2 : a_res) ? 1 : 0;
    ta.lin = lin;
    ta.total = total;
    ta.cnorm = idx->cnorm;
    {
      const char* e = std::getenv("RAIRS_COARSE_DBG");
      ta.dbg = e ? std::atoi(e) : 0;
      const char* z = std::getenv("RAIRS_COARSE_LAZY_NS");
      ta.lazy_ns = z ? (uint32_t)std::atoi(z) : 96u;
    }
    ta.out_v = vals;
    ta.out_i = ids;
    const dim3 tgrid = lin ? dim3((unsigned)G, 1u) : dim3((unsigned)mtiles, (unsigned)nsplit);
    RAIRS_CUDA_TRY(launch_topw(reg ? KR : 0, tgrid, dim3((unsigned)mtiles, (unsigned)nsplit), smem_k, s,
                               tmA, tmB, ta));
    RAIRS_CHECK_LAUNCH();
    if (debug_sync_enabled()) {
      char what[160];
      snprintf(what, sizeof(what), "coarse_topw_kernel (rows %lld..%lld of %lld, X=%p, Xc=%p)",
               (long long)r0, (long long)(r0 + nr), (long long)rows, (const void*)X, (const void*)Xc);
      RAIRS_TRY(debug_sync_point(s, what));
    }
    // exact fp64 recomputation of the (rare) uncertified rows (split path for
    // large nlist: its workspace now, the certify kernel lists the rows)
    ProbeArgs pa{};
    pa.X = Xc;
    pa.rows = nr;
    pa.d = d;
    pa.C = idx->centroids;
    pa.nl = nl;
    pa.L = L;
    pa.mode = mode;
    pa.lambda = lambda;
    pa.strict = strict;
    pa.out_idx = out_idx ? out_idx + r0 * L : nullptr;
    pa.l1 = l1 ? l1 + r0 : nullptr;
    pa.l2 = l2 ? l2 + r0 : nullptr;
    pa.only_flagged = flags;
    ProbeSplitBufs sb;
    {
      const rairs_status ps = probe_split_prepare(pa, sb, s);
      if (ps != RAIRS_OK) {
        cudaFreeAsync(vals, s); cudaFreeAsync(ids, s); cudaFreeAsync(flags, s);
        return ps;
      }
    }
    CertArgs ca{};
    ca.vals = vals;
    ca.ids = ids;
    ca.S = nsplit;
    ca.Wp1 = Wp1;
    ca.Wout = Wout;
    ca.X = Xc;
    ca.rows = nr;
    ca.d = d;
    ca.C = idx->centroids;
    ca.nl = nl;
    ca.L = L;
    ca.mode = mode;
    ca.lambda = lambda;
    ca.strict = strict;
    ca.cmax = idx->cmax;
    ca.npow_c = npow_c;
    ca.capped_kr = (capped || short_lists) ? KR : 0;
    ca.sorted_kr = reg ? KR : 0;
    ca.run = run;
    ca.npow_w = npow_w;
    ca.out_idx = out_idx ? out_idx + r0 * L : nullptr;
    ca.l1 = l1 ? l1 + r0 : nullptr;
    ca.l2 = l2 ? l2 + r0 : nullptr;
    ca.flags = flags;
    ca.nflag = nflag;
    ca.split_list = sb.on ? sb.list : nullptr;
    ca.split_count = reinterpret_cast<uint32_t*>(flags + nr + 1);
    // candidate-row staging (coalesced loads) when it fits next to the sort buffers
    const size_t stage_warp = round_up((size_t)std::min(W, nl) * (d + 4) * 4, 16) + (size_t)d * 8 + 16;
    ca.stage_off = round_up(csmem, 16);
    ca.stage_warp = stage_warp;
    ca.stage_rows = ((d & 3) == 0 && ca.stage_off + CT_WARPS * stage_warp <= 160 * 1024) ? 1 : 0;
    const size_t csmem_all = ca.stage_rows ? ca.stage_off + CT_WARPS * stage_warp : csmem;
    RAIRS_CUDA_TRY(cudaFuncSetAttribute(coarse_certify_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem_all));
    const int cgrid = (int)std::min<int64_t>(ceil_div(nr, CT_WARPS), 148 * 16);
    RAIRS_CUDA_TRY(launch_pdl(coarse_certify_kernel, dim3(cgrid), dim3(CT_THREADS), csmem_all, s, ca));
    RAIRS_DEBUG_POINT(s, "coarse_certify_kernel");
    rairs_status st = probe_split_launch(pa, sb, reinterpret_cast<const uint32_t*>(flags + nr + 1), flags, s);
    pa.flag_count = true;  // flags[nr]: rows the certify flagged (the split path may clear some)
    if (st == RAIRS_OK) st = launch_probe_exact(pa, s);   // remaining flagged rows
    if (st == RAIRS_OK && debug_sync_enabled()) st = debug_sync_point(s, "probe_exact fallback");
    probe_split_free(sb, s);
    cudaFreeAsync(vals, s);
    cudaFreeAsync(ids, s);
    cudaFreeAsync(flags, s);
    if (st != RAIRS_OK) return st;
  }
  return RAIRS_OK;
}

}  // namespace rairs
