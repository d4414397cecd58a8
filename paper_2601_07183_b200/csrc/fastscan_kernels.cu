// fastscan_kernels.cu -- query-major 4-bit fast scan with register LUTs (A3-A6).
//
// One WARP per query (queries claimed from an atomic counter by persistent
// warps), fused:
//   A3  ComputeLookupTable (LUT P:711-716) + uint8 quantisation (O2,
//       R2/R3): lane per subquantizer, fp32 with explicit rounding, written
//       to the warp's shared-memory LUT (16 B per subquantizer).
//   A4  SEIL work list (Alg. 5, order-free rule R9): every probed
//       list's owned range, plus each of its references (owner i -> list l)
//       whose owner is NOT probed (binary search in the sorted probe set).
//   A5  4-bit fast scan (PQFastScan P:729-737) on the GROUP layout: lane =
//       one 8-item nibble group, so one 32-bit code word holds the 8 items'
//       nibbles of ONE subquantizer m and the 16-entry LUT row of m sits in
//       four registers.  Four items are looked up per `prmt` pair (entries
//       0-7 and 8-15 of the row, selected by the low three nibble bits), a
//       third `prmt` in sign-replicate mode turns bit 3 of each nibble into a
//       byte mask that blends the two, and `dp4a` (fma pipe) adds each byte
//       into its item's exact u32 sum (R4: no wrap, any M).  Codes stream as
//       coalesced 16-B loads (a warp reads 512 contiguous-per-block bytes per
//       instruction), nothing is staged: each byte is used by one lane.
//   A6  top-bigK by the unique key (s << 32 | id) (rqueue P:1645, R5): items
//       with s <= tau are appended to a warp buffer as pre-keys (s, slot); a
//       full buffer is cut at the bigK-th SCORE by a radix select (ties kept,
//       no id loads); at the end the survivors' ids are loaded and the exact
//       top-bigK set is taken (ties at the cut score ranked by id).  Massive
//       score ties switch the query to exact mode (resolved keys, sort + cut).
// The candidate keys then go to the exact refine (search_kernels.cu).
//
// The group layout (`codes_g`, built from the cell-major layout by
// fastscan_prepare): per 32-slot block of 16*M_pad bytes, [m4 = m/4][group g
// = (slot/8)%4][4 words, m = 4 m4 + k]; word bits 4v..4v+3 = item slot%8 = v.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "index.cuh"
#include "lut_common.cuh"

namespace rairs {

constexpr int FS_RCAP = 64;      // ranges per scan batch (per warp)
constexpr int FS_MAXW = 8;       // warps per CTA (fewer when bigK needs more shared memory)
constexpr int FS_SLOTS = 64;     // claim-counter slots (concurrent searches)
// RAIRS_FS_DBG timing experiments (skip rounds / selection / loads) are only
// compiled in with -DRAIRS_FS_TIMING; the product kernel has no such branches.
#ifdef RAIRS_FS_TIMING
constexpr bool kFsTiming = true;
#else
constexpr bool kFsTiming = false;
#endif

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint4 ldg_nc_v4(const uint8_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// 8 lookups: items v = 0..7 of one nibble word w (subquantizer m, LUT row T)
__device__ __forceinline__ void lookup8(const uint4& T, uint32_t w, uint32_t (&acc)[8]) {
  const uint32_t x = w & 0x77777777u;          // low three bits of each nibble
  const uint32_t xh = __umulhi(x, 0x10000u);   // x >> 16 (items 4-7), on the fma pipe
  const uint32_t w4 = w << 4;
  // byte i = 0xFF iff bit 3 of nibble i: sign-replicate the byte holding it at bit 7
  const uint32_t m0 = prmt(w4, w, 0xD9C8u);
  const uint32_t m1 = prmt(w4, w, 0xFBEAu);
  const uint32_t lo0 = prmt(T.x, T.y, x), hi0 = prmt(T.z, T.w, x);
  const uint32_t lo1 = prmt(T.x, T.y, xh), hi1 = prmt(T.z, T.w, xh);
  const uint32_t r0 = (lo0 & ~m0) | (hi0 & m0);   // one LOP3
  const uint32_t r1 = (lo1 & ~m1) | (hi1 & m1);
  acc[0] = __dp4a(r0, 0x00000001u, acc[0]);
  acc[1] = __dp4a(r0, 0x00000100u, acc[1]);
  acc[2] = __dp4a(r0, 0x00010000u, acc[2]);
  acc[3] = __dp4a(r0, 0x01000000u, acc[3]);
  acc[4] = __dp4a(r1, 0x00000001u, acc[4]);
  acc[5] = __dp4a(r1, 0x00000100u, acc[5]);
  acc[6] = __dp4a(r1, 0x00010000u, acc[6]);
  acc[7] = __dp4a(r1, 0x01000000u, acc[7]);
}

// the same 8 lookups with the sums packed in pairs: dp2a adds byte 2p with
// weight 1 and byte 2p+1 with weight 2^15 into one u32, so items (2p, 2p+1)
// share an accumulator (item 2p in bits 0-14, exact while M_pad * 255 < 2^15,
// i.e. M_pad <= 128; item 2p+1 in bits 15-31): 4 instead of 8 fma-pipe
// instructions per word.  fs_unpack splits them after the group's last word.
__device__ __forceinline__ void lookup8p(const uint4& T, uint32_t w, uint32_t (&acc)[4]) {
  const uint32_t x = w & 0x77777777u;
  const uint32_t xh = __umulhi(x, 0x10000u);
  const uint32_t w4 = w << 4;
  const uint32_t m0 = prmt(w4, w, 0xD9C8u);
  const uint32_t m1 = prmt(w4, w, 0xFBEAu);
  const uint32_t lo0 = prmt(T.x, T.y, x), hi0 = prmt(T.z, T.w, x);
  const uint32_t lo1 = prmt(T.x, T.y, xh), hi1 = prmt(T.z, T.w, xh);
  const uint32_t r0 = (lo0 & ~m0) | (hi0 & m0);
  const uint32_t r1 = (lo1 & ~m1) | (hi1 & m1);
  acc[0] = __dp2a_lo(0x80000001u, r0, acc[0]);
  acc[1] = __dp2a_hi(0x80000001u, r0, acc[1]);
  acc[2] = __dp2a_lo(0x80000001u, r1, acc[2]);
  acc[3] = __dp2a_hi(0x80000001u, r1, acc[3]);
}

__device__ __forceinline__ void fs_unpack(const uint32_t (&p)[4], uint32_t (&acc)[8]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc[2 * i] = p[i] & 0x7FFFu;
    acc[2 * i + 1] = p[i] >> 15;
  }
}

struct FsArgs {
  const uint8_t* codes;        // group layout
  const uint32_t* slot_rows;
  const uint32_t* own_off;
  const uint32_t* own_cnt;
  const uint32_t* ref_ptr;
  const int32_t* ref_owner;
  const uint32_t* ref_start;
  const uint32_t* ref_cnt;
  const float* cbT;            // codebook transposed [16][dsub][M]
  int d, M, M_pad, dsub, shard_id, nshards;
  const float* queries;
  int64_t nq;
  const int32_t* probes;
  int nprobe, npp2, bigK, cap, hbits;
  uint64_t* out_keys;
  int64_t* dco;
  unsigned long long* dco_total;
  uint8_t* lut_q;
  float* lut_a;
  float* lut_b;
  int sorted_out;
  unsigned* ctr;               // [2]: query claims, warps finished (self-resetting)
  unsigned total_warps;
  // per-warp shared memory carve-up (bytes)
  int o_lut, o_cand, o_hist, o_ps, o_pre, o_r0, o_rs, o_rc, o_rg, warp_bytes;
  int cb_smem;                 // fs_lut_kernel: bytes of the per-CTA codebook copy (0: global)
  const uint4* luts;           // [nq][M_pad] quantised LUT rows (fs_lut_kernel)
  int pstride;                 // probes row stride (>= nprobe: a prefix of each probe list)
  const uint32_t* qlist;       // optional: scan only queries qlist[0 .. *qcount)
  const uint32_t* qcount;
  // threshold mode (list-major fused path): with nprobe = 1 the scanned items
  // are the members of the query's nearest list, a subset of U(q), so their
  // bigK-th smallest score bounds the query's bigK-th from above; written to
  // tau_out[q] (0xFFFFFFFF if the list has fewer than bigK items), no keys
  uint32_t* tau_out;
  // deferred finish: the scan kernel leaves each query's buffer (cap entries,
  // n | exact << 31 in defer_n) to fs_finish_kernel, a separate high-occupancy
  // pass, instead of selecting in place
  uint64_t* defer_buf;
  uint32_t* defer_n;
  // paper-literal SEIL layout (seil_paper.cu): paper = 1 -> codes / slot_rows
  // are that layout's and the work list follows Alg. 5
  int paper;
  const uint32_t* p_off;
  const uint32_t* p_shared;
  const uint32_t* p_misc;
  const uint32_t* p_other;
  const uint32_t* p_ref_start;
  const uint32_t* p_ref_cnt;
  int o_rl;                    // warp smem: misc list of each range (paper)
  const uint32_t* order;       // claim order of the queries (heavy first) or null
  int parts;                   // work items per query (small batches: the query's group
                               // tasks split into `parts` equal intervals, one warp each)
  const uint32_t* list_items;  // N_l for the cost estimate (or own_cnt)
  uint64_t cost_thr;           // a query is heavy when cost * nlist > cost_thr
  int nlist;
  int dbg;                     // timing experiments only (RAIRS_FS_DBG bits): 1 no rounds, 2 no LUT, 4 no finish
};

// ---- warp helpers -------------------------------------------------------------
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// smallest bin b of a 256-bin histogram with cumulative count >= K (K >= 1,
// total >= K); *below = the count of the bins before b
__device__ __forceinline__ uint32_t fs_bsel256(const uint32_t* hist, uint32_t K, uint32_t* below) {
  const int lane = lane_id();
  const uint4 h0 = reinterpret_cast<const uint4*>(hist)[lane * 2];  // hist is 16-B aligned
  const uint4 h1 = reinterpret_cast<const uint4*>(hist)[lane * 2 + 1];
  const uint32_t h[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
  const uint32_t loc = (h0.x + h0.y) + (h0.z + h0.w) + (h1.x + h1.y) + (h1.z + h1.w);
  const uint32_t inc = warp_incl_scan(loc);
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

// The K-th smallest SCORE (high 32 bits) among the entries of cand[0..n) whose
// score lies in [lo, lo + 2^w) (K <= their count): radix select over 8-bit
// digits.  *below_out = #entries in [lo, s*).  hist = 256 words of scratch.
__device__ __noinline__ uint32_t fs_kth_score(const uint64_t* cand, uint32_t n, uint32_t K, uint32_t lo,
                                              int w, uint32_t* hist, uint32_t* below_out) {
  const int lane = lane_id();
  uint32_t below = 0, need = K;
  for (;;) {
    const int sh = w > 8 ? w - 8 : 0;
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    const uint32_t span = 1u << w;
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t s = (uint32_t)(cand[i] >> 32);
      if (s >= lo && s - lo < span) atomicAdd(&hist[(s - lo) >> sh], 1u);
    }
    __syncwarp();
    uint32_t bl;
    const uint32_t b = fs_bsel256(hist, need, &bl);
    __syncwarp();
    below += bl;
    need -= bl;
    lo += b << sh;
    if (sh == 0) break;
    w = sh;
  }
  *below_out = below;
  return lo;
}

// stable in-place compaction of cand[0..n) to the entries with score <= smax
__device__ __noinline__ uint32_t fs_keep_le(uint64_t* cand, uint32_t n, uint32_t smax) {
  const int lane = lane_id();
  uint32_t out = 0;
  for (uint32_t i0 = 0; i0 < n; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint64_t v = i < n ? cand[i] : kKeyInf;
    const bool k = i < n && (uint32_t)(v >> 32) <= smax;
    const unsigned bal = __ballot_sync(0xffffffffu, k);
    __syncwarp();
    if (k) cand[out + __popc(bal & ((1u << lane) - 1u))] = v;
    out += __popc(bal);
  }
  __syncwarp();
  return out;
}

__device__ __noinline__ void fs_sort_u64(uint64_t* a, int n) {  // warp bitonic, n power of two
  const int lane = lane_id();
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (n >> 1); i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const uint64_t x = a[lo], y = a[hi];
        if ((x > y) == asc) { a[lo] = y; a[hi] = x; }
      }
      __syncwarp();
    }
  }
}

__device__ void fs_sort_i32(int32_t* a, int n) {
  const int lane = lane_id();
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (n >> 1); i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const int32_t x = a[lo], y = a[hi];
        if ((x > y) == asc) { a[lo] = y; a[hi] = x; }
      }
      __syncwarp();
    }
  }
}

// pre-keys (s << 32 | slot) of cand[i0..n) -> keys (s << 32 | global id)
__device__ __noinline__ void fs_resolve(const FsArgs& a, uint64_t* cand, uint32_t i0, uint32_t n) {
  const int lane = lane_id();
  for (uint32_t b = i0; b < n; b += 128) {  // four independent loads in flight per lane
    uint64_t v[4];
    uint32_t row[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = b + u * 32 + lane;
      v[u] = i < n ? cand[i] : 0ull;
      row[u] = i < n ? __ldg(a.slot_rows + (uint32_t)v[u]) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = b + u * 32 + lane;
      if (i < n)
        cand[i] = (v[u] & 0xFFFFFFFF00000000ull) |
                  (uint64_t)(row[u] * (uint32_t)a.nshards + (uint32_t)a.shard_id);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ bool fs_in_sorted(const int32_t* Ps, int npp2, int32_t x) {
  int lo = 0;  // largest index with Ps[idx] <= x, by a power-of-two descent
  for (int step = npp2 >> 1; step > 0; step >>= 1)
    if (Ps[lo + step] <= x) lo += step;
  return Ps[lo] == x;
}

// The lane task of a scan round: one 8-item group of a range of the batch.
struct FsTask {
  const uint8_t* gp;   // the group's 16-B column at m4 = 0 (a valid dummy when idle)
  uint32_t gi;         // group index (slot / 8)
  uint32_t vmask;      // items of the group inside the range (0 when idle)
  uint32_t ml;         // paper layout: the list whose misc area holds the group, else ~0
};

__device__ __forceinline__ FsTask fs_task(uint32_t t, uint32_t ng_tot, uint32_t nr, const uint32_t* rs,
                                          const uint32_t* rc, const uint32_t* rg, const uint8_t* codes,
                                          uint64_t blk_bytes) {
  FsTask k{codes, 0u, 0u, 0xFFFFFFFFu};
  if (t < ng_tot) {
    uint32_t lo = 0, hi = nr;  // largest r with rg[r] <= t
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (rg[mid] <= t) lo = mid; else hi = mid;
    }
    const uint32_t st = rs[lo], en = st + rc[lo];
    const uint32_t gi = (st >> 3) + (t - rg[lo]);
    const uint32_t g0 = gi * 8u;
    const uint32_t a0 = st > g0 ? st - g0 : 0u;
    const uint32_t a1 = min(en - g0, 8u);
    k.vmask = ((1u << a1) - 1u) & ~((1u << a0) - 1u);
    k.gi = gi;
    k.gp = codes + (uint64_t)(gi >> 2) * blk_bytes + (gi & 3) * 16;
  }
  return k;
}

// The lane tasks of one round (tasks t0 .. t0+31) without a per-lane search:
// r_lo = the range holding task t0; lane j looks at the start of range
// r_lo + 1 + j, the boundaries that fall inside the round are OR-reduced into
// a 32-bit mask, and lane L's range is r_lo + (boundaries at positions <= L).
// On return r_lo holds the range of task t0 + 32 (the next round's).
__device__ __forceinline__ FsTask fs_round_task(uint32_t t0, uint32_t& r_lo, uint32_t ng_tot, uint32_t nr,
                                                const uint32_t* rs, const uint32_t* rc, const uint32_t* rg,
                                                const uint32_t* rl, const uint8_t* codes, uint64_t blk_bytes) {
  const int lane = lane_id();
  uint32_t r, adv;
  const uint32_t e = r_lo + 1 <= nr ? rg[r_lo + 1] : 0xFFFFFFFFu;  // end of range r_lo
  if (e >= t0 + 32u) {  // the whole round inside range r_lo (warp-uniform)
    r = r_lo;
    adv = e == t0 + 32u ? 1u : 0u;
  } else {
    // lane j inspects range r_lo + 1 + j: the ranges that can start at
    // positions 1 .. 32 of the round (every range holds >= 1 task), so a range
    // starting right after 31 one-task ranges (position 32) is seen too and
    // r_lo keeps holding the next round's first task
    const uint32_t j = r_lo + 1u + (uint32_t)lane;
    uint32_t bit = 0, at32 = 0;
    if (j < nr) {
      const uint32_t d = rg[j] - t0;  // >= 1: range r_lo holds t0
      if (d < 32) bit = 1u << d;
      at32 = d == 32 ? 1u : 0u;
    }
    const uint32_t bits = __reduce_or_sync(0xffffffffu, bit);
    r = r_lo + __popc(bits & (0xFFFFFFFFu >> (31 - lane)));
    adv = __popc(bits) + (__ballot_sync(0xffffffffu, at32 != 0) ? 1u : 0u);
  }
  FsTask k{codes, 0u, 0u, 0xFFFFFFFFu};
  const uint32_t t = t0 + (uint32_t)lane;
  if (t < ng_tot) {
    const uint32_t st = rs[r], en = st + rc[r];
    if (rl) k.ml = rl[r];
    const uint32_t gi = (st >> 3) + (t - rg[r]);
    const uint32_t g0 = gi * 8u;
    const uint32_t a0 = st > g0 ? st - g0 : 0u;
    const uint32_t a1 = min(en - g0, 8u);
    k.vmask = ((1u << a1) - 1u) & ~((1u << a0) - 1u);
    k.gi = gi;
    k.gp = codes + (uint64_t)(gi >> 2) * blk_bytes + (gi & 3) * 16;
  }
  r_lo += adv;
  return k;
}

// the final top-bigK of one query's buffer (cold: one copy, not inlined)
__device__ __noinline__ uint32_t fs_finish(const FsArgs& a, uint64_t* cand, uint32_t* hist, uint32_t n,
                                           bool exact, int hsh, uint32_t cap) {
  const int lane = lane_id();
  const unsigned below_me = (1u << lane) - 1u;
  const uint32_t bigK = (uint32_t)a.bigK;
  uint32_t keep = n;
  if (exact) {
    for (uint32_t i = n + lane; i < cap; i += 32) cand[i] = kKeyInf;
    __syncwarp();
    fs_sort_u64(cand, (int)cap);
    return min(n, bigK);
  }
  if (n <= bigK) {
    fs_resolve(a, cand, 0, n);
    keep = n;
  } else {
    // level 1 from the incremental histogram (exact counts of the buffered
    // entries for every bin up to the threshold bin), then the score inside it
    uint32_t below1, below2;
    const uint32_t b1 = fs_bsel256(hist, bigK, &below1);
    __syncwarp();
    const uint32_t s_star = fs_kth_score(cand, n, bigK - below1, b1 << hsh, hsh, hist, &below2);
    const uint32_t below = below1 + below2;
    n = fs_keep_le(cand, n, s_star);  // the `below` keys with s < s*, and the ties at s*
    fs_resolve(a, cand, 0, n);
    const uint32_t need = bigK - below, nt = n - below;
    keep = bigK;
    if (nt > need) {  // rank the ties at s* by id (R5)
      if (nt <= 128) {
        uint64_t* tie = reinterpret_cast<uint64_t*>(hist);  // 128 keys of scratch
        uint32_t nk = 0, ntt = 0;
        for (uint32_t i0 = 0; i0 < n; i0 += 32) {  // stable partition: s < s* first
          const uint32_t i = i0 + lane;
          const uint64_t v = i < n ? cand[i] : kKeyInf;
          const bool lt = i < n && (uint32_t)(v >> 32) < s_star;
          const bool eq = i < n && !lt;
          const unsigned bl = __ballot_sync(0xffffffffu, lt), be = __ballot_sync(0xffffffffu, eq);
          __syncwarp();
          if (lt) cand[nk + __popc(bl & below_me)] = v;
          if (eq) tie[ntt + __popc(be & below_me)] = v;
          nk += __popc(bl);
          ntt += __popc(be);
        }
        __syncwarp();
        if (nt <= 32) {  // rank by counting (keys are unique)
          const uint64_t v = (uint32_t)lane < nt ? tie[lane] : kKeyInf;
          uint32_t rank = 0;
          for (uint32_t j = 0; j < nt; ++j) rank += tie[j] < v ? 1u : 0u;
          __syncwarp();
          if ((uint32_t)lane < nt && rank < need) cand[below + rank] = v;
        } else {
          for (uint32_t j = nt + lane; j < 128; j += 32) tie[j] = kKeyInf;
          __syncwarp();
          fs_sort_u64(tie, 128);
          for (uint32_t j = lane; j < need; j += 32) cand[below + j] = tie[j];
        }
      } else {  // many ties: sort the whole (resolved) buffer
        for (uint32_t i = n + lane; i < cap; i += 32) cand[i] = kKeyInf;
        __syncwarp();
        fs_sort_u64(cand, (int)cap);
      }
    }
  }
  __syncwarp();
  if (a.sorted_out && keep > 1) {
    int p2 = 1;
    while (p2 < (int)keep) p2 <<= 1;
    for (uint32_t i = keep + lane; i < (uint32_t)p2; i += 32) cand[i] = kKeyInf;
    __syncwarp();
    fs_sort_u64(cand, p2);
  }
  return keep;
}

// A full buffer: drop the entries above the bin threshold; if still too full,
// cut at the exact bigK-th score (ties kept, histogram rebuilt); if even that
// leaves too many (massive ties), switch to exact mode: resolved keys, sorted,
// cut to bigK.  Cold path.
struct FsSel {
  uint32_t n;        // buffered entries
  uint32_t bthr;     // items whose bin (s >> hsh) exceeds bthr cannot be in the top-bigK
  uint32_t tau;      // ... nor items with s > tau
  uint32_t hcount;   // entries counted in hist (appended so far, minus those dropped)
  uint32_t exact;    // massive-tie mode: the buffer holds resolved keys
  uint32_t hlast;    // hcount at the last bin-threshold refresh
  uint64_t tau_key;  // exact mode: keys >= tau_key are dropped
};

__device__ __noinline__ FsSel fs_compact(const FsArgs& a, uint64_t* cand, uint32_t* hist, int hsh,
                                         FsSel st, uint32_t round) {
  const int lane = lane_id();
  const uint32_t bigK = (uint32_t)a.bigK, cap = (uint32_t)a.cap;
  if (!st.exact) {
    // (1) drop bins above bthr
    uint32_t out = 0;
    for (uint32_t i0 = 0; i0 < st.n; i0 += 32) {
      const uint32_t i = i0 + lane;
      const uint64_t v = i < st.n ? cand[i] : kKeyInf;
      const uint32_t s = (uint32_t)(v >> 32);
      const bool k = i < st.n && (s >> hsh) <= st.bthr && s <= st.tau;
      const unsigned bal = __ballot_sync(0xffffffffu, k);
      __syncwarp();
      if (k) cand[out + __popc(bal & ((1u << lane) - 1u))] = v;
      out += __popc(bal);
    }
    __syncwarp();
    st.n = out;
    if (st.n + round <= cap) return st;
    // (2) exact bigK-th score, ties kept; rebuild the histogram
    uint32_t below;
    const uint32_t s_star = fs_kth_score(cand, st.n, bigK, 0u, a.hbits, hist, &below);
    st.n = fs_keep_le(cand, st.n, s_star);
    st.tau = s_star;
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    for (uint32_t i = lane; i < st.n; i += 32) atomicAdd(&hist[(uint32_t)(cand[i] >> 32) >> hsh], 1u);
    __syncwarp();
    st.hcount = st.n;
    st.hlast = 0u;
    if (st.n + round <= cap) return st;
    fs_resolve(a, cand, 0, st.n);
    st.exact = 1;
  }
  for (uint32_t i = st.n + lane; i < cap; i += 32) cand[i] = kKeyInf;
  __syncwarp();
  fs_sort_u64(cand, (int)cap);
  st.n = bigK;
  st.tau_key = cand[bigK - 1];
  st.tau = (uint32_t)(st.tau_key >> 32);
  return st;
}

// lane's 8 scores -> pass mask: valid items that can still be in the top-bigK
// (s <= lim = min(tau, the largest score of bin bthr))
__device__ __forceinline__ uint32_t fs_pass(const uint32_t (&acc)[8], uint32_t vmask, uint32_t lim) {
  uint32_t pm = 0;
#pragma unroll
  for (int v = 0; v < 8; ++v) pm |= (acc[v] <= lim ? 1u : 0u) << v;
  return pm & vmask;
}

// Paper layout, misc area of list ml (RemoveVectorIfVisited, Alg. 5 line 16):
// an item whose embedded other list was visited before ml -- probed with a
// smaller id (ascending visit order, reading R9) -- was scored there; drop it.
__device__ __forceinline__ uint32_t fs_paper_drop(const FsArgs& a, uint32_t pm, uint32_t gi, uint32_t ml,
                                                  const int32_t* Ps) {
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    if ((pm >> v) & 1u) {
      const uint32_t o = __ldg(a.p_other + gi * 8u + v);
      if (o < ml && fs_in_sorted(Ps, a.npp2, (int32_t)o)) pm &= ~(1u << v);
    }
  }
  return pm;
}

// exact (massive-tie) mode: drop the items whose resolved key is >= tau_key
__device__ __forceinline__ uint32_t fs_pass_exact(const FsArgs& a, const uint32_t (&accp)[8], uint32_t pm,
                                                  uint32_t gi, uint64_t tau_key) {
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    if ((pm >> v) & 1u) {
      const uint32_t row = __ldg(a.slot_rows + gi * 8u + v);
      const uint64_t key = ((uint64_t)accp[v] << 32) |
                           (uint64_t)(row * (uint32_t)a.nshards + (uint32_t)a.shard_id);
      if (key >= tau_key) pm &= ~(1u << v);
    }
  }
  return pm;
}

__device__ __forceinline__ void fs_put(const FsArgs& a, uint64_t* cand, uint32_t* hist, int hsh,
                                       const uint32_t (&acc)[8], uint32_t pm, uint32_t gi, bool exact,
                                       uint32_t& pos) {
  if (!exact) {  // warp-uniform; predicated stores, no branches
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const bool on = (pm >> v) & 1u;
      if (on) {
        atomicAdd(&hist[acc[v] >> hsh], 1u);
        cand[pos] = ((uint64_t)acc[v] << 32) | (uint64_t)(gi * 8u + v);
      }
      pos += on ? 1u : 0u;
    }
  } else {
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      if ((pm >> v) & 1u) {
        const uint32_t row = __ldg(a.slot_rows + gi * 8u + v);
        cand[pos++] = ((uint64_t)acc[v] << 32) |
                      (uint64_t)(row * (uint32_t)a.nshards + (uint32_t)a.shard_id);
      }
    }
  }
}

// exclusive prefix and total over the warp of a per-lane count c < 16 (four
// ballots instead of a shuffle chain)
__device__ __forceinline__ uint32_t fs_prefix16(uint32_t c, unsigned below_me, uint32_t& tot) {
  uint32_t pre = 0, t = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const unsigned m = __ballot_sync(0xffffffffu, (c >> b) & 1u);
    pre += (uint32_t)__popc(m & below_me) << b;
    t += (uint32_t)__popc(m) << b;
  }
  tot = t;
  return pre;
}

// The deferred exact top-bigK: one warp per query over the buffer the scan
// left (pre-keys with an s <= bin-threshold filter, or resolved keys in
// massive-tie mode): histogram of its scores, then fs_finish (exact bigK-th
// score, ids, ties by id).  Runs at high occupancy, apart from the lookups.
constexpr int FF_WARPS = 8;
constexpr uint32_t FF_CAPS = 512;  // shared-memory entries per warp (a buffer of up to `cap`
                                   // is cut to its bin threshold first; more: in global memory)
__global__ void __launch_bounds__(FF_WARPS * 32) fs_finish_kernel(const __grid_constant__ FsArgs a) {
  extern __shared__ __align__(16) uint8_t ff_smem[];
  const int lane = lane_id(), warp = warp_id();
  const unsigned below_me = (1u << lane) - 1u;
  const uint32_t cap = (uint32_t)a.cap, bigK = (uint32_t)a.bigK;
  const uint32_t caps = min(cap, FF_CAPS);
  uint64_t* cand = reinterpret_cast<uint64_t*>(ff_smem + (size_t)warp * (caps * 8 + 1024));
  uint32_t* hist = reinterpret_cast<uint32_t*>(cand + caps);
  const int hsh = a.hbits > 8 ? a.hbits - 8 : 0;
  pdl_wait();  // the scan kernel's buffers
  const int nw = blockDim.x >> 5;
  for (int64_t q = (int64_t)blockIdx.x * nw + warp; q < a.nq; q += (int64_t)gridDim.x * nw) {
    const uint32_t nx = a.defer_n[q];
    const uint32_t n = nx & 0x7FFFFFFFu;
    const bool exact = (nx >> 31) != 0;
    uint64_t* src = a.defer_buf + (size_t)q * cap;
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    uint64_t* buf = cand;  // where fs_finish works: shared memory, or the global buffer itself
    uint32_t m = n, bcap = caps;
    if (exact) {
      if (n <= caps) {
        for (uint32_t i = lane; i < n; i += 32) cand[i] = src[i];
      } else {
        buf = src;
        bcap = cap;
      }
    } else if (n <= caps) {
      // one pass (four 8-B loads in flight per lane): copy into shared memory
      // and histogram
      for (uint32_t i0 = 0; i0 < n; i0 += 128) {
        uint64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t i = i0 + 32u * u + lane;
          v[u] = i < n ? src[i] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t i = i0 + 32u * u + lane;
          if (i < n) {
            cand[i] = v[u];
            atomicAdd(&hist[(uint32_t)(v[u] >> 32) >> hsh], 1u);
          }
        }
      }
    } else {
      for (uint32_t i = lane; i < n; i += 32) atomicAdd(&hist[(uint32_t)(src[i] >> 32) >> hsh], 1u);
      __syncwarp();
      {
        // keep the entries whose bin is at most the bin of the bigK-th score
        uint32_t bl;
        const uint32_t bs = fs_bsel256(hist, bigK, &bl);
        uint32_t cnt = 0;
        for (uint32_t i = lane; i < n; i += 32) cnt += ((uint32_t)(src[i] >> 32) >> hsh) <= bs ? 1u : 0u;
        m = __reduce_add_sync(0xffffffffu, cnt);
        uint64_t* dst = cand;
        if (m > caps) {  // rare (a wide bin): compact in place in the global buffer
          dst = src;
          bcap = cap;
        }
        uint32_t out = 0;
        for (uint32_t i0 = 0; i0 < n; i0 += 32) {
          const uint32_t i = i0 + lane;
          const uint64_t v = i < n ? src[i] : kKeyInf;
          const bool k = i < n && ((uint32_t)(v >> 32) >> hsh) <= bs;
          const unsigned bal = __ballot_sync(0xffffffffu, k);
          __syncwarp();
          if (k) dst[out + __popc(bal & below_me)] = v;
          out += __popc(bal);
        }
        buf = dst;
      }
    }
    __syncwarp();
    const uint32_t keep = fs_finish(a, buf, hist, m, exact, hsh, bcap);
    for (uint32_t i = lane; i < bigK; i += 32) a.out_keys[q * bigK + i] = i < keep ? buf[i] : kKeyInf;
    __syncwarp();
  }
  pdl_trigger();
}

// Claim order for the scan (longest-first, two classes): a query whose probed
// lists hold more items than the batch's mean expectation (nprobe x mean N_l)
// is put at the front, the others at the back, so the persistent warps take
// the long queries first and the tail of the grid runs short ones.  Results do
// not depend on the order (each query is independent).
__global__ void fs_order_kernel(const __grid_constant__ FsArgs a, uint32_t* order) {
  pdl_wait();  // probes
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < a.nq) {
    const int32_t* pq = a.probes + q * a.pstride;
    uint64_t cost = 0;
    for (int i = 0; i < a.nprobe; ++i) cost += __ldg(a.list_items + __ldg(pq + i));
    if (cost * (uint64_t)a.nlist > a.cost_thr) order[atomicAdd(&a.ctr[2], 1u)] = (uint32_t)q;
    else order[a.nq - 1 - atomicAdd(&a.ctr[3], 1u)] = (uint32_t)q;
  }
  pdl_trigger();
}

// Split mode: query q's P parts each left their exact top-bigK keys, sorted
// (resolved (s, id) keys: unique); one warp per query merges them -- bigK
// rounds of a warp-wide minimum over the P list heads (P <= 64: lanes hold
// the heads of parts lane and lane + 32).
__global__ void __launch_bounds__(256) fs_merge_parts_kernel(const uint64_t* __restrict__ part_keys, int P,
                                                              int bigK, int64_t nq, uint64_t* __restrict__ out_keys) {
  const int lane = lane_id();
  const int64_t q = (int64_t)blockIdx.x * 8 + warp_id();
  pdl_wait();  // the parts' finish kernel
  if (q >= nq) return;
  const uint64_t* base = part_keys + (size_t)q * P * bigK;
  int i0 = 0, i1 = 0;
  uint64_t h0 = lane < P ? base[(size_t)lane * bigK] : kKeyInf;
  uint64_t h1 = lane + 32 < P ? base[(size_t)(lane + 32) * bigK] : kKeyInf;
  for (int i = 0; i < bigK; ++i) {
    uint64_t m = h0 < h1 ? h0 : h1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t x = __shfl_xor_sync(0xffffffffu, m, o);
      m = x < m ? x : m;
    }
    if (lane == 0) out_keys[q * bigK + i] = m;
    if (m == kKeyInf) continue;
    if (h0 == m) {
      h0 = ++i0 < bigK ? base[(size_t)lane * bigK + i0] : kKeyInf;
    } else if (h1 == m) {
      h1 = ++i1 < bigK ? base[(size_t)(lane + 32) * bigK + i1] : kKeyInf;
    }
  }
  pdl_trigger();
}

// A3 for every query of the batch, one warp per query (O2: lane per
// subquantizer, fp32 RN, ascending t; see build_lut in lut_common.cuh), into luts[q][M_pad].
// Needs only the queries, so under programmatic dependent launch it overlaps
// the coarse stage; it waits for that stage (griddepcontrol.wait) only before
// it exits, so its completion implies the probes are ready for the scan.
constexpr int FL_WARPS = 8;
__global__ void __launch_bounds__(FL_WARPS * 32) fs_lut_kernel(const __grid_constant__ FsArgs a, uint4* luts) {
  extern __shared__ __align__(16) uint8_t fl_smem[];
  const int lane = lane_id(), warp = warp_id();
  float* cbs = reinterpret_cast<float*>(fl_smem);
  if (a.cb_smem) {
    for (int i = threadIdx.x; i < a.cb_smem / 4; i += blockDim.x) cbs[i] = __ldg(a.cbT + i);
    __syncthreads();
  }
  const float* cb = a.cb_smem ? cbs : a.cbT;
  const LutArgs la{a.queries, a.d, a.M, a.M_pad, a.dsub, a.cbT, luts, a.lut_q, a.lut_a, a.lut_b};
  const bool keepT = a.M * 17 <= 16 * 1024 / 4;  // [16][M] + [M] floats of scratch fit 16 KB
  float* scratch = reinterpret_cast<float*>(fl_smem + a.cb_smem) + (size_t)warp * (keepT ? 17 * a.M : a.M);
  for (int64_t q = (int64_t)blockIdx.x * FL_WARPS + warp; q < a.nq; q += (int64_t)gridDim.x * FL_WARPS) {
    build_lut(la, q, luts + q * a.M_pad, scratch, cb, keepT);
    (void)lane;
  }
  pdl_wait();     // the coarse stage's probes are complete before this grid is
  if (a.order) {  // the scan's claim order (fs_order_kernel's work, one launch fewer)
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < a.nq;
         q += (int64_t)gridDim.x * blockDim.x) {
      const int32_t* pq = a.probes + q * a.pstride;
      uint64_t cost = 0;
      for (int i = 0; i < a.nprobe; ++i) cost += __ldg(a.list_items + __ldg(pq + i));
      uint32_t* ord = const_cast<uint32_t*>(a.order);
      if (cost * (uint64_t)a.nlist > a.cost_thr) ord[atomicAdd(&a.ctr[2], 1u)] = (uint32_t)q;
      else ord[a.nq - 1 - atomicAdd(&a.ctr[3], 1u)] = (uint32_t)q;
    }
  }
  pdl_trigger();
}


// One warp per query; see the file header.  A round scores 64 groups: lane
// tasks t0 + lane and t0 + 32 + lane (two independent chains per lane, one
// LUT row load per subquantizer for both).  Each group keeps a ring of two
// 16-B code loads in flight: consuming chunk c issues chunk c + 2, which past
// the group's end is chunk 0/1 of the lane's NEXT round's group, so a round's
// DRAM latency overlaps the previous round's lookups.
template <int MINB, int GPL, int NW, bool PK, int DR = 4>
__global__ void __launch_bounds__(NW * 32, MINB) fs_scan_kernel(const __grid_constant__ FsArgs a) {
  constexpr int D = DR / GPL;                // ring slots per group
  constexpr uint32_t FS_ROUND = 256u * GPL;  // items appended per round at most
  const int dbg = kFsTiming ? a.dbg : 0;
  extern __shared__ __align__(16) uint8_t fs_smem[];
  const int lane = lane_id(), warp = warp_id();
  uint8_t* wb = fs_smem + (size_t)warp * a.warp_bytes;
  uint4* lut = reinterpret_cast<uint4*>(wb + a.o_lut);
  uint64_t* cand = reinterpret_cast<uint64_t*>(wb + a.o_cand);
  uint32_t* hist = reinterpret_cast<uint32_t*>(wb + a.o_hist);
  int32_t* Ps = reinterpret_cast<int32_t*>(wb + a.o_ps);
  uint32_t* pre = reinterpret_cast<uint32_t*>(wb + a.o_pre);
  uint32_t* r0s = reinterpret_cast<uint32_t*>(wb + a.o_r0);
  uint32_t* rs = reinterpret_cast<uint32_t*>(wb + a.o_rs);
  uint32_t* rc = reinterpret_cast<uint32_t*>(wb + a.o_rc);
  uint32_t* rg = reinterpret_cast<uint32_t*>(wb + a.o_rg);
  uint32_t* rlp = a.paper ? reinterpret_cast<uint32_t*>(wb + a.o_rl) : nullptr;
  const int M4 = a.M_pad / 4;  // a multiple of 4 (M_pad % 16 == 0)
  const uint64_t blk_bytes = 16ull * (uint64_t)a.M_pad;
  const int np = a.nprobe;
  const uint32_t cap = (uint32_t)a.cap, bigK = (uint32_t)a.bigK;
  const int hsh = a.hbits > 8 ? a.hbits - 8 : 0;  // 256 score bins
  const unsigned below_me = (1u << lane) - 1u;
  pdl_wait();  // probes of the coarse stage

  for (;;) {
    uint32_t qq = 0;
    if (lane == 0) qq = atomicAdd(&a.ctr[0], 1u);
    qq = __shfl_sync(0xffffffffu, qq, 0);
    // a query subset (a.qlist / *a.qcount: the list-major path's overflowed
    // queries) or every query
    const uint32_t P = (uint32_t)a.parts;
    if (a.qlist ? qq >= *a.qcount : qq >= (uint64_t)a.nq * P) break;
    const uint32_t part = P > 1 ? qq % P : 0u;
    if (P > 1) qq /= P;  // split mode: no query subset, no claim order
    const int64_t q = a.qlist ? (int64_t)a.qlist[qq] : a.order ? (int64_t)a.order[qq] : (int64_t)qq;
    const int32_t* pq = a.probes + q * a.pstride;

    // the query's LUT rows (fs_lut_kernel) into the warp's shared memory by
    // cp.async: the copy runs while the probe set and range list are built
    for (int m = lane; m < a.M_pad; m += 32)
      cp_async16((uint32_t)__cvta_generic_to_shared(lut + m), a.luts + q * a.M_pad + m);
    cp_async_commit();

    // ---- probe set: sorted copy (membership, R9) + per-probe reference prefix ----
    for (int i = lane; i < a.npp2; i += 32) Ps[i] = i < np ? __ldg(pq + i) : INT_MAX;
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    if (a.npp2 > 1) fs_sort_i32(Ps, a.npp2);
    uint32_t nrefs = 0;
    for (int i0 = 0; i0 < np; i0 += 32) {
      const int i = i0 + lane;
      uint32_t nr = 0, r0 = 0;
      if (i < np) {
        const int l = __ldg(pq + i);
        r0 = __ldg(a.ref_ptr + l);
        nr = __ldg(a.ref_ptr + l + 1) - r0;
      }
      const uint32_t inc = warp_incl_scan(nr);
      if (i < np) { pre[i] = nrefs + inc - nr; r0s[i] = r0; }
      nrefs += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) pre[np] = nrefs;

    // ---- A3: LUT + uint8 quantisation (O2); T / mn scratch in the candidate buffer ----
    cp_async_wait0();  // the LUT rows (issued at the query's start)
    __syncwarp();

    // ---- A4 + A5 + A6 ----
    FsSel st{0u, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u, 0u, kKeyInf};
    uint32_t my_dco = 0;
    // sources: np owned ranges (paper layout: np shared-block ranges, then np
    // misc areas), then the probed lists' references
    const uint32_t npb = a.paper ? 2u * (uint32_t)np : (uint32_t)np;
    const uint32_t nsrc = npb + nrefs;
    // the slot range of source s (empty when it does not exist or R9 skips it)
    auto source = [&](uint32_t s, uint32_t& st0, uint32_t& cnt, uint32_t& ml) {
        st0 = 0;
        cnt = 0;
        ml = 0xFFFFFFFFu;
        if (s < npb) {
          const bool misc = s >= (uint32_t)np;  // paper layout only
          const int l = __ldg(pq + (misc ? s - (uint32_t)np : s));
          if (!a.paper) {
            st0 = __ldg(a.own_off + l);
            cnt = __ldg(a.own_cnt + l);
          } else if (!misc) {
            st0 = __ldg(a.p_off + l);
            cnt = __ldg(a.p_shared + l);
          } else {
            st0 = __ldg(a.p_off + l) + __ldg(a.p_shared + l);
            cnt = __ldg(a.p_misc + l);
            ml = (uint32_t)l;
          }
        } else if (s < nsrc) {
          const uint32_t e = s - npb;
          int lo = 0, hi = np;  // probe of reference e: largest i with pre[i] <= e
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pre[mid] <= e) lo = mid; else hi = mid;
          }
          const uint32_t j = r0s[lo] + (e - pre[lo]);
          const int32_t o = __ldg(a.ref_owner + j);
          if (!fs_in_sorted(Ps, a.npp2, o)) {  // R9: owner not probed -> scan the cell here
            st0 = __ldg((a.paper ? a.p_ref_start : a.ref_start) + j);
            cnt = __ldg((a.paper ? a.p_ref_cnt : a.ref_cnt) + j);
          }
        }
    };
    // split mode: the query's total group tasks G (this part takes
    // [part G / P, (part + 1) G / P)) and items (part 0 reports the DCO)
    uint64_t g_lo = 0, g_hi = ~0ull;
    if (P > 1) {
      uint64_t G = 0, I = 0;
      for (uint32_t sb = 0; sb < nsrc; sb += 32) {
        uint32_t st0, cnt, ml;
        source(sb + lane, st0, cnt, ml);
        const uint32_t g = cnt ? ((st0 + cnt - 1) >> 3) - (st0 >> 3) + 1 : 0u;
        G += __reduce_add_sync(0xffffffffu, g);
        I += __reduce_add_sync(0xffffffffu, cnt);
      }
      g_lo = (uint64_t)part * G / P;
      g_hi = (uint64_t)(part + 1) * G / P;
      if (part == 0 && lane == 0) my_dco = (uint32_t)I;  // summed over lanes below
    }
    uint64_t g_base = 0;  // global task index of the batch's first task
    uint32_t s0 = 0;
    for (;;) {
      // (1) a batch of ranges: s < np -> owned range of probe s; else reference s - np
      uint32_t nr = 0;
      while (s0 < nsrc && nr <= FS_RCAP - 32) {
        const uint32_t s = s0 + lane;
        uint32_t st0, cnt, ml;
        source(s, st0, cnt, ml);
        const bool has = cnt > 0;
        const unsigned bal = __ballot_sync(0xffffffffu, has);
        if (has) {
          const uint32_t p = nr + __popc(bal & below_me);
          rs[p] = st0;
          rc[p] = cnt;
          if (rlp) rlp[p] = ml;
        }
        nr += __popc(bal);
        s0 += 32;
      }
      if (nr == 0) break;
      __syncwarp();
      // (2) group prefix of the batch's ranges
      uint32_t ng_tot = 0;
      for (uint32_t r0 = 0; r0 < nr; r0 += 32) {
        const uint32_t r = r0 + lane;
        uint32_t g = 0;
        if (r < nr) {
          const uint32_t sr = rs[r], c = rc[r];
          g = ((sr + c - 1) >> 3) - (sr >> 3) + 1;
          if (P == 1) my_dco += c;
        }
        const uint32_t inc = warp_incl_scan(g);
        if (r < nr) rg[r] = ng_tot + inc - g;
        ng_tot += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) rg[nr] = ng_tot;
      __syncwarp();
      // (3) rounds of 32 * GPL groups: lane tasks t0 + 32 g + lane, g < GPL, over
      // the batch's tasks [t_beg, t_end) (split mode: this part's interval)
      uint32_t t_beg = 0, t_end = ng_tot;
      if (P > 1) {
        const uint64_t b0 = g_base, b1 = g_base + ng_tot;
        t_beg = (uint32_t)(min(max(g_lo, b0), b1) - b0);
        t_end = (uint32_t)(min(max(g_hi, b0), b1) - b0);
      }
      g_base += ng_tot;
      if (t_beg >= t_end) {
        __syncwarp();
        continue;
      }
      uint32_t r_lo = 0;  // range holding the first task of the next round to map
      if (t_beg > 0) {    // the range holding t_beg: ranges with rg[r] <= t_beg, minus one
        uint32_t c = 0;
        for (uint32_t r = lane; r < nr; r += 32) c += rg[r] <= t_beg ? 1u : 0u;
        r_lo = __reduce_add_sync(0xffffffffu, c) - 1u;
      }
      FsTask A[GPL];
#pragma unroll
      for (int g = 0; g < GPL; ++g) A[g] = fs_round_task(t_beg + 32u * g, r_lo, t_end, nr, rs, rc, rg, rlp, a.codes, blk_bytes);
      // per group a ring of D loop-carried chunk slots (chunk c in slot c % D),
      // each refilled right after it is consumed with the chunk D ahead (past
      // the group's end: chunk c % D of the lane's next-round group), so the
      // ring holds GPL * D = 4 16-B loads in flight and no register copies.
      // (A cp.async shared-memory ring measured 2x slower.)
      uint4 R[GPL][D];
#pragma unroll
      for (int g = 0; g < GPL; ++g)
#pragma unroll
        for (int s = 0; s < D; ++s) R[g][s] = ldg_nc_v4(A[g].gp + s * 64);
      for (uint32_t t0 = t_beg; t0 < ((dbg & 1) ? 0u : t_end); t0 += 32u * GPL) {
        FsTask nA[GPL];
#pragma unroll
        for (int g = 0; g < GPL; ++g)
          nA[g] = fs_round_task(t0 + 32u * (GPL + g), r_lo, t_end, nr, rs, rc, rg, rlp, a.codes, blk_bytes);
        uint32_t acc[GPL][8];
        uint32_t accp[GPL][4];
#pragma unroll
        for (int g = 0; g < GPL; ++g) {
#pragma unroll
          for (int v = 0; v < 8; ++v) acc[g][v] = 0u;
#pragma unroll
          for (int v = 0; v < 4; ++v) accp[g][v] = 0u;
        }
        // one iteration: chunks c .. c+D-1 consumed, each slot refilled from
        // `nxt` (chunk c+D+s of this group, or chunk s of the next round's)
        auto iter = [&](int c, const uint8_t* const (&nxt)[GPL]) {
          const uint4* L = lut + 4 * c;
          // the same chunks of the next round's groups into L2 (one round ahead
          // of their loads: the register ring alone covers L2 latency, not
          // DRAM's); a 128-B line holds two chunks of four groups
          if (!(dbg & 16))
#pragma unroll
            for (int g = 0; g < GPL; ++g)
#pragma unroll
              for (int s = 0; s < D; s += 2) prefetch_l2(nA[g].gp + (c + s) * 64);
#pragma unroll
          for (int s = 0; s < D; ++s) {
#pragma unroll
            for (int g = 0; g < GPL; ++g) {
              if (dbg & 32) R[g][s] = make_uint4(c, c * 3u, c * 5u, c * 7u);  // timing: no code loads
              if constexpr (PK) {
                lookup8p(L[4 * s + 0], R[g][s].x, accp[g]);
                lookup8p(L[4 * s + 1], R[g][s].y, accp[g]);
                lookup8p(L[4 * s + 2], R[g][s].z, accp[g]);
                lookup8p(L[4 * s + 3], R[g][s].w, accp[g]);
              } else {
                lookup8(L[4 * s + 0], R[g][s].x, acc[g]);
                lookup8(L[4 * s + 1], R[g][s].y, acc[g]);
                lookup8(L[4 * s + 2], R[g][s].z, acc[g]);
                lookup8(L[4 * s + 3], R[g][s].w, acc[g]);
              }
              if (!(dbg & 32)) R[g][s] = ldg_nc_v4(nxt[g] + s * 64);
            }
          }
        };
        // M4 % D == 0; the last iteration is peeled (its refills come from the
        // next round's groups), so the loop body has no address selects
#pragma unroll 1
        for (int c = 0; c < M4 - D; c += D) {
          const uint8_t* nxt[GPL];
#pragma unroll
          for (int g = 0; g < GPL; ++g) nxt[g] = A[g].gp + (c + D) * 64;
          iter(c, nxt);
        }
        {
          const uint8_t* nxt[GPL];
#pragma unroll
          for (int g = 0; g < GPL; ++g) nxt[g] = nA[g].gp;
          iter(M4 - D, nxt);
        }
        if constexpr (PK) {
#pragma unroll
          for (int g = 0; g < GPL; ++g) fs_unpack(accp[g], acc[g]);
        }
        if (dbg & 8) {  // timing experiment: no selection (scores folded into the DCO sum)
          uint32_t x = 0;
#pragma unroll
          for (int g = 0; g < GPL; ++g)
#pragma unroll
            for (int v = 0; v < 8; ++v) x += acc[g][v];
          my_dco += x & 1u;
#pragma unroll
          for (int g = 0; g < GPL; ++g) A[g] = nA[g];
          continue;
        }
        if (st.n + FS_ROUND > cap) st = fs_compact(a, cand, hist, hsh, st, FS_ROUND);
        // append (pre-key s << 32 | slot) every valid item that can be in the top-bigK
        const uint32_t lim = min(st.tau, st.bthr >= (0xFFFFFFFFu >> hsh) ? 0xFFFFFFFFu
                                                                          : ((st.bthr + 1u) << hsh) - 1u);
        // cheap first test: no score of the lane's groups (valid or not) <= lim
        uint32_t mn = acc[0][0];
#pragma unroll
        for (int g = 0; g < GPL; ++g)
#pragma unroll
          for (int v = 0; v < 8; ++v) mn = min(mn, acc[g][v]);
        if (__any_sync(0xffffffffu, mn <= lim)) {
          uint32_t pm[GPL], c = 0;
#pragma unroll
          for (int g = 0; g < GPL; ++g) {
            pm[g] = mn <= lim ? fs_pass(acc[g], A[g].vmask, lim) : 0u;
            if (pm[g] && A[g].ml != 0xFFFFFFFFu) pm[g] = fs_paper_drop(a, pm[g], A[g].gi, A[g].ml, Ps);
            if (st.exact && pm[g]) pm[g] = fs_pass_exact(a, acc[g], pm[g], A[g].gi, st.tau_key);
            c += __popc(pm[g]);
          }
          if (__any_sync(0xffffffffu, c != 0u)) {
            uint32_t tot;
            uint32_t pos = st.n;
            if constexpr (GPL == 1) {
              pos += fs_prefix16(c, below_me, tot);
            } else {
              const uint32_t inc = warp_incl_scan(c);
              tot = __shfl_sync(0xffffffffu, inc, 31);
              pos += inc - c;
            }
#pragma unroll
            for (int g = 0; g < GPL; ++g) fs_put(a, cand, hist, hsh, acc[g], pm[g], A[g].gi, st.exact, pos);
            st.n += tot;
            __syncwarp();
            if (!st.exact) {
              st.hcount += tot;
              // smallest bin whose cumulative count reaches bigK, refreshed once
              // 32 more entries are counted (a stale bin is a valid, looser cut)
              if (st.hcount >= bigK && st.hcount >= st.hlast + 32u) {
                uint32_t bl;
                st.bthr = fs_bsel256(hist, bigK, &bl);
                st.hlast = st.hcount;
              }
            }
          }
        }
#pragma unroll
        for (int g = 0; g < GPL; ++g) A[g] = nA[g];
      }
      __syncwarp();
    }

    // ---- exact top-bigK of the buffer (here, or deferred to fs_finish_kernel) ----
    if (a.defer_buf) {
      // only entries that can still be in the top-bigK (s <= the final bound;
      // resolved keys in exact mode are all kept)
      const size_t item = P > 1 ? (size_t)q * P + part : (size_t)q;
      uint64_t* dst = a.defer_buf + item * cap;
      const uint32_t lim = st.exact ? 0xFFFFFFFFu
                                    : min(st.tau, st.bthr >= (0xFFFFFFFFu >> hsh) ? 0xFFFFFFFFu
                                                                                 : ((st.bthr + 1u) << hsh) - 1u);
      uint32_t nout = 0;
      for (uint32_t i0 = 0; i0 < st.n; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint64_t v = i < st.n ? cand[i] : kKeyInf;
        const bool k = i < st.n && (uint32_t)(v >> 32) <= lim;
        const unsigned bal = __ballot_sync(0xffffffffu, k);
        if (k) dst[nout + __popc(bal & below_me)] = v;
        nout += __popc(bal);
      }
      st.n = nout;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) my_dco += __shfl_xor_sync(0xffffffffu, my_dco, o);
      if (lane == 0) {
        a.defer_n[item] = st.n | (st.exact ? 0x80000000u : 0u);
        if (a.dco && (P == 1 || part == 0)) a.dco[q] = (int64_t)my_dco;
        if (a.dco_total) atomicAdd(a.dco_total, (unsigned long long)my_dco);
      }
      __syncwarp();
      continue;
    }
    const uint32_t keep = (dbg & 4) ? 0u : fs_finish(a, cand, hist, st.n, st.exact != 0, hsh, cap);
    if (a.tau_out) {  // threshold mode: the bigK-th smallest score (an upper bound, see FsArgs)
      uint32_t mx = 0;
      for (uint32_t i = lane; i < keep; i += 32) mx = max(mx, (uint32_t)(cand[i] >> 32));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) a.tau_out[q] = keep == bigK ? mx : 0xFFFFFFFFu;
    } else {
      for (uint32_t i = lane; i < bigK; i += 32) a.out_keys[q * bigK + i] = i < keep ? cand[i] : kKeyInf;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_dco += __shfl_xor_sync(0xffffffffu, my_dco, o);
    if (lane == 0) {
      if (a.dco) a.dco[q] = (int64_t)my_dco;
      if (a.dco_total) atomicAdd(a.dco_total, (unsigned long long)my_dco);
    }
    __syncwarp();
  }
  // the last warp out resets the claim counters for the next launch on this slot
  if (lane == 0) {
    const unsigned done = atomicAdd(&a.ctr[1], 1u);
    if (done == a.total_warps - 1) {
      atomicExch(&a.ctr[0], 0u);
      atomicExch(&a.ctr[1], 0u);
      atomicExch(&a.ctr[2], 0u);
      atomicExch(&a.ctr[3], 0u);
    }
  }
}

// ---------------------------------------------------------------------------
// group layout from the cell-major layout (thread per (group, m4))
__global__ void fs_regroup_kernel(const uint64_t* __restrict__ codes64, int64_t n_groups, int NU,
                                  int M4, uint8_t* __restrict__ codes_g) {
  const int64_t total = n_groups * M4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = e / M4;
    const int m4 = (int)(e - gi * M4);
    uint32_t wd[4] = {0u, 0u, 0u, 0u};
    for (int v = 0; v < 8; ++v) {
      const int64_t slot = gi * 8 + v;
      const uint64_t w = codes64[((slot >> 5) * NU + (m4 >> 2)) * 32 + (slot & 31)];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int m = 4 * m4 + k;  // nibble (m & 15) of unit m >> 4
        wd[k] |= (uint32_t)((w >> (4 * (m & 15))) & 0xFu) << (4 * v);
      }
    }
    const int64_t blk = gi >> 2;
    uint4* dst = reinterpret_cast<uint4*>(codes_g + blk * (int64_t)(16 * 4 * M4) + (int64_t)m4 * 64 +
                                          (gi & 3) * 16);
    *dst = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  }
}

__global__ void fs_transpose_cb_kernel(const float* __restrict__ cb, int M, int dsub,
                                       float* __restrict__ cbT) {
  const int total = M * 16 * dsub;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int m = e / (16 * dsub), j = (e / dsub) % 16, t = e % dsub;
    cbT[((size_t)j * dsub + t) * M + m] = cb[e];
  }
}

rairs_status fastscan_prepare(rairs_index_s* idx, cudaStream_t s) {
  cudaFree(idx->codes_g);
  idx->codes_g = nullptr;
  idx->device_bytes -= idx->fs_bytes;
  idx->fs_bytes = 0;
  const int64_t slots = std::max<int64_t>(idx->n_slots, 32);
  const size_t bytes = (size_t)slots * idx->M_pad / 2;
  RAIRS_CUDA_TRY(cudaMalloc(&idx->codes_g, bytes));
  const int M4 = idx->M_pad / 4;
  const int64_t groups = slots / 8;
  const int64_t total = groups * M4;
  fs_regroup_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 32), 256, 0, s>>>(
      reinterpret_cast<const uint64_t*>(idx->codes), groups, idx->M_pad / 16, M4, idx->codes_g);
  RAIRS_CHECK_LAUNCH();
  if (!idx->cbT) {
    RAIRS_CUDA_TRY(cudaMalloc(&idx->cbT, (size_t)idx->M * 16 * idx->dsub * 4));
    fs_transpose_cb_kernel<<<(unsigned)ceil_div(idx->M * 16 * idx->dsub, 256), 256, 0, s>>>(
        idx->codebook, idx->M, idx->dsub, idx->cbT);
    RAIRS_CHECK_LAUNCH();
    RAIRS_CUDA_TRY(cudaMalloc(&idx->fs_ctr, FS_SLOTS * 4 * sizeof(unsigned)));
    RAIRS_CUDA_TRY(cudaMemsetAsync(idx->fs_ctr, 0, FS_SLOTS * 4 * sizeof(unsigned), s));
    idx->device_bytes += (size_t)idx->M * 16 * idx->dsub * 4 + FS_SLOTS * 16;
  }
  idx->fs_bytes = bytes;
  idx->device_bytes += bytes;
  return RAIRS_OK;
}

// ---------------------------------------------------------------------------
// experiment switch (RAIRS_FS_VARIANT): 0 = one group per lane per round,
// 2 CTAs/SM (128 registers); 1 = 3 CTAs/SM (80 registers, spills); 2 = two
// groups per lane per round (shared LUT rows; ptxas sinks the ring refills to
// the end of the iteration, so the loads stall: measured 7 % slower)
static int fs_variant() {
  static const int v = [] {
    const char* e = std::getenv("RAIRS_FS_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
static int fs_round_items() { return fs_variant() == 2 ? 512 : 256; }

// ring slots per lane: 6 when M_pad / 4 is a multiple of 6 and the sums are
// packed (c4: 6 chunks = 24 nibble words of lead per load, scan 232 -> 226 us),
// else 4 (RAIRS_FS_RING=4 forces 4)
static int fastscan_ring() {
  static const int v = [] {
    const char* e = std::getenv("RAIRS_FS_RING");
    return e ? std::atoi(e) : 6;
  }();
  return v;
}

// packed pair sums (lookup8p, M_pad <= 128); RAIRS_FS_PACK=0: one u32 per item
static bool fastscan_pack_on() {
  static const bool on = [] {
    const char* e = std::getenv("RAIRS_FS_PACK");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}

int fastscan_cap(int bigK, int M_pad);

static int fs_hbits(int M) {
  int b = 1;
  while (((int64_t)M * 255) >> b) ++b;
  return b;
}

struct FsPlan {
  FsArgs a;
  int warps;
  size_t smem;
};

static rairs_status fs_plan(const rairs_index_s* idx, const SearchArgs& sa, const FsExtra& ex, FsPlan& pl) {
  FsArgs& p = pl.a;
  p = FsArgs{};
  p.parts = 1;
  p.codes = idx->codes_g;
  p.slot_rows = idx->slot_rows;
  if (idx->seil_layout != 0) {
    if (!idx->p_codes_g) {
      set_error("fast scan: paper SEIL layout selected but not built");
      return RAIRS_E_INTERNAL;
    }
    p.paper = 1;
    p.codes = idx->p_codes_g;
    p.slot_rows = idx->p_slot_rows;
    p.p_off = idx->p_off;
    p.p_shared = idx->p_shared;
    p.p_misc = idx->p_misc;
    p.p_other = idx->p_other;
    p.p_ref_start = idx->p_ref_start;
    p.p_ref_cnt = idx->p_ref_cnt;
  }
  p.own_off = idx->own_off;
  p.own_cnt = idx->own_cnt;
  p.ref_ptr = idx->ref_ptr;
  p.ref_owner = idx->ref_owner;
  p.ref_start = idx->ref_start;
  p.ref_cnt = idx->ref_cnt;
  p.cbT = idx->cbT;
  p.d = idx->d;
  p.M = idx->M;
  p.M_pad = idx->M_pad;
  p.dsub = idx->dsub;
  p.shard_id = idx->shard_id;
  p.nshards = idx->nshards;
  p.queries = sa.queries;
  p.nq = sa.nq;
  p.probes = sa.probes;
  p.nprobe = ex.nprobe_eff > 0 ? ex.nprobe_eff : sa.nprobe;
  p.pstride = sa.nprobe;
  p.npp2 = next_pow2(p.nprobe);
  p.qlist = ex.qlist;
  p.qcount = ex.qcount;
  p.tau_out = ex.tau_out;
  p.defer_buf = ex.defer_buf;
  p.defer_n = ex.defer_n;
  p.bigK = sa.k * sa.refine_factor;
  p.cap = fastscan_cap(p.bigK, idx->M_pad);
  p.hbits = fs_hbits(idx->M);
  p.out_keys = sa.cand_keys;
  p.dco = ex.tau_out ? nullptr : sa.dco;
  p.dco_total = ex.tau_out ? nullptr : sa.counters;
  p.lut_q = sa.lut_q;
  p.lut_a = sa.lut_a;
  p.lut_b = sa.lut_b;
  p.sorted_out = sa.sorted_keys ? 1 : 0;
  {
    const char* e = std::getenv("RAIRS_FS_DBG");
    p.dbg = e ? std::atoi(e) : 0;
  }
  int o = 0;
  auto take = [&](int bytes, int align) {
    o = (int)round_up(o, align);
    const int at = o;
    o += bytes;
    return at;
  };
  p.o_lut = take(idx->M_pad * 16, 16);
  p.o_cand = take(p.cap * 8, 16);
  p.o_hist = take(256 * 4, 16);
  p.o_ps = take(p.npp2 * 4, 16);
  p.o_pre = take((p.nprobe + 1) * 4, 4);
  p.o_r0 = take(p.nprobe * 4, 4);
  p.o_rs = take(FS_RCAP * 4, 4);
  p.o_rc = take(FS_RCAP * 4, 4);
  p.o_rg = take((FS_RCAP + 1) * 4, 4);
  p.o_rl = p.paper ? take(FS_RCAP * 4, 4) : 0;
  p.warp_bytes = (int)round_up(o, 16);
  if (p.cap * 8 < idx->M * 4 + 16) {
    set_error("fast scan: candidate buffer smaller than the LUT scratch");
    return RAIRS_E_INTERNAL;
  }
  const int cbb = idx->M * 16 * idx->dsub * 4;
  p.cb_smem = cbb <= 160 * 1024 ? cbb : 0;  // fs_lut_kernel stages it (c3: 96 KB)
  p.luts = sa.luts;
  pl.warps = std::min<int>(FS_MAXW, (200 * 1024) / p.warp_bytes);
  if (pl.warps < 1) {
    set_error("fast scan: k * refine_factor / nprobe exceed the shared-memory budget");
    return RAIRS_E_UNSUPPORTED;
  }
  pl.smem = (size_t)pl.warps * p.warp_bytes;
  return RAIRS_OK;
}

template <int MINB, int GPL, int NW, bool PK, int DR = 4>
static rairs_status fs_launch(FsPlan& pl, cudaStream_t s) {
  pl.warps = std::min(pl.warps, NW);
  pl.smem = (size_t)pl.warps * pl.a.warp_bytes;
  RAIRS_CUDA_TRY(cudaFuncSetAttribute(fs_scan_kernel<MINB, GPL, NW, PK, DR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)pl.smem));
  int per_sm = 0;
  RAIRS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fs_scan_kernel<MINB, GPL, NW, PK, DR>,
                                                               pl.warps * 32, pl.smem));
  per_sm = std::max(per_sm, 1);
  const int64_t need = ceil_div(pl.a.nq * std::max(pl.a.parts, 1), pl.warps);  // work items
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, 148LL * per_sm));
  pl.a.total_warps = grid * (unsigned)pl.warps;
  RAIRS_CUDA_TRY(launch_pdl(fs_scan_kernel<MINB, GPL, NW, PK, DR>, dim3(grid), dim3(pl.warps * 32), pl.smem, s, pl.a));
  return RAIRS_OK;
}

rairs_status launch_fastscan(rairs_index_s* idx, const SearchArgs& sa, cudaStream_t s,
                             const FsExtra& ex) {
  if (sa.nq <= 0) return RAIRS_OK;
  if (!idx->codes_g || !idx->fs_ctr || !sa.luts) {
    set_error("fast scan: group layout or LUT workspace missing");
    return RAIRS_E_INTERNAL;
  }
  FsPlan pl;
  RAIRS_TRY(fs_plan(idx, sa, ex, pl));
  const unsigned slot = idx->fs_slot.fetch_add(1u) % FS_SLOTS;
  pl.a.ctr = idx->fs_ctr + 4 * slot;
  // small batches: each query's group tasks split over several warps
  const int P = (!ex.qlist && !ex.tau_out && ex.defer_buf) ? fastscan_parts(idx, sa.nq, sa.nprobe) : 1;
  pl.a.parts = P;
  if (P > 1 && sa.dco) RAIRS_CUDA_TRY(cudaMemsetAsync(sa.dco, 0, (size_t)sa.nq * 8, s));
  const bool use_order = fastscan_order_on() && P == 1 && !ex.qlist && sa.nq > 1;
  uint32_t* order = nullptr;
  struct OrderFree {
    uint32_t*& p;
    cudaStream_t s;
    ~OrderFree() { if (p) cudaFreeAsync(p, s); }
  } order_free{order, s};
  if (use_order) {
    RAIRS_CUDA_TRY(ws_malloc(&order, (size_t)sa.nq * 4, s));
    pl.a.order = order;
    pl.a.list_items = idx->list_items ? idx->list_items : idx->own_cnt;
    pl.a.nlist = (int)idx->nlist;
    const uint64_t total = idx->list_items ? (uint64_t)idx->sum_list_items : (uint64_t)idx->n_live;
    pl.a.cost_thr = (uint64_t)pl.a.nprobe * total;
  }
  if (!ex.luts_ready) {  // A3 for the whole batch (overlaps the coarse stage's tail under PDL);
                         // with the claim order computed after its wait on the coarse stage
    const bool keepT = idx->M * 17 <= 16 * 1024 / 4;
    const size_t lsm = (size_t)pl.a.cb_smem + (size_t)FL_WARPS * (keepT ? 17 : 1) * idx->M * 4;
    RAIRS_CUDA_TRY(cudaFuncSetAttribute(fs_lut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)lsm));
    // persistent: each CTA stages the codebook once for many queries
    int per_sm = 1;
    RAIRS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fs_lut_kernel, FL_WARPS * 32, lsm));
    per_sm = std::max(1, std::min(per_sm, 8));
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(sa.nq, FL_WARPS), 148LL * per_sm));
    RAIRS_CUDA_TRY(launch_pdl(fs_lut_kernel, dim3(g), dim3(FL_WARPS * 32), lsm, s, pl.a,
                              const_cast<uint4*>(sa.luts)));
  } else if (use_order) {
    const unsigned g = (unsigned)ceil_div(sa.nq, 256);
    RAIRS_CUDA_TRY(launch_pdl(fs_order_kernel, dim3(g), dim3(256), 0, s, pl.a, order));
  }
  const bool kev = sa.kev[0] && sa.kev_used && !ex.tau_out && !ex.qlist;
  if (kev) RAIRS_CUDA_TRY(cudaEventRecord(sa.kev[0], s));
  switch (fs_variant()) {
    case 1: RAIRS_TRY((fs_launch<3, 1, 8, false>(pl, s))); break;
    case 2: RAIRS_TRY((fs_launch<2, 2, 8, false>(pl, s))); break;
    default:
      if (idx->M_pad <= 128 && fastscan_pack_on() && fastscan_ring() == 6 && (idx->M_pad / 4) % 6 == 0)
        RAIRS_TRY((fs_launch<2, 1, 8, true, 6>(pl, s)));
      else if (idx->M_pad <= 128 && fastscan_pack_on()) RAIRS_TRY((fs_launch<2, 1, 8, true>(pl, s)));
      else RAIRS_TRY((fs_launch<2, 1, 8, false>(pl, s)));
      break;
  }
  if (kev) {
    RAIRS_CUDA_TRY(cudaEventRecord(sa.kev[1], s));
    *sa.kev_used = true;
  }
  if (pl.a.defer_buf) {
    const size_t per = (size_t)std::min<uint32_t>((uint32_t)pl.a.cap, FF_CAPS) * 8 + 1024;
    const int nw = (int)std::max<size_t>(1, std::min<size_t>(FF_WARPS, (200 * 1024) / per));
    const size_t fsm = (size_t)nw * per;
    RAIRS_CUDA_TRY(cudaFuncSetAttribute(fs_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)fsm));
    FsArgs fa = pl.a;  // split mode: one finish per (query, part), sorted, then a merge
    uint64_t* part_keys = nullptr;
    if (P > 1) {
      RAIRS_CUDA_TRY(ws_malloc(&part_keys, (size_t)sa.nq * P * pl.a.bigK * 8, s));
      fa.nq = sa.nq * P;
      fa.out_keys = part_keys;
      fa.sorted_out = 1;
    }
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(fa.nq, nw), 148 * 8));
    RAIRS_CUDA_TRY(launch_pdl(fs_finish_kernel, dim3(g), dim3(nw * 32), fsm, s, fa));
    if (P > 1) {
      const cudaError_t le = launch_pdl(fs_merge_parts_kernel, dim3((unsigned)ceil_div(sa.nq, 8)), dim3(256), 0, s,
                                        (const uint64_t*)part_keys, P, pl.a.bigK, sa.nq, pl.a.out_keys);
      cudaFreeAsync(part_keys, s);
      RAIRS_CUDA_TRY(le);
    }
  }
  return RAIRS_OK;
}

// Work items per query of the query-major scan: a small batch whose queries
// each score many items (c5 at nprobe 64: ~150k) splits each query's group
// tasks over P warps, P ~ expected items / 4k (each part then finds its own
// top-bigK: P x the selection work, so only when the scan work dominates),
// capped at 64 and at the resident warps; RAIRS_FS_PARTS overrides.
int fastscan_parts(const rairs_index_s* idx, int64_t nq, int nprobe) {
  if (const char* e = std::getenv("RAIRS_FS_PARTS"))  // read per search (tests force split mode)
    return std::max(1, std::min(64, std::atoi(e)));
  constexpr int64_t kWarps = 148 * 16;  // resident scan warps (2 CTAs x 8 warps per SM)
  if (nq <= 0 || nq * 2 > kWarps || idx->nlist <= 0) return 1;
  const double items = (double)nprobe *
                       ((double)(idx->list_items ? idx->sum_list_items : idx->n_live) / idx->nlist);
  const int64_t p = std::min<int64_t>({64, kWarps / nq, (int64_t)(items / 4096.0)});
  return (int)std::max<int64_t>(1, p);
}

// longest-first claim order for the scan (RAIRS_FS_ORDER=0: batch order)
bool fastscan_order_on() {
  static const bool on = [] {
    const char* e = std::getenv("RAIRS_FS_ORDER");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}

// Smallest candidate buffer: 1024 entries (fewer compactions: c4 scan -3 %)
// when two 8-warp CTAs still fit an SM's shared memory with it, else 512
// (RAIRS_FS_CAPMIN overrides).
static int fs_capmin(int M_pad) {
  static const int env = [] {
    const char* e = std::getenv("RAIRS_FS_CAPMIN");
    return e ? std::max(256, next_pow2(std::atoi(e))) : 0;
  }();
  if (env) return env;
  const int warp_bytes = M_pad * 16 + 1024 * 8 + 1024 + 2048;  // LUT + buffer + histogram + ranges
  return 2 * FS_MAXW * warp_bytes <= 220 * 1024 ? 1024 : 512;
}

int fastscan_cap(int bigK, int M_pad) {
  return std::max(fs_capmin(M_pad), next_pow2(bigK + fs_round_items() + 64));
}

}  // namespace rairs
