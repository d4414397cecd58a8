// search_kernels.cu -- the RAIRS query hot path on sm_100a.
//
// One CTA per query (grid-stride), fused:
//   K3  ComputeLookupTable (LUT P:711-716) + uint8 quantisation (R3)
//   K4  SEIL work list (Alg. 5, order-free dedup rule R9:
//       a reference (owner i -> list l) is scanned iff i is not probed)
//   K5  4-bit fast scan (PQFastScan P:729-737): lane = item of a 32-slot
//       block, codes streamed as 8-B units per lane (coalesced 256 B per warp
//       load), LUT rows in shared memory, exact u32 integer accumulation (R4)
//   A6  per-query top-bigK by the unique key (s << 32 | id) (rqueue P:1645;
//       R5): threshold filter into a shared-memory buffer, periodic exact
//       compaction by bitonic sort.
// then
//   K6  refine: exact fp64 distances of the bigK candidates,
//       top-k by (fp32 distance, id), one CTA per query.
//   K7  shard merge (O11).
#include <algorithm>

#include "index.cuh"
#include "tc_helpers.cuh"

namespace rairs {

constexpr int ST = 256;          // scan threads per CTA
constexpr int SNW = ST / 32;     // warps
constexpr int BPW = 8;           // blocks per warp per round
constexpr int ROUND = SNW * BPW * 32;  // max candidates appended per round
constexpr int RCAP = 512;        // ranges per work-list chunk

struct ScanParams {
  // index
  const uint64_t* codes64;
  const uint32_t* slot_rows;
  const uint32_t* own_off;
  const uint32_t* own_cnt;
  const uint32_t* ref_ptr;
  const int32_t* ref_owner;
  const uint32_t* ref_start;
  const uint32_t* ref_cnt;
  const float* codebook;
  int d, M, M_pad, dsub, nlist, shard_id, nshards;
  // query batch
  const float* queries;
  int64_t nq;
  const int32_t* probes;
  int nprobe, bigK, cap, hshift;
  uint64_t* out_keys;
  int64_t* dco;
  unsigned long long* dco_total;
  uint8_t* lut_q;
  float* lut_a;
  float* lut_b;
  // shared memory carve-up
  int off_lut, off_mn, off_span, off_bm, off_P, off_sp, off_rs, off_re, off_bp, off_hist, off_cand,
      smem;
};

// ---------------------------------------------------------------------------
// CTA-wide exclusive scan of n <= ST*4 u32 values in place; a[n] = total.
__device__ uint32_t cta_exclusive_scan(uint32_t* a, int n, uint32_t* warp_tot) {
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  constexpr int IPT = 4;
  uint32_t v[IPT];
  uint32_t local = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    int e = tid * IPT + i;
    v[i] = (e < n) ? a[e] : 0u;
    local += v[i];
  }
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = (lane < SNW) ? warp_tot[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < SNW) warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == SNW - 1) warp_tot[SNW] = wi;  // total
  }
  __syncthreads();
  uint32_t run = warp_tot[warp] + incl - local;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    int e = tid * IPT + i;
    if (e < n) a[e] = run;
    run += v[i];
  }
  const uint32_t total = warp_tot[SNW];
  if (tid == 0) a[n] = total;
  __syncthreads();
  return total;
}

// ---------------------------------------------------------------------------
// O2 / R2-R3: T[m][j] in fp32 with explicit rounding, ascending t, no FMA.
__device__ __forceinline__ float lut_T(const float* __restrict__ q,
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

// 8 lookups of one 32-bit word = 8 nibbles (subquantizers row0..row0+7).
// Even nibbles -> bytes of E, odd nibbles -> bytes of O; each byte is a
// 0..15 index into a 16-entry LUT row (LDS.U8 with an immediate row offset).
__device__ __forceinline__ uint32_t lookup8(const uint8_t* __restrict__ lutrow, uint32_t x) {
  const uint32_t E = x & 0x0F0F0F0Fu;
  const uint32_t O = (x >> 4) & 0x0F0F0F0Fu;
  uint32_t s0 = lutrow[0 * 16 + (E & 0xFFu)];
  uint32_t s1 = lutrow[1 * 16 + (O & 0xFFu)];
  uint32_t s2 = lutrow[2 * 16 + __byte_perm(E, 0, 0x4441)];
  uint32_t s3 = lutrow[3 * 16 + __byte_perm(O, 0, 0x4441)];
  uint32_t s4 = lutrow[4 * 16 + __byte_perm(E, 0, 0x4442)];
  uint32_t s5 = lutrow[5 * 16 + __byte_perm(O, 0, 0x4442)];
  uint32_t s6 = lutrow[6 * 16 + (E >> 24)];
  uint32_t s7 = lutrow[7 * 16 + (O >> 24)];
  return ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7));
}

__device__ __forceinline__ uint64_t ldg_stream_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

template <int NU>
__device__ __forceinline__ uint32_t score_block(const uint64_t* __restrict__ blkp,
                                                const uint8_t* __restrict__ lut, int lane,
                                                int nu_rt) {
  uint32_t acc = 0;
  if constexpr (NU > 0) {
    uint64_t w[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) w[u] = ldg_stream_u64(blkp + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      acc += lookup8(lut + (u * 16) * 16, (uint32_t)w[u]);
      acc += lookup8(lut + (u * 16 + 8) * 16, (uint32_t)(w[u] >> 32));
    }
  } else {
    for (int u = 0; u < nu_rt; ++u) {
      uint64_t w = ldg_stream_u64(blkp + u * 32 + lane);
      acc += lookup8(lut + (u * 16) * 16, (uint32_t)w);
      acc += lookup8(lut + (u * 16 + 8) * 16, (uint32_t)(w >> 32));
    }
  }
  return acc;
}

// ---------------------------------------------------------------------------
// A6 top-bigK selection state (per query, shared memory):
//  * hist[bin]: number of APPENDED candidates per score bin (bin = s >> hshift).
//    Every scanned item whose bin <= bthr is appended, and bthr only
//    decreases, so for bins <= bthr the histogram counts ALL scanned items.
//  * bthr: smallest bin with cumulative count >= bigK (conservative while
//    warps race; recomputed lock-free by the warp that crosses a counter).
//    Items in bins > bthr cannot be among the bigK smallest keys (the bin map
//    is monotone in s), so they are dropped without touching shared memory.
//  * tau: exact key threshold, only set by the (rare) sort fallback.
//  The final result is the exact sort of the survivors: unique keys
//  (s << 32 | id) make it independent of scheduling (R5).
constexpr int NBINS = 2048;

__device__ __forceinline__ uint32_t recompute_bthr(const uint32_t* hist, uint32_t upto,
                                                   uint32_t bigK) {
  // warp-cooperative: smallest b <= upto with sum_{i<=b} hist[i] >= bigK (else upto)
  const int lane = lane_id();
  uint32_t run = 0;
  for (uint32_t b0 = 0; b0 <= upto; b0 += 32) {
    const uint32_t b = b0 + lane;
    uint32_t v = (b <= upto) ? ((volatile const uint32_t*)hist)[b] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, run + v >= bigK && b <= upto);
    if (hit) return b0 + (uint32_t)(__ffs(hit) - 1);
    run += __shfl_sync(0xffffffffu, v, 31);
  }
  return upto;
}

// Drop candidates outside (bin <= bthr && key < tau); returns the new count.
// All threads; starts and ends with a barrier.  cap <= ST * 16.
__device__ uint32_t filter_cands(uint64_t* cand, uint32_t n, uint32_t bthr, uint64_t tau,
                                 int hshift, uint32_t* warp_tot) {
  constexpr int PER = 16;
  uint64_t v[PER];
  uint32_t keep = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const uint32_t e = threadIdx.x * PER + i;
    v[i] = (e < n) ? cand[e] : kKeyInf;
    const bool k = (e < n) && ((uint32_t)(v[i] >> (32 + hshift)) <= bthr) && (v[i] <= tau);
    if (!k) v[i] = kKeyInf;
    keep += k ? 1u : 0u;
  }
  // exclusive scan of per-thread counts
  const int lane = lane_id(), warp = warp_id();
  uint32_t incl = keep;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();  // everyone has read cand[] into registers
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = (lane < SNW) ? warp_tot[lane] : 0u, wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < SNW) warp_tot[lane] = wi - w;
    if (lane == SNW - 1) warp_tot[SNW] = wi;
  }
  __syncthreads();
  uint32_t pos = warp_tot[warp] + incl - keep;
#pragma unroll
  for (int i = 0; i < PER; ++i)
    if (v[i] != kKeyInf) cand[pos++] = v[i];
  const uint32_t total = warp_tot[SNW];
  __syncthreads();
  return total;
}

template <int NU>
__global__ void __launch_bounds__(ST, 4) scan_kernel(ScanParams p) {
  extern __shared__ __align__(16) unsigned char sm[];
  // The LUT lives in a static shared array when NU is known at compile time so
  // every LDS.U8 address is (nibble + constant) with no base-register add.
  __shared__ __align__(16) uint8_t lut_static[NU > 0 ? NU * 256 : 16];
  uint8_t* lut = (NU > 0) ? lut_static : (sm + p.off_lut);
  float* mn = reinterpret_cast<float*>(sm + p.off_mn);
  float* span = reinterpret_cast<float*>(sm + p.off_span);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(sm + p.off_bm);
  int32_t* P = reinterpret_cast<int32_t*>(sm + p.off_P);
  uint32_t* sp = reinterpret_cast<uint32_t*>(sm + p.off_sp);
  uint32_t* rs = reinterpret_cast<uint32_t*>(sm + p.off_rs);
  uint32_t* re = reinterpret_cast<uint32_t*>(sm + p.off_re);
  uint32_t* bp = reinterpret_cast<uint32_t*>(sm + p.off_bp);
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm + p.off_hist);
  uint64_t* cand = reinterpret_cast<uint64_t*>(sm + p.off_cand);
  __shared__ uint32_t warp_tot[SNW + 1];
  __shared__ unsigned int cand_cnt, bthr, since, dco_acc;
  __shared__ uint64_t tau;
  __shared__ float sh_S;

  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const int M = p.M, M16 = p.M * 16, MP16 = p.M_pad * 16;
  const int nu_rt = p.M_pad / 16;
  const int bm_words = (p.nlist + 31) >> 5;
  const int hshift = p.hshift;
  const uint32_t bigK = (uint32_t)p.bigK;
  const uint32_t recomp = max(32u, bigK / 2u);

  for (int64_t q = blockIdx.x; q < p.nq; q += gridDim.x) {
    const float* qv = p.queries + q * p.d;

    // ---------------- K3: LUT + uint8 quantisation (O2) ----------------
    // the first 4 * ST entries' T stay in registers for the quantisation pass
    float Tr[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int e0 = 0; e0 < M16; e0 += ST) {          // warp-uniform trip count
      const int e = e0 + tid;
      const bool act = e < M16;
      float T = act ? lut_T(qv, p.codebook, e >> 4, e & 15, p.dsub) : 0.0f;
      const int kk = e0 / ST;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (u == kk) Tr[u] = T;
      float lo = act ? T : __int_as_float(0x7f800000);
      float hi = act ? T : -__int_as_float(0x7f800000);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      if (act && (e & 15) == 0) {
        mn[e >> 4] = lo;
        span[e >> 4] = __fsub_rn(hi, lo);
      }
    }
    for (int w = tid; w < bm_words; w += ST) bitmap[w] = 0u;
    for (int w = tid; w < NBINS; w += ST) hist[w] = 0u;
    if (tid == 0) {
      cand_cnt = 0;
      bthr = NBINS - 1;
      since = 0;
      dco_acc = 0;
      tau = kKeyInf;
    }
    __syncthreads();
    if (warp == 0) {
      float s = 0.0f;
      for (int m = lane; m < M; m += 32) s = fmaxf(s, span[m]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, o));
      if (lane == 0) sh_S = s;
    }
    // probe set -> bitmap (R9 dedup needs "owner in P")
    for (int i = tid; i < p.nprobe; i += ST) {
      const int l = p.probes[q * p.nprobe + i];
      P[i] = l;
      atomicOr(&bitmap[l >> 5], 1u << (l & 31));
    }
    __syncthreads();
    const float S = sh_S;
    const float a = (S > 0.0f) ? __fdiv_rn(255.0f, S) : 1.0f;
    for (int e = tid; e < MP16; e += ST) {
      uint32_t v = 0;
      const int m = e >> 4;
      if (m < M && S > 0.0f) {
        const int kk = (e - tid) / ST;
        float T = 0.0f;  // the first pass's value (same function of the same inputs)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u == kk) T = Tr[u];
        if (kk >= 4) T = lut_T(qv, p.codebook, m, e & 15, p.dsub);
        const float t2 = __fmul_rn(__fsub_rn(T, mn[m]), a);
        v = (uint32_t)min(255, __float2int_rn(t2));
      }
      lut[e] = (uint8_t)v;
      if (p.lut_q && m < M) p.lut_q[q * M16 + e] = (uint8_t)v;
    }
    if (tid == 0) {
      if (p.lut_a) p.lut_a[q] = a;
      if (p.lut_b) {
        float b = 0.0f;
        for (int m = 0; m < M; ++m) b = __fadd_rn(b, mn[m]);
        p.lut_b[q] = b;
      }
    }
    // sources per probed list: 1 owned range + its references
    for (int i = tid; i < p.nprobe; i += ST) {
      const int l = P[i];
      sp[i] = 1u + (p.ref_ptr[l + 1] - p.ref_ptr[l]);
    }
    __syncthreads();
    const uint32_t nsrc_total = cta_exclusive_scan(sp, p.nprobe, warp_tot);

    uint32_t my_dco = 0;
    for (uint32_t cs = 0; cs < nsrc_total; cs += RCAP) {
      const int nsrc = (int)((nsrc_total - cs) < (uint32_t)RCAP ? (nsrc_total - cs) : (uint32_t)RCAP);
      // ---------------- K4: SEIL work list ----------------
      for (int i = tid; i < nsrc; i += ST) {
        const uint32_t s = cs + i;
        int lo = 0, hi = p.nprobe;  // largest pi with sp[pi] <= s
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (sp[mid] <= s) lo = mid; else hi = mid;
        }
        const int l = P[lo];
        const uint32_t sub = s - sp[lo];
        uint32_t st = 0, en = 0;
        if (sub == 0) {
          st = p.own_off[l];
          en = st + p.own_cnt[l];
        } else {
          const uint32_t j = p.ref_ptr[l] + sub - 1;
          const int o = p.ref_owner[j];
          if (!((bitmap[o >> 5] >> (o & 31)) & 1u)) {
            st = p.ref_start[j];
            en = st + p.ref_cnt[j];
          }
        }
        rs[i] = st;
        re[i] = en;
        bp[i] = (en > st) ? (((en - 1) >> 5) - (st >> 5) + 1) : 0u;
        my_dco += en - st;
      }
      __syncthreads();
      const uint32_t nblk = cta_exclusive_scan(bp, nsrc, warp_tot);

      // ---------------- K5 + A6: fast scan + threshold top-bigK ----------------
      int r = 0;  // per-warp cursor into the range list (monotone in b)
      for (uint32_t base = 0; base < nblk; base += SNW * BPW) {
        const uint64_t tau_r = tau;
#pragma unroll 1
        for (int kk = 0; kk < BPW; ++kk) {
          const uint32_t b = base + kk * SNW + warp;
          if (b >= nblk) break;
          while (bp[r + 1] <= b) ++r;
          const uint32_t st = rs[r], en = re[r];
          const uint32_t gblk = (st >> 5) + (b - bp[r]);
          const uint32_t slot = gblk * 32u + lane;
          const bool valid = (slot >= st) && (slot < en);
          const uint32_t s = score_block<NU>(p.codes64 + (size_t)gblk * nu_rt * 32, lut, lane, nu_rt);
          const uint32_t bin = s >> hshift;
          const bool maybe = valid && (bin <= *(volatile uint32_t*)&bthr);
          if (__any_sync(0xffffffffu, maybe)) {
            uint64_t key = kKeyInf;
            if (maybe) {
              const uint32_t row = p.slot_rows[slot];
              const uint32_t gid = row * (uint32_t)p.nshards + (uint32_t)p.shard_id;
              key = ((uint64_t)s << 32) | gid;
            }
            const bool pass = maybe && key < tau_r;
            const unsigned bal = __ballot_sync(0xffffffffu, pass);
            if (bal) {
              const unsigned c = (unsigned)__popc(bal);
              unsigned pos = 0, old = 0;
              if (lane == 0) {
                pos = atomicAdd(&cand_cnt, c);
                old = atomicAdd(&since, c);
              }
              pos = __shfl_sync(0xffffffffu, pos, 0);
              old = __shfl_sync(0xffffffffu, old, 0);
              if (pass) {
                cand[pos + __popc(bal & ((1u << lane) - 1u))] = key;
                atomicAdd(&hist[bin], 1u);
              }
              if (old < recomp && old + c >= recomp) {   // this warp refreshes bthr
                __syncwarp();
                const uint32_t nb = recompute_bthr(hist, *(volatile uint32_t*)&bthr, bigK);
                if (lane == 0) {
                  atomicMin(&bthr, nb);
                  atomicExch(&since, 0u);
                }
              }
            }
          }
        }
        __syncthreads();
        if (cand_cnt > (uint32_t)(p.cap - ROUND)) {
          if (warp == 0) {
            const uint32_t nb = recompute_bthr(hist, bthr, bigK);
            if (lane == 0) bthr = nb;
          }
          __syncthreads();
          const uint32_t nk = filter_cands(cand, cand_cnt, bthr, tau, hshift, warp_tot);
          if (tid == 0) cand_cnt = nk;
          __syncthreads();
          if (nk > (uint32_t)(p.cap - ROUND)) {  // pathological ties: exact sort fallback
            int np = 2;
            while (np < (int)nk) np <<= 1;
            for (int i = nk + tid; i < np; i += ST) cand[i] = kKeyInf;
            __syncthreads();
            cta_bitonic_sort_u64(cand, np);
            if (tid == 0) {
              cand_cnt = bigK;
              tau = cand[bigK - 1];
            }
            __syncthreads();
          }
        }
      }
      __syncthreads();
    }
    // DCO = |U_s(q)|: sum of scanned range lengths (valid items only)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_dco += __shfl_xor_sync(0xffffffffu, my_dco, o);
    if (lane == 0) atomicAdd(&dco_acc, my_dco);
    if (warp == 0) {
      const uint32_t nb = recompute_bthr(hist, bthr, bigK);
      if (lane == 0) bthr = nb;
    }
    __syncthreads();
    const uint32_t nk = filter_cands(cand, cand_cnt, bthr, tau, hshift, warp_tot);
    int np = 2;
    while (np < (int)nk) np <<= 1;
    for (int i = nk + tid; i < np; i += ST) cand[i] = kKeyInf;
    __syncthreads();
    cta_bitonic_sort_u64(cand, np);
    const int keep = (int)min(nk, bigK);
    for (int i = tid; i < p.bigK; i += ST)
      p.out_keys[q * p.bigK + i] = (i < keep) ? cand[i] : kKeyInf;
    if (tid == 0 && p.dco) p.dco[q] = (int64_t)dco_acc;
    if (tid == 0 && p.dco_total) atomicAdd(p.dco_total, (unsigned long long)dco_acc);
    __syncthreads();
  }
}

static int scan_smem_layout(ScanParams& p) {
  int o = 0;
  auto take = [&](int bytes, int align) {
    o = (int)round_up(o, align);
    int at = o;
    o += bytes;
    return at;
  };
  p.off_lut = take(p.M_pad * 16, 16);  // used only by the runtime-NU instance
  p.off_mn = take(p.M * 4, 16);
  p.off_span = take(p.M * 4, 16);
  p.off_bm = take(((p.nlist + 31) / 32) * 4, 16);
  p.off_P = take(p.nprobe * 4, 16);
  p.off_sp = take((p.nprobe + 1) * 4, 16);
  p.off_rs = take(RCAP * 4, 16);
  p.off_re = take(RCAP * 4, 16);
  p.off_bp = take((RCAP + 1) * 4, 16);
  p.off_hist = take(NBINS * 4, 16);
  p.off_cand = take(p.cap * 8, 16);
  p.smem = (int)round_up(o, 16);
  return p.smem;
}

template <int NU>
static rairs_status launch_scan_nu(ScanParams& p, cudaStream_t s) {
  RAIRS_CUDA_TRY(cudaFuncSetAttribute(scan_kernel<NU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      p.smem));
  const int grid = (int)std::min<int64_t>(p.nq, 1 << 30);
  scan_kernel<NU><<<grid, ST, p.smem, s>>>(p);
  RAIRS_CHECK_LAUNCH();
  return RAIRS_OK;
}

rairs_status launch_scan(const rairs_index_s* idx, const SearchArgs& a, cudaStream_t s) {
  if (a.nq <= 0) return RAIRS_OK;
  ScanParams p{};
  p.codes64 = reinterpret_cast<const uint64_t*>(idx->codes);
  p.slot_rows = idx->slot_rows;
  p.own_off = idx->own_off;
  p.own_cnt = idx->own_cnt;
  p.ref_ptr = idx->ref_ptr;
  p.ref_owner = idx->ref_owner;
  p.ref_start = idx->ref_start;
  p.ref_cnt = idx->ref_cnt;
  p.codebook = idx->codebook;
  p.d = idx->d;
  p.M = idx->M;
  p.M_pad = idx->M_pad;
  p.dsub = idx->dsub;
  p.nlist = idx->nlist;
  p.shard_id = idx->shard_id;
  p.nshards = idx->nshards;
  p.queries = a.queries;
  p.nq = a.nq;
  p.probes = a.probes;
  p.nprobe = a.nprobe;
  p.bigK = a.k * a.refine_factor;
  p.cap = next_pow2(p.bigK + ROUND);
  p.hshift = 0;
  while (((int64_t)p.M * 255) >> p.hshift >= NBINS) ++p.hshift;
  if (p.cap > ST * 16) {
    set_error("scan: k * refine_factor too large for the candidate buffer");
    return RAIRS_E_UNSUPPORTED;
  }
  p.out_keys = a.cand_keys;
  p.dco = a.dco;
  p.dco_total = a.counters;
  p.lut_q = a.lut_q;
  p.lut_a = a.lut_a;
  p.lut_b = a.lut_b;
  scan_smem_layout(p);
  if (p.smem > 220 * 1024) {
    set_error("scan: shared memory budget exceeded");
    return RAIRS_E_UNSUPPORTED;
  }
  switch (idx->M_pad / 16) {
    case 1: return launch_scan_nu<1>(p, s);
    case 2: return launch_scan_nu<2>(p, s);
    case 3: return launch_scan_nu<3>(p, s);
    case 4: return launch_scan_nu<4>(p, s);
    case 6: return launch_scan_nu<6>(p, s);
    case 8: return launch_scan_nu<8>(p, s);
    case 12: return launch_scan_nu<12>(p, s);
    case 24: return launch_scan_nu<24>(p, s);
    default: return launch_scan_nu<0>(p, s);
  }
}

// ---------------------------------------------------------------------------
// K6 refine: delta = fp32( sum_t ((double)q_t - (double)x_t)^2 ) in ascending t
// (O10), candidates ordered by the key (bits(delta) << 32 | id).
// The bigK candidate rows are gathered coalesced (one warp per row, 128-B
// segments) into a shared-memory tile of RT rows x RDC dims (odd row stride:
// conflict-free column reads); each thread then extends its own row's serial
// fp64 sum over the tile, so the summation order stays ascending in t.
constexpr int RT = 128;
constexpr int RDC = 128;           // dims per tile
constexpr int RSTRIDE = RDC + 1;

__global__ void __launch_bounds__(RT) refine_kernel(const uint64_t* __restrict__ keys,
                                                    int64_t nq, int bigK, int npow, int k,
                                                    const float* __restrict__ queries,
                                                    const float* __restrict__ X, int d, int G,
                                                    const uint32_t* __restrict__ labels,
                                                    unsigned long long* __restrict__ refined,
                                                    int64_t* __restrict__ out_ids,
                                                    float* __restrict__ out_dists) {
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
        for (int rb = 0; rb < 32; rb += 8) {
          float v[8][RDC / 32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t row = rows[warp * 32 + rb + i];
            const float* src = X + (size_t)(row == 0xFFFFFFFFu ? 0u : row) * d + t0;
#pragma unroll
            for (int j = 0; j < RDC / 32; ++j) {
              const int t = lane + 32 * j;
              v[i][j] = (row != 0xFFFFFFFFu && t < dc) ? __ldg(src + t) : 0.0f;
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
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
  __shared__ uint32_t nvalid;
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const int myrow = warp + 8 * lane;  // lane j (< 16) fetches the key of row warp + 8j
  const int nch = (bigK + RS_ROWS - 1) / RS_ROWS;
  // candidate rows are read once: evict them first from L2, so the gather does
  // not push out the score rows the concurrent selection streams
  uint64_t l2pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(l2pol));
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
      if (tid == 0) nvalid = 0;
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
    if (tid < crow) {
      const uint32_t g = gids[tid];
      uint64_t out = kKeyInf;
      if (g != 0xFFFFFFFFu) {
        const float4* xr = reinterpret_cast<const float4*>(tile + tid * RSF);
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
        atomicAdd(&nvalid, 1u);
      }
      rk[c * RS_ROWS + tid] = out;
    }
    __syncthreads();  // tile / gids free for the next unit; rk complete after the last chunk
    if (c == nch - 1) {
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
  refine_stage_kernel<D4><<<grid, RS_THREADS, smem, s>>>(a.cand_keys, a.nq, bigK, a.k, a.queries,
                                                          idx->X, idx->nshards, idx->labels,
                                                          a.counters ? a.counters + 1 : nullptr,
                                                          a.out_ids, a.out_dists);
  RAIRS_CHECK_LAUNCH();
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
  const int npow = next_pow2(std::max(bigK, 2));
  const size_t smem = (size_t)npow * 8 + (size_t)idx->d * 8 + (size_t)RT * RSTRIDE * 4 + RT * 4;
  if (smem > 220 * 1024) {
    set_error("refine: shared memory budget exceeded");
    return RAIRS_E_UNSUPPORTED;
  }
  RAIRS_CUDA_TRY(cudaFuncSetAttribute(refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  const int grid = (int)std::min<int64_t>(a.nq, 1 << 30);
  refine_kernel<<<grid, RT, smem, s>>>(a.cand_keys, a.nq, bigK, npow, a.k, a.queries, idx->X,
                                        idx->d, idx->nshards, idx->labels,
                                        a.counters ? a.counters + 1 : nullptr, a.out_ids, a.out_dists);
  RAIRS_CHECK_LAUNCH();
  return RAIRS_OK;
}

// ---------------------------------------------------------------------------
// K7 merge of G per-shard top-k lists: first k by (dist, id) (O11).
__global__ void merge_kernel(const int64_t* __restrict__ ids, const float* __restrict__ dists,
                             int G, int64_t nq, int k, int npow, int64_t* __restrict__ out_ids,
                             float* __restrict__ out_dists) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* key = reinterpret_cast<uint64_t*>(sm);
  for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
    for (int e = threadIdx.x; e < npow; e += blockDim.x) {
      uint64_t v = kKeyInf;
      if (e < G * k) {
        const int g = e / k, j = e - g * k;
        const int64_t id = ids[((int64_t)g * nq + q) * k + j];
        const float dd = dists[((int64_t)g * nq + q) * k + j];
        if (id >= 0) v = ((uint64_t)__float_as_uint(dd) << 32) | (uint64_t)(uint32_t)id;
      }
      key[e] = v;
    }
    __syncthreads();
    cta_bitonic_sort_u64(key, npow);
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      const uint64_t v = key[i];
      out_ids[q * k + i] = (v != kKeyInf) ? (int64_t)(uint32_t)(v & 0xFFFFFFFFu) : -1;
      out_dists[q * k + i] = (v != kKeyInf) ? __uint_as_float((uint32_t)(v >> 32))
                                            : __int_as_float(0x7f800000);
    }
    __syncthreads();
  }
}

rairs_status launch_merge(const int64_t* ids, const float* dists, int G, int64_t nq, int k,
                          int64_t* out_ids, float* out_dists, cudaStream_t s) {
  if (nq <= 0) return RAIRS_OK;
  const int npow = next_pow2(std::max(G * k, 2));
  const size_t smem = (size_t)npow * 8;
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
