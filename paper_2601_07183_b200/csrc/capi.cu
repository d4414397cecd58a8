// capi.cu -- extern "C" entry points of librairs.so (see include/rairs.h).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <new>
#include <string>

#include "index.cuh"

namespace rairs {
bool debug_sync_enabled() {
  static const bool on = [] {
    const char* e = getenv("RAIRS_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}
rairs_status debug_sync_point(cudaStream_t s, const char* what) {
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("after ") + what + ": " + cudaGetErrorString(e));
    return RAIRS_E_CUDA;
  }
  return RAIRS_OK;
}
}  // namespace rairs

namespace rairs {

static thread_local std::string g_err;

cudaError_t ws_malloc(void** p, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev], &props);
      if (e != cudaSuccess) {
        pools[dev] = nullptr;
        return e;
      }
      uint64_t thr = ~0ull;  // keep freed blocks (the pool is the library's)
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  return cudaMallocFromPoolAsync(p, bytes, pools[dev], s);
}
void set_error(const std::string& msg) { g_err = msg; }

static inline unsigned grid_for(int64_t n, int bs = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + bs - 1) / bs, 148 * 16));
}

__global__ void nonfinite_kernel(const float4* __restrict__ x, int64_t n4, unsigned* __restrict__ bad) {
  unsigned c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    c += !isfinite(v.x) + !isfinite(v.y) + !isfinite(v.z) + !isfinite(v.w);
  }
  if (c) atomicAdd(bad, c);
}

__global__ void nonfinite_tail_kernel(const float* __restrict__ x, int64_t n, unsigned* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) atomicAdd(bad, 1u);
}

// RAIRS_E_INVALID if any of the `count` floats at x (device) is NaN or +-inf
static rairs_status check_finite(const float* x, int64_t count, const char* what, cudaStream_t s) {
  unsigned* bad = nullptr;
  RAIRS_CUDA_TRY(ws_malloc(&bad, sizeof(unsigned), s));
  RAIRS_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(unsigned), s));
  const bool al = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int64_t n4 = al ? count / 4 : 0;
  if (n4 > 0) nonfinite_kernel<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const float4*>(x), n4, bad);
  if (count - 4 * n4 > 0)
    nonfinite_tail_kernel<<<grid_for(count - 4 * n4), 256, 0, s>>>(x + 4 * n4, count - 4 * n4, bad);
  unsigned h = 0;
  cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(bad, s);
  RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  if (h) {
    set_error(std::string(what) + " holds non-finite values");
    return RAIRS_E_INVALID;
  }
  return RAIRS_OK;
}

static rairs_status invalid(const std::string& msg) {
  set_error(msg);
  return RAIRS_E_INVALID;
}

static bool is_dev_ptr(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

#define REQUIRE_DEV(ptr, name)                                                   \
  do {                                                                           \
    if (!is_dev_ptr(ptr)) return invalid(std::string(name) + " must be a device pointer"); \
  } while (0)
#define OPTIONAL_DEV(ptr, name)                                                  \
  do {                                                                           \
    if ((ptr) != nullptr && !is_dev_ptr(ptr))                                    \
      return invalid(std::string(name) + " must be a device pointer or NULL");   \
  } while (0)

static rairs_status validate_params(const rairs_build_params* p, int64_t n, int32_t d) {
  if (!p) return invalid("params is NULL");
  if (n < 1) return invalid("n must be >= 1");
  if (d < 1) return invalid("d must be >= 1");
  if (p->nbits != 4) {
    set_error("only nbits = 4 is supported");
    return RAIRS_E_UNSUPPORTED;
  }
  if (p->nlist < 1 || p->nlist > 65536) return invalid("nlist must be in [1, 65536]");
  if (p->M < 1 || d % p->M != 0) return invalid("M must divide d");
  if (d / p->M > 8) {
    set_error("d/M > 8 is not supported");
    return RAIRS_E_UNSUPPORTED;
  }
  if (p->assignment != RAIRS_ASSIGN_SINGLE && p->assignment != RAIRS_ASSIGN_AIR &&
      p->assignment != RAIRS_ASSIGN_SOAR)
    return invalid("assignment must be RAIRS_ASSIGN_SINGLE, RAIRS_ASSIGN_AIR or RAIRS_ASSIGN_SOAR");
  if (p->nshards < 1 || p->shard_id < 0 || p->shard_id >= p->nshards)
    return invalid("need 0 <= shard_id < nshards");
  if (n >= (1ll << 30)) {
    set_error("more than 2^30 rows per shard is not supported");
    return RAIRS_E_UNSUPPORTED;
  }
  if ((int64_t)n * p->nshards >= 0xFFFFFFFFll) {
    set_error("global ids must fit in 32 bits");
    return RAIRS_E_UNSUPPORTED;
  }
  if (p->assignment != RAIRS_ASSIGN_SINGLE) {
    if (!(p->lambda >= 0.0f) || !std::isfinite(p->lambda)) return invalid("lambda must be finite and >= 0");
    int nc = std::min(p->n_cands, p->nlist);
    if (nc < 1) return invalid("n_cands must be >= 1");
    if (nc > 32) {
      set_error("n_cands > 32 is not supported");
      return RAIRS_E_UNSUPPORTED;
    }
    if (p->strict && nc < 2) return invalid("strict assignment needs n_cands >= 2 and nlist >= 2");
  }
  return RAIRS_OK;
}

static void free_index(rairs_index_s* x) {
  if (!x) return;
  cudaFree(x->centroids); cudaFree(x->codebook); cudaFree(x->X); cudaFree(x->l1); cudaFree(x->l2);
  cudaFree(x->codes); cudaFree(x->slot_rows); cudaFree(x->own_off); cudaFree(x->own_cnt);
  cudaFree(x->ref_ptr); cudaFree(x->ref_owner); cudaFree(x->ref_start); cudaFree(x->ref_cnt);
  cudaFree(x->cnorm); cudaFree(x->certify_fallbacks); cudaFree(x->counters);
  cudaFree(x->list_items); cudaFree(x->ref_item_off); cudaFree(x->list_base); cudaFree(x->list_ids);
  cudaFree(x->lm_order);
  cudaFree(x->codes_g); cudaFree(x->cbT); cudaFree(x->fs_ctr);
  seil_paper_free(x);
  cudaFree(x->live_bits);
  cudaFree(x->labels); cudaFree(x->lab_sorted); cudaFree(x->lab_rows);
  for (auto& st : x->aux) if (st) cudaStreamDestroy(st);
  for (auto& e : x->aux_ev) if (e) cudaEventDestroy(e);
  if (x->h2d) cudaStreamDestroy(x->h2d);
  for (auto& e : x->h2d_ev) if (e) cudaEventDestroy(e);
  for (auto& e : x->hq_ev) if (e) cudaEventDestroy(e);
  for (auto& b : x->hq_buf) cudaFree(b);
  delete x->hq_mu;
  delete x->aux_mu;
  for (auto& es : x->pending)
    for (int i = 0; i < 6; ++i) cudaEventDestroy(es.e[i]);
  for (auto e : x->pool) cudaEventDestroy(e);
  delete x;
}

// stage events (only when profiling is on)
struct StageEvents {
  rairs_index_s* idx;
  cudaStream_t s;
  rairs_index_s::EvSet ev{};
  bool on;
  StageEvents(rairs_index_s* i, cudaStream_t st) : idx(i), s(st), on(i->prof) {
    if (!on) return;
    std::lock_guard<std::mutex> lock(idx->prof_mu);
    for (int k = 0; k < 6; ++k) {
      if (!idx->pool.empty()) {
        ev.e[k] = idx->pool.back();
        idx->pool.pop_back();
      } else {
        cudaEventCreate(&ev.e[k]);
      }
    }
  }
  void mark(int k) {
    if (on) cudaEventRecord(ev.e[k], s);
  }
  void commit() {
    if (!on) return;
    std::lock_guard<std::mutex> lock(idx->prof_mu);
    idx->pending.push_back(ev);
  }
};

// rairs_search_host: 1 = the host queries are copied on the index's copy stream
// (into its query-buffer ring, overlapping the previous search), 0 = no copy
// stream, one copy on the search stream.  (Copying in 2-4 chunks with a coarse
// launch per chunk was measured slower: the extra coarse launches cost more than
// the earlier start.)
static int host_chunks(const rairs_index_s* idx, int64_t, int) { return idx->h2d ? 1 : 0; }

static rairs_status search_impl(rairs_index_s* idx, const float* queries, int64_t nq, int k,
                                int nprobe, int rf, int32_t* probes_out, uint8_t* lut_q,
                                float* lut_a, float* lut_b, uint32_t* cand_ids,
                                uint32_t* cand_scores, int64_t* dco, int64_t* out_ids,
                                float* out_dists, cudaStream_t s,
                                const float* queries_host = nullptr) {
  // queries_host != NULL: `queries` is a device buffer this call fills from it
  if (nq == 0) return RAIRS_OK;
  const int bigK = k * rf;
  int32_t* probes = probes_out;
  uint64_t* keys = nullptr;
  if (!probes) RAIRS_CUDA_TRY(ws_malloc(&probes, (size_t)nq * nprobe * 4, s));
  cudaError_t e = ws_malloc(&keys, (size_t)nq * bigK * 8, s);
  if (e != cudaSuccess) {
    if (!probes_out) cudaFreeAsync(probes, s);
    set_error(std::string("workspace: ") + cudaGetErrorString(e));
    return RAIRS_E_OOM;
  }
  SearchArgs a{};
  a.queries = queries;
  a.nq = nq;
  a.k = k;
  a.nprobe = nprobe;
  a.refine_factor = rf;
  a.probes = probes;
  a.cand_keys = keys;
  a.dco = dco;
  a.lut_q = lut_q;
  a.lut_a = lut_a;
  a.lut_b = lut_b;
  a.out_ids = out_ids;
  a.out_dists = out_dists;
  a.counters = idx->counters;
  idx->n_searches += 1;
  idx->n_queries += nq;

  StageEvents ev(idx, s);
  if (ev.on) {
    a.kev[0] = ev.ev.e[4];
    a.kev[1] = ev.ev.e[5];
    a.kev_used = &ev.ev.kern;
  }
  rairs_status st = RAIRS_OK;
  ev.mark(0);
  // coarse: P(q) = first nprobe lists by (D64, l)  (O1).  Tensor-core TF32
  // filter + exact fp64 certify (K1/K2), or the exact fp64 kernel directly.
  const int hchunks = queries_host ? host_chunks(idx, nq, nprobe) : 0;
  int64_t nk = 0;
  if (queries_host && hchunks == 0) {
    RAIRS_CUDA_TRY(cudaMemcpyAsync(const_cast<float*>(queries), queries_host,
                                   (size_t)nq * idx->d * 4, cudaMemcpyHostToDevice, s));
  }
  if (hchunks == 1 && queries_host) {
    // one copy on the copy stream (into the index's query-buffer ring): it
    // overlaps the previous search; this search waits for it
    std::lock_guard<std::mutex> lock(*idx->aux_mu);
    RAIRS_CUDA_TRY(cudaMemcpyAsync(const_cast<float*>(queries), queries_host,
                                   (size_t)nq * idx->d * 4, cudaMemcpyHostToDevice, idx->h2d));
    RAIRS_CUDA_TRY(cudaEventRecord(idx->h2d_ev[1], idx->h2d));
    RAIRS_CUDA_TRY(cudaStreamWaitEvent(s, idx->h2d_ev[1], 0));
  }
  bool small_done = false;
  if (idx->coarse_mode == 0 && nq <= coarse_small_rows()) {  // small batch (auto mode): exact fp64 coarse, split over CTAs
    ProbeArgs pa{};
    pa.X = queries;
    pa.rows = nq;
    pa.d = idx->d;
    pa.C = idx->centroids;
    pa.nl = idx->nlist;
    pa.L = nprobe;
    pa.mode = 0;
    pa.out_idx = probes;
    st = launch_probe_split_all(pa, s, &small_done);
    if (small_done) nk += 3;  // iota + split + merge
  }
  if (small_done || st != RAIRS_OK) {
  } else if (coarse_fused_ok(idx, nprobe)) {
    st = launch_coarse_fused(idx, queries, nq, nprobe, 0, 0.0, 0, probes, nullptr, nullptr,
                             idx->certify_fallbacks, s);
    nk += 3;  // topw + certify + exact fallback
  } else {
    ProbeArgs pa{};
    pa.X = queries;
    pa.rows = nq;
    pa.d = idx->d;
    pa.C = idx->centroids;
    pa.nl = idx->nlist;
    pa.L = nprobe;
    pa.mode = 0;
    pa.out_idx = probes;
    st = launch_probe_exact(pa, s);
    nk += 1;
  }
  ev.mark(1);
  bool refined = false;
  if (st == RAIRS_OK) {
    if (listmajor_ok(idx, nq, nprobe, bigK)) {
      a.fused_refine = true;
      a.sorted_keys = cand_ids != nullptr || cand_scores != nullptr;
      a.ev_selected = ev.on ? ev.ev.e[2] : nullptr;
      st = launch_listmajor(idx, a, s);
      const int chunks = (nq >= LM_NCH * LM_OVERLAP_MIN_Q && idx->aux[0]) ? LM_NCH : 1;
      nk += 6 + 2 * chunks;  // zero, count, scan, scatter, lut_tiles, tensor + (select, refine) x chunks
      refined = true;
    } else {
      a.sorted_keys = cand_ids != nullptr || cand_scores != nullptr;
      uint4* luts = nullptr;
      uint64_t* dbuf = nullptr;
      uint32_t* dn = nullptr;
      // the exact top-bigK in a separate pass (RAIRS_FS_DEFER=0: in the scan kernel)
      static const bool defer = [] {
        const char* e = std::getenv("RAIRS_FS_DEFER");
        return e ? std::atoi(e) != 0 : true;
      }();
      const size_t dcap = (size_t)fastscan_cap(bigK, idx->M_pad);
      const size_t dparts = (size_t)fastscan_parts(idx, nq, nprobe);  // split mode: one buffer per (query, part)
      cudaError_t le = ws_malloc(&luts, (size_t)nq * idx->M_pad * 16, s);
      if (le == cudaSuccess && defer) le = ws_malloc(&dbuf, (size_t)nq * dparts * dcap * 8, s);
      if (le == cudaSuccess && defer) le = ws_malloc(&dn, (size_t)nq * dparts * 4, s);
      if (le != cudaSuccess) {
        set_error(std::string("workspace: ") + cudaGetErrorString(le));
        st = RAIRS_E_OOM;
      } else {
        a.luts = luts;
        FsExtra ex;
        ex.defer_buf = dbuf;
        ex.defer_n = dn;
        st = launch_fastscan(idx, a, s, ex);
        nk += (defer ? 2 : 1) + (dparts > 1 && defer ? 1 : 0);  // + LUT (+ finish) (+ merge); the
                                                                // claim order comes from the LUT kernel
      }
      cudaFreeAsync(luts, s);
      cudaFreeAsync(dbuf, s);
      cudaFreeAsync(dn, s);
      nk += 1;
      ev.mark(2);
    }
  }
  if (st == RAIRS_OK && (cand_ids || cand_scores)) {
    st = launch_split_keys(keys, nq * bigK, cand_ids, cand_scores, s);
    nk += 1;
  }
  if (st == RAIRS_OK && !refined) {
    st = launch_refine(idx, a, s);
    nk += 1;
  }
  if (st == RAIRS_OK) idx->kernels += nk;
  ev.mark(3);
  ev.commit();
  if (!probes_out) cudaFreeAsync(probes, s);
  cudaFreeAsync(keys, s);
  if (st == RAIRS_OK) {
    idx->launches[0] += 1;
    idx->launches[1] += 1;
    idx->launches[2] += 1;
  }
  return st;
}

static rairs_status validate_search(rairs_index_t idx, int64_t nq, int32_t k, int32_t nprobe,
                                    int32_t rf) {
  if (!idx) return invalid("index is NULL");
  if (nq < 0) return invalid("nq must be >= 0");
  if (k < 1) return invalid("k must be >= 1");
  if (nprobe < 1 || nprobe > idx->nlist) return invalid("nprobe must be in [1, nlist]");
  if (nprobe > 1024) {
    set_error("nprobe > 1024 is not supported");
    return RAIRS_E_UNSUPPORTED;
  }
  if (rf < 1) return invalid("refine_factor must be >= 1");
  if ((int64_t)k * rf > 2048) {
    set_error("k * refine_factor > 2048 is not supported");
    return RAIRS_E_UNSUPPORTED;
  }
  return RAIRS_OK;
}

}  // namespace rairs

using namespace rairs;

extern "C" {

const char* rairs_last_error(void) { return g_err.c_str(); }
const char* rairs_version(void) { return "rairs-b200 0.1 (sm_100a)"; }

void rairs_default_params(rairs_build_params* p, int32_t nlist, int32_t M) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->nlist = nlist;
  p->M = M;
  p->nbits = 4;
  p->assignment = RAIRS_ASSIGN_AIR;
  p->lambda = 0.5f;
  p->n_cands = 10;
  p->strict = 0;
  p->kmeans_iters = 25;
  p->train_sample = 0;
  p->seed = 1234;
  p->shard_id = 0;
  p->nshards = 1;
}

rairs_status rairs_train(const float* base, int64_t n, int32_t d, const rairs_build_params* p,
                         void* stream, float* centroids_out, float* codebook_out) {
  RAIRS_TRY(validate_params(p, n, d));
  if (p->nlist > n) return invalid("nlist must be <= n");
  REQUIRE_DEV(base, "base");
  REQUIRE_DEV(centroids_out, "centroids_out");
  REQUIRE_DEV(codebook_out, "codebook_out");
  cudaStream_t s = (cudaStream_t)stream;
  const int iters = p->kmeans_iters > 0 ? p->kmeans_iters : 25;
  RAIRS_TRY(train_kmeans(base, n, d, p->nlist, iters, p->seed, p->train_sample, centroids_out, s));
  RAIRS_TRY(train_pq(base, n, d, p->M, iters, p->seed, 65536, codebook_out, s));
  return RAIRS_OK;
}

// Alg. 3 RairAssign (AIR, SOARL2) or single assignment of local rows
// [row0, row0 + cnt) of idx->X into idx->l1/l2, exact fp64 (O4). Tensor-core
// filter + certified fp64 re-rank for nlist > 256 (same result as the exact kernel).
static rairs_status assign_rows(rairs_index_s* idx, int64_t row0, int64_t cnt, cudaStream_t s) {
  if (cnt <= 0) return RAIRS_OK;
  const rairs_build_params* p = &idx->params;
  ProbeArgs pa{};
  pa.X = idx->X + row0 * idx->d;
  pa.rows = cnt;
  pa.d = idx->d;
  pa.C = idx->centroids;
  pa.nl = p->nlist;
  if (p->assignment != RAIRS_ASSIGN_SINGLE) {
    pa.mode = p->assignment == RAIRS_ASSIGN_SOAR ? 3 : 1;
    pa.L = std::min(p->n_cands, p->nlist);
    pa.lambda = (double)p->lambda;
    pa.strict = p->strict;
  } else {
    pa.mode = 2;
    pa.L = 1;
  }
  pa.l1 = idx->l1 + row0;
  pa.l2 = idx->l2 + row0;
  if (coarse_fused_ok(idx, pa.L) && idx->nlist > 256) {
    unsigned* fb = nullptr;
    RAIRS_CUDA_TRY(ws_malloc(&fb, sizeof(unsigned), s));
    RAIRS_CUDA_TRY(cudaMemsetAsync(fb, 0, sizeof(unsigned), s));
    rairs_status st = launch_coarse_fused(idx, pa.X, cnt, pa.L, pa.mode, pa.lambda, pa.strict,
                                          nullptr, pa.l1, pa.l2, fb, s);
    cudaFreeAsync(fb, s);
    if (st == RAIRS_OK && debug_sync_enabled()) st = debug_sync_point(s, "build: coarse assignment");
    return st;
  }
  return launch_probe_exact(pa, s);
}

rairs_status rairs_build_from_trained(const float* base, int64_t n, int32_t d, const int64_t* ids,
                                      const float* centroids, const float* codebook,
                                      const rairs_build_params* p, void* stream,
                                      rairs_index_t* out) {
  RAIRS_TRY(validate_params(p, n, d));
  if (!out) return invalid("out is NULL");
  REQUIRE_DEV(base, "base");
  REQUIRE_DEV(centroids, "centroids");
  REQUIRE_DEV(codebook, "codebook");
  OPTIONAL_DEV(ids, "ids");
  cudaStream_t s = (cudaStream_t)stream;
  RAIRS_TRY(check_finite(base, n * d, "base", s));            // before any index state exists
  if (ids) RAIRS_TRY(labels_validate(nullptr, ids, n, s));
  rairs_index_s* idx = new (std::nothrow) rairs_index_s();
  if (!idx) return RAIRS_E_OOM;
  {
    // (search workspaces: the library's own stream-ordered pool, ws_malloc)
  }
  cudaGetDevice(&idx->device);
  idx->n = n;
  idx->n_live = n;
  idx->cap_rows = n;
  idx->d = d;
  idx->nlist = p->nlist;
  idx->M = p->M;
  idx->M_pad = (int)round_up(p->M, 16);
  idx->dsub = d / p->M;
  idx->shard_id = p->shard_id;
  idx->nshards = p->nshards;
  idx->params = *p;
  rairs_status st = RAIRS_OK;
  auto fail = [&](rairs_status code) {
    free_index(idx);
    return code;
  };
#define B_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { set_error(std::string(#x) + ": " + cudaGetErrorString(_e)); return fail(_e == cudaErrorMemoryAllocation ? RAIRS_E_OOM : RAIRS_E_CUDA); } } while (0)
  const size_t cb_bytes = (size_t)p->M * 16 * idx->dsub * 4;
  B_TRY(cudaMalloc(&idx->centroids, (size_t)p->nlist * d * 4));
  B_TRY(cudaMalloc(&idx->codebook, cb_bytes));
  B_TRY(cudaMalloc(&idx->X, (size_t)n * d * 4));
  B_TRY(cudaMalloc(&idx->l1, n * 4));
  B_TRY(cudaMalloc(&idx->l2, n * 4));
  idx->device_bytes = (size_t)p->nlist * d * 4 + cb_bytes + (size_t)n * d * 4 + n * 8;
  B_TRY(cudaMemcpyAsync(idx->centroids, centroids, (size_t)p->nlist * d * 4, cudaMemcpyDeviceToDevice, s));
  B_TRY(cudaMemcpyAsync(idx->codebook, codebook, cb_bytes, cudaMemcpyDeviceToDevice, s));
  B_TRY(cudaMemcpyAsync(idx->X, base, (size_t)n * d * 4, cudaMemcpyDeviceToDevice, s));
  if (ids) {
    B_TRY(cudaMalloc(&idx->labels, (size_t)n * 4));
    idx->device_bytes += n * 12;  // labels + the sorted (label, row) table
    st = labels_store(idx, ids, 0, n, s);
    if (st != RAIRS_OK) return fail(st);
  }
  st = coarse_prepare(idx, s);
  if (st != RAIRS_OK) return fail(st);
  B_TRY(cudaMalloc(&idx->certify_fallbacks, sizeof(unsigned)));
  B_TRY(cudaMemsetAsync(idx->certify_fallbacks, 0, sizeof(unsigned), s));
  B_TRY(cudaMalloc(&idx->counters, 2 * sizeof(unsigned long long)));
  B_TRY(cudaMemsetAsync(idx->counters, 0, 2 * sizeof(unsigned long long), s));
  // Alg. 3 RairAssign (AIR / SOARL2) or single assignment, exact fp64 (O4)
  st = assign_rows(idx, 0, n, s);
  if (st != RAIRS_OK) return fail(st);
  // Alg. 4 SeilInsert (cell-major) + PQ encoding (O5) into the packed layout
  st = build_layout(idx, s);
  if (st != RAIRS_OK) return fail(st);
  st = listmajor_prepare(idx, s);
  if (st != RAIRS_OK) return fail(st);
  st = fastscan_prepare(idx, s);
  if (st != RAIRS_OK) return fail(st);
  B_TRY(cudaStreamSynchronize(s));
#undef B_TRY
  *out = idx;
  return RAIRS_OK;
}

rairs_status rairs_build_index(const float* base, int64_t n, int32_t d, const int64_t* ids,
                               const rairs_build_params* p, void* stream, rairs_index_t* out) {
  RAIRS_TRY(validate_params(p, n, d));
  if (p->nlist > n) return invalid("nlist must be <= n");
  REQUIRE_DEV(base, "base");
  OPTIONAL_DEV(ids, "ids");
  if (ids) RAIRS_TRY(labels_validate(nullptr, ids, n, (cudaStream_t)stream));
  cudaStream_t s = (cudaStream_t)stream;
  float *c = nullptr, *cb = nullptr;
  RAIRS_CUDA_TRY(cudaMalloc(&c, (size_t)p->nlist * d * 4));
  cudaError_t e = cudaMalloc(&cb, (size_t)p->M * 16 * (d / p->M) * 4);
  if (e != cudaSuccess) {
    cudaFree(c);
    set_error("codebook alloc failed");
    return RAIRS_E_OOM;
  }
  rairs_status st = rairs_train(base, n, d, p, stream, c, cb);
  if (st == RAIRS_OK) st = rairs_build_from_trained(base, n, d, ids, c, cb, p, stream, out);
  cudaStreamSynchronize(s);
  cudaFree(c);
  cudaFree(cb);
  return st;
}

rairs_status rairs_index_free(rairs_index_t idx) {
  if (!idx) return invalid("index is NULL");
  cudaDeviceSynchronize();
  free_index(idx);
  return RAIRS_OK;
}

rairs_status rairs_index_get_info(rairs_index_t idx, rairs_index_info* out) {
  if (!idx || !out) return invalid("NULL argument");
  out->n = idx->n;
  out->d = idx->d;
  out->nlist = idx->nlist;
  out->M = idx->M;
  out->M_pad = idx->M_pad;
  out->n_slots = idx->n_slots;
  out->n_cells = idx->n_cells;
  out->n_refs = idx->n_refs;
  out->n_double = idx->n_double;
  out->max_refs_per_list = idx->max_refs;
  out->shard_id = idx->shard_id;
  out->nshards = idx->nshards;
  out->device_bytes = idx->device_bytes;
  out->n_live = idx->n_live;
  out->has_ids = idx->labels != nullptr;
  return RAIRS_OK;
}

// ---- updates (NEXT-3; P:1393-1409 batched SeilInsert, P:1870-1880 delete) ----
__global__ void live_init_kernel(uint32_t* __restrict__ bits, int64_t words, int64_t n) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = w * 32;
    bits[w] = lo + 32 <= n ? 0xFFFFFFFFu : (lo >= n ? 0u : ((1u << (n - lo)) - 1u));
  }
}

// clear the live bit of every listed global id this shard holds; count the
// bits that were set (ids not held, out of range or already deleted are ignored)
__global__ void remove_ids_kernel(const int64_t* __restrict__ ids, int64_t m, int shard, int G,
                                  int64_t n, uint32_t* __restrict__ bits,
                                  unsigned long long* __restrict__ removed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = ids[i];
    if (id < 0 || id % G != shard) continue;
    const int64_t r = id / G;
    if (r >= n) continue;
    const uint32_t bit = 1u << (r & 31);
    const uint32_t old = atomicAnd(&bits[r >> 5], ~bit);
    if (old & bit) atomicAdd(removed, 1ull);
  }
}

__global__ void live_set_range_kernel(uint32_t* __restrict__ bits, int64_t r0, int64_t r1) {
  for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x)
    atomicOr(&bits[r >> 5], 1u << (r & 31));
}

static rairs_status relayout(rairs_index_s* idx, cudaStream_t s) {
  RAIRS_TRY(build_layout(idx, s));
  RAIRS_TRY(listmajor_prepare(idx, s));
  RAIRS_TRY(fastscan_prepare(idx, s));
  if (idx->seil_layout != 0) RAIRS_TRY(seil_paper_prepare(idx, s));
  RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  return RAIRS_OK;
}

static rairs_status grow_rows(rairs_index_s* idx, int64_t need, cudaStream_t s) {
  if (need <= idx->cap_rows) return RAIRS_OK;
  // 1/8 headroom: repeated batches amortise the copy without doubling 100M-row stores
  const int64_t cap = std::max<int64_t>(need, idx->cap_rows + idx->cap_rows / 8);
  const int d = idx->d;
  float* X = nullptr;
  int32_t *l1 = nullptr, *l2 = nullptr;
  uint32_t* bits = nullptr;
  auto undo = [&](cudaError_t e) {
    cudaFree(X); cudaFree(l1); cudaFree(l2); cudaFree(bits);
    set_error(std::string("rairs_add: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? RAIRS_E_OOM : RAIRS_E_CUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&X, (size_t)cap * d * 4)) != cudaSuccess) return undo(e);
  if ((e = cudaMalloc(&l1, (size_t)cap * 4)) != cudaSuccess) return undo(e);
  if ((e = cudaMalloc(&l2, (size_t)cap * 4)) != cudaSuccess) return undo(e);
  if (idx->live_bits && (e = cudaMalloc(&bits, (size_t)(cap + 31) / 32 * 4)) != cudaSuccess) return undo(e);
  uint32_t* lab = nullptr;
  if (idx->labels && (e = cudaMalloc(&lab, (size_t)cap * 4)) != cudaSuccess) {
    cudaFree(lab);
    return undo(e);
  }
  cudaMemcpyAsync(X, idx->X, (size_t)idx->n * d * 4, cudaMemcpyDeviceToDevice, s);
  cudaMemcpyAsync(l1, idx->l1, (size_t)idx->n * 4, cudaMemcpyDeviceToDevice, s);
  cudaMemcpyAsync(l2, idx->l2, (size_t)idx->n * 4, cudaMemcpyDeviceToDevice, s);
  if (bits) {
    cudaMemsetAsync(bits, 0, (size_t)(cap + 31) / 32 * 4, s);
    cudaMemcpyAsync(bits, idx->live_bits, (size_t)(idx->cap_rows + 31) / 32 * 4,
                    cudaMemcpyDeviceToDevice, s);
  }
  if (lab) cudaMemcpyAsync(lab, idx->labels, (size_t)idx->n * 4, cudaMemcpyDeviceToDevice, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) {
    cudaFree(lab);
    return undo(e);
  }
  cudaFree(idx->X); cudaFree(idx->l1); cudaFree(idx->l2); cudaFree(idx->live_bits);
  cudaFree(idx->labels);
  idx->X = X; idx->l1 = l1; idx->l2 = l2; idx->live_bits = bits; idx->labels = lab;
  if (lab) idx->device_bytes += (cap - idx->cap_rows) * 4;
  idx->device_bytes += (cap - idx->cap_rows) * ((int64_t)d * 4 + 8) +
                       (bits ? ((cap + 31) / 32 - (idx->cap_rows + 31) / 32) * 4 : 0);
  idx->cap_rows = cap;
  return RAIRS_OK;
}

rairs_status rairs_add(rairs_index_t idx, const float* x, int64_t n_add, const int64_t* ids,
                       int64_t* first_id, void* stream) {
  if (!idx) return invalid("index is NULL");
  if (n_add < 0) return invalid("n_add must be >= 0");
  if (n_add == 0) {
    if (first_id) *first_id = idx->n * idx->nshards + idx->shard_id;
    return RAIRS_OK;
  }
  REQUIRE_DEV(x, "x");
  OPTIONAL_DEV(ids, "ids");
  if ((ids != nullptr) != (idx->labels != nullptr))
    return invalid(idx->labels ? "this index holds caller ids: pass ids for the new rows"
                               : "this index numbers its rows itself: ids must be NULL");
  RAIRS_TRY(check_finite(x, n_add * idx->d, "x", (cudaStream_t)stream));
  if (ids) RAIRS_TRY(labels_validate(idx, ids, n_add, (cudaStream_t)stream));
  const int64_t n_new = idx->n + n_add;
  if (n_new >= (1ll << 30)) {
    set_error("more than 2^30 rows per shard is not supported");
    return RAIRS_E_UNSUPPORTED;
  }
  if (n_new * idx->nshards >= 0xFFFFFFFFll) {
    set_error("global ids must fit in 32 bits");
    return RAIRS_E_UNSUPPORTED;
  }
  cudaStream_t s = (cudaStream_t)stream;
  RAIRS_CUDA_TRY(cudaDeviceSynchronize());  // in-flight searches may read the old arrays
  RAIRS_TRY(grow_rows(idx, n_new, s));
  const int64_t r0 = idx->n;
  RAIRS_CUDA_TRY(cudaMemcpyAsync(idx->X + r0 * idx->d, x, (size_t)n_add * idx->d * 4,
                                 cudaMemcpyDeviceToDevice, s));
  if (idx->live_bits) {
    live_set_range_kernel<<<grid_for(n_add), 256, 0, s>>>(idx->live_bits, r0, n_new);
    RAIRS_CHECK_LAUNCH();
  }
  // new rows: Alg. 3 assignment (lines 1-12) with the index's trained centroids
  // (rows >= idx->n: nothing the index serves changes until the relayout)
  RAIRS_TRY(assign_rows(idx, r0, n_add, s));
  idx->n = n_new;
  idx->n_live += n_add;
  // Alg. 4 for the batch: cells, references and codes re-laid out (cell-major);
  // on failure the index keeps its previous rows and layout
  const rairs_status rl = relayout(idx, s);
  if (rl != RAIRS_OK) {
    idx->n = r0;
    idx->n_live -= n_add;
    relayout(idx, s);  // the previous layout (kept, or rebuilt if a later table failed)
    return rl;
  }
  if (ids) RAIRS_TRY(labels_store(idx, ids, r0, n_add, s));
  if (first_id) *first_id = r0 * idx->nshards + idx->shard_id;
  return RAIRS_OK;
}

rairs_status rairs_remove_ids(rairs_index_t idx, const int64_t* ids, int64_t n_ids,
                              int64_t* n_removed, void* stream) {
  if (!idx) return invalid("index is NULL");
  if (n_ids < 0) return invalid("n_ids must be >= 0");
  if (n_removed) *n_removed = 0;
  if (n_ids == 0) return RAIRS_OK;
  REQUIRE_DEV(ids, "ids");
  cudaStream_t s = (cudaStream_t)stream;
  RAIRS_CUDA_TRY(cudaDeviceSynchronize());
  const int64_t words = (idx->cap_rows + 31) / 32;
  if (!idx->live_bits) {
    RAIRS_CUDA_TRY(cudaMalloc(&idx->live_bits, (size_t)words * 4));
    live_init_kernel<<<grid_for(words), 256, 0, s>>>(idx->live_bits, words, idx->n);
    RAIRS_CHECK_LAUNCH();
    idx->device_bytes += words * 4;
  }
  unsigned long long* cnt = nullptr;
  int64_t* gids = nullptr;
  if (idx->labels) {  // caller ids -> internal global ids
    RAIRS_CUDA_TRY(ws_malloc(&gids, (size_t)n_ids * 8, s));
    RAIRS_TRY(labels_to_gids(idx, ids, n_ids, gids, s));
  }
  RAIRS_CUDA_TRY(ws_malloc(&cnt, sizeof(unsigned long long), s));
  RAIRS_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
  remove_ids_kernel<<<grid_for(n_ids), 256, 0, s>>>(gids ? gids : ids, n_ids, idx->shard_id,
                                                    idx->nshards, idx->n, idx->live_bits, cnt);
  RAIRS_CHECK_LAUNCH();
  if (gids) cudaFreeAsync(gids, s);
  unsigned long long h = 0;
  RAIRS_CUDA_TRY(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(cnt, s);
  RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  if (n_removed) *n_removed = (int64_t)h;
  if (h == 0) return RAIRS_OK;
  idx->n_live -= (int64_t)h;
  return relayout(idx, s);
}

rairs_status rairs_search(rairs_index_t idx, const float* queries, int64_t nq, int32_t k,
                          int32_t nprobe, int32_t refine_factor, int64_t* out_ids,
                          float* out_dists, int64_t* dco, void* stream) {
  RAIRS_TRY(validate_search(idx, nq, k, nprobe, refine_factor));
  if (nq == 0) return RAIRS_OK;
  REQUIRE_DEV(queries, "queries");
  REQUIRE_DEV(out_ids, "out_ids");
  REQUIRE_DEV(out_dists, "out_dists");
  OPTIONAL_DEV(dco, "dco");
  return search_impl(idx, queries, nq, k, nprobe, refine_factor, nullptr, nullptr, nullptr,
                     nullptr, nullptr, nullptr, dco, out_ids, out_dists, (cudaStream_t)stream);
}

static rairs_status search_host_impl(rairs_index_t idx, const float* queries_host, int64_t nq,
                                     int32_t k, int32_t nprobe, int32_t refine_factor,
                                     int64_t* out_ids_host, float* out_dists_host, void* stream,
                                     bool sync) {
  RAIRS_TRY(validate_search(idx, nq, k, nprobe, refine_factor));
  if (nq == 0) return RAIRS_OK;
  if (!queries_host || !out_ids_host || !out_dists_host) return invalid("NULL host buffer");
  cudaStream_t s = (cudaStream_t)stream;
  float* dq = nullptr;
  int64_t* di = nullptr;
  float* dd = nullptr;
  const size_t qb = (size_t)nq * idx->d * 4, ib = (size_t)nq * k * 8, db = (size_t)nq * k * 4;
  const bool chunked = host_chunks(idx, nq, nprobe) >= 1;  // copies on the copy stream
  std::unique_lock<std::mutex> lock;
  int slot = -1;
  if (chunked) {
    // chunked copies run on the copy stream, into one of the index's two query
    // buffers; it waits (on the device) until the search that last read the
    // buffer has finished, never for the rest of the search stream
    lock = std::unique_lock<std::mutex>(*idx->hq_mu);
    slot = idx->hq_next;
    idx->hq_next ^= 1;
    if (idx->hq_cap[slot] < qb) {
      RAIRS_CUDA_TRY(cudaDeviceSynchronize());
      cudaFree(idx->hq_buf[slot]);
      idx->hq_buf[slot] = nullptr;
      idx->hq_cap[slot] = 0;
      RAIRS_CUDA_TRY(cudaMalloc(&idx->hq_buf[slot], qb));
      idx->hq_cap[slot] = qb;
    }
    RAIRS_CUDA_TRY(cudaStreamWaitEvent(idx->h2d, idx->hq_ev[slot], 0));
    dq = idx->hq_buf[slot];
  } else {
    RAIRS_CUDA_TRY(ws_malloc(&dq, qb, s));
  }
  RAIRS_CUDA_TRY(ws_malloc(&di, ib, s));
  RAIRS_CUDA_TRY(ws_malloc(&dd, db, s));
  rairs_status st = search_impl(idx, dq, nq, k, nprobe, refine_factor, nullptr, nullptr, nullptr,
                                nullptr, nullptr, nullptr, nullptr, di, dd, s, queries_host);
  if (chunked) cudaEventRecord(idx->hq_ev[slot], s);  // the buffer is free again after this
  if (st == RAIRS_OK) {
    cudaMemcpyAsync(out_ids_host, di, ib, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(out_dists_host, dd, db, cudaMemcpyDeviceToHost, s);
  }
  if (!chunked) cudaFreeAsync(dq, s);
  cudaFreeAsync(di, s);
  cudaFreeAsync(dd, s);
  if (sync || st != RAIRS_OK) RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  return st;
}

rairs_status rairs_search_host(rairs_index_t idx, const float* queries_host, int64_t nq,
                               int32_t k, int32_t nprobe, int32_t refine_factor,
                               int64_t* out_ids_host, float* out_dists_host, void* stream) {
  return search_host_impl(idx, queries_host, nq, k, nprobe, refine_factor, out_ids_host,
                          out_dists_host, stream, true);
}

rairs_status rairs_search_host_async(rairs_index_t idx, const float* queries_host, int64_t nq,
                                     int32_t k, int32_t nprobe, int32_t refine_factor,
                                     int64_t* out_ids_host, float* out_dists_host, void* stream) {
  return search_host_impl(idx, queries_host, nq, k, nprobe, refine_factor, out_ids_host,
                          out_dists_host, stream, false);
}

rairs_status rairs_search_debug(rairs_index_t idx, const float* queries, int64_t nq, int32_t k,
                                int32_t nprobe, int32_t refine_factor, int32_t* probes,
                                uint8_t* lut_q, float* lut_a, float* lut_b, uint32_t* cand_ids,
                                uint32_t* cand_scores, int64_t* dco, int64_t* out_ids,
                                float* out_dists, void* stream) {
  RAIRS_TRY(validate_search(idx, nq, k, nprobe, refine_factor));
  if (nq == 0) return RAIRS_OK;
  REQUIRE_DEV(queries, "queries");
  OPTIONAL_DEV(probes, "probes");
  OPTIONAL_DEV(lut_q, "lut_q");
  OPTIONAL_DEV(lut_a, "lut_a");
  OPTIONAL_DEV(lut_b, "lut_b");
  OPTIONAL_DEV(cand_ids, "cand_ids");
  OPTIONAL_DEV(cand_scores, "cand_scores");
  OPTIONAL_DEV(dco, "dco");
  REQUIRE_DEV(out_ids, "out_ids");
  REQUIRE_DEV(out_dists, "out_dists");
  return search_impl(idx, queries, nq, k, nprobe, refine_factor, probes, lut_q, lut_a, lut_b,
                     cand_ids, cand_scores, dco, out_ids, out_dists, (cudaStream_t)stream);
}

rairs_status rairs_merge_topk(const int64_t* ids, const float* dists, int32_t G, int64_t nq,
                              int32_t k, int64_t* out_ids, float* out_dists, void* stream) {
  if (G < 1 || k < 1 || nq < 0) return invalid("need G >= 1, k >= 1, nq >= 0");
  if (nq == 0) return RAIRS_OK;
  REQUIRE_DEV(ids, "ids");
  REQUIRE_DEV(dists, "dists");
  REQUIRE_DEV(out_ids, "out_ids");
  REQUIRE_DEV(out_dists, "out_dists");
  return launch_merge(ids, dists, G, nq, k, out_ids, out_dists, (cudaStream_t)stream);
}

rairs_status rairs_exact_knn(const float* base, int64_t n, int32_t d, const float* queries,
                             int64_t nq, int32_t K, int64_t* out_ids, double* out_d64,
                             void* stream) {
  if (n < 1 || d < 1 || nq < 0) return invalid("need n >= 1, d >= 1, nq >= 0");
  if (K < 1 || K > n) return invalid("need 1 <= K <= n");
  if (K > 256) {
    set_error("K > 256 is not supported");
    return RAIRS_E_UNSUPPORTED;
  }
  if (nq == 0) return RAIRS_OK;
  REQUIRE_DEV(base, "base");
  REQUIRE_DEV(queries, "queries");
  OPTIONAL_DEV(out_ids, "out_ids");
  OPTIONAL_DEV(out_d64, "out_d64");
  ProbeArgs pa{};
  pa.X = queries;
  pa.rows = nq;
  pa.d = d;
  pa.C = base;
  pa.nl = n;
  pa.L = K;
  pa.mode = 0;
  pa.out_idx64 = out_ids;
  pa.out_d64 = out_d64;
  return launch_probe_exact(pa, (cudaStream_t)stream);
}

rairs_status rairs_export_trained(rairs_index_t idx, float* centroids, float* codebook,
                                  void* stream) {
  if (!idx) return invalid("index is NULL");
  OPTIONAL_DEV(centroids, "centroids");
  OPTIONAL_DEV(codebook, "codebook");
  cudaStream_t s = (cudaStream_t)stream;
  if (centroids)
    RAIRS_CUDA_TRY(cudaMemcpyAsync(centroids, idx->centroids, (size_t)idx->nlist * idx->d * 4,
                                   cudaMemcpyDeviceToDevice, s));
  if (codebook)
    RAIRS_CUDA_TRY(cudaMemcpyAsync(codebook, idx->codebook, (size_t)idx->M * 16 * idx->dsub * 4,
                                   cudaMemcpyDeviceToDevice, s));
  return RAIRS_OK;
}

rairs_status rairs_export_assignment(rairs_index_t idx, int32_t* l1, int32_t* l2, uint8_t* codes,
                                     void* stream) {
  if (!idx) return invalid("index is NULL");
  OPTIONAL_DEV(l1, "l1");
  OPTIONAL_DEV(l2, "l2");
  OPTIONAL_DEV(codes, "codes");
  cudaStream_t s = (cudaStream_t)stream;
  if (l1) RAIRS_CUDA_TRY(cudaMemcpyAsync(l1, idx->l1, idx->n * 4, cudaMemcpyDeviceToDevice, s));
  if (l2) RAIRS_CUDA_TRY(cudaMemcpyAsync(l2, idx->l2, idx->n * 4, cudaMemcpyDeviceToDevice, s));
  if (codes) RAIRS_TRY(export_codes(idx, codes, s));
  return RAIRS_OK;
}

rairs_status rairs_export_layout(rairs_index_t idx, int64_t* own_off, int64_t* own_cnt,
                                 int64_t* ref_ptr, int32_t* ref_owner, int64_t* ref_start,
                                 int64_t* ref_cnt, uint32_t* slot_rows, void* stream) {
  if (!idx) return invalid("index is NULL");
  OPTIONAL_DEV(own_off, "own_off");
  OPTIONAL_DEV(own_cnt, "own_cnt");
  OPTIONAL_DEV(ref_ptr, "ref_ptr");
  OPTIONAL_DEV(ref_owner, "ref_owner");
  OPTIONAL_DEV(ref_start, "ref_start");
  OPTIONAL_DEV(ref_cnt, "ref_cnt");
  OPTIONAL_DEV(slot_rows, "slot_rows");
  return export_layout64(idx, own_off, own_cnt, ref_ptr, ref_owner, ref_start, ref_cnt, slot_rows,
                         (cudaStream_t)stream);
}

rairs_status rairs_set_coarse_mode(rairs_index_t idx, int32_t mode) {
  if (!idx) return invalid("index is NULL");
  if (mode < 0 || mode > 2) return invalid("coarse mode must be 0 (auto), 1 (exact), 2 (tensor core)");
  idx->coarse_mode = mode;
  return RAIRS_OK;
}

rairs_status rairs_set_scan_mode(rairs_index_t idx, int32_t mode) {
  if (!idx) return invalid("index is NULL");
  if (mode < 0 || mode > 2) return invalid("scan mode must be 0 (auto), 1 (SIMT), 2 (list-major)");
  idx->scan_mode = mode;
  return RAIRS_OK;
}

rairs_status rairs_set_seil_layout(rairs_index_t idx, int32_t layout) {
  if (!idx) return invalid("index is NULL");
  if (layout < 0 || layout > 3)
    return invalid("SEIL layout must be 0 (cell-major), 1 (paper-literal), 2 (paper-literal for query-major "
                   "scans) or 3 (hybrid for query-major scans)");
  const int kind = layout == 3 ? 3 : 1;
  const int prev = idx->seil_layout;
  idx->seil_layout = layout;
  if (layout != 0 && (!idx->p_codes_g || idx->p_kind != kind)) {
    cudaStream_t s = nullptr;
    RAIRS_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    RAIRS_CUDA_TRY(cudaDeviceSynchronize());
    const rairs_status st = seil_paper_prepare(idx, s);
    cudaStreamDestroy(s);
    if (st != RAIRS_OK) {
      idx->seil_layout = idx->p_codes_g ? prev : 0;
      return st;
    }
  }
  if (layout == 0) seil_paper_free(idx);
  return RAIRS_OK;
}

rairs_status rairs_certify_fallbacks(rairs_index_t idx, int64_t* count, int32_t reset) {
  if (!idx || !count) return invalid("NULL argument");
  unsigned v = 0;
  RAIRS_CUDA_TRY(cudaMemcpy(&v, idx->certify_fallbacks, sizeof(unsigned), cudaMemcpyDeviceToHost));
  *count = v;
  if (reset) RAIRS_CUDA_TRY(cudaMemset(idx->certify_fallbacks, 0, sizeof(unsigned)));
  return RAIRS_OK;
}

rairs_status rairs_get_stats(rairs_index_t idx, rairs_stats* out, int32_t reset) {
  if (!idx || !out) return invalid("NULL argument");
  RAIRS_CUDA_TRY(cudaDeviceSynchronize());
  unsigned long long c[2] = {0, 0};
  unsigned fb = 0;
  RAIRS_CUDA_TRY(cudaMemcpy(c, idx->counters, sizeof(c), cudaMemcpyDeviceToHost));
  RAIRS_CUDA_TRY(cudaMemcpy(&fb, idx->certify_fallbacks, sizeof(fb), cudaMemcpyDeviceToHost));
  double ms[3] = {0, 0, 0};
  RAIRS_TRY(rairs_profile_read(idx, ms, nullptr, 0));
  out->searches = idx->n_searches;
  out->queries = idx->n_queries;
  out->dco_total = (int64_t)c[0];
  out->refine_total = (int64_t)c[1];
  out->certify_fallbacks = fb;
  out->ms_coarse = ms[0];
  out->ms_scan = ms[1];
  out->ms_refine = ms[2];
  if (reset) {
    RAIRS_CUDA_TRY(cudaMemset(idx->counters, 0, sizeof(c)));
    RAIRS_CUDA_TRY(cudaMemset(idx->certify_fallbacks, 0, sizeof(unsigned)));
    RAIRS_TRY(rairs_profile_read(idx, nullptr, nullptr, 1));
    idx->n_searches = 0;
    idx->n_queries = 0;
  }
  return RAIRS_OK;
}

rairs_status rairs_search_plan(rairs_index_t idx, int64_t nq, int32_t k, int32_t nprobe,
                               int32_t refine_factor, int32_t* coarse_path, int32_t* scan_path) {
  RAIRS_TRY(validate_search(idx, nq, k, nprobe, refine_factor));
  if (coarse_path) *coarse_path = coarse_fused_ok(idx, nprobe) ? 2 : 1;
  if (scan_path) *scan_path = listmajor_ok(idx, nq, nprobe, k * refine_factor) ? 2 : 1;
  return RAIRS_OK;
}

rairs_status rairs_profile_kernels(rairs_index_t idx, int64_t* kernels, int32_t reset) {
  if (!idx || !kernels) return invalid("NULL argument");
  *kernels = idx->kernels;
  if (reset) idx->kernels.store(0);
  return RAIRS_OK;
}

rairs_status rairs_profile_enable(rairs_index_t idx, int32_t on) {
  if (!idx) return invalid("index is NULL");
  idx->prof = on != 0;
  return RAIRS_OK;
}

rairs_status rairs_profile_read(rairs_index_t idx, double* ms3, int64_t* launches3,
                                int32_t reset) {
  if (!idx) return invalid("index is NULL");
  std::lock_guard<std::mutex> lock(idx->prof_mu);
  for (auto& es : idx->pending) {
    RAIRS_CUDA_TRY(cudaEventSynchronize(es.e[3]));
    for (int k = 0; k < 3; ++k) {
      float ms = 0.0f;
      RAIRS_CUDA_TRY(cudaEventElapsedTime(&ms, es.e[k], es.e[k + 1]));
      idx->ms[k] += ms;
    }
    if (es.kern) {
      float ms = 0.0f;
      RAIRS_CUDA_TRY(cudaEventElapsedTime(&ms, es.e[4], es.e[5]));
      idx->ms_kern += ms;
      idx->kern_launches += 1;
    }
    for (int k = 0; k < 6; ++k) idx->pool.push_back(es.e[k]);
  }
  idx->pending.clear();
  for (int k = 0; k < 3; ++k) {
    if (ms3) ms3[k] = idx->ms[k];
    if (launches3) launches3[k] = idx->launches[k];
  }
  if (reset) {
    for (int k = 0; k < 3; ++k) {
      idx->ms[k] = 0;
      idx->launches[k] = 0;
    }
  }
  return RAIRS_OK;
}

rairs_status rairs_profile_read_kernel(rairs_index_t idx, double* ms, int64_t* launches,
                                       int32_t reset) {
  if (!idx) return invalid("index is NULL");
  RAIRS_TRY(rairs_profile_read(idx, nullptr, nullptr, 0));  // drain pending events
  std::lock_guard<std::mutex> lock(idx->prof_mu);
  if (ms) *ms = idx->ms_kern;
  if (launches) *launches = idx->kern_launches;
  if (reset) {
    idx->ms_kern = 0;
    idx->kern_launches = 0;
  }
  return RAIRS_OK;
}

}  // extern "C"
