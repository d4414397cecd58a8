// index.cuh -- device-resident RAIRS index (one shard) and kernel launchers.
#pragma once

#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace rairs {
}  // namespace rairs

namespace rairs {
// batches of at least LM_NCH x LM_OVERLAP_MIN_Q queries run select + refine as
// LM_NCH concurrent query chunks on the index's auxiliary streams
constexpr int64_t LM_OVERLAP_MIN_Q = 2048;
constexpr int LM_NCH = 2;  // 4 measured: 19.12M vs 19.2-19.3M QPS
}  // namespace rairs

struct rairs_index_s {
  int device = 0;
  int64_t n = 0;            // local rows (inserted so far, deleted ones included)
  int64_t n_live = 0;       // rows not deleted (the ones the layout holds)
  int64_t cap_rows = 0;     // allocated rows of X / l1 / l2
  // deletion tombstones (NEXT-3): bit r of live_bits[r/32] = row r is live;
  // NULL until the first rairs_remove_ids (then every row < n is live)
  uint32_t* live_bits = nullptr;
  // caller-supplied ids (labels.cu): labels[r] of local row r (NULL: the
  // internal global ids r * G + shard are the ids), and the sorted
  // (label, row) table for deletes by label
  uint32_t* labels = nullptr;
  uint32_t* lab_sorted = nullptr;
  uint32_t* lab_rows = nullptr;
  int d = 0, nlist = 0, M = 0, M_pad = 0, dsub = 0;
  int shard_id = 0, nshards = 1;
  rairs_build_params params{};

  // trained state (fp32)
  float* centroids = nullptr;   // [nlist x d]
  float* codebook = nullptr;    // [M x 16 x dsub]
  // refine store: raw rows in insertion order
  float* X = nullptr;           // [n x d]
  // assignment (sorted pair per local row)
  int32_t* l1 = nullptr;
  int32_t* l2 = nullptr;

  // cell-major SEIL layout
  int64_t n_slots = 0;          // multiple of 32 per list
  uint8_t* codes = nullptr;     // [n_slots/32][M_pad/16][32 lanes][8 B]
  uint32_t* slot_rows = nullptr;  // [n_slots] local row or kSlotPad
  uint32_t* own_off = nullptr;  // [nlist] slot offset of list l's owned region
  uint32_t* own_cnt = nullptr;  // [nlist] items in it
  uint32_t* ref_ptr = nullptr;  // [nlist+1] CSR of references per list
  int32_t* ref_owner = nullptr; // [n_refs]
  uint32_t* ref_start = nullptr;  // [n_refs] slot
  uint32_t* ref_cnt = nullptr;  // [n_refs]
  int64_t n_refs = 0, n_cells = 0, n_double = 0;
  // coarse stage (K1/K2): fp32 ||c||^2, max ||c||, mode 0 auto / 1 exact / 2 tensor core
  float* cnorm = nullptr;
  double cmax = 0.0;
  int coarse_mode = 0;
  unsigned* certify_fallbacks = nullptr;  // device counter
  // rairs_get_stats: device counters [0] items scored (DCO), [1] candidates
  // refined; host counters of searches and queries
  unsigned long long* counters = nullptr;
  // host counters: searches may run concurrently on different streams (rairs.h)
  std::atomic<int64_t> n_searches{0}, n_queries{0};
  // list-major scan (NEXT-1): mode 0 auto / 1 SIMT query-major / 2 list-major
  int scan_mode = 0;
  uint32_t* list_items = nullptr;    // [nlist] N_l = own_cnt + sum of ref_cnt
  uint32_t* ref_item_off = nullptr;  // [n_refs] item offset inside the list-task
  int64_t max_list_items = 0;
  uint64_t* list_base = nullptr;     // [nlist + 1] prefix of N_l (into list_ids)
  uint32_t* list_ids = nullptr;      // [sum N_l] global id of item i of list-task l
  uint32_t* lm_order = nullptr;      // [nlist] lists by descending N_l (claim order)
  int64_t sum_list_items = 0;        // sum of N_l (mean list-task length = this / nlist)
  int max_refs = 0;
  // query-major register-LUT fast scan (fastscan_kernels.cu): the codes again in
  // the 8-item nibble-group layout, the codebook transposed [16][dsub][M], and
  // self-resetting query-claim counters (one pair per concurrent search slot)
  uint8_t* codes_g = nullptr;
  float* cbT = nullptr;
  unsigned* fs_ctr = nullptr;
  std::atomic<unsigned> fs_slot{0};
  int64_t fs_bytes = 0;
  // paper-literal SEIL layout (Alg. 4; seil_paper.cu), built on
  // demand: per list l, p_off[l] = region start (32-aligned), p_shared[l]
  // items in shared 32-item blocks, then p_misc[l] misc items (p_other: the
  // other list id embedded with each misc item, kNoOther in shared blocks);
  // p_ref_start / p_ref_cnt: the shared blocks each reference (ref_ptr /
  // ref_owner order) points at.  seil_layout 1 = searches use it (query-major
  // only), 2 = query-major searches use it, list-major ones the cell-major layout.
  // 3 = the hybrid layout in the same arrays (seil_paper.cu): each list's
  // cell-major owned range unchanged, then misc copies of the cross cells
  // (i < l, l) smaller than one 8-item group; larger cells stay references.
  // p_kind = the layout the p_* arrays hold (1 paper-literal, 3 hybrid).
  int seil_layout = 0;
  int p_kind = 0;
  uint8_t* p_codes_g = nullptr;
  uint32_t* p_slot_rows = nullptr;
  uint32_t* p_other = nullptr;
  uint32_t* p_off = nullptr;
  uint32_t* p_shared = nullptr;
  uint32_t* p_misc = nullptr;
  uint32_t* p_ref_start = nullptr;
  uint32_t* p_ref_cnt = nullptr;
  int64_t p_slots = 0, p_bytes = 0;
  int64_t device_bytes = 0;
  int64_t layout_bytes = 0, lm_bytes = 0;  // parts of device_bytes rebuilt by add/remove
  // two auxiliary streams + fork/join events (list-major select/refine overlap)
  cudaStream_t aux[rairs::LM_NCH] = {};
  cudaEvent_t aux_ev[1 + 2 * rairs::LM_NCH] = {};
  std::mutex* aux_mu = nullptr;  // one search at a time enqueues on the aux streams
  // host-query copy stream + events (rairs_search_host: chunked H2D / coarse overlap)
  cudaStream_t h2d = nullptr;
  cudaEvent_t h2d_ev[2] = {};
  // two device query buffers for host searches, reused in turn: a buffer is
  // refilled (on the copy stream) only after the search that read it is done
  // (hq_ev, recorded on the search stream) -- no per-call allocation, no host sync
  float* hq_buf[2] = {nullptr, nullptr};
  size_t hq_cap[2] = {0, 0};
  cudaEvent_t hq_ev[2] = {nullptr, nullptr};
  int hq_next = 0;
  std::mutex* hq_mu = nullptr;

  // stage profiling (CUDA events on the search stream); prof_mu guards the
  // event vectors and sums (concurrent searches)
  bool prof = false;
  struct EvSet { cudaEvent_t e[6]; bool kern = false; };  // e[4..5]: the dominant scan kernel
  std::mutex prof_mu;
  std::vector<EvSet> pending;
  std::vector<cudaEvent_t> pool;
  double ms[3] = {0, 0, 0};
  double ms_kern = 0;
  int64_t kern_launches = 0;
  std::atomic<int64_t> launches[3] = {{0}, {0}, {0}};
  std::atomic<int64_t> kernels{0};  // kernels launched by searches (rairs_profile_kernels)
};

namespace rairs {

// ---- build-side launchers (build_kernels.cu) -------------------------------
// Exact fp64 nearest-"lists" selection: for each of `rows` rows of X (row
// major [rows x d]) the first L of `nl` rows of C by (D64, index).
//   mode 0: write out_idx [rows x L] (i32) and optionally out_d64 [rows x L].
//   mode 1: AIR assignment (Alg. 3): L = n_cands; writes l1/l2 sorted pair.
//   mode 2: single assignment: l1 = l2 = nearest.
struct ProbeArgs {
  const float* X;
  int64_t rows;
  int d;
  const float* C;
  int64_t nl;
  int L;
  int mode;
  double lambda;
  int strict;
  int32_t* out_idx;    // mode 0 (i32) or NULL
  int64_t* out_idx64;  // mode 0 (i64) or NULL
  double* out_d64;     // mode 0, optional
  int32_t* l1;         // modes 1/2
  int32_t* l2;
  const int32_t* only_flagged;  // mode 0: process only row groups with a flagged row
  bool flag_count = false;      // only_flagged[rows] = number of flagged rows (0: exit at once)
};
rairs_status launch_probe_exact(const ProbeArgs& a, cudaStream_t s);
// every row through the split exact path when rows < PX_CAP and nlist is large
// (small search batches: no TF32 GEMM / certificate); *done = false otherwise
rairs_status launch_probe_split_all(const ProbeArgs& a, cudaStream_t s, bool* done);
// search batches of at most this many queries take launch_probe_split_all
// (RAIRS_COARSE_SMALL; 0 disables)
int coarse_small_rows();
// few flagged rows x many lists: split exact fallback (clears the flags it handles).
// prepare (before the certify kernel, which appends the flagged rows to
// b.list / *count itself), launch (programmatic dependent launches), free.
constexpr int PX_CAP = 2048;  // rows the split path takes per call (the rest: tiled kernel)
struct ProbeSplitBufs {
  uint32_t* list = nullptr;
  uint64_t* tk = nullptr;
  uint32_t* ti = nullptr;
  int per = 0, npow_s = 0, npow_m = 0;
  size_t sm_s = 0, sm_m = 0;
  bool on = false;
};
rairs_status probe_split_prepare(const ProbeArgs& a, ProbeSplitBufs& b, cudaStream_t s);
rairs_status probe_split_launch(const ProbeArgs& a, const ProbeSplitBufs& b, const uint32_t* count,
                                int32_t* flags, cudaStream_t s);
void probe_split_free(ProbeSplitBufs& b, cudaStream_t s);

rairs_status train_kmeans(const float* X, int64_t n, int d, int k, int iters, uint64_t seed,
                          int64_t max_train, float* centroids_out, cudaStream_t s);
rairs_status train_pq(const float* X, int64_t n, int d, int M, int iters, uint64_t seed,
                      int64_t max_train, float* codebook_out, cudaStream_t s);
rairs_status build_layout(rairs_index_s* idx, cudaStream_t s);
rairs_status export_codes(const rairs_index_s* idx, uint8_t* codes, cudaStream_t s);
rairs_status export_layout64(const rairs_index_s* idx, int64_t* own_off, int64_t* own_cnt,
                             int64_t* ref_ptr, int32_t* ref_owner, int64_t* ref_start,
                             int64_t* ref_cnt, uint32_t* slot_rows, cudaStream_t s);

// ---- caller-supplied ids (labels.cu) -------------------------------------------
// every id in [0, 2^32 - 2], no duplicates, none already held by idx (idx may be NULL)
rairs_status labels_validate(const rairs_index_s* idx, const int64_t* ids, int64_t m, cudaStream_t s);
// labels[row0 .. row0+m) = ids, then rebuild the sorted (label, row) table
rairs_status labels_store(rairs_index_s* idx, const int64_t* ids, int64_t row0, int64_t m, cudaStream_t s);
// labels -> internal global ids (-1 if not held)
rairs_status labels_to_gids(const rairs_index_s* idx, const int64_t* ids, int64_t m, int64_t* gids,
                            cudaStream_t s);

// ---- coarse stage (coarse_kernels.cu) ---------------------------------------
rairs_status coarse_prepare(rairs_index_s* idx, cudaStream_t s);
bool coarse_fused_ok(const rairs_index_s* idx, int L);
// first L lists of each row of X by (D64, l): mode 0 -> out_idx [rows x L];
// mode 1 -> RAIR pair (l1, l2); mode 2 -> single (l1 = l2 = nearest).
rairs_status launch_coarse_fused(const rairs_index_s* idx, const float* X, int64_t rows, int L,
                                 int mode, double lambda, int strict, int32_t* out_idx,
                                 int32_t* l1, int32_t* l2, unsigned* nflag, cudaStream_t s);

// ---- list-major tensor-core scan (listmajor_kernels.cu) ----------------------
rairs_status listmajor_prepare(rairs_index_s* idx, cudaStream_t s);
bool listmajor_ok(const rairs_index_s* idx, int64_t nq, int nprobe, int bigK);
struct SearchArgs;
rairs_status launch_listmajor(const rairs_index_s* idx, const SearchArgs& a, cudaStream_t s);


// ---- search-side launchers (search_kernels.cu) -----------------------------
struct SearchArgs {
  const float* queries;
  int64_t nq;
  int k, nprobe, refine_factor;
  int32_t* probes;       // [nq x nprobe] (workspace or debug output)
  uint64_t* cand_keys;   // [nq x bigK]   (workspace)
  int64_t* dco;          // [nq] or NULL
  uint8_t* lut_q;        // debug [nq x M x 16] or NULL
  float* lut_a;
  float* lut_b;
  int64_t* out_ids;
  float* out_dists;
  // list-major path: also run the refine (overlapped with the selection, in
  // query halves on the index's two auxiliary streams); record ev_selected on
  // the search stream once every query's candidates are final (stage timing)
  bool fused_refine = false;
  cudaEvent_t ev_selected = nullptr;
  unsigned long long* counters = nullptr;  // idx->counters (DCO, refined) or NULL
  // candidate keys wanted in (s, id) order (debug outputs); otherwise each
  // query's bigK keys may be written in any order (the refine ranks them)
  bool sorted_keys = false;
  const uint4* luts = nullptr;  // fast scan: [nq][M_pad] LUT rows workspace (16 B each)
  // profiling: events recorded right around the dominant scan kernel's launch
  // (fs_scan_kernel / lm_tensor_kernel); *kev_used set when recorded
  cudaEvent_t kev[2] = {nullptr, nullptr};
  bool* kev_used = nullptr;
};
// query-major register-LUT fast scan (fastscan_kernels.cu): A3-A6 fused
rairs_status fastscan_prepare(rairs_index_s* idx, cudaStream_t s);
struct FsExtra {
  int nprobe_eff = 0;                 // > 0: scan only the first nprobe_eff probes of each row
  const uint32_t* qlist = nullptr;    // scan only queries qlist[0 .. *qcount) (device)
  const uint32_t* qcount = nullptr;
  uint32_t* tau_out = nullptr;        // threshold mode (see FsArgs::tau_out)
  bool luts_ready = false;            // a.luts already holds every query's LUT
  uint64_t* defer_buf = nullptr;      // deferred finish workspace [nq][fastscan_cap(bigK, M_pad)]
  uint32_t* defer_n = nullptr;        // [nq]
};
bool fastscan_order_on();
int fastscan_parts(const rairs_index_s* idx, int64_t nq, int nprobe);  // work items per query (defer buffers: nq x parts)
// paper-literal SEIL layout (seil_paper.cu)
rairs_status seil_paper_prepare(rairs_index_s* idx, cudaStream_t s);
void seil_paper_free(rairs_index_s* idx);
int fastscan_cap(int bigK, int M_pad);
rairs_status launch_fastscan(rairs_index_s* idx, const SearchArgs& a, cudaStream_t s,
                             const FsExtra& ex = FsExtra{});
rairs_status launch_refine(const rairs_index_s* idx, const SearchArgs& a, cudaStream_t s);
rairs_status launch_merge(const int64_t* ids, const float* dists, int G, int64_t nq, int k,
                          int64_t* out_ids, float* out_dists, cudaStream_t s);
rairs_status launch_split_keys(const uint64_t* keys, int64_t count, uint32_t* ids,
                               uint32_t* scores, cudaStream_t s);

}  // namespace rairs
