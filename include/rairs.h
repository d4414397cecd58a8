/*
 * rairs.h -- C ABI of the B200 (sm_100a) RAIRS search library (librairs.so).
 *
 * RAIRS = RAIR redundant assignment + SEIL shared-cell lists over an IVF-PQ
 * 4-bit fast-scan index with exact refine (arXiv 2601.07183).  This library
 * implements the query-time hot path (Alg. 2 RairsSearch, P:938-947,
 * with Alg. 5 SeilSearch P:1613-1645) and the index build that feeds it
 * (Alg. 1 AddVectors P:914-924, Alg. 3 RairAssign P:1194-1206, Alg. 4
 * SeilInsert P:1517-1555 in its cell-major form, DESIGN.md "Readings" R10).
 *
 * Conventions (all entry points):
 *  - Every call returns rairs_status; on failure rairs_last_error() returns a
 *    thread-local message valid until the next call on that thread.  Arguments
 *    are validated before any device work; a failed call leaves the index
 *    unchanged.  No C++ exception crosses this boundary.
 *  - "dev" pointers must be CUDA device (or managed) memory on the current
 *    device; a host pointer there is RAIRS_E_INVALID.  "host" pointers are
 *    ordinary (pageable or pinned) host memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  All device work is enqueued on it; device outputs are valid
 *    after the stream is synchronised.  Calls taking host outputs synchronise
 *    the stream before returning.
 *  - Ownership: the caller owns every buffer it passes; the library owns the
 *    index (device memory) and frees it in rairs_index_free().
 *  - Vector ids: the build takes the rows of ONE shard.  With shard_id = s and
 *    nshards = G (vector partition id mod G), local row
 *    r is global id r*G + s.  Results report global ids (int64), ordered by
 *    (squared L2 distance, id) ascending; missing results are (-1, +inf).
 *  - Concurrency: search/export calls are read-only on the index and may run
 *    concurrently on different streams; build/free are exclusive.
 */
#ifndef RAIRS_H_
#define RAIRS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rairs_index_s* rairs_index_t;

typedef enum {
  RAIRS_OK = 0,
  RAIRS_E_INVALID = -1,     /* bad argument (checked before any device work) */
  RAIRS_E_OOM = -2,         /* device allocation failed */
  RAIRS_E_CUDA = -3,        /* CUDA runtime / launch error */
  RAIRS_E_UNSUPPORTED = -4, /* valid but not implemented (e.g. nbits != 4) */
  RAIRS_E_INTERNAL = -5
} rairs_status;

typedef enum {
  RAIRS_ASSIGN_SINGLE = 0, /* each vector in its nearest list only (IVFPQfs) */
  RAIRS_ASSIGN_AIR = 1,    /* RAIR second list by the AIR metric (Alg. 3) */
  RAIRS_ASSIGN_SOAR = 2    /* SOARL2 comparison strategy:
                              Alg. 3 with loss ||r'||^2 + lambda*(r.r'/||r||)^2
                              (Table 2); the term is 0 when ||r|| = 0.
                              Use strict = 1 for the paper's always-two-lists
                              SOARL2 (and lambda = 0, strict = 1 for NaiveRA). */
} rairs_assign;

typedef struct {
  int32_t nlist;        /* number of IVF lists, 1 <= nlist <= 65536, nlist <= n */
  int32_t M;            /* PQ subquantizers; d % M == 0; d/M <= 8 */
  int32_t nbits;        /* must be 4 (16 sub-centroids) */
  int32_t assignment;   /* rairs_assign */
  float lambda;         /* AIR / SOAR lambda (AIR: P:1083-1084, 0.5) */
  int32_t n_cands;      /* N_CANDS (10); clamped to nlist */
  int32_t strict;       /* 0 = RAIR (non-strict), 1 = SRAIR */
  int32_t kmeans_iters; /* Lloyd iterations for training (default 25) */
  int64_t train_sample; /* max training rows; 0 = min(n, 256*nlist) */
  uint64_t seed;        /* training seed */
  int32_t shard_id;     /* this index's shard s (0 <= s < nshards) */
  int32_t nshards;      /* G >= 1 */
} rairs_build_params;

/* Fill `p` with the paper's defaults for the given shape. */
void rairs_default_params(rairs_build_params* p, int32_t nlist, int32_t M);

typedef struct {
  int64_t n;            /* local rows in this shard */
  int32_t d, nlist, M, M_pad;
  int64_t n_slots;      /* code slots incl. padding (multiple of 32 per list) */
  int64_t n_cells;      /* distinct (l1,l2) cells */
  int64_t n_refs;       /* SEIL references (cells with l1 < l2) */
  int64_t n_double;     /* vectors assigned to two lists */
  int32_t max_refs_per_list;
  int32_t shard_id, nshards;
  int64_t device_bytes; /* index memory on the device */
  int64_t n_live;       /* rows not deleted (n counts every row ever inserted) */
  int32_t has_ids;      /* 1: the index holds caller-supplied ids (see build) */
} rairs_index_info;

/* ---- training (B1/B3; not part of the bit-exact contract) ----------------
 * Coarse k-means (nlist centroids) + PQ codebook (M x 16 x d/M) trained on
 * the GPU from `base` (dev, [n x d] fp32 row-major).  Outputs are dev
 * buffers [nlist*d] and [M*16*(d/M)] fp32.  Deterministic for fixed seed. */
rairs_status rairs_train(const float* base, int64_t n, int32_t d,
                         const rairs_build_params* p, void* stream,
                         float* centroids_out, float* codebook_out);

/* ---- build (Alg. 1 AddVectors with Alg. 3 + Alg. 4) ---------------------
 * base: dev [n x d] fp32, the rows of shard p->shard_id.  centroids: dev
 * [nlist x d]; codebook: dev [M x 16 x d/M].  Assignment (fp64, O4) and PQ
 * encoding (fp64, O5) are bit-exact functions of (base, centroids, codebook).
 * The raw rows are copied into the index (refine store).
 * ids: dev [n] int64 caller-supplied vector ids (SPEC's VectorSet ids),
 * or NULL: then row r of shard s has id r * nshards + s.  Caller ids must be
 * unique and in [0, 2^32 - 2]; they are what searches return and what
 * rairs_remove_ids takes.  Ties in the exact distance are broken by the id
 * returned; the candidate stage breaks score ties by insertion order (R5).
 * Errors: n < 1, d < 1, nlist > n or > 65536, d % M, nbits != 4, n > 2^30;
 * non-finite base values or ids out of range / duplicated (INVALID,
 * checked on the device before anything is allocated). */
rairs_status rairs_build_from_trained(const float* base, int64_t n, int32_t d, const int64_t* ids,
                                      const float* centroids, const float* codebook,
                                      const rairs_build_params* p, void* stream,
                                      rairs_index_t* out);

/* rairs_train + rairs_build_from_trained (ids: as above). */
rairs_status rairs_build_index(const float* base, int64_t n, int32_t d, const int64_t* ids,
                               const rairs_build_params* p, void* stream,
                               rairs_index_t* out);

rairs_status rairs_index_free(rairs_index_t idx);
rairs_status rairs_index_get_info(rairs_index_t idx, rairs_index_info* out);

/* ---- updates ------------------------------------------
 * Insert a batch (batched SeilInsert, Alg. 4): x is a dev
 * [n_add x d] fp32 batch; its rows get local rows n .. n+n_add-1, i.e. global
 * ids (n+i)*nshards + shard_id (first_id, host, optional, receives the first).
 * Each row is assigned with the index's build parameters and trained state
 * (Alg. 3, O4, bit-exact to a fresh build), and the cell-major layout, codes
 * and list tables are rebuilt on the device (the paper appends blocks and
 * reference entries per batch; the result -- U(q), scores, ids,
 * DCO -- is the same as for an index built over all live rows at once).
 * x is copied; the caller keeps ownership. Row storage grows by >= 1/8.
 * Synchronises the device first: no search may run on this index concurrently.
 * ids: dev [n_add] int64 caller ids of the new rows -- required when the index
 * was built with ids (unique, not yet held, in [0, 2^32 - 2]), NULL otherwise.
 * Errors: n_add < 0, x not a device pointer or non-finite, ids given / missing /
 * invalid (INVALID); > 2^30 rows per shard or global ids >= 2^32 (UNSUPPORTED); OOM
 * (the index is unchanged). */
rairs_status rairs_add(rairs_index_t idx, const float* x, int64_t n_add, const int64_t* ids,
                       int64_t* first_id, void* stream);

/* Delete by id: ids is a dev [n_ids] int64 array of the ids the
 * index returns (caller ids if it was built with them, else global ids); ids this
 * shard does not hold (id % nshards != shard_id, or beyond its rows) and ids
 * already deleted are ignored. *n_removed (host, optional) = rows deleted now.
 * Deleted rows leave the layout (no tombstone is ever scored: DCO, U(q) and
 * results equal those of an index built over the remaining rows with their
 * original ids); their raw rows stay in the refine store. Synchronises the
 * device first: no search may run on this index concurrently.
 * Errors: n_ids < 0, ids not a device pointer (INVALID). */
rairs_status rairs_remove_ids(rairs_index_t idx, const int64_t* ids, int64_t n_ids,
                              int64_t* n_removed, void* stream);

/* ---- search (Alg. 2 RairsSearch, batched) --------------------------------
 * queries: dev [nq x d] fp32.  bigK = k*refine_factor.
 * out_ids: dev [nq x k] int64 global ids; out_dists: dev [nq x k] fp32
 * squared L2 (reading R14).  dco: dev [nq] int64 or NULL -- number of items
 * scored per query on this shard (= |U_s(q)|, O12).
 * Errors: nq < 0, k < 1, nprobe < 1 or > nlist, refine_factor < 1,
 * k*refine_factor > 2048 (UNSUPPORTED), nprobe > 1024 (UNSUPPORTED). */
rairs_status rairs_search(rairs_index_t idx, const float* queries, int64_t nq, int32_t k,
                          int32_t nprobe, int32_t refine_factor, int64_t* out_ids,
                          float* out_dists, int64_t* dco, void* stream);

/* Same as rairs_search with HOST buffers: copies queries host->device, runs
 * the search, copies results device->host and synchronises `stream`.  The
 * queries are copied on the index's copy stream into one of two device
 * buffers it reuses in turn (a buffer is refilled once the search that read
 * it is done), so a call's copy can overlap the previous call's search.  Host
 * buffers should be pinned (page-locked). */
rairs_status rairs_search_host(rairs_index_t idx, const float* queries_host, int64_t nq,
                               int32_t k, int32_t nprobe, int32_t refine_factor,
                               int64_t* out_ids_host, float* out_dists_host, void* stream);

/* rairs_search_host without the final synchronisation: everything is
 * enqueued (results land in the host buffers once `stream` has completed the
 * call's work); queries_host and the outputs must stay valid and untouched
 * until then.  Back-to-back calls on one stream overlap the next batch's
 * host->device copy with the current batch's search.  Argument errors are
 * reported synchronously; on an error the stream is synchronised. */
rairs_status rairs_search_host_async(rairs_index_t idx, const float* queries_host, int64_t nq,
                                     int32_t k, int32_t nprobe, int32_t refine_factor,
                                     int64_t* out_ids_host, float* out_dists_host, void* stream);

/* Per-stage outputs for parity tests (dev pointers, any may be NULL):
 * probes [nq x nprobe] i32 (O1); lut_q [nq x M x 16] u8, lut_a/lut_b [nq] f32
 * (O2); cand_ids/cand_scores [nq x bigK] u32 (O9, global ids, padded with
 * 0xFFFFFFFF); dco [nq] i64; out_ids/out_dists as rairs_search. */
rairs_status rairs_search_debug(rairs_index_t idx, const float* queries, int64_t nq,
                                int32_t k, int32_t nprobe, int32_t refine_factor,
                                int32_t* probes, uint8_t* lut_q, float* lut_a, float* lut_b,
                                uint32_t* cand_ids, uint32_t* cand_scores, int64_t* dco,
                                int64_t* out_ids, float* out_dists, void* stream);

/* ---- shard merge (K7) -----------------------------------------------------
 * ids/dists: dev [G x nq x k] (per-shard results, e.g. after an NCCL
 * all_gather); ids are full 64-bit values (any id >= 0; negative = padding).
 * Output: dev [nq x k], the first k of the union by (dist, id), padded with
 * (-1, +inf).  O11.  G * k <= 16384 (UNSUPPORTED otherwise). */
rairs_status rairs_merge_topk(const int64_t* ids, const float* dists, int32_t G, int64_t nq,
                              int32_t k, int64_t* out_ids, float* out_dists, void* stream);

/* ---- exact k-NN ground truth (B7) ------------------------------------------
 * First K rows of base by (D64(q,x), id) (O13) -- fp64 ordered distances.
 * base: dev [n x d], queries: dev [nq x d]; out: dev [nq x K] int64 ids and
 * fp64 distances (either may be NULL).  K <= 256. */
rairs_status rairs_exact_knn(const float* base, int64_t n, int32_t d, const float* queries,
                             int64_t nq, int32_t K, int64_t* out_ids, double* out_d64,
                             void* stream);

/* ---- exports for parity tests ---------------------------------------------
 * rairs_export_trained: dev [nlist x d] centroids, dev [M x 16 x d/M] codebook.
 * rairs_export_assignment: dev [n] l1, l2 (sorted pair) and dev [n x M]
 *   unpacked codes per local row (any may be NULL).
 * rairs_export_layout: cell-major SEIL (dev, any may be NULL):
 *   own_off/own_cnt [nlist] i64 (slot offset, item count of list l's owned
 *   region = its cells (l, j>=l)); ref_ptr [nlist+1] i64 CSR over lists;
 *   ref_owner [n_refs] i32, ref_start [n_refs] i64 (slot), ref_cnt [n_refs] i64;
 *   slot_rows [n_slots] u32 (local row, 0xFFFFFFFF = padding). */
rairs_status rairs_export_trained(rairs_index_t idx, float* centroids, float* codebook,
                                  void* stream);
rairs_status rairs_export_assignment(rairs_index_t idx, int32_t* l1, int32_t* l2,
                                     uint8_t* codes, void* stream);
rairs_status rairs_export_layout(rairs_index_t idx, int64_t* own_off, int64_t* own_cnt,
                                 int64_t* ref_ptr, int32_t* ref_owner, int64_t* ref_start,
                                 int64_t* ref_cnt, uint32_t* slot_rows, void* stream);

/* ---- coarse stage mode ------------------------------------------------------
 * 0 = auto (tensor-core TF32 filter + fp64 certification when d % 4 == 0 and
 * nlist >= 64, else exact fp64); 1 = exact fp64 only; 2 = tensor-core path
 * whenever d % 4 == 0.  Every mode returns exactly the O1 probe set.
 * rairs_certify_fallbacks: queries whose TF32 filter could not be certified
 * and were recomputed exactly (host out; synchronises the device). */
rairs_status rairs_set_coarse_mode(rairs_index_t idx, int32_t mode);
rairs_status rairs_certify_fallbacks(rairs_index_t idx, int64_t* count, int32_t reset);

/* Search statistics since the index was built or last reset (SURVEY §8(b)
 * rairs_stats): searches and queries run, items scored (DCO, O12 / R17, summed
 * over queries and shards' calls on this index), candidates refined (exact
 * distances computed, A7), queries whose coarse stage fell back to the exact
 * kernel, and stage times in ms (CUDA events; 0 unless rairs_profile_enable).
 * Synchronises the device.  reset != 0 zeroes everything after reading. */
typedef struct {
  int64_t searches, queries;
  int64_t dco_total, refine_total, certify_fallbacks;
  double ms_coarse, ms_scan, ms_refine;
} rairs_stats;
rairs_status rairs_get_stats(rairs_index_t idx, rairs_stats* out, int32_t reset);

/* ---- scan mode --------------------------------------------------------------
 * 0 = auto (list-major when the batch probes each list >= 3 times on average
 * and its limits hold, else query-major), 1 = query-major fast scan (one warp
 * per query: LUT rows in registers, prmt lookups, dp4a sums over an 8-item
 * nibble-group code layout, SEIL range list, exact top-bigK), 2 = list-major:
 * (query, probe) pairs grouped by list, scores of each list's items for all its
 * queries as one exact u8 x u8 -> s32 tcgen05 contraction of one-hot codes and
 * quantised LUTs (the paper's query-batch cache optimisation).
 * Both modes produce identical candidates. */
rairs_status rairs_set_scan_mode(rairs_index_t idx, int32_t mode);

/* ---- SEIL list layout (NEXT-2) ----------------------------------------------
 * 0 = cell-major (default, reading R10): list l owns its cells (l, j >= l)
 * contiguously, remainders included, and list j holds (owner, slot, count)
 * references to the cells (i < j, j); every vector is stored once.
 * 1 = paper-literal SEIL (Alg. 4 SeilInsert): per
 * cell floor(n/32) 32-item blocks stored once in list i and referenced from
 * list j, the n % 32 remainder items duplicated into both lists'
 * miscellaneous areas with the other list id embedded; searched per Alg. 5
 * (SeilSearch) with the lists visited in ascending id (reading
 * R9): references skipped when their owner was visited, misc items dropped
 * after scoring when their other list was visited.  Same candidates and
 * results as layout 0; the per-query DCO is the paper's DCO_paperSEIL (misc
 * items scored in both lists).  Layout 1 is built from layout 0 when selected
 * (host-side map + one device gather; synchronous, extra device memory about
 * n * (M/2 + 8) bytes), rebuilt by rairs_add / rairs_remove_ids while
 * selected, freed when 0 is selected; searches then take the query-major
 * scan.  2 = both layouts kept: query-major scans read the paper-literal one
 * (its remainders sit in contiguous misc areas instead of many short
 * references, so fewer partially filled 8-item groups are scanned: c4 scan
 * -6 %), list-major scans (rairs_set_scan_mode) the cell-major one.
 * 3 = hybrid (not in the paper; same results, U(q) of R9): query-major scans
 * read, per list, its cell-major owned range followed by copies of the cross
 * cells (i < l, l) with fewer than 8 items (one nibble group), each dropped
 * after scoring when its owner i was probed (RemoveVectorIfVisited, Alg. 5
 * line 16); larger cells stay references.  DCO = the cell-major DCO + the
 * copied items whose owner was also probed.  List-major scans read the
 * cell-major layout.
 * Errors: RAIRS_E_INVALID (NULL index, layout not 0..3), RAIRS_E_OOM,
 * RAIRS_E_CUDA. */
rairs_status rairs_set_seil_layout(rairs_index_t idx, int32_t layout);

/* ---- stage timing (CUDA events on the search stream) ----------------------
 * When enabled, every search records events around its stages on its stream;
 * rairs_profile_read synchronises and returns the accumulated milliseconds
 * and launch counts since the last reset:
 *   ms[0] coarse (probe selection), ms[1] scan (LUT + SEIL work list +
 *   fast-scan + top-bigK), ms[2] refine; launches[i] likewise. */
rairs_status rairs_profile_enable(rairs_index_t idx, int32_t on);
rairs_status rairs_profile_read(rairs_index_t idx, double* ms3, int64_t* launches3,
                                int32_t reset);
/* The dominant scan kernel's own device time (fs_scan_kernel on the
 * query-major path, lm_tensor_kernel on the list-major one) from events
 * recorded right around its launch while profiling is enabled: accumulated
 * milliseconds (*ms) and launches (*launches) since the last reset. */
rairs_status rairs_profile_read_kernel(rairs_index_t idx, double* ms, int64_t* launches,
                                       int32_t reset);
/* Number of CUDA kernels the library launched for searches on this index
 * since the last reset (host-side count, always on): *kernels receives it;
 * reset != 0 zeroes the counter. RAIRS_E_INVALID on NULL arguments. */
rairs_status rairs_profile_kernels(rairs_index_t idx, int64_t* kernels, int32_t reset);

/* Which kernels a search of nq queries with these parameters would use (no
 * device work): *coarse_path = 1 exact fp64 probe kernel, 2 tensor-core TF32
 * filter + certification; *scan_path = 1 SIMT query-major scan, 2 list-major
 * tcgen05 scan (scan mode auto: list-major when nq*nprobe >= 3*nlist, i.e. a
 * probed list is shared by several queries, and its limits hold). Either
 * pointer may be NULL. Same validation as rairs_search. */
rairs_status rairs_search_plan(rairs_index_t idx, int64_t nq, int32_t k, int32_t nprobe,
                               int32_t refine_factor, int32_t* coarse_path, int32_t* scan_path);

const char* rairs_last_error(void);
const char* rairs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RAIRS_H_ */
