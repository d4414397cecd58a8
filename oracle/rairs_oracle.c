/*
 * rairs_oracle.c -- plain, slow, obviously-correct CPU oracle for the RAIRS
 * query-time hot path (arXiv 2601.07183).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2601_07183_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Compiled with  gcc -O2 -ffp-contract=off -fopenmp  (x86-64 SSE2 scalar
 * IEEE single/double, round-to-nearest-even, no FMA contraction).
 *
 * Every function cites the passage it follows:
 *   P:n  = /root/reference/PAPER.md line n,  S:n = SPEC.md line n,
 *   O1..O13, R1..R21 = SURVEY.md §8(c) definitions / readings (restated in
 *   DESIGN.md "Readings").
 * "fp64 ordered sum" = operands widened exactly to double, summed left to
 * right over t, every op rounded to nearest, no FMA.
 *
 * Parity pins live in tests/test_oracle_*.py (brute force, closed forms,
 * invariants, library routines).  Parity-unpinned functions: oracle_kmeans /
 * oracle_pq_train (training, O3) are outside the bit-exact contract; they are
 * pinned only by invariants (nlist=1 -> mean, objective non-increasing).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL -1
#define OR_ENOMEM -2

/* ------------------------------------------------------------------ utils */

int oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* splitmix64: seeded PRNG used only by the training routines (O3). */
static uint64_t sm64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* O1 / O13 distance: D64(v,c) = sum_t ((double)v_t - (double)c_t)^2, fp64
 * ordered (P:679-682 squared Euclidean distance). */
static double d64(const float* a, const float* b, int d) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) {
        double df = (double)a[t] - (double)b[t];
        double sq = df * df;
        s = s + sq;
    }
    return s;
}

typedef struct { double dist; int64_t id; } dist_id;

static int cmp_dist_id(const void* pa, const void* pb) {
    const dist_id* a = (const dist_id*)pa;
    const dist_id* b = (const dist_id*)pb;
    if (a->dist < b->dist) return -1;
    if (a->dist > b->dist) return 1;
    return (a->id < b->id) ? -1 : (a->id > b->id) ? 1 : 0;
}

/* ------------------------------------------------------------ O1: probes */
/* FindNearestLists (Alg.2 line 5; "top-nprobe nearest
 * lists"): order all lists by (D64(q,c_l), l) -- ties by list id --
 * and return the first nprobe.  Plain definition: full sort of nlist. */
static void probe_one(const float* q, int d, const float* cent, int nlist,
                      int nprobe, dist_id* scratch, int32_t* out) {
    for (int l = 0; l < nlist; ++l) {
        scratch[l].dist = d64(q, cent + (int64_t)l * d, d);
        scratch[l].id = l;
    }
    qsort(scratch, (size_t)nlist, sizeof(dist_id), cmp_dist_id);
    for (int p = 0; p < nprobe; ++p) out[p] = (int32_t)scratch[p].id;
}

int oracle_probe(const float* q, int64_t nq, int d, const float* cent, int nlist,
                 int nprobe, int32_t* probes) {
    if (nprobe < 1 || nprobe > nlist || d < 1) return OR_EINVAL;
    int err = OR_OK;
#pragma omp parallel
    {
        dist_id* scratch = (dist_id*)malloc(sizeof(dist_id) * (size_t)nlist);
        if (!scratch) {
#pragma omp atomic write
            err = OR_ENOMEM;
        } else {
#pragma omp for schedule(dynamic, 4)
            for (int64_t i = 0; i < nq; ++i)
                probe_one(q + i * d, d, cent, nlist, nprobe, scratch, probes + i * nprobe);
        }
        free(scratch);
    }
    return err;
}

/* ---------------------------------------------------- O4: AIR assignment */
/* RairAssign (Alg.3):
 *   cand = first N_C lists of O1 applied to v          (line 2)
 *   residual0 = centroid0 - v, residual = centroid - v (lines 3-7, fp64)
 *   loss[i] = L2sqr(residual) + lambda * InnerProd(residual0, residual) (line 8)
 *   listID1 = cand[0]; start = strict ? 1 : 0          (lines 9-10)
 *   listID2 = cand[first argmin loss[start..N_C-1]]    (line 11; ties -> nearer)
 *   return sorted pair                                  (line 12)
 * mode 0 = single assignment (l1 = l2 = nearest list).
 * mode 2 = SOARL2: the same steps with line 8's loss
 *   replaced by Table 2's SOAR formula:
 *   loss[i] = L2sqr(residual) + lambda * (InnerProd(residual0, residual) / ||residual0||)^2,
 *   ||residual0|| = sqrt of the ordered fp64 sum of squares; the projection term
 *   is 0 when ||residual0|| = 0 (then residual0 . residual = 0). */
static void assign_one(const float* v, int d, const float* cent, int nlist, int mode,
                       double lambda, int n_cands, int strict, dist_id* scratch,
                       double* r0, double* r, int32_t* o1, int32_t* o2) {
    for (int l = 0; l < nlist; ++l) {
        scratch[l].dist = d64(v, cent + (int64_t)l * d, d);
        scratch[l].id = l;
    }
    qsort(scratch, (size_t)nlist, sizeof(dist_id), cmp_dist_id);
    int c0 = (int)scratch[0].id;
    if (mode == 0) { *o1 = c0; *o2 = c0; return; }
    const float* cen0 = cent + (int64_t)c0 * d;
    for (int t = 0; t < d; ++t) r0[t] = (double)cen0[t] - (double)v[t];
    double rr = 0.0;
    for (int t = 0; t < d; ++t) { double sq = r0[t] * r0[t]; rr = rr + sq; }
    int start = strict ? 1 : 0;
    int best = -1;
    double best_loss = 0.0;
    for (int i = start; i < n_cands; ++i) {
        const float* ci = cent + scratch[i].id * d;
        for (int t = 0; t < d; ++t) r[t] = (double)ci[t] - (double)v[t];
        double l2sqr = 0.0, ip = 0.0;
        for (int t = 0; t < d; ++t) { double sq = r[t] * r[t]; l2sqr = l2sqr + sq; }
        for (int t = 0; t < d; ++t) { double pr = r0[t] * r[t]; ip = ip + pr; }
        double loss;
        if (mode == 2) {
            double proj = rr == 0.0 ? 0.0 : ip / sqrt(rr);
            loss = rr == 0.0 ? l2sqr : l2sqr + lambda * (proj * proj);
        } else {
            double term = lambda * ip;
            loss = l2sqr + term;
        }
        if (best < 0 || loss < best_loss) { best = i; best_loss = loss; }
    }
    int c2 = (int)scratch[best].id;
    *o1 = c0 < c2 ? c0 : c2;
    *o2 = c0 < c2 ? c2 : c0;
}

int oracle_assign(const float* x, int64_t n, int d, const float* cent, int nlist,
                  int mode, double lambda, int n_cands, int strict,
                  int32_t* l1, int32_t* l2) {
    if (nlist < 1 || d < 1 || mode < 0 || mode > 2) return OR_EINVAL;
    if (n_cands > nlist) n_cands = nlist;                 /* N_C = min(10, nlist) */
    if (n_cands < 1 || (strict && n_cands < 2 && mode != 0)) return OR_EINVAL;
    int err = OR_OK;
#pragma omp parallel
    {
        dist_id* scratch = (dist_id*)malloc(sizeof(dist_id) * (size_t)nlist);
        double* r0 = (double*)malloc(sizeof(double) * (size_t)d);
        double* r = (double*)malloc(sizeof(double) * (size_t)d);
        if (!scratch || !r0 || !r) {
#pragma omp atomic write
            err = OR_ENOMEM;
        } else {
#pragma omp for schedule(dynamic, 64)
            for (int64_t i = 0; i < n; ++i)
                assign_one(x + i * d, d, cent, nlist, mode, lambda, n_cands, strict,
                           scratch, r0, r, l1 + i, l2 + i);
        }
        free(scratch); free(r0); free(r);
    }
    return err;
}

/* ---------------------------------------------------------- O5: encode */
/* PQ encoding ("encodes a vector as its sub-vectors' cluster IDs"):
 * code_m(x) = first j minimising sum_t ((double)x_{m*dsub+t} - (double)C[m][j][t])^2
 * (fp64 ordered; ties -> smaller j).  codes is [n x M] unpacked u8. */
int oracle_encode(const float* x, int64_t n, int d, const float* codebook, int M,
                  uint8_t* codes) {
    if (M < 1 || d % M != 0) return OR_EINVAL;
    int dsub = d / M;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        for (int m = 0; m < M; ++m) {
            const float* xs = x + i * d + (int64_t)m * dsub;
            int bj = 0;
            double bd = 0.0;
            for (int j = 0; j < 16; ++j) {
                double dd = d64(xs, codebook + ((int64_t)m * 16 + j) * dsub, dsub);
                if (j == 0 || dd < bd) { bj = j; bd = dd; }
            }
            codes[i * M + m] = (uint8_t)bj;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------- O2: LUT + uint8 */
/* ComputeLookupTable (LUT definition P:711-716 "the squared distance
 * between the query sub-vector and all cluster centroids"), with the uint8
 * quantisation reading R3:
 *  1. T[m][j] = sum_{t<dsub} (q_{m dsub+t} - C[m][j][t])^2 in fp32, each
 *     sub/mul/add rounded to nearest, ascending t, no FMA (R2).
 *  2. mn_m = min_j T[m][j];  S = max_m (max_j T[m][j] - mn_m).
 *  3. a = 255/S (fp32 division); if S == 0: all Qv = 0 and a = 1.
 *  4. Qv[m][j] = min(255, rint((T[m][j] - mn_m) * a)), half-to-even.
 *  5. b = sum_m mn_m (fp32, ascending m).  Estimate = b + s/a (info only). */
static void lut_one(const float* q, int d, const float* codebook, int M,
                    float* T, uint8_t* Qv, float* a_out, float* b_out) {
    int dsub = d / M;
    for (int m = 0; m < M; ++m) {
        for (int j = 0; j < 16; ++j) {
            const float* c = codebook + ((int64_t)m * 16 + j) * dsub;
            float acc = 0.0f;
            for (int t = 0; t < dsub; ++t) {
                float diff = q[m * dsub + t] - c[t];
                float sq = diff * diff;
                acc = acc + sq;
            }
            T[m * 16 + j] = acc;
        }
    }
    float S = 0.0f, b = 0.0f;
    float* mn = (float*)malloc(sizeof(float) * (size_t)M);
    for (int m = 0; m < M; ++m) {
        float lo = T[m * 16], hi = T[m * 16];
        for (int j = 1; j < 16; ++j) {
            if (T[m * 16 + j] < lo) lo = T[m * 16 + j];
            if (T[m * 16 + j] > hi) hi = T[m * 16 + j];
        }
        mn[m] = lo;
        float span = hi - lo;
        if (span > S) S = span;
    }
    for (int m = 0; m < M; ++m) b = b + mn[m];
    float a = 1.0f;
    if (S > 0.0f) a = 255.0f / S;
    for (int m = 0; m < M; ++m) {
        for (int j = 0; j < 16; ++j) {
            int v = 0;
            if (S > 0.0f) {
                float t1 = T[m * 16 + j] - mn[m];
                float t2 = t1 * a;
                float r = nearbyintf(t2);          /* default mode: half-to-even */
                v = (int)r;
                if (v > 255) v = 255;
            }
            Qv[m * 16 + j] = (uint8_t)v;
        }
    }
    free(mn);
    *a_out = a;
    *b_out = b;
}

int oracle_lut(const float* q, int64_t nq, int d, const float* codebook, int M,
               uint8_t* Qv, float* a, float* b) {
    if (M < 1 || d % M != 0) return OR_EINVAL;
#pragma omp parallel
    {
        float* T = (float*)malloc(sizeof(float) * (size_t)M * 16);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < nq; ++i)
            lut_one(q + i * d, d, codebook, M, T, Qv + i * M * 16, a + i, b + i);
        free(T);
    }
    return OR_OK;
}

/* ------------------------------------------------- O7-O11: the search */
/* Members Mem_l = {x : l1(x) = l  or  l2(x) = l} as CSR (ids ascending). */
typedef struct { int64_t* ptr; int64_t* idx; } csr_t;

static int build_members(const int32_t* l1, const int32_t* l2, int64_t n, int nlist,
                         csr_t* out) {
    int64_t* ptr = (int64_t*)calloc((size_t)nlist + 1, sizeof(int64_t));
    if (!ptr) return OR_ENOMEM;
    for (int64_t i = 0; i < n; ++i) {
        ptr[l1[i] + 1]++;
        if (l2[i] != l1[i]) ptr[l2[i] + 1]++;
    }
    for (int l = 0; l < nlist; ++l) ptr[l + 1] += ptr[l];
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ptr[nlist] ? ptr[nlist] : 1));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)nlist);
    if (!idx || !fill) { free(ptr); free(idx); free(fill); return OR_ENOMEM; }
    memcpy(fill, ptr, sizeof(int64_t) * (size_t)nlist);
    for (int64_t i = 0; i < n; ++i) {
        idx[fill[l1[i]]++] = i;
        if (l2[i] != l1[i]) idx[fill[l2[i]]++] = i;
    }
    free(fill);
    out->ptr = ptr;
    out->idx = idx;
    return OR_OK;
}

static int cmp_u64(const void* pa, const void* pb) {
    uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    return a < b ? -1 : a > b ? 1 : 0;
}

typedef struct { float dist; int64_t id; } fdist_id;

static int cmp_fdist_id(const void* pa, const void* pb) {
    const fdist_id* a = (const fdist_id*)pa;
    const fdist_id* b = (const fdist_id*)pb;
    if (a->dist < b->dist) return -1;
    if (a->dist > b->dist) return 1;
    return (a->id < b->id) ? -1 : (a->id > b->id) ? 1 : 0;
}

/*
 * oracle_search: Alg.2 RairsSearch for a batch, by the plain
 * definitions:
 *   P(q)   = O1 probes;  LUT = O2;
 *   U(q)   = {x : l1(x) in P or l2(x) in P}  computed from Mem_l with a
 *            seen-bitmap -- NO SEIL logic (SEIL reaches exactly this set:
 *            P:1418-1446, reading R9/R10);
 *   s(q,x) = sum_m Qv[m][code_m(x)] exact integer (O8);
 *   shard s = {x : id mod G == s} (O11);  U_s = U ∩ shard s;
 *   Cand_s = the min(bigK, |U_s|) smallest (s, id) pairs (rqueue; O9);
 *   delta  = (float) D64(q, x)  (refine P:719-726, 944; O10);
 *   R_s    = first k of Cand_s by (delta, id), padded (-1, +inf) (R13);
 *   result = first k of  U_s R_s  by (delta, id) (O11; G = 1 -> R_0).
 *   dco_s  = |U_s|  (O12, valid items only, R17).
 * Outputs (any may be NULL):
 *   probes  [nq*nprobe] i32        Qv [nq*M*16] u8   a, b [nq] f32
 *   cand_ids/cand_scores [nq*G*bigK] u32 (pad 0xFFFFFFFF)   dco [nq*G] i64
 *   shard_ids/shard_dists [nq*G*k]  (R_s)     out_ids/out_dists [nq*k]
 */
int oracle_search(const float* X, int64_t n, int d,
                  const int32_t* l1, const int32_t* l2, const uint8_t* codes, int M,
                  const float* cent, int nlist, const float* codebook,
                  const float* queries, int64_t nq, int k, int nprobe,
                  int refine_factor, int G,
                  int32_t* probes, uint8_t* Qv_out, float* a_out, float* b_out,
                  uint32_t* cand_ids, uint32_t* cand_scores, int64_t* dco,
                  int64_t* shard_ids, float* shard_dists,
                  int64_t* out_ids, float* out_dists) {
    if (k < 1 || nprobe < 1 || nprobe > nlist || refine_factor < 1 || G < 1 ||
        M < 1 || d % M != 0 || n < 0)
        return OR_EINVAL;
    const int bigK = k * refine_factor;
    csr_t mem;
    int err = build_members(l1, l2, n, nlist, &mem);
    if (err) return err;
#pragma omp parallel
    {
        dist_id* scratch = (dist_id*)malloc(sizeof(dist_id) * (size_t)nlist);
        int32_t* P = (int32_t*)malloc(sizeof(int32_t) * (size_t)nprobe);
        float* T = (float*)malloc(sizeof(float) * (size_t)M * 16);
        uint8_t* Qv = (uint8_t*)malloc((size_t)M * 16);
        uint8_t* seen = (uint8_t*)calloc((size_t)(n ? n : 1), 1);
        int64_t* U = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
        uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n ? n : 1));
        fdist_id* cand = (fdist_id*)malloc(sizeof(fdist_id) * (size_t)bigK);
        fdist_id* allr = (fdist_id*)malloc(sizeof(fdist_id) * (size_t)G * k);
#pragma omp for schedule(dynamic, 1)
        for (int64_t qi = 0; qi < nq; ++qi) {
            const float* q = queries + qi * d;
            float a, b;
            probe_one(q, d, cent, nlist, nprobe, scratch, P);
            lut_one(q, d, codebook, M, T, Qv, &a, &b);
            if (probes) memcpy(probes + qi * nprobe, P, sizeof(int32_t) * (size_t)nprobe);
            if (Qv_out) memcpy(Qv_out + qi * M * 16, Qv, (size_t)M * 16);
            if (a_out) a_out[qi] = a;
            if (b_out) b_out[qi] = b;
            /* U(q) from the member lists, each id once (seen-bitmap). */
            int64_t nu = 0;
            for (int p = 0; p < nprobe; ++p) {
                int l = P[p];
                for (int64_t e = mem.ptr[l]; e < mem.ptr[l + 1]; ++e) {
                    int64_t x = mem.idx[e];
                    if (!seen[x]) { seen[x] = 1; U[nu++] = x; }
                }
            }
            for (int64_t e = 0; e < nu; ++e) seen[U[e]] = 0;
            int nall = 0;
            for (int s = 0; s < G; ++s) {
                /* U_s with integer scores, as (s << 32 | id) keys. */
                int64_t nk = 0;
                for (int64_t e = 0; e < nu; ++e) {
                    int64_t x = U[e];
                    if (x % G != s) continue;
                    uint32_t sc = 0;
                    for (int m = 0; m < M; ++m) sc += Qv[m * 16 + codes[x * M + m]];
                    keys[nk++] = ((uint64_t)sc << 32) | (uint64_t)x;
                }
                if (dco) dco[qi * G + s] = nk;
                qsort(keys, (size_t)nk, sizeof(uint64_t), cmp_u64);
                int nc = nk < bigK ? (int)nk : bigK;
                for (int c = 0; c < bigK; ++c) {
                    int64_t o = (qi * G + s) * (int64_t)bigK + c;
                    if (cand_ids) cand_ids[o] = c < nc ? (uint32_t)(keys[c] & 0xFFFFFFFFu) : 0xFFFFFFFFu;
                    if (cand_scores) cand_scores[o] = c < nc ? (uint32_t)(keys[c] >> 32) : 0xFFFFFFFFu;
                }
                /* refine */
                for (int c = 0; c < nc; ++c) {
                    int64_t x = (int64_t)(keys[c] & 0xFFFFFFFFu);
                    cand[c].dist = (float)d64(q, X + x * d, d);
                    cand[c].id = x;
                }
                qsort(cand, (size_t)nc, sizeof(fdist_id), cmp_fdist_id);
                for (int r = 0; r < k; ++r) {
                    int64_t o = (qi * G + s) * (int64_t)k + r;
                    int64_t id = r < nc ? cand[r].id : -1;
                    float dist = r < nc ? cand[r].dist : INFINITY;
                    if (shard_ids) shard_ids[o] = id;
                    if (shard_dists) shard_dists[o] = dist;
                    if (r < nc) allr[nall++] = cand[r];
                }
            }
            qsort(allr, (size_t)nall, sizeof(fdist_id), cmp_fdist_id);
            for (int r = 0; r < k; ++r) {
                if (out_ids) out_ids[qi * k + r] = r < nall ? allr[r].id : -1;
                if (out_dists) out_dists[qi * k + r] = r < nall ? allr[r].dist : INFINITY;
            }
        }
        free(scratch); free(P); free(T); free(Qv); free(seen); free(U); free(keys);
        free(cand); free(allr);
    }
    free(mem.ptr);
    free(mem.idx);
    return OR_OK;
}

/* ----------------------------------------------------- O12: DCO variants */
/* For comparison with the paper only (P:2090-2096, P:1437-1446,
 * cost P:1713-1719):
 *   dco_noseil[q]    = sum_{l in P} |Mem_l|
 *   dco_paperseil[q] = sum_{cells (i<=j): i in P or j in P} 32*floor(n_ij/32)
 *                    + sum_{l in P} sum_{cells c containing l} (n_c mod 32)
 * (paper layout: full 32-item blocks stored once and skipped via reference
 * entries; misc remainders stored in both lists and always scanned). */
typedef struct { int32_t i, j; } cellkey;
static int cmp_cell(const void* pa, const void* pb) {
    const cellkey* a = (const cellkey*)pa;
    const cellkey* b = (const cellkey*)pb;
    if (a->i != b->i) return a->i < b->i ? -1 : 1;
    return (a->j < b->j) ? -1 : (a->j > b->j) ? 1 : 0;
}

int oracle_dco_variants(const int32_t* l1, const int32_t* l2, int64_t n, int nlist,
                        const int32_t* probes, int64_t nq, int nprobe,
                        int64_t* dco_noseil, int64_t* dco_paperseil) {
    cellkey* ck = (cellkey*)malloc(sizeof(cellkey) * (size_t)(n ? n : 1));
    int64_t* memsz = (int64_t*)calloc((size_t)nlist, sizeof(int64_t));
    if (!ck || !memsz) { free(ck); free(memsz); return OR_ENOMEM; }
    for (int64_t x = 0; x < n; ++x) {
        ck[x].i = l1[x]; ck[x].j = l2[x];
        memsz[l1[x]]++;
        if (l2[x] != l1[x]) memsz[l2[x]]++;
    }
    qsort(ck, (size_t)n, sizeof(cellkey), cmp_cell);
    /* distinct cells with sizes */
    int64_t ncell = 0;
    cellkey* cells = (cellkey*)malloc(sizeof(cellkey) * (size_t)(n ? n : 1));
    int64_t* csz = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    for (int64_t x = 0; x < n; ++x) {
        if (ncell > 0 && cells[ncell - 1].i == ck[x].i && cells[ncell - 1].j == ck[x].j) {
            csz[ncell - 1]++;
        } else {
            cells[ncell] = ck[x];
            csz[ncell] = 1;
            ncell++;
        }
    }
#pragma omp parallel
    {
        uint8_t* inP = (uint8_t*)calloc((size_t)nlist, 1);
#pragma omp for schedule(dynamic, 4)
        for (int64_t q = 0; q < nq; ++q) {
            const int32_t* P = probes + q * nprobe;
            for (int p = 0; p < nprobe; ++p) inP[P[p]] = 1;
            int64_t a = 0, b = 0;
            for (int p = 0; p < nprobe; ++p) a += memsz[P[p]];
            for (int64_t c = 0; c < ncell; ++c) {
                int ii = cells[c].i, jj = cells[c].j;
                int64_t full = 32 * (csz[c] / 32), rem = csz[c] % 32;
                if (inP[ii] || inP[jj]) b += full;
                if (inP[ii]) b += rem;
                if (jj != ii && inP[jj]) b += rem;
            }
            if (dco_noseil) dco_noseil[q] = a;
            if (dco_paperseil) dco_paperseil[q] = b;
            for (int p = 0; p < nprobe; ++p) inP[P[p]] = 0;
        }
        free(inP);
    }
    free(ck); free(memsz); free(cells); free(csz);
    return OR_OK;
}

/* ---------------------------------------------------- O13: exact k-NN */
/* Ground truth (P:2087-2089 recall; S:62 ties by smaller id): the first K of
 * all x ordered by (D64(q,x), id).  Kept as a sorted array of the K best,
 * insertion when a candidate beats the current K-th. */
int oracle_exact_knn(const float* X, int64_t n, int d, const float* queries, int64_t nq,
                     int K, int64_t* gt_ids, double* gt_d64) {
    if (K < 1 || K > n) return OR_EINVAL;
#pragma omp parallel
    {
        dist_id* best = (dist_id*)malloc(sizeof(dist_id) * (size_t)K);
#pragma omp for schedule(dynamic, 1)
        for (int64_t qi = 0; qi < nq; ++qi) {
            const float* q = queries + qi * d;
            int cnt = 0;
            for (int64_t x = 0; x < n; ++x) {
                dist_id e;
                e.dist = d64(q, X + x * d, d);
                e.id = x;
                if (cnt == K && cmp_dist_id(&e, &best[K - 1]) >= 0) continue;
                int pos = cnt < K ? cnt : K - 1;
                while (pos > 0 && cmp_dist_id(&e, &best[pos - 1]) < 0) {
                    best[pos] = best[pos - 1];
                    --pos;
                }
                best[pos] = e;
                if (cnt < K) ++cnt;
            }
            for (int r = 0; r < K; ++r) {
                gt_ids[qi * K + r] = best[r].id;
                if (gt_d64) gt_d64[qi * K + r] = best[r].dist;
            }
        }
        free(best);
    }
    return OR_OK;
}

/* ------------------------------------------------ O3: training (unpinned
 * bit-wise; outside the parity contract, R16).  Lloyd k-means in fp64:
 * init = k distinct training points chosen by a seeded partial Fisher-Yates
 * shuffle; each iteration assigns every point to its nearest centroid by
 * (D64, l), recomputes centroids as fp64 means (summed in point order), and
 * re-seeds an empty cluster from the largest cluster's centroid with a
 * +-1/1024 relative perturbation (the largest keeps -, the empty gets +).
 * P:501-502 ("computes nlist clusters"), P:705-707 (PQ sub-quantisers). */
static int kmeans_core(const float* x, int64_t n, int d, int k, int iters, uint64_t seed,
                       float* cent_out, double* obj_trace) {
    if (k < 1 || n < k || d < 1 || iters < 0) return OR_EINVAL;
    double* c = (double*)malloc(sizeof(double) * (size_t)k * d);
    float* cf = (float*)malloc(sizeof(float) * (size_t)k * d);
    double* sum = (double*)malloc(sizeof(double) * (size_t)k * d);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    int32_t* asg = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    double* pd = (double*)malloc(sizeof(double) * (size_t)n);
    if (!c || !cf || !sum || !cnt || !asg || !perm || !pd) {
        free(c); free(cf); free(sum); free(cnt); free(asg); free(perm); free(pd);
        return OR_ENOMEM;
    }
    uint64_t st = seed;
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    for (int i = 0; i < k; ++i) {
        int64_t j = i + (int64_t)(sm64(&st) % (uint64_t)(n - i));
        int64_t tmp = perm[i]; perm[i] = perm[j]; perm[j] = tmp;
        for (int t = 0; t < d; ++t) c[(int64_t)i * d + t] = (double)x[perm[i] * d + t];
    }
    for (int it = 0; it <= iters; ++it) {
        for (int64_t i = 0; i < (int64_t)k * d; ++i) cf[i] = (float)c[i];
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            int bl = 0;
            double bd = 0.0;
            for (int l = 0; l < k; ++l) {
                double dd = d64(x + i * d, cf + (int64_t)l * d, d);
                if (l == 0 || dd < bd) { bl = l; bd = dd; }
            }
            asg[i] = bl;
            pd[i] = bd;
        }
        double obj = 0.0;
        for (int64_t i = 0; i < n; ++i) obj += pd[i];
        if (obj_trace) obj_trace[it] = obj;
        if (it == iters) break;
        memset(sum, 0, sizeof(double) * (size_t)k * d);
        memset(cnt, 0, sizeof(int64_t) * (size_t)k);
        for (int64_t i = 0; i < n; ++i) {
            cnt[asg[i]]++;
            for (int t = 0; t < d; ++t) sum[(int64_t)asg[i] * d + t] += (double)x[i * d + t];
        }
        for (int l = 0; l < k; ++l)
            if (cnt[l] > 0)
                for (int t = 0; t < d; ++t) c[(int64_t)l * d + t] = sum[(int64_t)l * d + t] / (double)cnt[l];
        for (int l = 0; l < k; ++l) {
            if (cnt[l] > 0) continue;
            int big = 0;
            for (int j = 1; j < k; ++j) if (cnt[j] > cnt[big]) big = j;
            for (int t = 0; t < d; ++t) {
                double v = c[(int64_t)big * d + t];
                double eps = (v != 0.0 ? fabs(v) : 1.0) / 1024.0;
                c[(int64_t)l * d + t] = v + eps;
                c[(int64_t)big * d + t] = v - eps;
            }
            cnt[l] = cnt[big] / 2;
            cnt[big] -= cnt[l];
        }
    }
    for (int64_t i = 0; i < (int64_t)k * d; ++i) cent_out[i] = (float)c[i];
    free(c); free(cf); free(sum); free(cnt); free(asg); free(perm); free(pd);
    return OR_OK;
}

int oracle_kmeans(const float* x, int64_t n, int d, int k, int iters, uint64_t seed,
                  float* centroids, double* obj_trace) {
    return kmeans_core(x, n, d, k, iters, seed, centroids, obj_trace);
}

/* PQ training: M independent 16-means on the dsub-dim sub-vectors
 * ("for each dimension group, PQ partitions the sub-vectors into
 * (e.g., 16) clusters (e.g., using K-means)").  codebook is [M x 16 x dsub]. */
int oracle_pq_train(const float* x, int64_t n, int d, int M, int iters, uint64_t seed,
                    float* codebook) {
    if (M < 1 || d % M != 0 || n < 16) return OR_EINVAL;
    int dsub = d / M;
    float* sub = (float*)malloc(sizeof(float) * (size_t)n * dsub);
    if (!sub) return OR_ENOMEM;
    for (int m = 0; m < M; ++m) {
        for (int64_t i = 0; i < n; ++i)
            for (int t = 0; t < dsub; ++t) sub[i * dsub + t] = x[i * d + (int64_t)m * dsub + t];
        int e = kmeans_core(sub, n, dsub, 16, iters, seed + 0x1000003ull * (uint64_t)(m + 1),
                            codebook + (int64_t)m * 16 * dsub, NULL);
        if (e) { free(sub); return e; }
    }
    free(sub);
    return OR_OK;
}
