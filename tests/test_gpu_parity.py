"""GPU (CUDA path, through the C ABI) vs CPU oracle parity. Needs a B200.

The oracle trains the coarse centroids and the PQ codebook (training is outside
the bit-exact contract, R16); the GPU index is built from that
trained state (rairs_build_from_trained) and everything downstream must match:
  * assignment (l1, l2) and PQ codes: bit-exact (O4, O5)
  * probes, LUT Qv / a / b, candidate (score, id) keys, DCO: bit-exact
  * refined distances: within 1e-4 relative (they are in fact bit-equal:
    both sides sum in fp64 in ascending t and round once)
  * final ids: identical
Inputs come from synth/ (seeded); no expected value comes from the CUDA path.
"""
import numpy as np
import pytest

from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

if not gpu_available():  # collected on CPU too; skip at import of fixtures
    pytest.skip("no CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import get_config, make_dataset  # noqa: E402

DEV = torch.device("cuda:0")
U32 = 0xFFFFFFFF


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


class Case:
    """Oracle-trained index of one config (CPU) + the GPU index built from it."""

    def __init__(self, oracle, name, n=None, nq=None, train_rows=20000, iters=6,
                 assignment="air", strict=False, lam=0.5):
        spec = get_config(name)
        self.spec = spec
        X, Q = make_dataset(spec, n=n, nq=nq)
        self.X, self.Q = X, Q
        rows = X[np.random.default_rng(5).permutation(X.shape[0])[:min(train_rows, X.shape[0])]]
        self.cent = oracle.kmeans(rows, spec.nlist, iters=iters, seed=11)
        self.cb = oracle.pq_train(rows, spec.M, iters=iters, seed=12)
        self.l1, self.l2 = oracle.assign(X, self.cent, assignment, lam=lam, strict=strict)
        self.codes = oracle.encode(X, self.cb)
        self.assignment, self.strict, self.lam = assignment, strict, lam

    def gpu_index(self, shard_id=0, nshards=1):
        rows = np.arange(shard_id, self.X.shape[0], nshards)
        return rb.Index.build(_t(self.X[rows]), self.spec.nlist, self.spec.M,
                              assignment=self.assignment.upper(), strict=self.strict,
                              lambda_=self.lam,
                              centroids=_t(self.cent), codebook=_t(self.cb),
                              shard_id=shard_id, nshards=nshards)


_CACHE = {}


def case(oracle, name, **kw):
    key = (name, tuple(sorted(kw.items())))
    if key not in _CACHE:
        _CACHE[key] = Case(oracle, name, **kw)
    return _CACHE[key]


def gpu_search(idx, Q, k, nprobe, rf, scan="auto"):
    idx.set_scan_mode(scan)
    out = idx.search_debug(_t(Q), k, nprobe, rf)
    torch.cuda.synchronize()
    r = {key: v.cpu().numpy() for key, v in out.items()}
    # the plain entry point (no debug outputs: the list-major selection writes
    # each query's top-bigK set unordered) must return the same results
    ids, dists, dco = idx.search(_t(Q), k, nprobe, rf, return_dco=True)
    assert np.array_equal(ids.cpu().numpy(), r["ids"]), "plain search ids differ from debug"
    assert np.array_equal(dists.cpu().numpy(), r["dists"]), "plain search dists differ"
    assert np.array_equal(dco.cpu().numpy(), r["dco"]), "plain search DCO differs"
    r["cand_ids"] = r["cand_ids"].view(np.uint32)
    r["cand_scores"] = r["cand_scores"].view(np.uint32)
    return r


def assert_search_equal(g, o, rows=None, shard=0):
    sel = slice(None) if rows is None else rows
    assert np.array_equal(g["probes"], o["probes"][sel]), "probe sets differ (O1)"
    assert np.array_equal(g["Qv"], o["Qv"][sel]), "quantised LUT differs (O2)"
    assert np.array_equal(g["a"], o["a"][sel]) and np.array_equal(g["b"], o["b"][sel])
    assert np.array_equal(g["dco"], o["dco"][sel][:, shard]), "DCO differs (O12)"
    assert np.array_equal(g["cand_scores"], o["cand_scores"][sel][:, shard]), "scores differ (O8/O9)"
    assert np.array_equal(g["cand_ids"], o["cand_ids"][sel][:, shard]), "candidate ids differ (O9)"
    oi = o["shard_ids"][sel][:, shard] if "shard_ids" in o else o["ids"][sel]
    od = o["shard_dists"][sel][:, shard] if "shard_dists" in o else o["dists"][sel]
    assert np.array_equal(g["ids"], oi), "final ids differ (O10)"
    fin = np.isfinite(od)
    assert np.array_equal(np.isfinite(g["dists"]), fin)
    assert np.allclose(g["dists"][fin], od[fin], rtol=1e-4, atol=0), "refined distances (1e-4)"


# ------------------------------------------------------------------ build
@pytest.mark.parametrize("name", ["c0", "c0s", "c1", "c1s"])
def test_build_assignment_codes_layout(oracle_mod, name):
    c = case(oracle_mod, name)
    idx = c.gpu_index()
    l1, l2, codes = [t.cpu().numpy() for t in idx.export_assignment()]
    assert np.array_equal(l1, c.l1) and np.array_equal(l2, c.l2), "AIR assignment (O4)"
    assert np.array_equal(codes, c.codes), "PQ codes (O5)"
    check_layout(idx, c.l1, c.l2)
    info = idx.info()
    assert info["n_double"] == int(np.sum(c.l1 != c.l2))


def check_layout(idx, l1, l2):
    """O6 (i)-(iv): stored once; owned region = cells (l, j>=l) in (l2, row)
    order; references = cells (i<j) with their slot range; padding at ends."""
    L = {k: v.cpu().numpy() for k, v in idx.export_layout().items()}
    rows = L["slot_rows"].view(np.uint32)
    valid = rows != U32
    n = l1.shape[0]
    assert valid.sum() == n and np.array_equal(np.sort(rows[valid]), np.arange(n))      # (i)
    nl = L["own_off"].shape[0]
    for l in range(nl):
        off, cnt = int(L["own_off"][l]), int(L["own_cnt"][l])
        mine = np.nonzero(l1 == l)[0]
        order = mine[np.lexsort((mine, l2[mine]))]
        assert np.array_equal(rows[off:off + cnt], order)                             # (ii)
        end = off + ((cnt + 31) // 32) * 32
        assert (rows[off + cnt:end] == U32).all()                                      # (iv)
        refs = []
        for e in range(int(L["ref_ptr"][l]), int(L["ref_ptr"][l + 1])):
            refs.append((int(L["ref_owner"][e]), int(L["ref_start"][e]), int(L["ref_cnt"][e])))
        expect = []
        for i in range(l):
            cell = np.nonzero((l1 == i) & (l2 == l))[0]
            if cell.size:
                expect.append((i, cell.size))
        assert [(o, c) for o, _, c in refs] == expect                                  # (iii)
        for o, s, cn in refs:
            got = rows[s:s + cn]
            assert (l1[got] == o).all() and (l2[got] == l).all()


# ----------------------------------------------------------------- search
SEARCH_CASES = [
    ("c0", 5, 4, 4), ("c0s", 5, 4, 4), ("c0s", 5, 16, 2), ("c0s", 1, 1, 1),
    ("c1", 10, 8, 4), ("c1", 10, 1, 4), ("c1", 10, 64, 4),
    ("c1s", 10, 8, 4), ("c1s", 10, 16, 10), ("c1s", 1, 3, 100), ("c1s", 100, 8, 1),
    ("c1s", 100, 8, 4),   # top-100 workload: K_FACTOR 4, bigK 400
]


@pytest.mark.parametrize("scan", ["simt", "listmajor"])
@pytest.mark.parametrize("name,k,nprobe,rf", SEARCH_CASES)
def test_search_parity(oracle_mod, name, k, nprobe, rf, scan):
    c = case(oracle_mod, name)
    idx = c.gpu_index()
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, k, nprobe, rf)
    g = gpu_search(idx, c.Q, k, nprobe, rf, scan)
    assert_search_equal(g, o)


@pytest.mark.parametrize("scan", ["simt", "listmajor"])
def test_search_parity_many_queries(oracle_mod, scan):
    # 2,000 queries x nprobe 16 over 64 lists: ~500 queries per list -> 8 LUT/query
    # tiles per list-task in the list-major kernel; several queries per CTA in the
    # pipelined refine kernel
    c = case(oracle_mod, "c1s", nq=2000)
    idx = c.gpu_index()
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, 10, 16, 10)
    assert_search_equal(gpu_search(idx, c.Q, 10, 16, 10, scan), o)


@pytest.mark.parametrize("k,rf", [(10, 10), (100, 4)])
def test_search_parity_overlapped_halves(oracle_mod, k, rf):
    # >= 2 * LM_OVERLAP_MIN_Q queries: the list-major path selects and refines
    # two query halves on the index's auxiliary streams (odd count: unequal halves)
    c = case(oracle_mod, "c1s", nq=4503)
    idx = c.gpu_index()
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, k, 8, rf)
    assert_search_equal(gpu_search(idx, c.Q, k, 8, rf, "listmajor"), o)
    # the plain search entry point (fused refine, no debug outputs) agrees too
    idx.set_scan_mode("listmajor")
    ids, dists = idx.search(_t(c.Q), k, 8, rf)
    assert np.array_equal(ids.cpu().numpy(), o["ids"])


def test_search_modes_single_and_strict(oracle_mod):
    for kw in ({"assignment": "single"}, {"assignment": "air", "strict": True}):
        c = case(oracle_mod, "c1s", **kw)
        idx = c.gpu_index()
        l1, l2, _ = [t.cpu().numpy() for t in idx.export_assignment()]
        assert np.array_equal(l1, c.l1) and np.array_equal(l2, c.l2)
        o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, 10, 8, 4)
        assert_search_equal(gpu_search(idx, c.Q, 10, 8, 4), o)


@pytest.mark.parametrize("name,n", [("c1s", None), ("c2pl", 60000)])
def test_soarl2_and_naivera_assignment(oracle_mod, name, n):
    # NEXT-2 comparison strategies on the same kernels: SOARL2 (Table 2's SOAR loss,
    # P:1100, strict) and NaiveRA (AIR with lambda 0, strict).
    # c2pl (nlist 1024) builds through the tensor-core filter + certify path.
    for kw in ({"assignment": "soar", "strict": True, "lam": 1.0},
               {"assignment": "air", "strict": True, "lam": 0.0}):
        c = case(oracle_mod, name, n=n, **kw)
        idx = c.gpu_index()
        l1, l2, _ = [t.cpu().numpy() for t in idx.export_assignment()]
        assert np.array_equal(l1, c.l1) and np.array_equal(l2, c.l2), kw
        assert (l1 != l2).all()                       # strict: always two lists
        o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q[:500], 10, 8, 4)
        assert_search_equal(gpu_search(idx, c.Q[:500], 10, 8, 4), o)
        idx.free()


def test_exhaustive_reduction_equals_exact_knn(oracle_mod):
    # nprobe = nlist, bigK >= n  ->  exact k-NN (BJ invariant)
    c = case(oracle_mod, "c0s", n=2000)
    idx = c.gpu_index()
    k = 5
    rf = (c.X.shape[0] + k - 1) // k  # bigK >= n (bigK <= 2048 supported)
    g = gpu_search(idx, c.Q, k, c.spec.nlist, rf)
    gt, _ = oracle_mod.exact_knn(c.X, c.Q, k)
    assert np.array_equal(g["ids"], gt)
    assert (g["dco"] == c.X.shape[0]).all()


def test_edge_cases(oracle_mod):
    c = case(oracle_mod, "c1s")
    idx = c.gpu_index()
    # queries equal to base rows, a single query, and an empty batch
    Qs = c.X[[0, 17, 999]]
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, Qs, 3, 2, 7)
    assert_search_equal(gpu_search(idx, Qs, 3, 2, 7), o)
    o1 = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q[:1], 10, 8, 4)
    assert_search_equal(gpu_search(idx, c.Q[:1], 10, 8, 4), o1)
    ids, dists = idx.search(_t(c.Q[:0]), 10, 8, 4)
    assert ids.shape == (0, 10)
    # search == search_host == search_debug results
    ids, dists = idx.search(_t(c.Q), 10, 8, 4)
    hi, hd = idx.search_host(c.Q, 10, 8, 4)
    assert np.array_equal(ids.cpu().numpy(), hi) and np.array_equal(dists.cpu().numpy(), hd)


def test_padding_when_universe_smaller_than_k(oracle_mod):
    c = case(oracle_mod, "c0")
    idx = c.gpu_index()
    # k larger than any single list (3000 rows / 16 lists), nprobe=1 -> (-1, inf) tail
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, 1000, 1, 1)
    g = gpu_search(idx, c.Q, 1000, 1, 1)
    assert_search_equal(g, o)
    assert (g["ids"] == -1).any()


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_parity(oracle_mod, G):
    c = case(oracle_mod, "c1s")
    k, nprobe, rf = 10, 8, 4
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, k, nprobe, rf, nshards=G)
    per_ids, per_d = [], []
    for s in range(G):
        idx = c.gpu_index(shard_id=s, nshards=G)
        g = gpu_search(idx, c.Q, k, nprobe, rf)
        assert_search_equal(g, o, shard=s)
        per_ids.append(g["ids"])
        per_d.append(g["dists"])
    mi, md = rb.merge_topk(_t(np.stack(per_ids)), _t(np.stack(per_d)))
    assert np.array_equal(mi.cpu().numpy(), o["ids"])
    assert np.allclose(md.cpu().numpy(), o["dists"], rtol=1e-4)


def test_exact_knn_kernel(oracle_mod):
    c = case(oracle_mod, "c1")
    ids, d64 = rb.exact_knn(_t(c.X), _t(c.Q), 10)
    gi, gd = oracle_mod.exact_knn(c.X, c.Q, 10)
    assert np.array_equal(ids.cpu().numpy(), gi)
    assert np.array_equal(d64.cpu().numpy(), gd)


def test_errors_are_reported():
    X = torch.randn(500, 16, device=DEV)
    with pytest.raises(rb.RairsError):
        rb.build_index(X, nlist=8, M=5)                       # M does not divide d
    with pytest.raises(rb.RairsError):
        rb.build_index(X, nlist=8, M=8, nbits=8)              # nbits != 4
    with pytest.raises(rb.RairsError):
        rb.build_index(X, nlist=1000, M=8)                    # nlist > n
    idx = rb.build_index(X, nlist=8, M=8, kmeans_iters=3)
    q = torch.randn(4, 16, device=DEV)
    for bad in (dict(k=0, nprobe=2), dict(k=3, nprobe=9), dict(k=3, nprobe=0)):
        with pytest.raises(rb.RairsError):
            idx.search(q, refine_factor=2, **bad)
    with pytest.raises(TypeError):
        idx.search(q.cpu(), 3, 2)                             # host tensor on the device API


def test_gpu_training_properties():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((4000, 16)).astype(np.float32)
    c1, b1 = rb.train(_t(X), 1, 8, kmeans_iters=3, train_sample=4000)
    assert np.allclose(c1.cpu().numpy()[0], X.astype(np.float64).mean(0), atol=1e-5)
    ca, ba = rb.train(_t(X), 32, 8, kmeans_iters=5, seed=3)
    cb_, bb = rb.train(_t(X), 32, 8, kmeans_iters=5, seed=3)
    assert torch.equal(ca, cb_) and torch.equal(ba, bb)           # deterministic
    assert torch.isfinite(ca).all() and torch.isfinite(ba).all()


# ------------------------------------------ BJ full sizes, sampled queries
@pytest.mark.parametrize("scan", ["simt", "listmajor"])
@pytest.mark.parametrize("name,nprobe", [("c2", 16), ("c2pl", 4), ("c2pl", 64)])
def test_full_size_sampled(oracle_mod, name, nprobe, scan):
    """BJ configs[1] at full size (1M x 128, 10k queries) in the bench's launch
    configuration; the oracle recomputes a sample of 200 queries one by one."""
    c = case(oracle_mod, name, train_rows=32768, iters=4)
    spec = c.spec
    idx = c.gpu_index()
    rng = np.random.default_rng(7)
    sample = np.sort(rng.choice(c.Q.shape[0], 200, replace=False))
    g = gpu_search(idx, c.Q, spec.k, nprobe, spec.refine_factor, scan)   # all 10k queries
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q[sample], spec.k, nprobe,
                          spec.refine_factor)
    gs = {key: v[sample] for key, v in g.items()}
    assert_search_equal(gs, o)
    # assignment and codes on a sample of rows
    l1, l2, codes = [t.cpu().numpy() for t in idx.export_assignment()]
    assert np.array_equal(l1, c.l1) and np.array_equal(l2, c.l2)
    assert np.array_equal(codes, c.codes)


# ------------------------------------- coarse stage: tensor-core path == O1
@pytest.mark.parametrize("name,nprobes", [("c1s", [1, 8, 32]), ("c2pl", [1, 4, 16, 64, 128])])
def test_coarse_tensor_core_path_equals_exact(oracle_mod, name, nprobes):
    """K1 (tcgen05 TF32 GEMM) + K2 (fp64 certify) must give exactly O1's probe
    sets; the certification must succeed for almost every query (otherwise the
    GEMM is not doing the work and every query falls back to fp64)."""
    kw = dict(train_rows=32768, iters=4) if name.startswith("c2") else {}
    c = case(oracle_mod, name, **kw)
    idx = c.gpu_index()
    Qd = _t(c.Q)
    sample = np.arange(0, c.Q.shape[0], max(1, c.Q.shape[0] // 200))
    for npb in nprobes:
        idx.set_coarse_mode("exact")
        pe = idx.search_debug(Qd, c.spec.k, npb, 2)["probes"].cpu().numpy()
        idx.set_coarse_mode("tensor")
        idx.certify_fallbacks(reset=True)
        pt = idx.search_debug(Qd, c.spec.k, npb, 2)["probes"].cpu().numpy()
        fb = idx.certify_fallbacks(reset=True)
        assert np.array_equal(pe, pt)
        assert fb <= max(2, 0.02 * c.Q.shape[0]), f"{fb} uncertified queries at nprobe {npb}"
        po = oracle_mod.probe(c.Q[sample], c.cent, npb)
        assert np.array_equal(pt[sample], po)
    idx.set_coarse_mode("auto")


@pytest.mark.parametrize("scan", ["simt", "listmajor"])
def test_massive_score_ties(oracle_mod, scan):
    """Many identical vectors -> identical codes and scores: exercises the
    exact-sort fallback of the top-bigK selection (keys unique by id)."""
    rng = np.random.default_rng(21)
    base = rng.standard_normal((12, 16)).astype(np.float32)
    X = base[rng.integers(0, 12, 6000)] + 0.0
    Q = base[rng.integers(0, 12, 30)] + rng.standard_normal((30, 16)).astype(np.float32) * 0.01
    cent = oracle_mod.kmeans(X, 16, iters=3, seed=1)
    cb = oracle_mod.pq_train(X, 8, iters=3, seed=2)
    l1, l2 = oracle_mod.assign(X, cent, "air")
    codes = oracle_mod.encode(X, cb)
    idx = rb.Index.build(_t(X), 16, 8, centroids=_t(cent), codebook=_t(cb))
    for k, nprobe, rf in ((10, 4, 10), (5, 16, 20), (50, 8, 8)):
        o = oracle_mod.search(X, l1, l2, codes, cent, cb, Q, k, nprobe, rf)
        assert_search_equal(gpu_search(idx, Q, k, nprobe, rf, scan), o)


# ------------------------------- BJ configs[3] at full size (10M x 96), sampled
def test_c4_full_size_sampled_properties(oracle_mod):
    """BJ configs[3] at full size: 10M x 96 drawn on the device, nlist 16,384,
    M 48, the bench's launch configuration (all 10k queries in one batch,
    list-major scan). The index is GPU-trained (outside the bit-exact contract,
    R16); the oracle then checks, from the exported trained state and the same
    input rows, on samples it can compute one by one:
      O4/O5  assignment and codes of 4,000 sampled rows;
      O1/O2  probe sets and the quantised LUT of 64 sampled queries;
      O8     every returned candidate's integer score, from the oracle's own
             encode of that row;
      O9     completeness on a 20,000-row sample: every sampled row of U(q)
             whose key (s, id) is below the bigK-th candidate key is a candidate;
      O10    the final ids are the first k candidates by (delta, id), delta the
             fp64 ordered sum rounded to fp32 (1e-4 relative)."""
    from synth.gpu_generators import make_dataset_torch
    spec = get_config("c4")
    k, nprobe, rf = spec.k, 2, spec.refine_factor
    bigK = k * rf
    Xd, Qd = make_dataset_torch(spec, DEV)
    idx = rb.build_index(Xd, spec.nlist, spec.M, train_sample=64 * spec.nlist, kmeans_iters=10)
    idx.set_scan_mode("listmajor")
    assert idx.scan_path(spec.nq, k, nprobe, rf) == "listmajor"
    out = idx.search_debug(Qd, k, nprobe, rf)
    torch.cuda.synchronize()
    rng = np.random.default_rng(11)
    qs = np.sort(rng.choice(spec.nq, 64, replace=False))
    g = {key: v.cpu().numpy()[qs] for key, v in out.items()}
    g["cand_ids"] = g["cand_ids"].view(np.uint32)
    g["cand_scores"] = g["cand_scores"].view(np.uint32)
    cent, cb = [t.cpu().numpy() for t in idx.export_trained()]
    l1, l2, codes = [t.cpu().numpy() for t in idx.export_assignment()]
    Q = Qd.cpu().numpy()[qs]
    rows = np.sort(rng.choice(spec.n, 20000, replace=False))
    Xs = Xd[torch.from_numpy(rows).to(DEV)].cpu().numpy()
    # O4 / O5 on 4,000 of the sampled rows
    ol1, ol2 = oracle_mod.assign(Xs[:4000], cent, "air")
    assert np.array_equal(l1[rows[:4000]], ol1) and np.array_equal(l2[rows[:4000]], ol2)
    assert np.array_equal(codes[rows[:4000]], oracle_mod.encode(Xs[:4000], cb))
    # O1 / O2
    assert np.array_equal(g["probes"], oracle_mod.probe(Q, cent, nprobe))
    Qv, a, b = oracle_mod.lut(Q, cb)
    assert np.array_equal(g["Qv"], Qv) and np.array_equal(g["a"], a) and np.array_equal(g["b"], b)
    # O8: candidate scores from the oracle's encode of the candidate rows
    srow_l1, srow_l2 = oracle_mod.assign(Xs, cent, "air")
    scodes = oracle_mod.encode(Xs, cb)
    for i in range(len(qs)):
        cid = g["cand_ids"][i]
        valid = cid != 0xFFFFFFFF
        cx = Xd[torch.from_numpy(cid[valid].astype(np.int64)).to(DEV)].cpu().numpy()
        cc = oracle_mod.encode(cx, cb).astype(np.int64)
        s = Qv[i][np.arange(spec.M)[None, :], cc].sum(1)
        assert np.array_equal(s, g["cand_scores"][i][valid].astype(np.int64)), "O8 scores"
        assert np.all(np.diff(s * 2**32 + cid[valid].astype(np.int64)) > 0), "keys sorted"
        # O9 completeness on the row sample
        P = set(g["probes"][i].tolist())
        inU = np.array([(x in P) or (y in P) for x, y in zip(srow_l1, srow_l2)])
        ss = Qv[i][np.arange(spec.M)[None, :], scodes.astype(np.int64)].sum(1)
        kmax = s[-1] * 2**32 + int(cid[valid][-1]) if valid.sum() == bigK else np.inf
        must = inU & (ss * 2**32 + rows < kmax)
        assert set(rows[must].tolist()) <= set(cid[valid].tolist()), "O9 completeness"
        # O10: refine = first k candidates by (fp32(fp64 ordered sum), id)
        acc = np.zeros(cx.shape[0], np.float64)
        qd = Q[i].astype(np.float64)
        for t in range(spec.d):
            df = qd[t] - cx[:, t].astype(np.float64)
            acc = acc + df * df
        delta = acc.astype(np.float32)
        order = np.lexsort((cid[valid], delta))[:k]
        assert np.array_equal(g["ids"][i], cid[valid][order].astype(np.int64)), "O10 ids"
        assert np.allclose(g["dists"][i], delta[order], rtol=1e-4, atol=0), "O10 distances"
    idx.free()


def test_exact_fallback_split_path_large_nlist(oracle_mod):
    """8,192 centroids packed in a tiny ball far from the origin: the TF32
    filter can never certify (its error bound dwarfs the distance gaps), so
    every query and every base row goes through the exact fallback -- the
    split path (first 2,048 flagged rows per chunk) and the tiled kernel (the
    rest). Probes and the RAIR assignment must equal O1 / O4 exactly."""
    rng = np.random.default_rng(3)
    center = rng.standard_normal(32).astype(np.float32)
    center *= np.float32(100.0 / np.linalg.norm(center))
    cent = (center + np.float32(1e-3) * rng.standard_normal((8192, 32))).astype(np.float32)
    X = (center + np.float32(2e-3) * rng.standard_normal((6000, 32))).astype(np.float32)
    Q = (center + np.float32(2e-3) * rng.standard_normal((300, 32))).astype(np.float32)
    cb = oracle_mod.pq_train(X, 8, iters=2, seed=1)
    idx = rb.Index.build(_t(X), 8192, 8, centroids=_t(cent), codebook=_t(cb))
    l1, l2, _ = [t.cpu().numpy() for t in idx.export_assignment()]
    ol1, ol2 = oracle_mod.assign(X, cent, "air")
    assert np.array_equal(l1, ol1) and np.array_equal(l2, ol2)
    Qd = _t(Q)
    idx.set_coarse_mode("tensor")
    for npb in (1, 10, 64):
        idx.certify_fallbacks(reset=True)
        pt = idx.search_debug(Qd, 10, npb, 2)["probes"].cpu().numpy()
        fb = idx.certify_fallbacks(reset=True)
        assert fb == Q.shape[0], f"expected every query uncertified, got {fb}"
        assert np.array_equal(pt, oracle_mod.probe(Q, cent, npb))
    idx.free()


@pytest.mark.parametrize("scan", ["simt", "listmajor"])
def test_parity_dsub4_padded_M(oracle_mod, scan):
    """d/M = 4 (as BJ configs[2]) with M = 24 (not a multiple of 16: the LUT
    has zero rows up to M_pad = 32, the code units are padded), AIR + SEIL."""
    rng = np.random.default_rng(17)
    means = rng.standard_normal((24, 96)).astype(np.float32)
    X = (means[rng.integers(0, 24, 5000)] + 0.8 * rng.standard_normal((5000, 96))).astype(np.float32)
    Q = (means[rng.integers(0, 24, 300)] + 0.8 * rng.standard_normal((300, 96))).astype(np.float32)
    cent = oracle_mod.kmeans(X, 32, iters=4, seed=5)
    cb = oracle_mod.pq_train(X, 24, iters=4, seed=6)
    l1, l2 = oracle_mod.assign(X, cent, "air")
    codes = oracle_mod.encode(X, cb)
    idx = rb.Index.build(_t(X), 32, 24, centroids=_t(cent), codebook=_t(cb))
    gl1, gl2, gcodes = [t.cpu().numpy() for t in idx.export_assignment()]
    assert np.array_equal(gl1, l1) and np.array_equal(gl2, l2) and np.array_equal(gcodes, codes)
    for k, nprobe, rf in ((10, 4, 10), (5, 12, 4)):
        o = oracle_mod.search(X, l1, l2, codes, cent, cb, Q, k, nprobe, rf)
        assert_search_equal(gpu_search(idx, Q, k, nprobe, rf, scan), o)
    idx.free()


def test_coarse_capped_lists_large_nprobe(oracle_mod):
    """nlist 4,096 (16 column tiles) and nprobe 48 / 96: W + 1 > 32, so the
    top-W epilogue keeps capped 32-entry register lists per (row, split, half)
    and K2 certifies against the smallest full list's 32nd value. Probe sets
    must equal the exact kernel's and O1 on a sample."""
    rng = np.random.default_rng(9)
    means = rng.standard_normal((512, 32)).astype(np.float32)
    X = (means[rng.integers(0, 512, 60000)] + 0.5 * rng.standard_normal((60000, 32))).astype(np.float32)
    Q = (means[rng.integers(0, 512, 2000)] + 0.5 * rng.standard_normal((2000, 32))).astype(np.float32)
    cent = X[rng.choice(X.shape[0], 4096, replace=False)].copy()
    cb = oracle_mod.pq_train(X[:20000], 8, iters=2, seed=1)
    idx = rb.Index.build(_t(X), 4096, 8, centroids=_t(cent), codebook=_t(cb))
    Qd = _t(Q)
    sample = np.arange(0, Q.shape[0], 20)
    for npb in (48, 96):
        idx.set_coarse_mode("exact")
        pe = idx.search_debug(Qd, 10, npb, 2)["probes"].cpu().numpy()
        idx.set_coarse_mode("tensor")
        idx.certify_fallbacks(reset=True)
        pt = idx.search_debug(Qd, 10, npb, 2)["probes"].cpu().numpy()
        fb = idx.certify_fallbacks(reset=True)
        assert np.array_equal(pe, pt)
        assert fb <= 0.05 * Q.shape[0], f"{fb} uncertified queries at nprobe {npb}"
        assert np.array_equal(pt[sample], oracle_mod.probe(Q[sample], cent, npb))
    idx.free()


# ------------------------------------------------------------ updates (NEXT-3)
def _oracle_on_rows(oracle, c, rows, Q, k, nprobe, rf):
    """Oracle search over the live subset X[rows] (same trained state), with
    its row indices mapped back to the original ids. The map is increasing, so
    every (s, id) / (delta, id) order is preserved."""
    o = oracle.search(c.X[rows], c.l1[rows], c.l2[rows], c.codes[rows], c.cent, c.cb, Q,
                      k, nprobe, rf)
    ci = o["cand_ids"]
    o["cand_ids"] = np.where(ci != U32, rows[np.minimum(ci, rows.size - 1)], U32).astype(np.uint32)
    for key in ("ids", "shard_ids"):
        ids = o[key]
        o[key] = np.where(ids >= 0, rows[np.clip(ids, 0, rows.size - 1)], -1)
    return o


@pytest.mark.parametrize("scan", ["simt", "listmajor"])
def test_insert_batches_equal_full_build(oracle_mod, scan):
    # paper protocol shape: build on 80 % of the rows, then insert
    # the rest in five batches; the index must equal a build over every row
    c = case(oracle_mod, "c1s")
    n = c.X.shape[0]
    n0 = int(0.8 * n)
    idx = rb.Index.build(_t(c.X[:n0]), c.spec.nlist, c.spec.M, assignment="AIR",
                         centroids=_t(c.cent), codebook=_t(c.cb))
    bounds = np.linspace(n0, n, 6).astype(int)
    for b0, b1 in zip(bounds[:-1], bounds[1:]):
        assert idx.add(_t(c.X[b0:b1])) == b0
    info = idx.info()
    assert info["n"] == n and info["n_live"] == n
    l1, l2, codes = [t.cpu().numpy() for t in idx.export_assignment()]
    assert np.array_equal(l1, c.l1) and np.array_equal(l2, c.l2) and np.array_equal(codes, c.codes)
    check_layout(idx, c.l1, c.l2)
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, 10, 8, 4)
    assert_search_equal(gpu_search(idx, c.Q, 10, 8, 4, scan), o)
    idx.free()


@pytest.mark.parametrize("scan", ["simt", "listmajor"])
def test_delete_then_insert_parity(oracle_mod, scan):
    # deletes in three batches (with repeats, negative and out-of-range ids),
    # then one insert: results equal the oracle over the live rows
    c = case(oracle_mod, "c1s")
    n = c.X.shape[0]
    n0 = n - 1000
    idx = rb.Index.build(_t(c.X[:n0]), c.spec.nlist, c.spec.M, assignment="AIR",
                         centroids=_t(c.cent), codebook=_t(c.cb))
    rng = np.random.default_rng(77)
    dead = rng.choice(n0, size=n0 // 5, replace=False)
    total = 0
    for part in np.array_split(dead, 3):
        extra = np.array([-1, n0 + 5000, int(part[0])], np.int64)   # ignored / repeated
        total += idx.remove_ids(torch.from_numpy(np.concatenate([part, extra])))
    assert total == dead.size
    assert idx.remove_ids(torch.from_numpy(dead[:10])) == 0        # already deleted
    assert idx.add(_t(c.X[n0:])) == n0
    live = np.ones(n, bool)
    live[dead] = False
    rows = np.nonzero(live)[0]
    info = idx.info()
    assert info["n"] == n and info["n_live"] == rows.size
    L = idx.export_layout()
    stored = L["slot_rows"].cpu().numpy().view(np.uint32)
    assert np.array_equal(np.sort(stored[stored != U32]), rows)      # stored once, live only
    o = _oracle_on_rows(oracle_mod, c, rows, c.Q, 10, 8, 4)
    assert_search_equal(gpu_search(idx, c.Q, 10, 8, 4, scan), o)
    idx.free()


def test_sharded_insert_and_delete_ids(oracle_mod):
    # shard s of G holds global ids = row * G + s; an insert continues that
    # numbering and deletes ignore ids of other shards
    c = case(oracle_mod, "c1s")
    G, s = 2, 1
    rows_all = np.arange(s, c.X.shape[0], G)
    half = rows_all.size // 2
    idx = rb.Index.build(_t(c.X[rows_all[:half]]), c.spec.nlist, c.spec.M, assignment="AIR",
                         centroids=_t(c.cent), codebook=_t(c.cb), shard_id=s, nshards=G)
    assert idx.add(_t(c.X[rows_all[half:]])) == half * G + s
    ids = torch.arange(0, 200, dtype=torch.int64)                   # 100 ours, 100 not
    assert idx.remove_ids(ids) == 100
    # shard s's global ids are the original rows s, s+G, ...: compare with the
    # oracle over its live rows (ids < 200 deleted), ids mapped back
    live = rows_all[rows_all >= 200]
    o = _oracle_on_rows(oracle_mod, c, live, c.Q[:300], 10, 8, 4)
    assert_search_equal(gpu_search(idx, c.Q[:300], 10, 8, 4), o)
    idx.free()


def test_search_host_copy_stream(oracle_mod):
    # rairs_search_host(_async) copies the host queries on the index's copy
    # stream into a two-slot device buffer ring (tensor-core coarse path,
    # nlist 1024): same results as the device entry point, and as the oracle
    c = case(oracle_mod, "c2pl", n=60000)
    idx = c.gpu_index()
    Q = c.Q[:9001]
    ids, dists = idx.search(_t(Q), 10, 4, 10)
    hi, hd = idx.search_host(Q, 10, 4, 10)
    assert np.array_equal(ids.cpu().numpy(), hi) and np.array_equal(dists.cpu().numpy(), hd)
    # the async entry point, twice back to back on one stream, then one sync
    outs = [(torch.empty((Q.shape[0], 10), dtype=torch.int64).pin_memory().numpy(),
             torch.empty((Q.shape[0], 10), dtype=torch.float32).pin_memory().numpy()) for _ in range(2)]
    qh = torch.from_numpy(Q).pin_memory().numpy()
    for o_i, o_d in outs:
        idx.search_host_async(qh, 10, 4, 10, o_i, o_d)
    torch.cuda.synchronize()
    for o_i, o_d in outs:
        assert np.array_equal(o_i, hi) and np.array_equal(o_d, hd)
    rows = np.r_[0:50, 2200:2300, 8950:9001]
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, Q[rows], 10, 4, 10)
    assert np.array_equal(hi[rows], o["ids"])
    idx.free()


def test_caller_ids(oracle_mod):
    # SURVEY §8(b) `ids`: caller-supplied vector ids are returned by searches
    # and taken by deletes; invalid ids are rejected before any mutation
    c = case(oracle_mod, "c1s")
    n = c.X.shape[0]
    n0 = n - 500
    rng = np.random.default_rng(9)
    lab = rng.choice(2**32 - 1, size=n, replace=False).astype(np.int64)
    idx = rb.Index.build(_t(c.X[:n0]), c.spec.nlist, c.spec.M, assignment="AIR",
                         centroids=_t(c.cent), codebook=_t(c.cb), ids=_t(lab[:n0]))
    assert idx.info()["has_ids"] == 1
    with pytest.raises(rb.RairsError):                      # a held id
        idx.add(_t(c.X[n0:]), ids=_t(np.r_[lab[n0:-1], lab[0]]))
    with pytest.raises(rb.RairsError):                      # ids required
        idx.add(_t(c.X[n0:]))
    assert idx.info()["n"] == n0                            # unchanged
    idx.add(_t(c.X[n0:]), ids=_t(lab[n0:]))
    dead = rng.choice(n, size=n // 10, replace=False)
    assert idx.remove_ids(torch.from_numpy(lab[dead])) == dead.size
    unknown = np.setdiff1d(np.arange(n, dtype=np.int64), lab)
    assert idx.remove_ids(torch.from_numpy(unknown)) == 0   # ids the index does not hold
    live = np.ones(n, bool)
    live[dead] = False
    rows = np.nonzero(live)[0]
    o = _oracle_on_rows(oracle_mod, c, rows, c.Q, 10, 8, 4)
    ids, dists = idx.search(_t(c.Q), 10, 8, 4)
    ids, dists = ids.cpu().numpy(), dists.cpu().numpy()
    want = np.where(o["ids"] >= 0, lab[np.maximum(o["ids"], 0)], -1)
    assert np.array_equal(ids, want) and np.array_equal(dists, o["dists"])
    idx.free()
    Xb = c.X[:n0].copy()
    Xb[7, 3] = np.nan                                       # non-finite input
    with pytest.raises(rb.RairsError):
        rb.Index.build(_t(Xb), c.spec.nlist, c.spec.M, centroids=_t(c.cent), codebook=_t(c.cb))
    idx = c.gpu_index()
    with pytest.raises(rb.RairsError):
        idx.add(_t(np.full((3, c.X.shape[1]), np.inf, np.float32)))
    assert idx.info()["n"] == c.X.shape[0]
    idx.free()
    for bad in (np.r_[lab[:n0 - 1], lab[0]], np.r_[lab[:n0 - 1], -5], np.r_[lab[:n0 - 1], 2**32 - 1]):
        with pytest.raises(rb.RairsError):
            rb.Index.build(_t(c.X[:n0]), c.spec.nlist, c.spec.M, centroids=_t(c.cent),
                           codebook=_t(c.cb), ids=_t(bad))


def test_search_stats(oracle_mod):
    # rairs_get_stats (SURVEY §8(b) rairs_stats): DCO total = the per-query DCO
    # sum, refined = the valid candidates, on both scan paths
    c = case(oracle_mod, "c1s")
    idx = c.gpu_index()
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, 10, 8, 4)
    idx.stats(reset=True)
    for scan in ("simt", "listmajor"):
        idx.set_scan_mode(scan)
        idx.search(_t(c.Q), 10, 8, 4)
    st = idx.stats(reset=True)
    nq = c.Q.shape[0]
    assert st["searches"] == 2 and st["queries"] == 2 * nq
    assert st["dco_total"] == 2 * int(o["dco"].sum())
    assert st["refine_total"] == 2 * int(np.minimum(o["dco"][:, 0], 40).sum())
    assert idx.stats()["dco_total"] == 0


def test_air_seil_direction_vs_single():
    # SURVEY §8(c) "parity unpinned" directional checks:
    # on the paper-like c2pl data, at the first swept nprobe reaching recall
    # 10@10 >= 0.9, AIR + SEIL needs <= 0.95x single assignment's DCO and
    # <= 0.7x its nprobe. Same trained state for both; 2,000 queries.
    from synth import get_config, make_dataset
    spec = get_config("c2pl")
    X, Q = make_dataset(spec, nq=2000)
    Xd, Qd = _t(X), _t(Q)
    gt_ids, gt_d = rb.exact_knn(Xd, Qd, 10)
    air = rb.build_index(Xd, spec.nlist, spec.M, assignment="AIR")
    cent, cb = air.export_trained()
    single = rb.Index.build(Xd, spec.nlist, spec.M, assignment="single", centroids=cent, codebook=cb)

    def first(idx):
        for npb in (1, 2, 3, 4, 5, 6, 8, 10, 12, 16):
            ids, dists, dco = idx.search(Qd, 10, npb, 10, return_dco=True)
            hit = (ids[:, :, None] == gt_ids[:, None, :]).any(-1)
            tie = (dists == gt_d[:, 9:10].float()) & (ids >= 0)
            rec = float((hit | tie).float().mean().item())
            if rec >= 0.9:
                return npb, float(dco.double().mean().item())
        raise AssertionError("recall 0.9 not reached")

    (pa, da), (ps, ds) = first(air), first(single)
    assert da <= 0.95 * ds, (pa, da, ps, ds)
    assert pa <= 0.7 * ps, (pa, ps)
    air.free()
    single.free()
