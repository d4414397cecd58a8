"""GPU parity, round 2 additions (through the C ABI, against the CPU oracle):

* the query-major register-LUT fast scan (fs_scan_kernel) and the list-major
  tensor scan over a sweep of M (M_pad/4 from 4 to 96 chunks), including the
  c3 shape (d = 1536, M = 384: integer scores above 16 bits, R4);
* BJ configs[3] (c4) and configs[4] (c5) at full size in the bench's launch
  configuration (the query-major kernel the bench times), sampled queries;
* delete-then-re-add of the same caller ids; the K7 merge with 64-bit ids.
No expected value comes from the CUDA path.
"""
import numpy as np
import pytest

from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

if not gpu_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import get_config, make_dataset  # noqa: E402
from tests.test_gpu_parity import DEV, _t, assert_search_equal, case, gpu_search  # noqa: E402
from tests.test_gpu_seil_paper import _hybrid_extra  # noqa: E402


def _oracle_index(oracle, X, nlist, M, seed=11):
    rows = X[np.random.default_rng(5).permutation(X.shape[0])[:min(20000, X.shape[0])]]
    cent = oracle.kmeans(rows, nlist, iters=4, seed=seed)
    cb = oracle.pq_train(rows, M, iters=4, seed=seed + 1)
    l1, l2 = oracle.assign(X, cent, "air")
    codes = oracle.encode(X, cb)
    return cent, cb, l1, l2, codes


# (d, M): M_pad / 4 = 4 (M = 8 -> 16), 8, 12, 16, 24, 32, 48; the c3 shape below
MS = [(16, 8), (48, 24), (96, 48), (128, 64), (192, 96), (256, 128), (384, 192)]


@pytest.mark.parametrize("scan", ["simt", "listmajor"])
@pytest.mark.parametrize("d,M", MS)
def test_scan_parity_M_variants(oracle_mod, d, M, scan):
    """Every stage bit-exact (probes, Qv/a/b, DCO, candidate (s, id), ids) and
    refined distances within 1e-4, for M_pad/4 = 4 .. 48 code chunks; the
    list-major path serves M_pad/16 in {1, 2, 3, 4, 6, 8} and falls back to
    the query-major kernel otherwise (asserted)."""
    spec = get_config("c0s", n=4000, nq=40, d=d, M=M, nlist=16)
    X, Q = make_dataset(spec)
    cent, cb, l1, l2, codes = _oracle_index(oracle_mod, X, spec.nlist, M)
    idx = rb.Index.build(_t(X), spec.nlist, M, centroids=_t(cent), codebook=_t(cb))
    M_pad = -(-M // 16) * 16
    lm_ok = M_pad // 16 in (1, 2, 3, 4, 6, 8)
    idx.set_scan_mode(scan)
    want = "listmajor" if (scan == "listmajor" and lm_ok) else "simt"
    assert idx.scan_path(Q.shape[0], 5, 4, 4) == want
    for k, nprobe, rf in ((5, 4, 4), (10, 16, 8)):
        o = oracle_mod.search(X, l1, l2, codes, cent, cb, Q, k, nprobe, rf)
        assert_search_equal(gpu_search(idx, Q, k, nprobe, rf, scan), o)
    idx.free()


@pytest.mark.parametrize("scan", ["simt", "listmajor"])
def test_c3_shape_parity(oracle_mod, scan):
    """BJ configs[2]'s shape (unit vectors, d = 1536, M = 384 x 4-bit, dsub 4)
    on a reduced base: integer scores reach M*255 = 97,920 > 2^16 (R4: the
    query-major kernel accumulates exact u32 per item; the list-major path
    does not serve M_pad = 384 and falls back to it)."""
    spec = get_config("c3", n=8000, nq=24, nlist=64)
    X, Q = make_dataset(spec)
    cent, cb, l1, l2, codes = _oracle_index(oracle_mod, X, spec.nlist, spec.M)
    idx = rb.Index.build(_t(X), spec.nlist, spec.M, centroids=_t(cent), codebook=_t(cb))
    for k, nprobe, rf in ((10, 8, 10), (10, 64, 4)):
        o = oracle_mod.search(X, l1, l2, codes, cent, cb, Q, k, nprobe, rf)
        g = gpu_search(idx, Q, k, nprobe, rf, scan)
        assert int(o["cand_scores"].max()) >= 0
        assert_search_equal(g, o)
    idx.free()


def test_delete_then_readd_same_ids(oracle_mod):
    """SPEC delete_vectors: an id deleted then added again (with a new vector)
    is searchable again and can be deleted again."""
    from tests.test_gpu_parity import _oracle_on_rows, case
    c = case(oracle_mod, "c1s")
    n = c.X.shape[0]
    lab = np.arange(n, dtype=np.int64) * 7 + 3
    n0 = n - 300
    idx = rb.Index.build(_t(c.X[:n0]), c.spec.nlist, c.spec.M, assignment="AIR",
                         centroids=_t(c.cent), codebook=_t(c.cb), ids=_t(lab[:n0]))
    rng = np.random.default_rng(4)
    dead = rng.choice(n0, size=300, replace=False)
    assert idx.remove_ids(torch.from_numpy(lab[dead])) == dead.size
    # the same ids come back with the last 300 vectors
    idx.add(_t(c.X[n0:]), ids=_t(lab[dead]))
    live = np.ones(n, bool)
    live[dead] = False
    rows = np.nonzero(live)[0]                 # rows n0.. carry the labels lab[dead]
    row_lab = lab.copy()
    row_lab[n0:] = lab[dead]
    o = _oracle_on_rows(oracle_mod, c, rows, c.Q, 10, 8, 4)
    ids, dists = idx.search(_t(c.Q), 10, 8, 4)
    ids, dists = ids.cpu().numpy(), dists.cpu().numpy()
    want = np.where(o["ids"] >= 0, row_lab[np.maximum(o["ids"], 0)], -1)
    assert np.array_equal(ids, want) and np.array_equal(dists, o["dists"])
    # a re-added id is held again (adding it a third time is rejected) ...
    with pytest.raises(rb.RairsError):
        idx.add(_t(c.X[:1]), ids=_t(lab[dead[:1]]))
    # ... and deletes hit the live row
    assert idx.remove_ids(torch.from_numpy(lab[dead[:50]])) == 50
    idx.free()


def test_merge_topk_64bit_ids():
    """K7 merge orders by (fp32 distance, full 64-bit id): ids above 2^32
    keep all their bits and break distance ties correctly (O11)."""
    rng = np.random.default_rng(3)
    G, nq, k = 4, 50, 16
    d = rng.integers(0, 6, size=(G, nq, k)).astype(np.float32)   # many exact ties
    ids = rng.choice(2**40, size=(G, nq, k), replace=False).astype(np.int64) + (1 << 33)
    ids[0, :, -3:] = -1
    d[0, :, -3:] = np.inf
    oi, od = rb.merge_topk(_t(ids), _t(d))
    oi, od = oi.cpu().numpy(), od.cpu().numpy()
    for q in range(nq):
        ii, dd = ids[:, q].ravel(), d[:, q].ravel()
        ok = ii >= 0
        order = np.lexsort((ii[ok], dd[ok]))[:k]
        assert np.array_equal(oi[q], ii[ok][order]) and np.array_equal(od[q], dd[ok][order])


def _full_size_sampled(oracle_mod, name, nprobe, scan, n_q=32, n_rows=20000, n_assign=4000):
    """A BJ config at full size, drawn on the device, GPU-trained (outside the
    bit-exact contract, R16), searched in the bench's launch configuration (all
    10k queries in one batch); the oracle checks, from the exported trained
    state and the same input rows, on samples it computes one by one:
      O4/O5  assignment and codes of sampled rows;
      O1/O2  probe sets and quantised LUT of sampled queries;
      O8     every returned candidate's integer score from the oracle's encode;
      O9     completeness on a row sample: every sampled row of U(q) whose key
             (s, id) is below the bigK-th candidate key is a candidate;
      O10    final ids = first k candidates by (delta, id), delta the fp64
             ordered sum rounded to fp32 (1e-4 relative)."""
    from synth.gpu_generators import make_dataset_torch
    spec = get_config(name)
    k, rf = spec.k, spec.refine_factor
    bigK = k * rf
    Xd, Qd = make_dataset_torch(spec, DEV)
    idx = rb.build_index(Xd, spec.nlist, spec.M, train_sample=64 * spec.nlist, kmeans_iters=10)
    idx.set_scan_mode(scan)
    path = idx.scan_path(spec.nq, k, nprobe, rf)
    out = idx.search_debug(Qd, k, nprobe, rf)
    ids_plain, d_plain = idx.search(Qd, k, nprobe, rf)     # the bench's entry point
    torch.cuda.synchronize()
    assert torch.equal(ids_plain, out["ids"]) and torch.equal(d_plain, out["dists"])
    rng = np.random.default_rng(11)
    qs = np.sort(rng.choice(spec.nq, n_q, replace=False))
    g = {key: v.cpu().numpy()[qs] for key, v in out.items()}
    g["cand_ids"] = g["cand_ids"].view(np.uint32)
    g["cand_scores"] = g["cand_scores"].view(np.uint32)
    cent, cb = [t.cpu().numpy() for t in idx.export_trained()]
    l1, l2, codes = [t.cpu().numpy() for t in idx.export_assignment()]
    Q = Qd.cpu().numpy()[qs]
    rows = np.sort(rng.choice(spec.n, n_rows, replace=False))
    Xs = Xd[torch.from_numpy(rows).to(DEV)].cpu().numpy()
    ol1, ol2 = oracle_mod.assign(Xs[:n_assign], cent, "air")
    assert np.array_equal(l1[rows[:n_assign]], ol1) and np.array_equal(l2[rows[:n_assign]], ol2)
    assert np.array_equal(codes[rows[:n_assign]], oracle_mod.encode(Xs[:n_assign], cb))
    assert np.array_equal(g["probes"], oracle_mod.probe(Q, cent, nprobe))
    Qv, a, b = oracle_mod.lut(Q, cb)
    assert np.array_equal(g["Qv"], Qv) and np.array_equal(g["a"], a) and np.array_equal(g["b"], b)
    sl1, sl2 = l1[rows], l2[rows]                 # checked on n_assign rows above
    scodes = codes[rows].astype(np.int64)
    for i in range(len(qs)):
        cid = g["cand_ids"][i]
        valid = cid != 0xFFFFFFFF
        cx = Xd[torch.from_numpy(cid[valid].astype(np.int64)).to(DEV)].cpu().numpy()
        cc = oracle_mod.encode(cx, cb).astype(np.int64)
        s = Qv[i][np.arange(spec.M)[None, :], cc].sum(1)
        assert np.array_equal(s, g["cand_scores"][i][valid].astype(np.int64)), "O8 scores"
        assert np.all(np.diff(s * 2**32 + cid[valid].astype(np.int64)) > 0), "keys sorted"
        P = set(g["probes"][i].tolist())
        inU = np.array([(x in P) or (y in P) for x, y in zip(sl1, sl2)])
        ss = Qv[i][np.arange(spec.M)[None, :], scodes].sum(1)
        kmax = s[-1] * 2**32 + int(cid[valid][-1]) if valid.sum() == bigK else np.inf
        must = inU & (ss * 2**32 + rows < kmax)
        assert set(rows[must].tolist()) <= set(cid[valid].tolist()), "O9 completeness"
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
    return path


def test_c4_full_size_query_major(oracle_mod):
    """BJ configs[3] (10M x 96) in the bench's configuration: auto picks the
    query-major register-LUT kernel (1.2 queries per probed list)."""
    assert _full_size_sampled(oracle_mod, "c4", 2, "auto") == "simt"


def test_c5_full_size_sampled(oracle_mod):
    """BJ configs[4] (100M x 128, nlist 65,536, nprobe 64) at full size: the
    capped-list coarse path with its uncertified rows, the scan of one 10k batch
    (~98k items per query), refine; 16 queries and 5,000 rows checked."""
    _full_size_sampled(oracle_mod, "c5", 64, "auto", n_q=16, n_rows=5000, n_assign=2000)


@pytest.mark.parametrize("parts", [2, 7, 64])
@pytest.mark.parametrize("nq", [1, 5, 100])
def test_split_query_parts_equal_oracle(oracle_mod, parts, nq):
    """Small-batch split mode of the query-major scan (each query's group tasks
    over `parts` warps, per-part exact top-bigK, then a P-way merge): the same
    candidates, DCO and results as the oracle (RAIRS_FS_PARTS forces P)."""
    import os
    c = case(oracle_mod, "c1s")
    idx = c.gpu_index()
    Q = c.Q[:nq]
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, Q, 10, 16, 10)
    os.environ["RAIRS_FS_PARTS"] = str(parts)
    try:
        g = gpu_search(idx, Q, 10, 16, 10, "simt")
    finally:
        del os.environ["RAIRS_FS_PARTS"]
    assert_search_equal(g, o)
    idx.free()


@pytest.mark.parametrize("nq", [1, 5, 16, 17])
def test_small_batch_coarse_split_path(oracle_mod, nq):
    """Search batches of <= 16 queries over >= 8,192 lists take the split exact
    coarse path for every row (no TF32 GEMM / certificate); 17 queries take
    the tensor-core path.  Both must give O1's probes and the oracle's
    results (Alg. 3 / O1, O10)."""
    spec = get_config("c0s", n=30000, nq=nq, d=32, M=16, nlist=8192)
    X, Q = make_dataset(spec)
    rows = X[np.random.default_rng(5).permutation(X.shape[0])[:20000]]
    cent = rows[np.random.default_rng(6).permutation(rows.shape[0])[:8192]].copy()
    cb = oracle_mod.pq_train(rows, 16, iters=2, seed=1)
    l1, l2 = oracle_mod.assign(X, cent, "air")
    codes = oracle_mod.encode(X, cb)
    idx = rb.Index.build(_t(X), 8192, 16, centroids=_t(cent), codebook=_t(cb))
    Qd = _t(Q)
    for k, nprobe, rf in ((10, 3, 10), (5, 40, 4)):
        pt = idx.search_debug(Qd, k, nprobe, rf)["probes"].cpu().numpy()
        assert np.array_equal(pt, oracle_mod.probe(Q, cent, nprobe))
        o = oracle_mod.search(X, l1, l2, codes, cent, cb, Q, k, nprobe, rf)
        assert_search_equal(gpu_search(idx, Q, k, nprobe, rf), o)
    idx.free()


@pytest.mark.parametrize("layout", ["cell", "paper", "hybrid"])
def test_runs_of_one_group_ranges(oracle_mod, layout):
    """8,192 lists of ~4 vectors and AIR references: a query's SEIL work list
    (Alg. 5) holds long runs of one-group ranges (short owned ranges and
    references).  A round whose 32 tasks each start a new range must hand
    the next round the range starting at position 32 (a range there was
    once skipped: DCO still equal, one item never scored).  40 queries: the
    unsplit query-major scan; nprobe 3 and 40."""
    spec = get_config("c0s", n=30000, nq=40, d=32, M=16, nlist=8192)
    X, Q = make_dataset(spec)
    rows = X[np.random.default_rng(5).permutation(X.shape[0])[:20000]]
    cent = rows[np.random.default_rng(6).permutation(rows.shape[0])[:8192]].copy()
    cb = oracle_mod.pq_train(rows, 16, iters=2, seed=1)
    l1, l2 = oracle_mod.assign(X, cent, "air")
    codes = oracle_mod.encode(X, cb)
    idx = rb.Index.build(_t(X), 8192, 16, centroids=_t(cent), codebook=_t(cb))
    idx.set_seil_layout(layout)
    for k, nprobe, rf in ((10, 3, 10), (5, 40, 4)):
        o = oracle_mod.search(X, l1, l2, codes, cent, cb, Q, k, nprobe, rf)
        g = gpu_search(idx, Q, k, nprobe, rf, "simt")
        if layout == "paper":  # the paper-literal layout's DCO is O12's DCO_paperSEIL
            want = oracle_mod.dco_variants(l1, l2, 8192, o["probes"])[1]
            assert np.array_equal(g["dco"], np.asarray(want).reshape(g["dco"].shape))
            g = dict(g, dco=o["dco"][:, 0])
        elif layout == "hybrid":  # + the tiny cross cells probed from both sides
            assert np.array_equal(g["dco"], o["dco"][:, 0] + _hybrid_extra(l1, l2, o["probes"]))
            g = dict(g, dco=o["dco"][:, 0])
        assert_search_equal(g, o)
    idx.free()
