"""Paper-literal SEIL layout on the GPU (NEXT-2; Alg. 4 SeilInsert P:1480-1560,
Alg. 5 SeilSearch P:1604-1649) against the CPU oracle.

The paper layout stores each cell's full 32-item blocks once and duplicates
the remainders into both lists' miscellaneous areas; searched per Alg. 5 with
the lists visited in ascending id (reading R9) it must return exactly the
oracle's candidates and results (U(q) is the same set), while the number of
scored items is the paper's DCO_paperSEIL: the oracle's O12 formula
(oracle_dco_variants), pinned independently by tests/seil_paper_sim.py."""
import numpy as np
import pytest

from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

if not gpu_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2601_07183_b200 as rb  # noqa: E402
from tests.test_gpu_parity import _t, assert_search_equal, case, gpu_search  # noqa: E402


def _check_paper(oracle_mod, c, idx, k, nprobe, rf, X=None, l1=None, l2=None, codes=None):
    X = c.X if X is None else X
    l1 = c.l1 if l1 is None else l1
    l2 = c.l2 if l2 is None else l2
    codes = c.codes if codes is None else codes
    o = oracle_mod.search(X, l1, l2, codes, c.cent, c.cb, c.Q, k, nprobe, rf)
    g = gpu_search(idx, c.Q, k, nprobe, rf, "simt")
    _, paper = oracle_mod.dco_variants(l1, l2, c.spec.nlist, o["probes"])
    assert np.array_equal(g["dco"], paper), "DCO differs from DCO_paperSEIL (O12)"
    g["dco"] = o["dco"][:, 0]  # the rest must equal the cell-major oracle exactly
    assert_search_equal(g, o)
    return o, paper


@pytest.mark.parametrize("name,k,nprobe,rf", [
    ("c0s", 5, 4, 4), ("c1", 10, 8, 4), ("c1s", 10, 8, 4), ("c1s", 10, 16, 10),
    ("c1s", 1, 3, 100), ("c1s", 100, 8, 4), ("c1", 10, 64, 4),
])
def test_paper_seil_search_equals_oracle(oracle_mod, name, k, nprobe, rf):
    c = case(oracle_mod, name)
    idx = c.gpu_index()
    idx.set_seil_layout("paper")
    o, paper = _check_paper(oracle_mod, c, idx, k, nprobe, rf)
    # the paper layout scores every remainder item in each probed list holding it
    assert (paper >= o["dco"][:, 0]).all()
    # back to cell-major: its own DCO again (O12 cell-major = |U(q)| pieces)
    idx.set_seil_layout("cell")
    assert_search_equal(gpu_search(idx, c.Q, k, nprobe, rf, "simt"), o)
    idx.free()


def test_paper_seil_forced_listmajor_takes_query_major(oracle_mod):
    c = case(oracle_mod, "c1s")
    idx = c.gpu_index()
    idx.set_seil_layout("paper")
    assert idx.scan_path(c.Q.shape[0], 10, 8, 4) == "simt"
    idx.set_scan_mode("listmajor")
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, 10, 8, 4)
    g = gpu_search(idx, c.Q, 10, 8, 4, "listmajor")
    _, paper = oracle_mod.dco_variants(c.l1, c.l2, c.spec.nlist, o["probes"])
    assert np.array_equal(g["dco"], paper)
    idx.free()


def test_paper_seil_rebuilt_by_insert_and_delete(oracle_mod):
    # the layout follows rairs_add / rairs_remove_ids while selected
    c = case(oracle_mod, "c1s")
    n = c.X.shape[0]
    n0 = int(0.7 * n)
    idx = rb.Index.build(_t(c.X[:n0]), c.spec.nlist, c.spec.M, assignment="AIR",
                         centroids=_t(c.cent), codebook=_t(c.cb))
    idx.set_seil_layout("paper")
    assert idx.add(_t(c.X[n0:])) == n0
    _check_paper(oracle_mod, c, idx, 10, 8, 4)
    # delete every 7th row: the oracle over the live rows (ids keep their row)
    dead = np.arange(0, n, 7)
    assert idx.remove_ids(_t(dead.astype(np.int64))) == dead.size
    live = np.setdiff1d(np.arange(n), dead)
    o = oracle_mod.search(c.X[live], c.l1[live], c.l2[live], c.codes[live], c.cent, c.cb, c.Q, 10, 8, 4)
    g = gpu_search(idx, c.Q, 10, 8, 4, "simt")
    _, paper = oracle_mod.dco_variants(c.l1[live], c.l2[live], c.spec.nlist, o["probes"])
    assert np.array_equal(g["dco"], paper)
    ids = np.where(o["ids"] >= 0, live[np.maximum(o["ids"], 0)], -1)
    assert np.array_equal(g["ids"], ids)
    fin = np.isfinite(o["dists"])
    assert np.allclose(g["dists"][fin], o["dists"][fin], rtol=1e-4, atol=0)
    idx.free()


def test_seil_layout_auto_per_scan_path(oracle_mod):
    # auto: query-major scans read the paper layout (DCO_paperSEIL), list-major
    # scans the cell-major one (the oracle's cell-major DCO); results identical
    c = case(oracle_mod, "c1s")
    idx = c.gpu_index()
    idx.set_seil_layout("auto")
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, 10, 8, 4)
    _, paper = oracle_mod.dco_variants(c.l1, c.l2, c.spec.nlist, o["probes"])
    g = gpu_search(idx, c.Q, 10, 8, 4, "simt")
    assert np.array_equal(g["dco"], paper)
    g["dco"] = o["dco"][:, 0]
    assert_search_equal(g, o)
    assert_search_equal(gpu_search(idx, c.Q, 10, 8, 4, "listmajor"), o)
    idx.free()


def _hybrid_extra(l1, l2, probes, tiny=8):
    """Items the hybrid layout scores beyond the cell-major DCO: per query, the
    items of every cross cell {a < b} with fewer than `tiny` items whose two
    lists were both probed (the copy in b's misc area is scored, then dropped)."""
    a = np.minimum(l1, l2).astype(np.int64)
    b = np.maximum(l1, l2).astype(np.int64)
    cross = a != b
    keys, n = np.unique(a[cross] * (1 << 32) + b[cross], return_counts=True)
    keys, n = keys[n < tiny], n[n < tiny]
    ca, cb = keys >> 32, keys & 0xFFFFFFFF
    out = np.zeros(probes.shape[0], dtype=np.int64)
    for q in range(probes.shape[0]):
        P = probes[q][probes[q] >= 0]
        out[q] = int(n[np.isin(ca, P) & np.isin(cb, P)].sum())
    return out


@pytest.mark.parametrize("name,k,nprobe,rf", [
    ("c0s", 5, 4, 4), ("c1s", 10, 8, 4), ("c1s", 1, 3, 100), ("c1s", 100, 16, 10), ("c1", 10, 64, 4),
])
def test_hybrid_seil_search_equals_oracle(oracle_mod, name, k, nprobe, rf):
    # hybrid layout (not in the paper): same U(q) and results as the cell-major
    # oracle; DCO = cell-major DCO + the tiny cross cells probed from both sides
    c = case(oracle_mod, name)
    idx = c.gpu_index()
    idx.set_seil_layout("hybrid")
    o = oracle_mod.search(c.X, c.l1, c.l2, c.codes, c.cent, c.cb, c.Q, k, nprobe, rf)
    g = gpu_search(idx, c.Q, k, nprobe, rf, "simt")
    extra = _hybrid_extra(c.l1, c.l2, o["probes"])
    assert np.array_equal(g["dco"], o["dco"][:, 0] + extra)
    g["dco"] = o["dco"][:, 0]
    assert_search_equal(g, o)
    # list-major scans read the cell-major layout: its own DCO (large k*rf
    # takes the query-major scan even when list-major is forced)
    idx.set_scan_mode("listmajor")
    if idx.scan_path(c.Q.shape[0], k, nprobe, rf) == "listmajor":
        assert_search_equal(gpu_search(idx, c.Q, k, nprobe, rf, "listmajor"), o)
    # paper <-> hybrid switches rebuild the layout
    idx.set_seil_layout("paper")
    _check_paper(oracle_mod, c, idx, k, nprobe, rf)
    idx.set_seil_layout("hybrid")
    g = gpu_search(idx, c.Q, k, nprobe, rf, "simt")
    assert np.array_equal(g["dco"], o["dco"][:, 0] + extra)
    idx.free()


def test_hybrid_seil_rebuilt_by_insert_and_delete(oracle_mod):
    c = case(oracle_mod, "c1s")
    n = c.X.shape[0]
    n0 = int(0.6 * n)
    idx = rb.Index.build(_t(c.X[:n0]), c.spec.nlist, c.spec.M, assignment="AIR",
                         centroids=_t(c.cent), codebook=_t(c.cb))
    idx.set_seil_layout("hybrid")
    assert idx.add(_t(c.X[n0:])) == n0
    dead = np.arange(3, n, 5)
    assert idx.remove_ids(_t(dead.astype(np.int64))) == dead.size
    live = np.setdiff1d(np.arange(n), dead)
    o = oracle_mod.search(c.X[live], c.l1[live], c.l2[live], c.codes[live], c.cent, c.cb, c.Q, 10, 8, 4)
    g = gpu_search(idx, c.Q, 10, 8, 4, "simt")
    assert np.array_equal(g["dco"], o["dco"][:, 0] + _hybrid_extra(c.l1[live], c.l2[live], o["probes"]))
    ids = np.where(o["ids"] >= 0, live[np.maximum(o["ids"], 0)], -1)
    assert np.array_equal(g["ids"], ids)
    fin = np.isfinite(o["dists"])
    assert np.allclose(g["dists"][fin], o["dists"][fin], rtol=1e-4, atol=0)
    idx.free()
