"""ctypes binding for the plain CPU oracle (``rairs_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs. The product package
``paper_2601_07183_b200`` never imports this module (and vice versa).

Every wrapper takes/returns host numpy arrays; see rairs_oracle.c for the
passage each routine follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_F64 = ctypes.c_double
_U64 = ctypes.c_uint64


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "rairs_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "ORACLE_CC=gcc"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_set_threads.argtypes = [_I32]
        L.oracle_max_threads.argtypes = []
        L.oracle_probe.argtypes = [_P, _I64, _I32, _P, _I32, _I32, _P]
        L.oracle_assign.argtypes = [_P, _I64, _I32, _P, _I32, _I32, _F64, _I32, _I32, _P, _P]
        L.oracle_encode.argtypes = [_P, _I64, _I32, _P, _I32, _P]
        L.oracle_lut.argtypes = [_P, _I64, _I32, _P, _I32, _P, _P, _P]
        L.oracle_search.argtypes = ([_P, _I64, _I32, _P, _P, _P, _I32, _P, _I32, _P, _P, _I64,
                                     _I32, _I32, _I32, _I32] + [_P] * 11)
        L.oracle_dco_variants.argtypes = [_P, _P, _I64, _I32, _P, _I64, _I32, _P, _P]
        L.oracle_exact_knn.argtypes = [_P, _I64, _I32, _P, _I64, _I32, _P, _P]
        L.oracle_kmeans.argtypes = [_P, _I64, _I32, _I32, _I32, _U64, _P, _P]
        L.oracle_pq_train.argtypes = [_P, _I64, _I32, _I32, _I32, _U64, _P]
        _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with status {rc}")


def set_threads(n: int) -> int:
    return lib().oracle_set_threads(int(n))


def max_threads() -> int:
    return lib().oracle_max_threads()


def probe(queries, centroids, nprobe: int) -> np.ndarray:
    """O1: P(q) = first nprobe lists by (D64, l)."""
    q, c = _f32(queries), _f32(centroids)
    out = np.empty((q.shape[0], nprobe), np.int32)
    _check(lib().oracle_probe(_ptr(q), q.shape[0], q.shape[1], _ptr(c), c.shape[0], nprobe,
                              _ptr(out)), "probe")
    return out


def assign(x, centroids, mode: str = "air", lam: float = 0.5, n_cands: int = 10,
           strict: bool = False):
    """O4: (l1, l2) sorted pair per vector (Alg. 3); mode "soar" = SOARL2
    (Table 2's SOAR loss in Alg. 3's place)."""
    xx, c = _f32(x), _f32(centroids)
    n = xx.shape[0]
    l1 = np.empty(n, np.int32)
    l2 = np.empty(n, np.int32)
    m = {"single": 0, "air": 1, "soar": 2}[mode]
    _check(lib().oracle_assign(_ptr(xx), n, xx.shape[1], _ptr(c), c.shape[0], m, float(lam),
                               int(n_cands), int(bool(strict)), _ptr(l1), _ptr(l2)), "assign")
    return l1, l2


def encode(x, codebook) -> np.ndarray:
    """O5: unpacked codes [n x M] uint8."""
    xx, cb = _f32(x), _f32(codebook)
    M = cb.shape[0]
    out = np.empty((xx.shape[0], M), np.uint8)
    _check(lib().oracle_encode(_ptr(xx), xx.shape[0], xx.shape[1], _ptr(cb), M, _ptr(out)),
           "encode")
    return out


def lut(queries, codebook):
    """O2: (Qv [nq x M x 16] u8, a [nq] f32, b [nq] f32)."""
    q, cb = _f32(queries), _f32(codebook)
    nq, M = q.shape[0], cb.shape[0]
    Qv = np.empty((nq, M, 16), np.uint8)
    a = np.empty(nq, np.float32)
    b = np.empty(nq, np.float32)
    _check(lib().oracle_lut(_ptr(q), nq, q.shape[1], _ptr(cb), M, _ptr(Qv), _ptr(a), _ptr(b)),
           "lut")
    return Qv, a, b


def search(X, l1, l2, codes, centroids, codebook, queries, k: int, nprobe: int,
           refine_factor: int, nshards: int = 1) -> Dict[str, np.ndarray]:
    """O7-O12 end to end (Alg. 2 by plain definitions), emulating G shards."""
    XX, q = _f32(X), _f32(queries)
    c, cb = _f32(centroids), _f32(codebook)
    a1, a2 = _i32(l1), _i32(l2)
    cd = np.ascontiguousarray(codes, dtype=np.uint8)
    n, d = XX.shape
    nq, M, G = q.shape[0], cb.shape[0], int(nshards)
    bigK = k * refine_factor
    r = {
        "probes": np.empty((nq, nprobe), np.int32),
        "Qv": np.empty((nq, M, 16), np.uint8),
        "a": np.empty(nq, np.float32),
        "b": np.empty(nq, np.float32),
        "cand_ids": np.empty((nq, G, bigK), np.uint32),
        "cand_scores": np.empty((nq, G, bigK), np.uint32),
        "dco": np.empty((nq, G), np.int64),
        "shard_ids": np.empty((nq, G, k), np.int64),
        "shard_dists": np.empty((nq, G, k), np.float32),
        "ids": np.empty((nq, k), np.int64),
        "dists": np.empty((nq, k), np.float32),
    }
    _check(lib().oracle_search(
        _ptr(XX), n, d, _ptr(a1), _ptr(a2), _ptr(cd), M, _ptr(c), c.shape[0], _ptr(cb),
        _ptr(q), nq, int(k), int(nprobe), int(refine_factor), G,
        _ptr(r["probes"]), _ptr(r["Qv"]), _ptr(r["a"]), _ptr(r["b"]), _ptr(r["cand_ids"]),
        _ptr(r["cand_scores"]), _ptr(r["dco"]), _ptr(r["shard_ids"]), _ptr(r["shard_dists"]),
        _ptr(r["ids"]), _ptr(r["dists"])), "search")
    return r


def dco_variants(l1, l2, nlist: int, probes):
    """O12: (dco_noseil, dco_paperseil) per query."""
    a1, a2, P = _i32(l1), _i32(l2), _i32(probes)
    nq, nprobe = P.shape
    a = np.empty(nq, np.int64)
    b = np.empty(nq, np.int64)
    _check(lib().oracle_dco_variants(_ptr(a1), _ptr(a2), a1.shape[0], int(nlist), _ptr(P), nq,
                                     nprobe, _ptr(a), _ptr(b)), "dco_variants")
    return a, b


def exact_knn(X, queries, K: int):
    """O13: (ids [nq x K] i64, D64 [nq x K] f64) by (D64, id)."""
    XX, q = _f32(X), _f32(queries)
    ids = np.empty((q.shape[0], K), np.int64)
    dd = np.empty((q.shape[0], K), np.float64)
    _check(lib().oracle_exact_knn(_ptr(XX), XX.shape[0], XX.shape[1], _ptr(q), q.shape[0], int(K),
                                  _ptr(ids), _ptr(dd)), "exact_knn")
    return ids, dd


def kmeans(x, k: int, iters: int = 25, seed: int = 1234, return_trace: bool = False):
    """O3 (training; outside the bit-exact contract)."""
    xx = _f32(x)
    out = np.empty((k, xx.shape[1]), np.float32)
    trace = np.empty(iters + 1, np.float64)
    _check(lib().oracle_kmeans(_ptr(xx), xx.shape[0], xx.shape[1], int(k), int(iters),
                               int(seed) & (2**64 - 1), _ptr(out), _ptr(trace)), "kmeans")
    return (out, trace) if return_trace else out


def pq_train(x, M: int, iters: int = 25, seed: int = 4321) -> np.ndarray:
    """O3 PQ codebook [M x 16 x dsub] (training; outside the bit-exact contract)."""
    xx = _f32(x)
    d = xx.shape[1]
    out = np.empty((M, 16, d // M), np.float32)
    _check(lib().oracle_pq_train(_ptr(xx), xx.shape[0], d, int(M), int(iters),
                                 int(seed) & (2**64 - 1), _ptr(out)), "pq_train")
    return out


def recall(ids: np.ndarray, gt_ids: np.ndarray, gt_d64: np.ndarray, X, queries,
           k: int) -> float:
    """recall k@k with SPEC's tie acceptance: a returned
    id whose D64 equals the k-th ground-truth distance also counts."""
    XX, q = _f32(X), _f32(queries)
    hits = 0
    for i in range(ids.shape[0]):
        g = set(int(v) for v in gt_ids[i, :k])
        kth = gt_d64[i, k - 1]
        for v in ids[i, :k]:
            v = int(v)
            if v < 0:
                continue
            if v in g:
                hits += 1
            else:
                df = q[i].astype(np.float64) - XX[v].astype(np.float64)
                dd = np.cumsum(df * df)[-1]          # fp64 ordered sum (O1/O13)
                if dd == kth:
                    hits += 1
    return hits / float(ids.shape[0] * k)
