"""Python face of the C ABI: build_index / Index.search (BASELINE north_star).

Argument marshalling only -- every step of the search path runs in the CUDA
kernels of librairs.so. PyTorch provides device memory and streams.
"""
from __future__ import annotations

import ctypes
from typing import Dict, Optional, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import BuildParams, IndexInfo, Stats, check, lib


def _dev_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    return t.detach().to(torch.float32).contiguous()


def _dev_ids(ids: Optional[torch.Tensor], n: int, device) -> Optional[torch.Tensor]:
    if ids is None:
        return None
    t = torch.as_tensor(ids).to(device=device, dtype=torch.int64).contiguous()
    if t.dim() != 1 or t.shape[0] != n:
        raise ValueError(f"ids must be a 1-D tensor of {n} ids")
    return t


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream: Optional[torch.cuda.Stream] = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_params(nlist: int, M: int, nbits: int = 4, assignment: str = "AIR",
                lambda_: float = 0.5, n_cands: int = 10, strict: bool = False,
                kmeans_iters: int = 25, train_sample: int = 0, seed: int = 1234,
                shard_id: int = 0, nshards: int = 1) -> BuildParams:
    p = BuildParams()
    lib().rairs_default_params(ctypes.byref(p), int(nlist), int(M))
    p.nbits = int(nbits)
    a = assignment.upper()
    modes = {"SINGLE": 0, "AIR": 1, "SOAR": 2, "SOARL2": 2}
    if a not in modes:
        raise ValueError("assignment must be 'AIR', 'single' or 'SOAR'")
    p.assignment = modes[a]
    p.lambda_ = float(lambda_)
    p.n_cands = int(n_cands)
    p.strict = int(bool(strict))
    p.kmeans_iters = int(kmeans_iters)
    p.train_sample = int(train_sample)
    p.seed = int(seed) & (2**64 - 1)
    p.shard_id = int(shard_id)
    p.nshards = int(nshards)
    return p


def train(base: torch.Tensor, nlist: int, M: int, **kw) -> Tuple[torch.Tensor, torch.Tensor]:
    """GPU k-means + PQ codebook training (rairs_train)."""
    base = _dev_f32(base, "base")
    n, d = base.shape
    p = make_params(nlist, M, **kw)
    cent = torch.empty((nlist, d), dtype=torch.float32, device=base.device)
    cb = torch.empty((M, 16, d // M), dtype=torch.float32, device=base.device)
    check(lib().rairs_train(_ptr(base), n, d, ctypes.byref(p), _stream(), _ptr(cent), _ptr(cb)),
          "rairs_train")
    return cent, cb


class Index:
    """One shard of a RAIRS index on one GPU (rairs_index_t)."""

    def __init__(self, handle: ctypes.c_void_p, device: torch.device):
        self._h = handle
        self.device = device
        info = self.info()
        self.n, self.d, self.nlist, self.M = info["n"], info["d"], info["nlist"], info["M"]
        self.shard_id, self.nshards = info["shard_id"], info["nshards"]

    # ------------------------------------------------------------ build
    @staticmethod
    def build(base: torch.Tensor, nlist: int, M: int, nbits: int = 4, assignment: str = "AIR",
              centroids: Optional[torch.Tensor] = None, codebook: Optional[torch.Tensor] = None,
              ids: Optional[torch.Tensor] = None, **kw) -> "Index":
        """ids: optional [n] int64 caller ids (unique, in [0, 2^32 - 2]); searches
        then return them and remove_ids takes them."""
        base = _dev_f32(base, "base")
        n, d = base.shape
        p = make_params(nlist, M, nbits=nbits, assignment=assignment, **kw)
        h = ctypes.c_void_p()
        idt = _dev_ids(ids, n, base.device)
        if centroids is None and codebook is None:
            check(lib().rairs_build_index(_ptr(base), n, d, _ptr(idt), ctypes.byref(p), _stream(),
                                          ctypes.byref(h)), "rairs_build_index")
        else:
            cent = _dev_f32(centroids, "centroids")
            cb = _dev_f32(codebook, "codebook")
            check(lib().rairs_build_from_trained(_ptr(base), n, d, _ptr(idt), _ptr(cent), _ptr(cb),
                                                 ctypes.byref(p), _stream(), ctypes.byref(h)),
                  "rairs_build_from_trained")
        return Index(h, base.device)

    def free(self):
        if self._h is not None and self._h.value:
            check(lib().rairs_index_free(self._h), "rairs_index_free")
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def info(self) -> Dict[str, int]:
        inf = IndexInfo()
        check(lib().rairs_index_get_info(self._h, ctypes.byref(inf)), "rairs_index_get_info")
        return {f: getattr(inf, f) for f, _ in IndexInfo._fields_}

    # ---------------------------------------------------------- updates
    def add(self, x: torch.Tensor, ids: Optional[torch.Tensor] = None) -> int:
        """Insert a batch (rairs_add); returns the global id of its first row
        (row i gets first_id + i * nshards). ids: the new rows' caller ids,
        required iff the index was built with ids."""
        xx = _dev_f32(x, "x")
        if xx.shape[1] != self.d:
            raise ValueError(f"x must be [n, {self.d}]")
        idt = _dev_ids(ids, xx.shape[0], xx.device)
        first = ctypes.c_int64(0)
        check(lib().rairs_add(self._h, _ptr(xx), xx.shape[0], _ptr(idt), ctypes.byref(first),
                              _stream()), "rairs_add")
        self.n = self.info()["n"]
        return int(first.value)

    def remove_ids(self, ids: torch.Tensor) -> int:
        """Delete rows by global id (rairs_remove_ids); returns how many this
        shard held and deleted now."""
        t = ids.to(device=self.device, dtype=torch.int64).contiguous()
        removed = ctypes.c_int64(0)
        check(lib().rairs_remove_ids(self._h, _ptr(t), t.numel(), ctypes.byref(removed),
                                     _stream()), "rairs_remove_ids")
        return int(removed.value)

    def stats(self, reset: bool = False) -> Dict[str, float]:
        """rairs_get_stats: searches, queries, DCO and refined totals, coarse
        fallbacks, stage ms (synchronises the device)."""
        st = Stats()
        check(lib().rairs_get_stats(self._h, ctypes.byref(st), int(bool(reset))), "rairs_get_stats")
        return {f: getattr(st, f) for f, _ in Stats._fields_}

    # ----------------------------------------------------------- search
    def search(self, queries: torch.Tensor, k: int, nprobe: int, refine_factor: int = 10,
               return_dco: bool = False, stream: Optional[torch.cuda.Stream] = None):
        """Batched Alg. 2 search on this shard. Returns (ids i64, dists f32) [nq x k]."""
        q = _dev_f32(queries, "queries")
        nq = q.shape[0]
        ids = torch.empty((nq, k), dtype=torch.int64, device=q.device)
        dists = torch.empty((nq, k), dtype=torch.float32, device=q.device)
        dco = torch.empty((nq,), dtype=torch.int64, device=q.device) if return_dco else None
        check(lib().rairs_search(self._h, _ptr(q), nq, int(k), int(nprobe), int(refine_factor),
                                 _ptr(ids), _ptr(dists), _ptr(dco), _stream(stream)),
              "rairs_search")
        return (ids, dists, dco) if return_dco else (ids, dists)

    def search_host(self, queries: np.ndarray, k: int, nprobe: int, refine_factor: int = 10,
                    out_ids: Optional[np.ndarray] = None, out_dists: Optional[np.ndarray] = None):
        """Host buffers in/out (rairs_search_host: H2D + search + D2H + sync)."""
        q = np.ascontiguousarray(queries, dtype=np.float32)
        nq = q.shape[0]
        ids = out_ids if out_ids is not None else np.empty((nq, k), np.int64)
        dists = out_dists if out_dists is not None else np.empty((nq, k), np.float32)
        check(lib().rairs_search_host(self._h, q.ctypes.data_as(ctypes.c_void_p), nq, int(k),
                                      int(nprobe), int(refine_factor),
                                      ids.ctypes.data_as(ctypes.c_void_p),
                                      dists.ctypes.data_as(ctypes.c_void_p), _stream()),
              "rairs_search_host")
        return ids, dists

    def search_host_async(self, queries: np.ndarray, k: int, nprobe: int, refine_factor: int,
                          out_ids: np.ndarray, out_dists: np.ndarray):
        """rairs_search_host_async: enqueue H2D + search + D2H on the current
        stream and return; the (pinned) host buffers are filled once the
        stream reaches this point (synchronise it before reading them)."""
        q = np.ascontiguousarray(queries, dtype=np.float32)
        if not (out_ids.flags.c_contiguous and out_dists.flags.c_contiguous):
            raise ValueError("output buffers must be C-contiguous")
        check(lib().rairs_search_host_async(self._h, q.ctypes.data_as(ctypes.c_void_p), q.shape[0],
                                            int(k), int(nprobe), int(refine_factor),
                                            out_ids.ctypes.data_as(ctypes.c_void_p),
                                            out_dists.ctypes.data_as(ctypes.c_void_p), _stream()),
              "rairs_search_host_async")

    def search_debug(self, queries: torch.Tensor, k: int, nprobe: int,
                     refine_factor: int = 10) -> Dict[str, torch.Tensor]:
        q = _dev_f32(queries, "queries")
        nq, dev = q.shape[0], q.device
        bigK = k * refine_factor
        r = {
            "probes": torch.empty((nq, nprobe), dtype=torch.int32, device=dev),
            "Qv": torch.empty((nq, self.M, 16), dtype=torch.uint8, device=dev),
            "a": torch.empty((nq,), dtype=torch.float32, device=dev),
            "b": torch.empty((nq,), dtype=torch.float32, device=dev),
            "cand_ids": torch.empty((nq, bigK), dtype=torch.int32, device=dev),
            "cand_scores": torch.empty((nq, bigK), dtype=torch.int32, device=dev),
            "dco": torch.empty((nq,), dtype=torch.int64, device=dev),
            "ids": torch.empty((nq, k), dtype=torch.int64, device=dev),
            "dists": torch.empty((nq, k), dtype=torch.float32, device=dev),
        }
        check(lib().rairs_search_debug(
            self._h, _ptr(q), nq, int(k), int(nprobe), int(refine_factor), _ptr(r["probes"]),
            _ptr(r["Qv"]), _ptr(r["a"]), _ptr(r["b"]), _ptr(r["cand_ids"]), _ptr(r["cand_scores"]),
            _ptr(r["dco"]), _ptr(r["ids"]), _ptr(r["dists"]), _stream()), "rairs_search_debug")
        return r

    # ---------------------------------------------------------- exports
    def export_trained(self) -> Tuple[torch.Tensor, torch.Tensor]:
        cent = torch.empty((self.nlist, self.d), dtype=torch.float32, device=self.device)
        cb = torch.empty((self.M, 16, self.d // self.M), dtype=torch.float32, device=self.device)
        check(lib().rairs_export_trained(self._h, _ptr(cent), _ptr(cb), _stream()),
              "rairs_export_trained")
        return cent, cb

    def export_assignment(self) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
        l1 = torch.empty((self.n,), dtype=torch.int32, device=self.device)
        l2 = torch.empty((self.n,), dtype=torch.int32, device=self.device)
        codes = torch.zeros((self.n, self.M), dtype=torch.uint8, device=self.device)  # deleted rows: 0
        check(lib().rairs_export_assignment(self._h, _ptr(l1), _ptr(l2), _ptr(codes), _stream()),
              "rairs_export_assignment")
        return l1, l2, codes

    def export_layout(self) -> Dict[str, torch.Tensor]:
        info = self.info()
        nl, nr, ns = info["nlist"], info["n_refs"], info["n_slots"]
        dev = self.device
        r = {
            "own_off": torch.empty((nl,), dtype=torch.int64, device=dev),
            "own_cnt": torch.empty((nl,), dtype=torch.int64, device=dev),
            "ref_ptr": torch.empty((nl + 1,), dtype=torch.int64, device=dev),
            "ref_owner": torch.empty((max(nr, 1),), dtype=torch.int32, device=dev),
            "ref_start": torch.empty((max(nr, 1),), dtype=torch.int64, device=dev),
            "ref_cnt": torch.empty((max(nr, 1),), dtype=torch.int64, device=dev),
            "slot_rows": torch.empty((max(ns, 1),), dtype=torch.int32, device=dev),
        }
        check(lib().rairs_export_layout(self._h, *[_ptr(r[k]) for k in
                                                   ("own_off", "own_cnt", "ref_ptr", "ref_owner",
                                                    "ref_start", "ref_cnt", "slot_rows")],
                                        _stream()), "rairs_export_layout")
        for key in ("ref_owner", "ref_start", "ref_cnt"):
            r[key] = r[key][:nr]
        r["slot_rows"] = r["slot_rows"][:ns]
        return r

    # ---------------------------------------------------- coarse stage
    COARSE_MODES = {"auto": 0, "exact": 1, "tensor": 2}

    def set_coarse_mode(self, mode: str = "auto"):
        """auto | exact (fp64 only) | tensor (TF32 tcgen05 filter + fp64 certify)."""
        check(lib().rairs_set_coarse_mode(self._h, self.COARSE_MODES[mode]), "rairs_set_coarse_mode")

    SCAN_MODES = {"auto": 0, "simt": 1, "listmajor": 2}

    def set_scan_mode(self, mode: str = "auto"):
        """auto | simt (query-major LUT-lookup scan) | listmajor (tcgen05 one-hot x LUT)."""
        check(lib().rairs_set_scan_mode(self._h, self.SCAN_MODES[mode]), "rairs_set_scan_mode")

    SEIL_LAYOUTS = {"cell": 0, "paper": 1, "auto": 2, "hybrid": 3}

    def set_seil_layout(self, layout: str = "cell"):
        """cell (cell-major SEIL, every vector stored once) | paper (the paper's
        layout: shared 32-item blocks + duplicated misc areas, Alg. 4/5; query-major
        scan only) | auto (both kept: query-major scans read the paper layout,
        list-major scans the cell-major one) | hybrid (query-major scans read each
        list's cell-major range plus copies of the cross cells below 8 items,
        dropped when their owner was probed; list-major scans the cell-major
        layout)."""
        check(lib().rairs_set_seil_layout(self._h, self.SEIL_LAYOUTS[layout]), "rairs_set_seil_layout")

    def certify_fallbacks(self, reset: bool = True) -> int:
        v = ctypes.c_int64()
        check(lib().rairs_certify_fallbacks(self._h, ctypes.byref(v), int(bool(reset))),
              "rairs_certify_fallbacks")
        return int(v.value)

    # ------------------------------------------------------- profiling
    def profile_enable(self, on: bool = True):
        check(lib().rairs_profile_enable(self._h, int(bool(on))), "rairs_profile_enable")

    def profile_read(self, reset: bool = True) -> Dict[str, object]:
        ms = (ctypes.c_double * 3)()
        nl = (ctypes.c_int64 * 3)()
        check(lib().rairs_profile_read(self._h, ms, nl, int(bool(reset))), "rairs_profile_read")
        return {"ms": {"coarse": ms[0], "scan": ms[1], "refine": ms[2]},
                "launches": {"coarse": nl[0], "scan": nl[1], "refine": nl[2]}}

    def profile_read_kernel(self, reset: bool = True) -> Dict[str, float]:
        """The dominant scan kernel's own time (ms) and launches (profiling on)."""
        ms = ctypes.c_double()
        nl = ctypes.c_int64()
        check(lib().rairs_profile_read_kernel(self._h, ctypes.byref(ms), ctypes.byref(nl),
                                              int(bool(reset))), "rairs_profile_read_kernel")
        return {"ms": ms.value, "launches": nl.value}

    def scan_path(self, nq: int, k: int, nprobe: int, refine_factor: int) -> str:
        """'listmajor' or 'simt': the scan kernels a search of nq queries uses."""
        sp = ctypes.c_int32()
        check(lib().rairs_search_plan(self._h, nq, k, nprobe, refine_factor, None,
                                      ctypes.byref(sp)), "rairs_search_plan")
        return "listmajor" if sp.value == 2 else "simt"

    def kernels_launched(self, reset: bool = True) -> int:
        """Kernels the library launched for searches since the last reset."""
        v = ctypes.c_int64()
        check(lib().rairs_profile_kernels(self._h, ctypes.byref(v), int(bool(reset))),
              "rairs_profile_kernels")
        return int(v.value)


def build_index(base: torch.Tensor, nlist: int, M: int, nbits: int = 4,
                assignment: str = "AIR", **kw) -> Index:
    """BASELINE north_star API: build_index(base, nlist, M, nbits=4, assignment)."""
    return Index.build(base, nlist, M, nbits=nbits, assignment=assignment, **kw)


def merge_topk(ids: torch.Tensor, dists: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
    """[G, nq, k] per-shard results -> [nq, k] global top-k by (dist, id) (K7)."""
    ids = ids.contiguous()
    dists = dists.to(torch.float32).contiguous()
    G, nq, k = ids.shape
    oi = torch.empty((nq, k), dtype=torch.int64, device=ids.device)
    od = torch.empty((nq, k), dtype=torch.float32, device=ids.device)
    check(lib().rairs_merge_topk(_ptr(ids), _ptr(dists), G, nq, k, _ptr(oi), _ptr(od), _stream()),
          "rairs_merge_topk")
    return oi, od


def exact_knn(base: torch.Tensor, queries: torch.Tensor, K: int) -> Tuple[torch.Tensor, torch.Tensor]:
    """Ground truth (B7): first K by (fp64 ordered distance, id)."""
    b = _dev_f32(base, "base")
    q = _dev_f32(queries, "queries")
    ids = torch.empty((q.shape[0], K), dtype=torch.int64, device=q.device)
    dd = torch.empty((q.shape[0], K), dtype=torch.float64, device=q.device)
    check(lib().rairs_exact_knn(_ptr(b), b.shape[0], b.shape[1], _ptr(q), q.shape[0], int(K),
                                _ptr(ids), _ptr(dd), _stream()), "rairs_exact_knn")
    return ids, dd
