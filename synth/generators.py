"""Synthetic stand-ins for the paper's workloads (BASELINE.json `configs`).

The paper's datasets (SIFT1M/1B, MSong, GIST, OpenAI-5M, T2I; PAPER.md
Table 2) are not available; these generators produce inputs of
the same shape and value structure. Recipes follow SURVEY.md §8(d):

* ``c1``  BJ configs[0]: 64 N(0, I_32) means, x = mu_z + 0.3 g, 20k base,
          100 queries, numpy default_rng(0); draw order = means, base labels,
          base noise, query labels, query noise.
* ``c1s`` c1 with sigma = 3.0 (weak structure, ~57 % AIR double assignment:
          exercises reference skipping and ragged SEIL ranges).
* ``c2``  BJ configs[1]: SIFT1M shape. mu_{c,t} = 255 u^2, u ~ U(0,1),
          x = clip(round(mu_z + 16 g), 0, 255) as float32.
* ``c2pl`` paper-like variant of c2 that carries the QPS@recall headline:
          rank-16 clusters x = mu_z + B_z g (g ~ N(0, I_16), B_z entries
          N(0, sigma^2/16), sigma = 48 calibrated), natural clusters =
          nlist/16 = 64, rounded/clipped to [0, 255] like c2.
* ``c3``  BJ configs[2]: 1536-d unit vectors, x = normalize(mu_z + s g),
          mu_c = normalize(N(0, I)), s = 0.6/sqrt(d) (cos(x, mu) ~ 0.85).

Queries are fresh draws from the same mixture (never copies of base rows).
Only numpy's PCG64 is used; the same (config, seed) always yields the same
arrays, on any machine.
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Tuple

import numpy as np


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    name: str
    n: int
    d: int
    nq: int
    nlist: int
    M: int
    k: int
    nprobe: int              # default / bench nprobe
    refine_factor: int
    kind: str                # generator family
    sigma: float
    seed: int
    nclusters: int           # mixture components (natural clusters)
    rank: int = 0            # low-rank subspace dim for "-pl" variants
    note: str = ""


CONFIGS = {
    # tiny unit-test config (not a BJ config): runs through the oracle in ms
    "c0": ConfigSpec("c0", 3000, 16, 40, 16, 8, 5, 4, 4, "gauss", 1.0, 7, 16,
                     note="unit-test size"),
    "c0s": ConfigSpec("c0s", 3000, 16, 40, 16, 8, 5, 4, 4, "gauss", 3.0, 7, 16,
                      note="unit-test size, weak structure"),
    "c1": ConfigSpec("c1", 20000, 32, 100, 64, 16, 10, 8, 4, "gauss", 0.3, 0, 64,
                     note="BJ configs[0]"),
    "c1s": ConfigSpec("c1s", 20000, 32, 100, 64, 16, 10, 8, 4, "gauss", 3.0, 0, 64,
                      note="c1 with sigma=3 (SURVEY §8(d) parity stress)"),
    "c2": ConfigSpec("c2", 1_000_000, 128, 10_000, 1024, 64, 10, 16, 10, "bytes",
                     16.0, 2, 1024, note="BJ configs[1]"),
    # sigma / natural clusters frozen from tools/calibrate_pl.py (profiles/calibration_c2pl.jsonl):
    # AIR double-assigns 45.8 %, single recall10@10 at nprobe 1 = 0.47, AIR reaches 0.95
    # at nprobe 4 (DCO 5.5k) vs single at nprobe 8 (DCO 8.2k).
    "c2pl": ConfigSpec("c2pl", 1_000_000, 128, 10_000, 1024, 64, 10, 4, 10,
                       "bytes_lowrank", 48.0, 2, 64, rank=16,
                       note="paper-like c2 (SURVEY §8(d) '-pl')"),
    "c3": ConfigSpec("c3", 1_000_000, 1536, 10_000, 4096, 384, 10, 32, 10, "sphere",
                     0.6 / np.sqrt(1536.0), 3, 4096, note="BJ configs[2]"),
    # large configs: drawn on the device by synth.gpu_generators (torch Philox)
    "c4": ConfigSpec("c4", 10_000_000, 96, 10_000, 16384, 48, 10, 32, 10, "aniso",
                     1.0, 4, 16384, note="BJ configs[3]"),
    "c5": ConfigSpec("c5", 100_000_000, 128, 10_000, 65536, 64, 10, 64, 10, "gauss_gpu",
                     0.25, 5, 65536, note="BJ configs[4] (one 10k batch of the 100k queries)"),
    # paper-like variants of the device-drawn / high-d configs (SURVEY §8(d) "-pl"):
    # rank-16 clusters, natural clusters = nlist/16; sigma frozen from
    # tools/calibrate_pl.py on 1M-row samples (profiles/calibration_<config>.jsonl):
    #   c4pl sigma 2.0: AIR double-assigns 42.9 %, single recall10@10 at nprobe 1 = 0.56,
    #        AIR reaches 0.95 at nprobe 3 (DCO 2.6k) vs single at nprobe 5 (0.967)
    #   c5pl sigma 1.0: 47.6 %, single 0.47, AIR 0.95 at nprobe 4 (DCO 8.8k) vs single at 6
    #   c3pl sigma 0.016 (~0.6/sqrt(d) per dimension, as c3): 40.4 %, single 0.37,
    #        AIR 0.95 at nprobe 6 (DCO 1.95k) vs single at 8
    "c4pl": ConfigSpec("c4pl", 10_000_000, 96, 10_000, 16384, 48, 10, 3, 10, "aniso_lowrank_gpu",
                       2.0, 4, 1024, rank=16, note="paper-like c4"),
    "c5pl": ConfigSpec("c5pl", 100_000_000, 128, 10_000, 65536, 64, 10, 4, 10, "lowrank_gpu",
                       1.0, 5, 4096, rank=16, note="paper-like c5"),
    "c3pl": ConfigSpec("c3pl", 1_000_000, 1536, 10_000, 4096, 384, 10, 6, 10, "sphere_lowrank_gpu",
                       0.016, 3, 256, rank=16, note="paper-like c3"),
}

GPU_KINDS = ("aniso", "gauss_gpu", "lowrank_gpu", "aniso_lowrank_gpu", "sphere_lowrank_gpu")


def get_config(name: str, **overrides) -> ConfigSpec:
    spec = CONFIGS[name]
    if overrides:
        spec = dataclasses.replace(spec, **overrides)
    return spec


def _normal(rng: np.random.Generator, shape) -> np.ndarray:
    return rng.standard_normal(shape, dtype=np.float32)


def _draw_gauss(rng, spec: ConfigSpec, means: np.ndarray, count: int) -> np.ndarray:
    z = rng.integers(0, spec.nclusters, size=count)
    g = _normal(rng, (count, spec.d))
    return (means[z] + np.float32(spec.sigma) * g).astype(np.float32)


def _draw_bytes(rng, spec: ConfigSpec, means: np.ndarray, count: int) -> np.ndarray:
    z = rng.integers(0, spec.nclusters, size=count)
    g = _normal(rng, (count, spec.d))
    x = means[z] + np.float32(spec.sigma) * g
    return np.clip(np.rint(x), 0, 255).astype(np.float32)


def _draw_bytes_lowrank(rng, spec: ConfigSpec, means, bases, count: int) -> np.ndarray:
    z = rng.integers(0, spec.nclusters, size=count)
    g = _normal(rng, (count, spec.rank))
    x = np.empty((count, spec.d), dtype=np.float32)
    order = np.argsort(z, kind="stable")
    zs = z[order]
    bounds = np.searchsorted(zs, np.arange(spec.nclusters + 1))
    for c in range(spec.nclusters):
        rows = order[bounds[c]:bounds[c + 1]]
        if rows.size:
            x[rows] = means[c] + g[rows] @ bases[c].T
    return np.clip(np.rint(x), 0, 255).astype(np.float32)


def _draw_sphere(rng, spec: ConfigSpec, means: np.ndarray, count: int,
                 chunk: int = 65536) -> np.ndarray:
    z = rng.integers(0, spec.nclusters, size=count)
    x = np.empty((count, spec.d), dtype=np.float32)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        v = means[z[s:e]] + np.float32(spec.sigma) * _normal(rng, (e - s, spec.d))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        x[s:e] = v
    return x


def make_dataset(spec: ConfigSpec, n: Optional[int] = None,
                 nq: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    """Return (base [n x d] float32, queries [nq x d] float32), C-contiguous.

    ``n``/``nq`` override the sizes (draw order is unchanged, so a smaller n
    yields different rows than a prefix of the full draw).
    """
    n = spec.n if n is None else n
    nq = spec.nq if nq is None else nq
    rng = np.random.default_rng(spec.seed)
    if spec.kind == "gauss":
        means = _normal(rng, (spec.nclusters, spec.d))
        base = _draw_gauss(rng, spec, means, n)
        qry = _draw_gauss(rng, spec, means, nq)
    elif spec.kind == "bytes":
        u = rng.random((spec.nclusters, spec.d), dtype=np.float32)
        means = (255.0 * u * u).astype(np.float32)
        base = _draw_bytes(rng, spec, means, n)
        qry = _draw_bytes(rng, spec, means, nq)
    elif spec.kind == "bytes_lowrank":
        u = rng.random((spec.nclusters, spec.d), dtype=np.float32)
        means = (255.0 * u * u).astype(np.float32)
        bases = (_normal(rng, (spec.nclusters, spec.d, spec.rank))
                 * np.float32(spec.sigma / np.sqrt(spec.rank))).astype(np.float32)
        base = _draw_bytes_lowrank(rng, spec, means, bases, n)
        qry = _draw_bytes_lowrank(rng, spec, means, bases, nq)
    elif spec.kind == "sphere":
        means = _normal(rng, (spec.nclusters, spec.d))
        means /= np.linalg.norm(means, axis=1, keepdims=True)
        base = _draw_sphere(rng, spec, means, n)
        qry = _draw_sphere(rng, spec, means, nq)
    elif spec.kind in GPU_KINDS:
        import torch
        from .gpu_generators import make_dataset_torch
        b, q = make_dataset_torch(spec, torch.device("cpu"), n=n, nq=nq)
        return b.numpy(), q.numpy()
    else:
        raise ValueError(f"unknown generator kind {spec.kind!r}")
    return np.ascontiguousarray(base), np.ascontiguousarray(qry)


def shard_rows(n: int, shard_id: int, nshards: int) -> np.ndarray:
    """Global ids owned by a shard under the partition shard(x) = id mod G
    (SURVEY §8(c) O11, §8(e)); local row r <-> global id r*G + shard_id."""
    return np.arange(shard_id, n, nshards, dtype=np.int64)
