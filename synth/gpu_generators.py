"""Seeded synthetic stand-ins for BASELINE.json's large configs, drawn on a torch
device ("c4 ... GPU-generated", "c5 ... generated on GPU").

Holds NO arithmetic of the RAIRS method: only mixture sampling. numpy would
take minutes (and 51 GB of host RAM) for c5, so these draw with torch's
counter-based Philox generator on the device; the same (config, seed, device
type, torch version) always yields the same tensors. Both the CUDA path and
the oracle consume the SAME drawn tensors (copied to host for the oracle).

* ``c4``  BJ configs[3]: 10M x 96, 16,384 clusters, means N(0, I_96),
          anisotropic per-cluster covariance R_c diag(lam_c) R_c^T with lam
          log-uniform on [0.05, 1] and R_c Haar-orthogonal (sign-fixed QR of a
          Gaussian); x = mu_z + R_z (sqrt(lam_z) * g).
* ``c5``  BJ configs[4]: 100M x 128, 65,536 clusters, means N(0, I_128)
          (mean spread s = 1, a reading: BJ gives only sigma), x = mu_z + 0.25 g.
* paper-like variants (SURVEY §8(d) "-pl"): rank-16 clusters x = mu_z + B_z g,
  g ~ N(0, I_16), B_z entries N(0, sigma^2/16) (per-point energy sigma^2 d as
  in BJ), natural clusters = nlist/16 so list boundaries cut through them:
  ``c4pl`` keeps c4's anisotropy inside the subspace (B_z columns scaled by
  sqrt(lambda), lambda log-uniform on [0.05, 1]); ``c5pl`` means N(0, I);
  ``c3pl`` unit-normalised, means normalize(N(0, I)).  sigma calibrated by
  tools/calibrate_pl.py (profiles/calibration_<config>.jsonl).
Queries are fresh draws from the same mixture.
"""
from __future__ import annotations

import math
from typing import Optional, Tuple

import torch

from .generators import ConfigSpec


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _aniso_bases(C: int, d: int, g: torch.Generator, device) -> Tuple[torch.Tensor, torch.Tensor]:
    means = torch.randn(C, d, generator=g, device=device)
    lo, hi = math.log(0.05), math.log(1.0)
    lam = torch.exp(lo + (hi - lo) * torch.rand(C, d, generator=g, device=device))
    B = torch.empty(C, d, d, device=device)
    for c0 in range(0, C, 2048):                      # Haar: QR of a Gaussian, sign-fixed
        G = torch.randn(min(2048, C - c0), d, d, generator=g, device=device)
        Qm, Rm = torch.linalg.qr(G)
        sgn = torch.sign(torch.diagonal(Rm, dim1=-2, dim2=-1))
        sgn[sgn == 0] = 1.0
        Qm = Qm * sgn[:, None, :]
        B[c0:c0 + Qm.shape[0]] = Qm * lam[c0:c0 + Qm.shape[0]].sqrt()[:, None, :]
    return means, B


def _draw_aniso(count: int, means, B, g, device, chunk: int = 1 << 21) -> torch.Tensor:
    C, d = means.shape
    out = torch.empty(count, d, device=device)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        z = torch.randint(0, C, (e - s,), generator=g, device=device)
        gg = torch.randn(e - s, d, generator=g, device=device)
        order = torch.argsort(z)
        zs = z[order]
        x = torch.empty(e - s, d, device=device)
        # group rows by cluster and apply each cluster's B_z (padded batched matmul)
        cnt = torch.bincount(zs, minlength=C)
        start = torch.cumsum(cnt, 0) - cnt
        pos = torch.arange(e - s, device=device) - start[zs]
        width = int(cnt.max().item())
        P = torch.zeros(C, width, d, device=device)
        P[zs, pos] = gg[order]
        Y = torch.bmm(P, B.transpose(1, 2))           # row vector g -> (B g)^T = g^T B^T
        x[order] = Y[zs, pos] + means[zs]
        out[s:e] = x
        del P, Y
    return out


def _draw_gauss(count: int, means, sigma: float, g, device, chunk: int = 1 << 23) -> torch.Tensor:
    C, d = means.shape
    out = torch.empty(count, d, device=device)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        z = torch.randint(0, C, (e - s,), generator=g, device=device)
        out[s:e] = means[z] + sigma * torch.randn(e - s, d, generator=g, device=device)
    return out


def _lowrank_bases(C: int, d: int, r: int, sigma: float, aniso: bool, g, device) -> torch.Tensor:
    B = torch.randn(C, d, r, generator=g, device=device) * (sigma / math.sqrt(r))
    if aniso:  # c4's anisotropy inside the subspace: columns scaled by sqrt(lambda)
        lo, hi = math.log(0.05), math.log(1.0)
        lam = torch.exp(lo + (hi - lo) * torch.rand(C, r, generator=g, device=device))
        B = B * lam.sqrt()[:, None, :]
    return B


def _draw_lowrank(count: int, means, B, g, device, normalize: bool) -> torch.Tensor:
    C, d = means.shape
    r = B.shape[2]
    chunk = max(4096, min(1 << 21, (1 << 30) // (d * r * 4)))
    out = torch.empty(count, d, device=device)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        z = torch.randint(0, C, (e - s,), generator=g, device=device)
        gg = torch.randn(e - s, r, 1, generator=g, device=device)
        x = means[z] + torch.bmm(B[z], gg).squeeze(-1)
        if normalize:
            x = x / x.norm(dim=1, keepdim=True)
        out[s:e] = x
    return out


def make_dataset_torch(spec: ConfigSpec, device, n: Optional[int] = None,
                       nq: Optional[int] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """(base [n x d] float32, queries [nq x d] float32) on `device`."""
    n = spec.n if n is None else n
    nq = spec.nq if nq is None else nq
    g = _gen(spec.seed, device)
    if spec.kind == "aniso":
        means, B = _aniso_bases(spec.nclusters, spec.d, g, device)
        base = _draw_aniso(n, means, B, g, device)
        qry = _draw_aniso(nq, means, B, g, device)
    elif spec.kind == "gauss_gpu":
        means = torch.randn(spec.nclusters, spec.d, generator=g, device=device)
        base = _draw_gauss(n, means, spec.sigma, g, device)
        qry = _draw_gauss(nq, means, spec.sigma, g, device)
    elif spec.kind in ("lowrank_gpu", "aniso_lowrank_gpu", "sphere_lowrank_gpu"):
        means = torch.randn(spec.nclusters, spec.d, generator=g, device=device)
        sphere = spec.kind == "sphere_lowrank_gpu"
        if sphere:
            means = means / means.norm(dim=1, keepdim=True)
        B = _lowrank_bases(spec.nclusters, spec.d, spec.rank, spec.sigma,
                           spec.kind == "aniso_lowrank_gpu", g, device)
        base = _draw_lowrank(n, means, B, g, device, sphere)
        qry = _draw_lowrank(nq, means, B, g, device, sphere)
    else:
        raise ValueError(f"{spec.name}: kind {spec.kind!r} is drawn by synth.make_dataset (numpy)")
    return base.contiguous(), qry.contiguous()
