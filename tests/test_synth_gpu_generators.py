"""CPU checks of the device-side generators for BASELINE.json configs[3]/[4]
(synth/gpu_generators.py), run on the CPU device at small sizes: determinism,
shapes, and the mixture structure the recipe states (DESIGN.md input recipe)."""
import math

import torch

from synth import get_config
from synth.gpu_generators import _aniso_bases, _gen, make_dataset_torch


def test_deterministic_and_shapes():
    for name in ("c4", "c5"):
        spec = get_config(name)
        a = make_dataset_torch(spec, torch.device("cpu"), n=3000, nq=17)
        b = make_dataset_torch(spec, torch.device("cpu"), n=3000, nq=17)
        assert a[0].shape == (3000, spec.d) and a[1].shape == (17, spec.d)
        assert a[0].dtype == torch.float32
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
        assert torch.isfinite(a[0]).all()


def test_c4_covariance_is_rotated_loguniform_spectrum():
    # B_c = R_c diag(sqrt(lam_c)) with R_c orthogonal: B_c B_c^T has eigenvalues lam_c,
    # all inside [0.05, 1] (BJ configs[3]: "eigenvalues log-uniform 0.05-1")
    g = _gen(4, torch.device("cpu"))
    means, B = _aniso_bases(8, 96, g, torch.device("cpu"))
    for c in range(8):
        R = B[c] / B[c].norm(dim=0, keepdim=True)          # columns of R_c
        assert torch.allclose(R.T @ R, torch.eye(96), atol=1e-4)
        ev = torch.linalg.eigvalsh((B[c] @ B[c].T).double())
        assert ev.min() > 0.05 - 1e-4 and ev.max() < 1.0 + 1e-4
        # log-uniform: log-eigenvalues spread over most of [log .05, 0]
        assert ev.min() < 0.1 and ev.max() > 0.8


def test_c5_within_cluster_spread():
    # x = mu_z + 0.25 g: the distance of a point to its nearest mean is ~ 0.25 sqrt(d)
    spec = get_config("c5")
    X, _ = make_dataset_torch(spec, torch.device("cpu"), n=2000, nq=1)
    g = _gen(spec.seed, torch.device("cpu"))
    means = torch.randn(spec.nclusters, spec.d, generator=g)
    d2 = torch.cdist(X[:200], means).min(dim=1).values
    expect = 0.25 * math.sqrt(spec.d)
    assert abs(float(d2.mean()) - expect) < 0.1 * expect
