"""CPU tests of bench.py's host logic: the recall definition (O13 with the tie
acceptance of S:498), the --k / --refine-factor overrides, and the reference
arm's JSON keys matching the CUDA arm's."""
import argparse

import torch

import bench


def test_recall_at_k_counts_ties_at_the_kth_distance():
    gt_ids = torch.tensor([[0, 1, 2]])
    gt_d = torch.tensor([[1.0, 2.0, 3.0]], dtype=torch.float64)
    # id 7 is not in GT but its distance equals the k-th GT distance -> counts
    ids = torch.tensor([[0, 7, 9]])
    dists = torch.tensor([[1.0, 3.0, 4.0]])
    assert abs(bench.recall_at_k(ids, gt_ids, gt_d, dists, 3) - 2 / 3) < 1e-12
    # padding (-1, +inf) never counts
    ids = torch.tensor([[0, -1, -1]])
    dists = torch.tensor([[1.0, float("inf"), float("inf")]])
    assert abs(bench.recall_at_k(ids, gt_ids, gt_d, dists, 3) - 1 / 3) < 1e-12


def test_spec_overrides_top100():
    ns = argparse.Namespace(k=100, refine_factor=4)
    assert bench.spec_overrides(ns) == {"k": 100, "refine_factor": 4}
    assert bench.spec_overrides(argparse.Namespace(k=None, refine_factor=None)) == {}


def test_strategies_cover_the_paper_comparison():
    # NEXT-2 comparison strategies plus the single-assignment baseline
    assert set(bench.STRATEGIES) == {"single", "naivera", "soarl2", "srair"}
    assert bench.STRATEGIES["naivera"]["lambda_"] == 0.0 and bench.STRATEGIES["naivera"]["strict"]
    assert bench.STRATEGIES["soarl2"]["assignment"] == "SOAR"
