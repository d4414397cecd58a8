"""Repro: GPU k-means (tensor-core assignment path) at large nlist."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402

nlist = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 300000
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(rows, 128, generator=g, device="cuda")
c, cb = rb.train(X, nlist, 64, kmeans_iters=2, train_sample=rows)
torch.cuda.synchronize()
print("train OK", nlist, rows, float(c.abs().sum()))
