"""Repro: GPU training on c5-distributed data (rows drawn like BJ configs[4])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import get_config  # noqa: E402
from synth.gpu_generators import make_dataset_torch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
spec = get_config("c5")
X, Q = make_dataset_torch(spec, torch.device("cuda"), n=n, nq=10)
c, cb = rb.train(X, spec.nlist, spec.M, kmeans_iters=2, train_sample=64 * spec.nlist)
torch.cuda.synchronize()
print("train OK", n, float(c.abs().sum()))
