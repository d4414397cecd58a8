"""c5 geometry (nlist 65,536, d 128, 10k queries) on a 4M-row base: the coarse
stage costs the same as at 100M (it depends on nq x nlist only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import get_config  # noqa: E402
from synth.gpu_generators import make_dataset_torch  # noqa: E402

spec = get_config("c5")
X, Q = make_dataset_torch(spec, torch.device("cuda"), n=8_000_000, nq=10_000)
idx = rb.build_index(X, spec.nlist, spec.M, train_sample=64 * spec.nlist, kmeans_iters=10)
idx.certify_fallbacks(reset=True)
for npb in (64, 64):
    idx.search(Q, 10, npb, 10)
torch.cuda.synchronize()
print("uncertified per search", idx.certify_fallbacks(reset=True) / 2)
torch.cuda.synchronize()
print("ok")
