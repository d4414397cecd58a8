"""BJ configs[4] at full size (100M x 128, nlist 65,536): build, then searches
of one 10k-query batch at nprobe 64 -- for ncu DRAM-traffic captures of the
fast-scan stage (codes stream from HBM at this size)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import get_config  # noqa: E402
from synth.gpu_generators import make_dataset_torch  # noqa: E402

spec = get_config("c5")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
X, Q = make_dataset_torch(spec, torch.device("cuda"))
idx = rb.build_index(X, spec.nlist, spec.M, train_sample=64 * spec.nlist, kmeans_iters=10)
del X
torch.cuda.empty_cache()
for i in range(reps):
    if i == reps - 1:
        torch.cuda.nvtx.range_push("search")   # ncu --nvtx --nvtx-include "search/"
    idx.search(Q, spec.k, 64, spec.refine_factor)
    if i == reps - 1:
        torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok", idx.info()["n_slots"])
