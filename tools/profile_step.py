"""Build one index and run a few search batches (for ncu launch lists / captures).

  python tools/profile_step.py [config] [nprobe] [scan_mode] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import get_config, make_dataset  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2pl"
spec = get_config(cfg)
npb = int(sys.argv[2]) if len(sys.argv) > 2 else spec.nprobe
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
dev = torch.device("cuda:0")
from synth import GPU_KINDS  # noqa: E402
if spec.kind in GPU_KINDS:  # c4 / c5: drawn on the device
    from synth.gpu_generators import make_dataset_torch
    Xd, Qd = make_dataset_torch(spec, dev)
    kw = dict(train_sample=64 * spec.nlist, kmeans_iters=10)
else:
    X, Q = make_dataset(spec)
    Xd, Qd = torch.from_numpy(X).to(dev), torch.from_numpy(Q).to(dev)
    kw = {}
idx = rb.build_index(Xd, spec.nlist, spec.M, **kw)
del Xd
idx.set_scan_mode(mode)
if os.environ.get("COARSE_DBG"):  # timing experiments of the search's coarse kernel only
    os.environ["RAIRS_COARSE_DBG"] = os.environ["COARSE_DBG"]
torch.cuda.synchronize()
for i in range(reps):
    if i == reps - 1:
        torch.cuda.nvtx.range_push("search")   # ncu --nvtx --nvtx-include "search/"
    ids, dists = idx.search(Qd, spec.k, npb, spec.refine_factor)
    if i == reps - 1:
        torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("profile_step OK", cfg, npb, mode, reps, ids.shape)
