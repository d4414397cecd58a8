"""Time the scan stage of one config/nprobe with CUDA events (library stage profiling).
  python tools/time_fs.py [config] [nprobe] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import GPU_KINDS, get_config, make_dataset  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
spec = get_config(cfg)
npb = int(sys.argv[2]) if len(sys.argv) > 2 else spec.nprobe
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
dev = torch.device("cuda:0")
if spec.kind in GPU_KINDS:
    from synth.gpu_generators import make_dataset_torch
    Xd, Qd = make_dataset_torch(spec, dev)
    kw = dict(train_sample=64 * spec.nlist, kmeans_iters=10)
else:
    X, Q = make_dataset(spec)
    Xd, Qd = torch.from_numpy(X).to(dev), torch.from_numpy(Q).to(dev)
    kw = {}
idx = rb.build_index(Xd, spec.nlist, spec.M, **kw)
del Xd
mode = os.environ.get("SCAN_MODE", "auto")
if os.environ.get("COARSE_DBG"):  # timing experiments of the search's coarse kernel only
    os.environ["RAIRS_COARSE_DBG"] = os.environ["COARSE_DBG"]
idx.set_scan_mode(mode)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for _ in range(3):
    idx.search(Qd, spec.k, npb, spec.refine_factor)
torch.cuda.synchronize()
idx.profile_enable(True)
idx.profile_read(reset=True)
for _ in range(reps):
    flush.zero_()
    idx.search(Qd, spec.k, npb, spec.refine_factor)
torch.cuda.synchronize()
p = idx.profile_read(reset=True)
print(cfg, npb, mode, {k: round(v / reps, 4) for k, v in p["ms"].items()},
      "uncertified/search", round(idx.certify_fallbacks(reset=True) / (reps + 3), 1))
