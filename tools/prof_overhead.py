"""Step time of one config with and without the library's stage profiling
(CUDA events between the search's kernels):  python tools/prof_overhead.py [cfg] [nprobe]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import get_config  # noqa: E402
from synth.gpu_generators import make_dataset_torch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
spec = get_config(cfg)
npb = int(sys.argv[2]) if len(sys.argv) > 2 else spec.nprobe
dev = torch.device("cuda:0")
Xd, Qd = make_dataset_torch(spec, dev)
idx = rb.build_index(Xd, spec.nlist, spec.M, train_sample=64 * spec.nlist, kmeans_iters=10)
del Xd
idx.set_seil_layout(os.environ.get("LAYOUT", "auto"))
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream()


def run(prof, steps=10):
    for _ in range(3):
        idx.search(Qd, spec.k, npb, spec.refine_factor)
    idx.profile_enable(prof)
    t = 0.0
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        idx.search(Qd, spec.k, npb, spec.refine_factor)
        b.record(st)
        b.synchronize()
        t += a.elapsed_time(b)
    idx.profile_enable(False)
    idx.profile_read(reset=True)
    return t / steps


for rep in range(2):
    print(cfg, "prof off %.4f ms  prof on %.4f ms" % (run(False), run(True)))
