"""Single-query and small-batch search latency (device events) of one config:
  python tools/lat_1q.py [config] [nprobe] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import GPU_KINDS, get_config, make_dataset  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
spec = get_config(cfg)
npb = int(sys.argv[2]) if len(sys.argv) > 2 else spec.nprobe
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
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
st = torch.cuda.current_stream()
for nq in (1, 8, 64):
    ts = []
    for i in range(reps + 3):
        q = Qd[i * nq:(i + 1) * nq]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        idx.search(q, spec.k, npb, spec.refine_factor)
        b.record(st)
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    idx.profile_enable(True)
    idx.profile_read(reset=True)
    for i in range(10):
        idx.search(Qd[i * nq:(i + 1) * nq], spec.k, npb, spec.refine_factor)
    torch.cuda.synchronize()
    p = idx.profile_read(reset=True)
    idx.profile_enable(False)
    print(cfg, "nprobe", npb, "nq", nq, "p50 %.4f ms  p99 %.4f ms" % (np.percentile(ts, 50), np.percentile(ts, 99)),
          "path", idx.scan_path(nq, spec.k, npb, spec.refine_factor),
          "stages (profiled)", {k: round(v / 10, 4) for k, v in p["ms"].items()})
