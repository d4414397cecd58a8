"""Wall-clock breakdown of one search batch through the device and host C-ABI entry points."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_07183_b200 as rb
from synth import get_config, make_dataset
spec = get_config(sys.argv[1] if len(sys.argv) > 1 else "c2pl")
X, Q = make_dataset(spec)
dev = torch.device("cuda:0")
idx = rb.build_index(torch.from_numpy(X).to(dev), spec.nlist, spec.M)
Qd = torch.from_numpy(Q).to(dev)
npb = int(sys.argv[2]) if len(sys.argv) > 2 else spec.nprobe
for _ in range(3): idx.search(Qd, spec.k, npb, spec.refine_factor)
torch.cuda.synchronize()
for name, fn in [("device", lambda: idx.search(Qd, spec.k, npb, spec.refine_factor)),
                 ("host", lambda: idx.search_host(qh, spec.k, npb, spec.refine_factor, oi, od))]:
    qh = torch.from_numpy(Q).pin_memory().numpy()
    oi = torch.empty((Q.shape[0], spec.k), dtype=torch.int64).pin_memory().numpy()
    od = torch.empty((Q.shape[0], spec.k), dtype=torch.float32).pin_memory().numpy()
    ts = []
    for _ in range(10):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(name, "median ms", round(1e3 * float(np.median(ts)), 3), "min", round(1e3 * min(ts), 3))
# enqueue-only cost (no sync)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): idx.search(Qd, spec.k, npb, spec.refine_factor)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("enqueue ms/call", round(1e3 * (t1 - t0) / 10, 3), "total ms/call", round(1e3 * (t2 - t0) / 10, 3))
