"""c5 (100M x 128, BJ nprobe 64): one 10k batch on the list-major (default),
list-major fused and query-major scan paths; device time per search.
  python tools/c5_paths.py [nprobe]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_07183_b200 as rb
from synth import get_config
from synth.gpu_generators import make_dataset_torch
spec = get_config("c5")
npb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda:0")
Xd, Qd = make_dataset_torch(spec, dev)
Qd = Qd[:10000].contiguous()
idx = rb.build_index(Xd, spec.nlist, spec.M)
for mode in ("auto", "simt", "listmajor"):
    idx.set_scan_mode(mode)
    for _ in range(2): idx.search(Qd, spec.k, npb, spec.refine_factor)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): idx.search(Qd, spec.k, npb, spec.refine_factor)
    e1.record(); e1.synchronize()
    print(mode, idx.scan_path(Qd.shape[0], spec.k, npb, spec.refine_factor), "ms/search", round(e0.elapsed_time(e1) / 3, 3), flush=True)
