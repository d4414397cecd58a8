"""Where the e2e (host buffers) time goes: device search time, host enqueue
time of one search, raw pinned H2D / D2H copies, and rairs_search_host wall.

  python tools/e2e_breakdown.py [config] [nprobe]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from synth import get_config, make_dataset  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2pl"
spec = get_config(cfg)
npb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
X, Q = make_dataset(spec)
dev = torch.device("cuda:0")
idx = rb.build_index(torch.from_numpy(X).to(dev), spec.nlist, spec.M)
Qd = torch.from_numpy(Q).to(dev)
k, rf = spec.k, spec.refine_factor
for _ in range(5):
    idx.search(Qd, k, npb, rf)
torch.cuda.synchronize()
R = 20


def med(xs):
    return float(np.median(xs)) * 1e3


dev_t, enq_t, host_t, h2d_t, d2h_t, plain_wall = [], [], [], [], [], []
qh = torch.from_numpy(Q).pin_memory()
oi = torch.empty((Q.shape[0], k), dtype=torch.int64).pin_memory()
od = torch.empty((Q.shape[0], k), dtype=torch.float32).pin_memory()
for _ in range(R):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    idx.search(Qd, k, npb, rf)
    t1 = time.perf_counter()
    e1.record()
    e1.synchronize()
    t2 = time.perf_counter()
    dev_t.append(e0.elapsed_time(e1) / 1e3)
    enq_t.append(t1 - t0)
    plain_wall.append(t2 - t0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    idx.search_host(qh.numpy(), k, npb, rf, oi.numpy(), od.numpy())
    host_t.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Qd.copy_(qh, non_blocking=True)
    torch.cuda.synchronize()
    h2d_t.append(time.perf_counter() - t0)
    ids = torch.empty((Q.shape[0], k), dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    oi.copy_(ids, non_blocking=True)
    od.copy_(ids.float(), non_blocking=True)
    torch.cuda.synchronize()
    d2h_t.append(time.perf_counter() - t0)
# serving mode: back-to-back rairs_search_host_async calls, one sync at the end
outs = [(torch.empty((Q.shape[0], k), dtype=torch.int64).pin_memory(),
         torch.empty((Q.shape[0], k), dtype=torch.float32).pin_memory()) for _ in range(2)]
for i in range(4):
    idx.search_host_async(qh.numpy(), k, npb, rf, outs[i % 2][0].numpy(), outs[i % 2][1].numpy())
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(R):
    idx.search_host_async(qh.numpy(), k, npb, rf, outs[i % 2][0].numpy(), outs[i % 2][1].numpy())
t_enq = time.perf_counter() - t0
torch.cuda.synchronize()
t_pipe = time.perf_counter() - t0
# copies alone, back to back (H2D of every batch + D2H of every result)
t0 = time.perf_counter()
for i in range(R):
    Qd.copy_(qh, non_blocking=True)
    outs[i % 2][0].copy_(ids, non_blocking=True)
torch.cuda.synchronize()
t_copy = time.perf_counter() - t0
side = torch.cuda.Stream()
with torch.cuda.stream(side):   # the same on a non-default (non-legacy) stream
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(R):
        idx.search_host_async(qh.numpy(), k, npb, rf, outs[i % 2][0].numpy(), outs[i % 2][1].numpy())
    torch.cuda.synchronize()
    t_side = time.perf_counter() - t0
print(f"pipelined async on a side stream: {1e3 * t_side / R:.3f} ms/step")
# manual overlap: device-buffer searches on the default stream, H2D copies of
# the next batch into a second device buffer on a copy stream
cs = torch.cuda.Stream()
Qd2 = torch.empty_like(Qd)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(R):
    with torch.cuda.stream(cs):
        (Qd2 if i % 2 else Qd).copy_(qh, non_blocking=True)
    idx.search(Qd if i % 2 else Qd2, k, npb, rf)
torch.cuda.synchronize()
print(f"manual overlap (search + concurrent H2D): {1e3 * (time.perf_counter() - t0) / R:.3f} ms/step")
print(f"pipelined async: {1e3 * t_pipe / R:.3f} ms/step (host enqueue {1e3 * t_enq / R:.3f} ms/step); "
      f"copies alone {1e3 * t_copy / R:.3f} ms/step")
print(f"device search {med(dev_t):.3f} ms | host enqueue {med(enq_t):.3f} ms | plain search wall "
      f"{med(plain_wall):.3f} ms | search_host wall {med(host_t):.3f} ms | pinned H2D "
      f"{Q.nbytes/1e6:.1f} MB {med(h2d_t):.3f} ms | D2H {med(d2h_t):.3f} ms")
