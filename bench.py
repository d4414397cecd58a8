#!/usr/bin/env python
"""Benchmark: batched RAIRS search (IVFPQ fast-scan + AIR + SEIL + refine) on B200.

Step = one pass of the whole hot path (coarse probe selection,
LUT + uint8 quantisation, SEIL work list, 4-bit fast scan, top-bigK, exact
refine; plus the NCCL all_gather + top-k merge when N > 1) over one batch of
10,000 synthetic queries with the index resident in HBM.

Default workload: BASELINE.json configs[3] "c4" -- the largest BJ config
that fits one B200 with its codes streaming from HBM (10M x 96, 16,384-cluster
anisotropic Gaussian mixture drawn on the device, nlist 16,384, PQ M=48 x
4-bit, AIR+SEIL, k=10, refine x10) -- at the smallest swept nprobe whose
recall10@10 >= 0.95 (BJ metric "QPS at recall10@10=0.95").  Side lines: the
same index at k=1 (BJ configs[3] asks for k=1 and k=10), single-query
latency, and the AIR+SEIL vs single / NaiveRA / SOARL2 / SRAIR comparison.
Other configs: --config c2pl | c2 | c3 | c5 | ...

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
--gpus N > 1 without a torch.distributed environment re-launches this script
under `python -m torch.distributed.run --nproc-per-node N` (one rank per GPU,
NCCL); the index is sharded by id mod N, every rank searches its shard, the
per-shard top-k are exchanged by one NCCL all_gather and merged by the K7
kernel (strong scaling: total work fixed).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NPROBE_SWEEP = [1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 24, 32, 48, 64, 96, 128]
L2_FLUSH_BYTES = 256 << 20   # > 126 MB L2


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def recall_at_k(ids, gt_ids, gt_d64, dists, k):
    """recall k@k; a returned id counts if it is in GT or its fp32 distance
    equals fp32(k-th GT distance) (tie acceptance)."""
    import torch
    hit = (ids[:, :, None] == gt_ids[:, None, :k]).any(-1)
    kth = gt_d64[:, k - 1].to(torch.float32)[:, None]
    tie = (dists == kth) & (ids >= 0)
    return float((hit | tie).float().sum().item()) / (ids.shape[0] * k)


def plateaued(sweep, n=3, eps=5e-4):
    """True when the last n swept points gained less than eps recall: the
    raw-PQ + refine_factor cap of separated mixtures, which more
    nprobe cannot lift."""
    if len(sweep) <= n:
        return False
    return sweep[-1]["recall"] - sweep[-1 - n]["recall"] < eps


def spec_overrides(args):
    """--k / --refine-factor (the paper's top-100 workload uses k 100 with
    K_FACTOR 4)."""
    ov = {}
    if args.k:
        ov["k"] = args.k
    if args.refine_factor:
        ov["refine_factor"] = args.refine_factor
    return ov


def build_workload(args, rank, world, dev):
    """Synthetic inputs + index. Host-drawn configs (c1-c3, c2pl) come from
    synth.make_dataset; the large BJ configs (c4: 10M x 96, c5: 100M x 128) are
    drawn on the device (synth.gpu_generators) -- every rank draws the same
    tensors and keeps its id-mod-N shard."""
    import torch
    import paper_2601_07183_b200 as rb
    from synth import GPU_KINDS, get_config, make_dataset
    spec = get_config(args.config, **spec_overrides(args))
    t0 = time.time()
    if spec.kind in GPU_KINDS:
        from synth.gpu_generators import make_dataset_torch
        Xd, Qd = make_dataset_torch(spec, dev)
        Q = Qd.cpu().numpy()
        # host copy only for the CPU-oracle baseline (rank 0, N = 1)
        X = Xd.cpu().numpy() if (world == 1 and not args.no_cpu_baseline) else None
        Xl = Xd if world == 1 else Xd[rank::world].contiguous()
    else:
        X, Q = make_dataset(spec)
        Xd = None
        rows = np.arange(rank, X.shape[0], world)
        Xl = torch.from_numpy(X[rows]).to(dev)
        Qd = torch.from_numpy(Q).to(dev)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    # exact ground truth (fp64, GPU) on a query sample, before the build frees memory
    nq_gt = Q.shape[0] if args.gt_queries <= 0 else min(Q.shape[0], args.gt_queries)
    Xfull = Xd if Xd is not None else torch.from_numpy(X).to(dev)
    gt_ids, gt_d64 = rb.exact_knn(Xfull, Qd[:nq_gt].contiguous(), spec.k)
    torch.cuda.synchronize()
    del Xfull
    # training for large nlist: a 64*nlist sample and 10 Lloyd iterations (R16;
    # training is outside the bit-exact contract)
    kw = {}
    if spec.nlist >= 4096:
        kw = dict(train_sample=64 * spec.nlist, kmeans_iters=10)
    t0 = time.time()
    if world == 1:
        idx = rb.build_index(Xl, spec.nlist, spec.M, assignment=args.assignment, **kw)
        torch.cuda.synchronize()
    else:
        from paper_2601_07183_b200.distributed import ShardedIndex
        if Xd is not None:
            Xtrain = Xd if rank == 0 else None
        else:
            Xtrain = torch.from_numpy(X).to(dev) if rank == 0 else None
        sh = ShardedIndex.build(Xl, spec.n, spec.nlist, spec.M, train_base=Xtrain,
                                assignment=args.assignment, **kw)
        idx = sh.local
        del Xtrain
    # SEIL list layout searched (default hybrid: cell-major + copies of the tiny cross cells)
    idx.set_seil_layout(args.seil_layout)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    del Xd, Xl
    torch.cuda.empty_cache()
    return spec, X, Q, Qd, idx, gen_s, build_s, gt_ids, gt_d64, nq_gt


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2601_07183_b200 as rb
    from paper_2601_07183_b200.distributed import sharded_merge

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # RAIRS_BENCH_BACKEND=gloo + RAIRS_BENCH_ONE_GPU=1: a functional run of the
    # N-rank path with every rank on cuda:0 (NCCL refuses two ranks per device);
    # timings of such a run are not scaling numbers
    backend = os.environ.get("RAIRS_BENCH_BACKEND", "nccl")
    gpu = 0 if os.environ.get("RAIRS_BENCH_ONE_GPU") == "1" else local_rank
    if world > 1:
        torch.cuda.set_device(gpu)
        dist.init_process_group(backend)
    dev = torch.device("cuda", gpu)
    spec, X, Q, Qd, idx, gen_s, build_s, gt_ids, gt_d64, nq_gt = build_workload(args, rank, world, dev)
    k, rf = spec.k, spec.refine_factor

    def step(nprobe, with_dco=False):
        if with_dco:
            ids, dists, dco = idx.search(Qd, k, nprobe, rf, return_dco=True)
        else:
            ids, dists = idx.search(Qd, k, nprobe, rf)
            dco = None
        if world > 1:
            ids, dists = sharded_merge(ids, dists)
        return ids, dists, dco

    # recall sweep -> headline nprobe (smallest with recall >= 0.95)
    sweep = []
    chosen = None
    for npb in [p for p in NPROBE_SWEEP if p <= spec.nlist]:
        ids, dists, _ = step(npb)
        r = recall_at_k(ids[:nq_gt], gt_ids, gt_d64, dists[:nq_gt], k)
        sweep.append({"nprobe": npb, "recall": round(r, 4)})
        if args.nprobe is None and r >= 0.95:
            chosen = npb
            break
        if plateaued(sweep) and (args.nprobe is None or npb >= args.nprobe):
            break
    if args.nprobe is not None:
        chosen = args.nprobe
    if chosen is None:  # 0.95 not reached: the smallest nprobe of the recall plateau
        best = max(p["recall"] for p in sweep)
        chosen = min(p["nprobe"] for p in sweep if p["recall"] >= best - 5e-4)
    ids, dists, dco = step(chosen, with_dco=True)
    recall = recall_at_k(ids[:nq_gt], gt_ids, gt_d64, dists[:nq_gt], k)
    dco_local = int(dco.sum().item())
    dco_total = dco_local
    if world > 1:
        t = torch.tensor([dco_local], dtype=torch.int64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t)
        dco_total = int(t.item())

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        flush.zero_()
        step(chosen)
    torch.cuda.synchronize()

    # ---------------- timed region (device events per step, L2 flushed between) ----------
    # The library's stage profiling records CUDA events between the search's
    # kernels, which breaks their programmatic-dependent-launch overlap (+26 us
    # per c4 step, tools/prof_overhead.py): the timed region runs without it,
    # and a second pass of the same K steps (same protocol) records the stage
    # times and the dominant kernel's own events for the roofline.
    idx.profile_enable(False)
    idx.kernels_launched(reset=True)
    idx.certify_fallbacks(reset=True)
    clk = ClockSampler(gpu)
    clk.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    torch.cuda.nvtx.range_push("timed")    # (for ncu --nvtx-include timed/; no-op otherwise)
    for i in range(args.steps):
        flush.zero_()                      # untimed: outside the step's events
        ev[i][0].record(stream)
        step(chosen)
        ev[i][1].record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clocks = clk.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kernels = idx.kernels_launched(reset=True) + (args.steps if world > 1 else 0)  # + K7 merge
    fallbacks = idx.certify_fallbacks(reset=True)
    # profile pass: the same K steps with stage events and the scan kernel's events
    idx.profile_enable(True)
    idx.profile_read(reset=True)
    idx.profile_read_kernel(reset=True)
    pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        pev[i][0].record(stream)
        step(chosen)
        pev[i][1].record(stream)
    torch.cuda.synchronize()
    prof_step_ms = sum(a.elapsed_time(b) for a, b in pev) / args.steps
    prof = idx.profile_read(reset=True)
    kprof = idx.profile_read_kernel(reset=True)   # the dominant scan kernel alone
    idx.profile_enable(False)
    t_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([t_ms], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    nq = Q.shape[0]
    qps = nq * args.steps / (t_ms / 1e3)

    # ---------------- e2e: host buffers through the C ABI (H2D + search + D2H) ----------
    e2e = None
    if world == 1:
        import torch as _t
        qh_t = _t.from_numpy(Q).pin_memory()
        oi_t = _t.empty((nq, k), dtype=_t.int64).pin_memory()
        od_t = _t.empty((nq, k), dtype=_t.float32).pin_memory()
        qh, oi, od = qh_t.numpy(), oi_t.numpy(), od_t.numpy()   # the tensors keep them pinned
        for _ in range(2):
            idx.search_host(qh, k, chosen, rf, oi, od)
        e_times = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            idx.search_host(qh, k, chosen, rf, oi, od)   # syncs the stream
            e_times.append(time.perf_counter() - t0)
        sync_v = nq * args.steps / sum(e_times)
        # serving mode: rairs_search_host_async back to back, batches alternating
        # between two streams (the header's concurrent-search contract), so the
        # H2D of batch i+1 (the library's copy stream) and the D2H of batch i
        # overlap the search of the other batch; L2 flush before every step
        # inside the timed region, on the step's stream; one synchronisation at
        # the end
        pinned = [(_t.empty((nq, k), dtype=_t.int64).pin_memory(),
                   _t.empty((nq, k), dtype=_t.float32).pin_memory()) for _ in range(2)]
        outs = [(a.numpy(), b.numpy()) for a, b in pinned]    # `pinned` keeps them alive
        streams = [_t.cuda.Stream(), _t.cuda.Stream()]
        # warm-up in the same back-to-back pattern, so the library's workspace
        # pool has grown to two concurrent searches before the timed region
        for i in range(max(4, args.warmup)):
            with _t.cuda.stream(streams[i % 2]):
                flush.zero_()
                idx.search_host_async(qh, k, chosen, rf, *outs[i % 2])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.steps):
            with _t.cuda.stream(streams[i % 2]):
                flush.zero_()
                idx.search_host_async(qh, k, chosen, rf, *outs[i % 2])
        torch.cuda.synchronize()
        pipe_v = nq * args.steps / (time.perf_counter() - t0)
        e2e = {"value": round(pipe_v, 1), "unit": "queries/s",
               "h2d_bytes_per_step": int(Q.nbytes), "d2h_bytes_per_step": int(nq * k * 12),
               "mode": "pipelined: rairs_search_host_async per step from pinned host memory, "
                       "batches alternating between two streams, results copied back to pinned "
                       "host memory every step, L2 flush per step inside the timed region, one sync "
                       "at the end",
               "sync_value": round(sync_v, 1),
               "sync_mode": "rairs_search_host per step (H2D + search + D2H + stream sync)"}

    if world > 1:
        # N GPUs: the sharded public API (ShardedIndex search = per-shard search +
        # NCCL all_gather + K7 merge) with host buffers: every rank copies the
        # batch in from pinned memory, rank 0 copies the merged result out
        qh_t = torch.from_numpy(Q).pin_memory()
        oi_t = torch.empty((nq, k), dtype=torch.int64).pin_memory()
        od_t = torch.empty((nq, k), dtype=torch.float32).pin_memory()
        def host_step():
            Qd.copy_(qh_t, non_blocking=True)
            ids_, dists_, _ = step(chosen)
            if rank == 0:
                oi_t.copy_(ids_, non_blocking=True)
                od_t.copy_(dists_, non_blocking=True)
        for _ in range(2):
            host_step()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            host_step()
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                          device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e = {"value": round(nq * args.steps / float(el.item()), 1), "unit": "queries/s",
               "h2d_bytes_per_step": int(Q.nbytes) * world, "d2h_bytes_per_step": int(nq * k * 12),
               "mode": "sharded public API per step: pinned H2D of the batch on every rank, "
                       "search + all_gather + merge, D2H of the merged top-k on rank 0; "
                       "wall clock, max over ranks"}

    # ---------------- one query at a time (paper's latency workload) ------------
    lat = None
    if world == 1 and args.latency_queries > 0:
        nl = min(args.latency_queries, Q.shape[0])
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        for i in range(5):
            idx.search(Qd[i:i + 1], k, chosen, rf)
        ts = []
        for i in range(nl):
            ev0.record(stream)
            idx.search(Qd[i:i + 1], k, chosen, rf)
            ev1.record(stream)
            ev1.synchronize()
            ts.append(ev0.elapsed_time(ev1))
        ts = np.array(ts)
        lat = {"queries": nl, "nprobe": chosen, "p50_ms": round(float(np.percentile(ts, 50)), 4),
               "p99_ms": round(float(np.percentile(ts, 99)), 4),
               "scan_path": idx.scan_path(1, k, chosen, rf)}

    # ---------------- roofline of the dominant stage (the fast scan, A3-A6) ----------------
    peak, peak_src = load_peaks()
    scan_mode = idx.scan_path(Q.shape[0], k, chosen, rf)
    scan_ms = prof["ms"]["scan"] / max(1, prof["launches"]["scan"])
    kern_ms = kprof["ms"] / kprof["launches"] if kprof["launches"] else scan_ms
    roof = scan_roofline(idx, spec, scan_mode, dco_local, Qd, k, chosen, rf, kern_ms, peak, peak_src,
                         args.config)
    roof["stage_ms"] = round(scan_ms, 4)
    roof["stage_frac"] = round(roof["algorithmic_bytes_per_launch"] / (scan_ms / 1e3) / 1e9 / peak, 4)
    roof_alu = None
    if scan_mode == "simt":
        # the query-major scan is bound by instruction issue, not HBM:
        # its work in 4-bit LUT lookup-accumulates (DCO x M) against the issue
        # ceiling of the kernel's word formulation -- per nibble word (8
        # lookups) 9 alu-pipe instructions (and, 6 prmt, 2 lop3) at 0.5
        # warp-instructions/clk/SMSP (tools/micro/pipe_rates.cu): 18 cycles
        # with the pair-packed dp2a sums (M_pad <= 128: ~6 fma-pipe
        # instructions), 20 cycles with one dp4a per item (~10 on the fma-heavy
        # pipe) -- x 32 lanes x 4 SMSPs x SMs x the SM clock sampled in the
        # timed region
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        clk = (clocks or {}).get("sm_mhz") or 1965.0
        m_pad = -(-spec.M // 16) * 16
        cyc = 18.0 if (m_pad <= 128 and os.environ.get("RAIRS_FS_PACK", "1") != "0") else 20.0
        peak_l = 8.0 / cyc * 32 * 4 * nsm * clk * 1e6
        ach_l = dco_local * spec.M / (kern_ms / 1e3)
        roof_alu = {"bound": "alu", "kernel": "fs_scan_kernel", "achieved": round(ach_l / 1e12, 3),
                    "peak": round(peak_l / 1e12, 3), "unit": "T lookups/s", "frac": round(ach_l / peak_l, 4),
                    "algorithmic_ops_per_launch": int(dco_local * spec.M),
                    "peak_derivation": "8 lookups / %d clk / SMSP x 32 lanes x 4 SMSPs x %d SMs x %.0f MHz"
                                       % (cyc, nsm, clk)}

    # ---------------- AIR + SEIL vs single assignment (the paper's comparison) ----
    vs_single = None
    if world == 1 and args.compare_single and X is not None:
        steps = max(3, args.steps // 2)
        vs_single = {name: compare_strategy(kw, idx, X, Qd, spec, gt_ids, gt_d64, nq_gt, flush,
                                            stream, steps)
                     for name, kw in STRATEGIES.items()}
        vs_single["air"] = {"nprobe": chosen, "recall": round(recall, 4),
                            "qps": round(qps, 1), "dco_per_query": round(dco_total / nq, 1),
                            "double_assigned_frac": round(idx.info()["n_double"] / max(1, spec.n), 4)}
        for name in STRATEGIES:
            if name != "single":
                vs_single[f"dco_ratio_{name}_over_single"] = round(
                    vs_single[name]["dco_per_query"] / max(1.0, vs_single["single"]["dco_per_query"]), 3)
        vs_single["dco_ratio_air_over_single"] = round(
            vs_single["air"]["dco_per_query"] / max(1.0, vs_single["single"]["dco_per_query"]), 3)

    k1 = None
    if world == 1 and args.k1 and k > 1:
        k1 = side_k1(idx, Qd, spec, gt_ids, gt_d64, nq_gt, flush, stream, args.steps)

    seil_layouts = None
    if world == 1 and args.seil_paper:
        seil_layouts = side_seil_layouts(idx, args.seil_layout, Qd, k, chosen, rf, gt_ids, gt_d64,
                                         nq_gt, flush, stream, args.steps, dco_total / nq, qps)

    updates = None
    if world == 1 and args.updates and X is not None and spec.n <= 2_000_000:
        updates = update_throughput(idx, X, spec, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(spec, X, Q, chosen)

    if rank == 0:
        info = idx.info()
        line = {
            "metric": f"QPS at recall{k}@{k}>=0.95 ({spec.name}: {spec.n:,} x {spec.d}, nlist {spec.nlist}, "
                      f"PQ {spec.M}x4b, AIR+SEIL, refine x{rf})",
            "value": round(qps, 1), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": spec.name, "n": spec.n, "d": spec.d, "nq_per_batch": nq,
                       "nlist": spec.nlist, "M": spec.M, "nbits": 4, "k": k, "refine_factor": rf,
                       "nprobe": chosen,
                       "assignment": args.assignment + "+SEIL(" + {"cell": "cell-major", "paper": "paper-literal",
                                                                 "auto": "paper-literal for query-major, "
                                                                         "cell-major for list-major",
                                                                 "hybrid": "hybrid: cell-major + copies of "
                                                                           "cross cells below 8 items"}[args.seil_layout] + ")",
                       "parallelism": f"index sharded id mod {world}" if world > 1 else "1 GPU",
                       "l2": "flushed (256 MB write) between timed steps, outside the step events"},
            "recall%d@%d" % (k, k): round(recall, 4), "recall_sweep": sweep,
            "dco_per_query": round(dco_total / nq, 1),
            "dco_per_s": round(dco_total * args.steps / (t_ms / 1e3), 1),
            "stage_ms_per_step": {kk: round(v / args.steps, 4) for kk, v in prof["ms"].items()},
            "profile_pass": {"ms_per_step": round(prof_step_ms, 4),
                             "note": "stage_ms_per_step and the roofline kernel time come from a second "
                                     "pass of the same K steps with the library's stage/kernel events on "
                                     "(they break the kernels' PDL overlap, so `value` is timed without them)"},
            "roofline": roof,
            "roofline_alu": roof_alu,
            "e2e": e2e, "gpu_launches": kernels,
            "coarse_uncertified_per_step": round(fallbacks / args.steps, 1),
            "latency_1q": lat,
            "air_vs_single": vs_single,
            "k1": k1,
            "seil_layouts": seil_layouts,
            "updates": updates,
            "clocks": clocks, "wall_s_timed_region": round(wall, 4),
            "build_s": round(build_s, 2), "datagen_s": round(gen_s, 2),
            "index": {k2: info[k2] for k2 in ("n", "n_slots", "n_cells", "n_refs", "n_double",
                                              "max_refs_per_list", "device_bytes")},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def scan_roofline(idx, spec, scan_mode, dco_local, Qd, k, nprobe, rf, scan_ms, peak, peak_src, cfg):
    """Roofline of the fast-scan stage (A3-A6), bytes it must read per launch:
    * query-major register-LUT scan (fs_scan_kernel): every scored item's codes
      are read once per query that scores it -- sum_q DCO(q) * M/2;
    * list-major tensor scan: each probed list-task's codes once per batch plus
      the score rows it materialises (written once, read twice).
    `traffic` is the stage's DRAM bytes per launch from an ncu capture
    (profiles/traffic_<cfg>.json), and `frac_dram` = traffic / time / peak."""
    import torch
    M2 = spec.M // 2
    if scan_mode == "listmajor":
        # the kernel timed is lm_tensor_kernel: it reads each probed list-task's
        # codes once per batch (N_l = owned items + referenced items) and writes
        # the u16 score rows (2 B per scored (item, query) pair = DCO)
        plist = probed_list_items(idx, Qd, k, nprobe, rf)
        alg = plist * M2 + dco_local * 2
        kern = ("lm_tensor_kernel (tcgen05 kind::i8 one-hot x LUT, bound by the one-hot expansion "
                "into TMEM); time from events right around its launch")
        unit = (f"M/2 = {M2} B per probed list-task item (codes once per batch: {int(plist)} items) "
                "+ 2 B per scored (item, query) pair (u16 score rows written)")
    else:
        alg = dco_local * M2
        kern = ("fs_scan_kernel (query-major: SEIL work list + register-LUT prmt/dp4a fast scan "
                "+ threshold filter, one warp per query); time from events right around its launch")
        unit = f"M/2 = {M2} B per DCO (each scored item's codes, once per query)"
    achieved = alg / (scan_ms / 1e3) / 1e9
    traffic, traffic_src, frac_dram = None, None, None
    tp = os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            if tj.get("scan_path") in (None, scan_mode) and tj.get("nprobe") in (None, nprobe):
                kname = "lm_tensor_kernel" if scan_mode == "listmajor" else "fs_scan_kernel"
                kk = tj.get("kernels", {}).get(kname)
                traffic = kk["dram_bytes_per_search"] if kk else tj.get("dram_bytes_per_launch")
                traffic_src = tj.get("source")
        except Exception:
            traffic = None
    if traffic:
        frac_dram = round(traffic / (scan_ms / 1e3) / 1e9 / peak, 4)
    return {"bound": "hbm", "kernel": kern, "scan_path": scan_mode,
            "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "frac_dram": frac_dram,
            "traffic_source": traffic_src, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": int(alg), "algorithmic_bytes_per_unit": unit,
            "avg_launch_ms": round(scan_ms, 4),
            "stage": "fast-scan stage A3-A6 = LUT kernel + scan kernel + finish/selection"}


def probed_list_items(idx, Qd, k, nprobe, rf):
    """Items of the list-tasks the batch probes (each distinct probed list l
    once: its owned items + the items of its references), from the exported
    layout and one debug search's probe sets."""
    import torch
    L = idx.export_layout()
    nl = L["own_cnt"].shape[0]
    refs = torch.zeros(nl, dtype=torch.int64, device=L["own_cnt"].device)
    if L["ref_cnt"].numel():
        lst = torch.repeat_interleave(torch.arange(nl, device=refs.device), L["ref_ptr"][1:] - L["ref_ptr"][:-1])
        refs.index_add_(0, lst, L["ref_cnt"])
    n_l = L["own_cnt"] + refs
    probes = idx.search_debug(Qd, k, nprobe, rf)["probes"].reshape(-1).long()
    used = torch.zeros(nl, dtype=torch.bool, device=refs.device)
    used[probes] = True
    del L
    return float(n_l[used].sum().item())


def side_k1(idx, Qd, spec, gt_ids, gt_d64, nq_gt, flush, stream, steps):
    """BJ configs[3] asks for k=1 as well as k=10: the same index and protocol,
    k = 1 with K_FACTOR 10, smallest swept nprobe with
    recall1@1 >= 0.95, device-timed steps (L2 flushed between them).  When
    K_FACTOR 10 plateaus below 0.95 (bigK = 10 PQ candidates hold the true
    nearest neighbour too rarely: a raw-PQ cap, not an nprobe one), the
    refine factor is raised (25, 50, 100) until the target is reached; the
    K_FACTOR 10 plateau is kept in the line as `k_factor_10`."""
    import torch
    nq = Qd.shape[0]

    def sweep_rf(rf):
        chosen, rec, sweep = None, None, []
        for npb in [p for p in NPROBE_SWEEP if p <= spec.nlist]:
            ids, dists = idx.search(Qd, 1, npb, rf)
            r = recall_at_k(ids[:nq_gt], gt_ids, gt_d64, dists[:nq_gt], 1)
            sweep.append({"nprobe": npb, "recall": round(r, 4)})
            chosen, rec = npb, r
            if r >= 0.95 or plateaued(sweep):
                break
        return chosen, rec, sweep

    def timed(rf, npb):
        for _ in range(3):
            idx.search(Qd, 1, npb, rf)
        t = 0.0
        for _ in range(steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            idx.search(Qd, 1, npb, rf)
            e1.record(stream)
            e1.synchronize()
            t += e0.elapsed_time(e1)
        return t / steps

    rf0 = spec.refine_factor
    chosen, rec, sweep = sweep_rf(rf0)
    ms = timed(rf0, chosen)
    line = {"metric": "QPS at recall1@1>=0.95", "k": 1, "refine_factor": rf0, "nprobe": chosen,
            "recall1@1": round(rec, 4), "recall_sweep": sweep,
            "value": round(nq / (ms / 1e3), 1), "unit": "queries/s", "ms_per_step": round(ms, 4)}
    if rec >= 0.95:
        return line
    base = dict(line)
    for rf in (25, 50, 100):
        chosen, rec, sweep = sweep_rf(rf)
        ms = timed(rf, chosen)
        line = {"metric": "QPS at recall1@1>=0.95", "k": 1, "refine_factor": rf, "nprobe": chosen,
                "recall1@1": round(rec, 4), "recall_sweep": sweep,
                "value": round(nq / (ms / 1e3), 1), "unit": "queries/s", "ms_per_step": round(ms, 4)}
        if rec >= 0.95:
            break
    line["k_factor_10"] = {k: base[k] for k in ("refine_factor", "nprobe", "recall1@1", "value", "ms_per_step")}
    line["k_factor_10"]["note"] = "K_FACTOR 10 (P:2016-2017) plateaus below 0.95 on this data"
    return line


def side_seil_layouts(idx, main_layout, Qd, k, nprobe, rf, gt_ids, gt_d64, nq_gt, flush, stream, steps,
                      dco_main, qps_main):
    """The same index over the other SEIL list layouts (NEXT-2): cell-major (R10:
    every vector stored once, remainders in the owner's cell, short references),
    the paper-literal one (Alg. 4/5: shared 32-item blocks stored once,
    remainders duplicated into both lists' misc areas) and the hybrid one
    (cell-major ranges + copies of the cross cells below 8 items); same
    candidates and recall; DCO per query and QPS under the main line's
    protocol (device events, L2 flushed between steps)."""
    import torch
    simt = idx.scan_path(Qd.shape[0], k, nprobe, rf) == "simt"
    main_name = {"cell": "cell", "paper": "paper", "auto": "paper", "hybrid": "hybrid"}[main_layout] \
        if simt else "cell"
    nq = Qd.shape[0]
    res = {main_name: {"qps": round(qps_main, 1), "dco_per_query": round(dco_main, 1), "main_line": True}}
    for other in ("cell", "paper", "hybrid"):
        if other == main_name:
            continue
        bytes0 = idx.info()["device_bytes"]
        idx.set_seil_layout(other)
        extra = idx.info()["device_bytes"] - bytes0
        try:
            ids, dists, dco = idx.search(Qd, k, nprobe, rf, return_dco=True)
            rec = recall_at_k(ids[:nq_gt], gt_ids, gt_d64, dists[:nq_gt], k)
            for _ in range(3):
                idx.search(Qd, k, nprobe, rf)
            t = 0.0
            for _ in range(steps):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                idx.search(Qd, k, nprobe, rf)
                e1.record(stream)
                e1.synchronize()
                t += e0.elapsed_time(e1)
        finally:
            idx.set_seil_layout(main_layout)
        res[other] = {"qps": round(nq * steps / (t / 1e3), 1),
                      "dco_per_query": round(float(dco.sum().item()) / nq, 1),
                      "recall": round(rec, 4), "main_line": False, "device_bytes_delta_of_switch": int(extra)}
    res["nprobe"] = nprobe
    res["scan_path"] = idx.scan_path(Qd.shape[0], k, nprobe, rf)
    for o in ("paper", "hybrid"):
        res[f"dco_ratio_{o}_over_cell"] = round(res[o]["dco_per_query"] / max(1.0, res["cell"]["dco_per_query"]), 4)
        res[f"qps_ratio_{o}_over_cell"] = round(res[o]["qps"] / max(1.0, res["cell"]["qps"]), 4)
    return res


# redundant-assignment strategies compared on the same trained state (SURVEY
# §8(f) NEXT-2; the paper's Fig. 7b/c and ablation):
# name -> Index.build keywords
STRATEGIES = {
    "single": {"assignment": "single"},                               # IVFPQfs
    "naivera": {"assignment": "AIR", "lambda_": 0.0, "strict": True},
    "soarl2": {"assignment": "SOAR", "lambda_": 1.0, "strict": True},
    "srair": {"assignment": "AIR", "lambda_": 0.5, "strict": True},
}


def compare_strategy(kw, idx, X, Qd, spec, gt_ids, gt_d64, nq_gt, flush, stream, steps):
    """An index of another assignment strategy from the SAME trained
    centroids/codebook: the smallest swept nprobe reaching recall >= 0.95, its
    QPS (same timing protocol, fewer steps) and DCO per query."""
    import torch
    import paper_2601_07183_b200 as rb
    k, rf = spec.k, spec.refine_factor
    cent, cb = idx.export_trained()
    Xd = torch.from_numpy(X).to(Qd.device)
    ids_ = rb.Index.build(Xd, spec.nlist, spec.M, centroids=cent, codebook=cb, **kw)
    del Xd
    n_double = ids_.info()["n_double"]
    chosen, rec, swp = None, None, []
    for npb in [p for p in NPROBE_SWEEP if p <= spec.nlist]:
        ids, dists = ids_.search(Qd, k, npb, rf)
        r = recall_at_k(ids[:nq_gt], gt_ids, gt_d64, dists[:nq_gt], k)
        chosen, rec = npb, r
        swp.append({"nprobe": npb, "recall": r})
        if r >= 0.95 or plateaued(swp):
            break
    _, _, dco = ids_.search(Qd, k, chosen, rf, return_dco=True)
    for _ in range(3):
        ids_.search(Qd, k, chosen, rf)
    t = 0.0
    for _ in range(steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ids_.search(Qd, k, chosen, rf)
        e1.record(stream)
        e1.synchronize()
        t += e0.elapsed_time(e1)
    nq = Qd.shape[0]
    ids_.free()
    return {"nprobe": chosen, "recall": round(rec, 4), "qps": round(nq * steps / (t / 1e3), 1),
            "dco_per_query": round(float(dco.sum().item()) / nq, 1),
            "double_assigned_frac": round(n_double / max(1, X.shape[0]), 4)}


def update_throughput(idx, X, spec, dev):
    """NEXT-3 side line, the paper's protocol: an index of 80 % of
    the rows (same trained state) takes five insert batches of 4 % each, then
    the full index loses five delete batches of 4 % each; rows per second of
    rairs_add / rairs_remove_ids (assignment + device re-layout included),
    for AIR+SEIL and for single assignment (the paper's IVFPQfs baseline)."""
    import torch
    import paper_2601_07183_b200 as rb
    cent, cb = idx.export_trained()
    n = X.shape[0]
    n0, bs = int(0.8 * n), int(0.04 * n)
    out = {"protocol": f"build {n0}, 5 inserts of {bs}; build {n}, 5 deletes of {bs} (P:2286-2292)"}
    Xd = torch.from_numpy(X).to(dev)
    perm = torch.from_numpy(np.random.default_rng(3).permutation(n)[:5 * bs]).to(dev)
    for name, kw in (("air", {"assignment": "AIR"}), ("single", {"assignment": "single"})):
        a = rb.Index.build(Xd[:n0], spec.nlist, spec.M, centroids=cent, codebook=cb, **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for b in range(5):
            a.add(Xd[n0 + b * bs:n0 + (b + 1) * bs])
        torch.cuda.synchronize()
        ins = 5 * bs / (time.perf_counter() - t0)
        a.free()
        a = rb.Index.build(Xd, spec.nlist, spec.M, centroids=cent, codebook=cb, **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for b in range(5):
            a.remove_ids(perm[b * bs:(b + 1) * bs])
        torch.cuda.synchronize()
        dele = 5 * bs / (time.perf_counter() - t0)
        a.free()
        out[name] = {"inserts_per_s": round(ins, 1), "deletes_per_s": round(dele, 1)}
    del Xd
    out["air_over_single"] = {k: round(out["air"][k] / out["single"][k], 3)
                              for k in ("inserts_per_s", "deletes_per_s")}
    return out


ORACLE_MAX_ROWS = 1_000_000
# the CUDA arm's measured recall-0.95 nprobe per config (the reference arm does no sweep)
REF_NPROBE = {"c4": 2, "c2pl": 4}


def oracle_sample_index(spec, X, iters=4, seed=11, n_full=None):
    """The CPU oracle's own index (oracle/: k-means + PQ training, Alg. 3
    assignment, O5 encode) of the workload, or of a bounded uniform sample of
    it: configs above 1M rows keep their first 1M rows (i.i.d. draws, so a
    uniform sample) and scale nlist by the same factor, which keeps the mean
    list size -- hence the per-query scan work at a given nprobe -- of the full
    workload.  Nothing here comes from the CUDA path."""
    import oracle
    n = X.shape[0] if n_full is None else n_full
    if n > ORACLE_MAX_ROWS:
        Xs = np.ascontiguousarray(X[:ORACLE_MAX_ROWS])
        nlist = max(1, int(round(spec.nlist * ORACLE_MAX_ROWS / n)))
        note = (f"uniform {ORACLE_MAX_ROWS:,}-row sample of the {n:,}-row base, nlist {nlist} "
                f"(mean list size of the full config)")
    else:
        Xs, nlist, note = X, spec.nlist, f"full {n:,}-row base, nlist {spec.nlist}"
    rows = Xs[np.random.default_rng(5).permutation(Xs.shape[0])[:min(Xs.shape[0], max(32768, 32 * nlist))]]
    cent = oracle.kmeans(rows, nlist, iters=iters, seed=seed)
    cb = oracle.pq_train(rows, spec.M, iters=iters, seed=seed + 1)
    l1, l2 = oracle.assign(Xs, cent, "air")
    codes = oracle.encode(Xs, cb)
    return Xs, l1, l2, codes, cent, cb, nlist, note


def cpu_baseline(spec, X, Q, nprobe, target_s=10.0):
    """The CPU oracle (oracle/, plain C + OpenMP, never tuned) on the host
    cores, on its own index of the same workload (oracle_sample_index; build
    untimed), oracle_search timed on a bounded query sample (~10 s)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    Xs, l1, l2, codes, cent, cb, nlist, note = oracle_sample_index(spec, X)
    sample = 100
    t0 = time.perf_counter()
    oracle.search(Xs, l1, l2, codes, cent, cb, Q[:sample], spec.k, nprobe, spec.refine_factor)
    dt = time.perf_counter() - t0
    if dt < target_s / 2:   # grow the sample toward ~10 s of CPU work, bounded by the batch
        sample = int(min(Q.shape[0], sample * max(1.0, target_s / max(dt, 1e-3))))
        t0 = time.perf_counter()
        oracle.search(Xs, l1, l2, codes, cent, cb, Q[:sample], spec.k, nprobe, spec.refine_factor)
        dt = time.perf_counter() - t0
    return {"value": round(sample / dt, 2), "unit": "queries/s", "cores": cores, "kind": "oracle",
            "sample": f"first {sample} of the {Q.shape[0]} queries, nprobe {nprobe}, oracle index "
                      f"of the {note} (built untimed)"}


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from synth import GPU_KINDS, get_config, make_dataset
    spec = get_config(args.config, **spec_overrides(args))
    if spec.kind in GPU_KINDS:   # the same seeded draw as the CUDA arm (input generation only)
        import torch
        from synth.gpu_generators import make_dataset_torch
        dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
        Xd, Qd = make_dataset_torch(spec, dev, n=min(spec.n, ORACLE_MAX_ROWS))
        X, Q = Xd.cpu().numpy(), Qd.cpu().numpy()
        del Xd, Qd
    else:
        X, Q = make_dataset(spec)
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    Xs, l1, l2, codes, cent, cb, nlist_s, note = oracle_sample_index(spec, X, n_full=spec.n)
    nprobe = args.nprobe or REF_NPROBE.get(spec.name, spec.nprobe)
    sample = 1000
    for _ in range(args.warmup):
        oracle.search(Xs, l1, l2, codes, cent, cb, Q[:64], spec.k, nprobe, spec.refine_factor)
    times = []
    for i in range(args.steps):
        qs = Q[(i * sample) % Q.shape[0]:][:sample]
        t0 = time.perf_counter()
        oracle.search(Xs, l1, l2, codes, cent, cb, qs, spec.k, nprobe, spec.refine_factor)
        times.append(time.perf_counter() - t0)
    v = sample * args.steps / sum(times)
    k = spec.k
    line = {"impl": "reference",
            # the same metric / unit / direction / config keys as the CUDA arm's line
            "metric": f"QPS at recall{k}@{k}>=0.95 ({spec.name}: {spec.n:,} x {spec.d}, nlist {spec.nlist}, "
                      f"PQ {spec.M}x4b, AIR+SEIL, refine x{spec.refine_factor})",
            "value": round(v, 2), "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * sum(times) / args.steps, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": spec.name, "n": spec.n, "d": spec.d,
                       "nq_per_batch": int(Q.shape[0]), "nlist": spec.nlist, "M": spec.M,
                       "nbits": 4, "k": spec.k, "refine_factor": spec.refine_factor,
                       "nprobe": nprobe, "assignment": args.assignment + "+SEIL(cell-major)",
                       "parallelism": f"CPU oracle, {cores} host threads",
                       "queries_per_step": sample, "oracle_index": note},
            "cpu_baseline": {"value": round(v, 2), "unit": "queries/s", "cores": cores,
                             "kind": "oracle",
                             "sample": f"{sample} queries per step (bounded sample of the 10k batch) "
                                       f"on the oracle index of the {note}"},
            "e2e": {"value": round(v, 2), "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c4")
    ap.add_argument("--assignment", default="AIR", choices=["AIR", "single"])
    ap.add_argument("--nprobe", type=int, default=None)
    ap.add_argument("--k", type=int, default=None,
                    help="override the config's k (top-100 workload: --k 100 --refine-factor 4)")
    ap.add_argument("--refine-factor", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--compare-single", type=int, default=1,
                    help="also measure single / NaiveRA / SOARL2 / SRAIR indexes on the same "
                         "trained state (air_vs_single)")
    ap.add_argument("--updates", type=int, default=1,
                    help="insert/delete throughput side line (paper protocol, n <= 2M)")
    ap.add_argument("--latency-queries", type=int, default=200,
                    help="single-query searches timed for p50/p99 latency (0 = skip)")
    ap.add_argument("--gt-queries", type=int, default=0,
                    help="queries with exact ground truth for recall (0 = all)")
    ap.add_argument("--k1", type=int, default=1,
                    help="side line: the same index at k=1 (BJ configs[3]: k=1 and k=10)")
    ap.add_argument("--seil-layout", default="hybrid", choices=["cell", "paper", "auto", "hybrid"],
                    help="SEIL list layout searched (rairs_set_seil_layout): cell-major (R10), "
                         "paper-literal (Alg. 4/5), or auto = paper-literal for query-major scans, "
                         "cell-major for list-major, or hybrid (cell-major + copies of cross cells "
                         "below 8 items). The other layouts are measured in seil_layouts.")
    ap.add_argument("--seil-paper", type=int, default=1,
                    help="side line: the same index searched over the other SEIL layouts "
                         "(cell-major, paper-literal Alg. 4/5, hybrid) at the chosen nprobe")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (NCCL ranks)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
               "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
