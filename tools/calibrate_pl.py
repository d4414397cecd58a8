"""Calibrate the paper-like ("-pl") generator of a config:
pick (sigma, natural clusters) so that AIR double-assigns 40-65 % of vectors,
single-assignment recall10@10 at nprobe=1 is < 0.9, and recall 0.95 is
reached inside the nprobe sweep at refine x10. Runs on one GPU; prints one
JSON line per candidate."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2601_07183_b200 as rb  # noqa: E402
from bench import NPROBE_SWEEP, recall_at_k  # noqa: E402
from synth import GPU_KINDS, get_config, make_dataset  # noqa: E402


def main():
    base = sys.argv[1] if len(sys.argv) > 1 else "c2pl"
    grid = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [[24, 64], [48, 64], [64, 64], [48, 16], [96, 16]]
    dev = torch.device("cuda:0")
    nmax = int(os.environ.get("CAL_N", "1000000"))   # calibrate on a <= 1M-row sample
    for sigma, nat in grid:
        spec0 = get_config(base)
        n = min(spec0.n, nmax)
        scale = n / spec0.n
        nlist = max(16, int(round(spec0.nlist * scale)))
        spec = get_config(base, sigma=float(sigma), nclusters=max(1, int(round(nat * scale))),
                          n=n, nlist=nlist)
        t0 = time.time()
        if spec.kind in GPU_KINDS:
            from synth.gpu_generators import make_dataset_torch
            Xd, Qd = make_dataset_torch(spec, dev)
        else:
            X, Q = make_dataset(spec)
            Xd, Qd = torch.from_numpy(X).to(dev), torch.from_numpy(Q).to(dev)
        gt, gd = rb.exact_knn(Xd, Qd, spec.k)
        cent, cb = rb.train(Xd, spec.nlist, spec.M)
        row = {"config": base, "sigma": sigma, "natural_clusters": nat, "n": n, "nlist": nlist,
               "natural_clusters_sample": spec.nclusters}
        for mode in ("AIR", "single"):
            idx = rb.Index.build(Xd, spec.nlist, spec.M, assignment=mode, centroids=cent, codebook=cb)
            info = idx.info()
            rec = {}
            for npb in NPROBE_SWEEP:
                ids, dists, dco = idx.search(Qd, spec.k, npb, spec.refine_factor, return_dco=True)
                rec[npb] = (round(recall_at_k(ids, gt, gd, dists, spec.k), 4),
                            round(float(dco.double().mean()), 1))
                if rec[npb][0] >= 0.99:
                    break
            row[mode] = {"double_frac": round(info["n_double"] / info["n"], 4),
                         "refs_per_list": round(info["n_refs"] / info["nlist"], 2),
                         "recall_dco": rec}
            idx.free()
        row["secs"] = round(time.time() - t0, 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
