import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as oracle_mod
import paper_2601_07183_b200 as rb
from synth import get_config, make_dataset
from tests.test_gpu_parity import gpu_search, _t
nq = 40
spec = get_config("c0s", n=30000, nq=nq, d=32, M=16, nlist=8192)
X, Q = make_dataset(spec)
rows = X[np.random.default_rng(5).permutation(X.shape[0])[:20000]]
cent = rows[np.random.default_rng(6).permutation(rows.shape[0])[:8192]].copy()
cb = oracle_mod.pq_train(rows, 16, iters=2, seed=1)
l1, l2 = oracle_mod.assign(X, cent, "air")
codes = oracle_mod.encode(X, cb)
idx = rb.Index.build(_t(X), 8192, 16, centroids=_t(cent), codebook=_t(cb))
res = []
for lay in ("cell", "paper", "hybrid"):
    idx.set_seil_layout(lay)
    for k, nprobe, rf in ((10, 3, 10), (5, 40, 4), (5, 8, 4), (5, 16, 4), (5, 24, 4)):
        o = oracle_mod.search(X, l1, l2, codes, cent, cb, Q, k, nprobe, rf)
        g = gpu_search(idx, Q, k, nprobe, rf, "simt")
        ocs = o["cand_scores"][:, 0]
        bad = [i for i in range(nq) if not np.array_equal(g["cand_scores"][i], ocs[i])]
        res.append((lay, k, nprobe, rf, len(bad)))
print(os.environ.get("TAG", ""), res, flush=True)
