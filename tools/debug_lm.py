import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_07183_b200 as rb
from synth import get_config, make_dataset
name = sys.argv[1]; npb = int(sys.argv[2]); nqs = int(sys.argv[3]) if len(sys.argv) > 3 else None
spec = get_config(name)
X, Q = make_dataset(spec, nq=nqs)
dev = torch.device("cuda:0")
idx = rb.build_index(torch.from_numpy(X).to(dev), spec.nlist, spec.M)
Qd = torch.from_numpy(Q).to(dev)
res = {}
for mode in ("simt", "listmajor"):
    idx.set_scan_mode(mode)
    r = idx.search_debug(Qd, spec.k, npb, spec.refine_factor)
    torch.cuda.synchronize()
    res[mode] = {k: v.cpu().numpy() for k, v in r.items()}
a, b = res["simt"], res["listmajor"]
for key in ("probes", "Qv", "dco", "cand_scores", "cand_ids", "ids"):
    eq = np.all(a[key].reshape(a[key].shape[0], -1) == b[key].reshape(b[key].shape[0], -1), axis=1)
    print(key, "queries differing:", int((~eq).sum()), "of", eq.size)
    if key == "cand_scores" and (~eq).any():
        q = int(np.nonzero(~eq)[0][0])
        print(" first bad query", q, "probes", a["probes"][q])
        print(" simt", a["cand_scores"][q][:20].view(np.uint32), a["cand_ids"][q][:20].view(np.uint32))
        print(" lm  ", b["cand_scores"][q][:20].view(np.uint32), b["cand_ids"][q][:20].view(np.uint32))
        sa = set(zip(a["cand_scores"][q].view(np.uint32), a["cand_ids"][q].view(np.uint32)))
        sb = set(zip(b["cand_scores"][q].view(np.uint32), b["cand_ids"][q].view(np.uint32)))
        print(" only simt", sorted(sa - sb)[:10]); print(" only lm", sorted(sb - sa)[:10])
