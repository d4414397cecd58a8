"""The sharded search end to end in two processes: each rank
builds its id-mod-2 shard with the CUDA library from the trained state rank 0
broadcasts, searches it with the CUDA kernels, the per-shard top-k are
exchanged by all_gather and merged by the K7 kernel (rairs_merge_topk).  Only
one GPU is available here, so both ranks share cuda:0 and talk over gloo (NCCL
refuses two ranks on one device); the ranks' kernels never wait on each other.
Compared with the oracle's G = 2 shard emulation (O11)."""
import os
import socket

import numpy as np
import pytest

from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

if not gpu_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, payload, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_07183_b200.distributed import ShardedIndex, shard_rows
        dev = torch.device("cuda", 0)
        X = payload["X"]
        rows = shard_rows(X.shape[0], rank, world).numpy()
        base = torch.from_numpy(X[rows]).to(dev)
        cent = torch.from_numpy(payload["cent"]) if rank == 0 else torch.zeros(payload["cent"].shape)
        cb = torch.from_numpy(payload["cb"]) if rank == 0 else torch.zeros(payload["cb"].shape)
        sh = ShardedIndex.from_trained(base, X.shape[0], cent.to(dev), cb.to(dev))
        Qd = torch.from_numpy(payload["Q"]).to(dev)
        res = []
        for k, nprobe, rf in payload["cases"]:
            ids, dists = sh.search(Qd, k, nprobe, rf)
            res.append((ids.cpu().numpy(), dists.cpu().numpy()))
        # inserts continue the id-mod-G numbering; deletes are summed over ranks
        first = sh.add(torch.from_numpy(payload["Xadd"]).to(dev))
        deleted = sh.remove_ids(torch.arange(0, 100, dtype=torch.int64))
        ids, dists = sh.search(Qd, 10, 8, 4)
        torch.cuda.synchronize()
        out_q.put((rank, res, first, deleted, ids.cpu().numpy(), dists.cpu().numpy()))
        sh.local.free()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_process_sharded_search_matches_oracle(oracle_mod):
    from synth import get_config, make_dataset
    spec = get_config("c1s")
    X, Q = make_dataset(spec)
    n = X.shape[0] - 400
    Xb, Xadd = X[:n], X[n:]
    rng = np.random.default_rng(5)
    rows = X[rng.permutation(n)[:20000]]
    cent = oracle_mod.kmeans(rows, spec.nlist, iters=6, seed=11)
    cb = oracle_mod.pq_train(rows, spec.M, iters=6, seed=12)
    cases = [(10, 8, 4), (5, 16, 10), (20, 4, 2)]
    payload = {"X": Xb, "Q": Q, "cent": cent, "cb": cb, "cases": cases, "Xadd": Xadd}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, payload, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = {}
    for _ in range(2):
        r, res, first, deleted, ids, dists = q.get(timeout=500)
        outs[r] = (res, first, deleted, ids, dists)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    l1, l2 = oracle_mod.assign(Xb, cent, "air")
    codes = oracle_mod.encode(Xb, cb)
    for ci, (k, nprobe, rf) in enumerate(cases):
        o = oracle_mod.search(Xb, l1, l2, codes, cent, cb, Q, k, nprobe, rf, nshards=2)
        for r in range(2):                      # every rank holds the merged result
            ids, dists = outs[r][0][ci]
            assert np.array_equal(ids, o["ids"]), f"merged ids (rank {r}, case {ci})"
            fin = np.isfinite(o["dists"])
            assert np.array_equal(np.isfinite(dists), fin)
            assert np.allclose(dists[fin], o["dists"][fin], rtol=1e-4, atol=0)
    assert outs[0][1] == outs[1][1] == n                   # first global id of the insert
    assert outs[0][2] == outs[1][2] == 100                 # ids 0..99, summed over shards
    # after the insert and the deletes: O11 emulated shard by shard -- the
    # oracle over each shard's live rows (global id x on shard x mod 2; local
    # order = global id order, so (s, id) ties break alike), per-shard top-k,
    # then the global first k by (distance, id)
    live = np.arange(X.shape[0])
    live = live[live >= 100]
    per = []
    for sh in range(2):
        rows = live[live % 2 == sh]
        Xs = X[rows]
        sl1, sl2 = oracle_mod.assign(Xs, cent, "air")
        o = oracle_mod.search(Xs, sl1, sl2, oracle_mod.encode(Xs, cb), cent, cb, Q, 10, 8, 4)
        per.append((np.where(o["ids"] >= 0, rows[np.maximum(o["ids"], 0)], -1), o["dists"]))
    ids, dists = outs[0][3], outs[0][4]
    assert np.array_equal(ids, outs[1][3]) and np.array_equal(dists, outs[1][4])
    for i in range(Q.shape[0]):
        pool = sorted((float(per[sh][1][i, j]), int(per[sh][0][i, j]))
                      for sh in range(2) for j in range(10) if per[sh][0][i, j] >= 0)[:10]
        assert [p[1] for p in pool] == ids[i][:len(pool)].tolist(), f"query {i}"
        assert np.allclose(dists[i][:len(pool)], [p[0] for p in pool], rtol=1e-4, atol=0)
