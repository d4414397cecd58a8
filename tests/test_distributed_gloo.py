"""Multi-process (world_size 2, gloo, CPU) tests of the sharding plumbing in
paper_2601_07183_b200/distributed.py: id-mod-G partition, broadcast of the
trained state, all_gather layout [G, nq, k] and the global top-k merge (O11).
Per-shard results come from the CPU oracle's shard emulation; the merge used
here is a plain sort (the product merge is the CUDA K7 kernel, covered by
tests/test_gpu_parity.py::test_sharded_parity)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sort_merge(all_ids, all_d):
    G, nq, k = all_ids.shape
    oi = torch.full((nq, k), -1, dtype=torch.int64)
    od = torch.full((nq, k), float("inf"))
    for q in range(nq):
        pool = sorted((float(all_d[g, q, j]), int(all_ids[g, q, j]))
                      for g in range(G) for j in range(k) if all_ids[g, q, j] >= 0)[:k]
        for j, (dd, ii) in enumerate(pool):
            oi[q, j], od[q, j] = ii, dd
    return oi, od


def _worker(rank, world, port, payload, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_07183_b200.distributed import (broadcast_trained, shard_rows,
                                                      sharded_merge)
        ids = torch.from_numpy(payload["shard_ids"][:, rank, :].copy())
        dists = torch.from_numpy(payload["shard_dists"][:, rank, :].copy())
        mi, md = sharded_merge(ids, dists, merge=_sort_merge)
        cent = torch.from_numpy(payload["cent"].copy()) if rank == 0 else torch.zeros(payload["cent"].shape)
        cb = torch.from_numpy(payload["cb"].copy()) if rank == 0 else torch.zeros(payload["cb"].shape)
        broadcast_trained(cent, cb, src=0)
        rows = shard_rows(payload["n"], rank, world).numpy()
        out_q.put((rank, mi.numpy(), md.numpy(), cent.numpy(), cb.numpy(), rows))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_merge_matches_oracle(oracle_mod):
    from synth import get_config, make_dataset
    spec = get_config("c1s")
    X, Q = make_dataset(spec, nq=20)
    cent = oracle_mod.kmeans(X, spec.nlist, iters=4, seed=3)
    cb = oracle_mod.pq_train(X, spec.M, iters=4, seed=4)
    l1, l2 = oracle_mod.assign(X, cent, "air")
    codes = oracle_mod.encode(X, cb)
    G = 2
    o = oracle_mod.search(X, l1, l2, codes, cent, cb, Q, 10, 8, 4, nshards=G)
    payload = {"shard_ids": o["shard_ids"], "shard_dists": o["shard_dists"], "cent": cent,
               "cb": cb, "n": X.shape[0]}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, G, port, payload, q)) for r in range(G)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(G):
        r = q.get(timeout=240)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(G):
        mi, md, c, b, rows = res[r]
        assert np.array_equal(mi, o["ids"])                     # O11 on every rank
        assert np.allclose(md, o["dists"], rtol=1e-6)
        assert np.array_equal(c, cent) and np.array_equal(b, cb)  # trained state broadcast
        assert np.array_equal(rows, np.arange(r, X.shape[0], G))  # id mod G partition
    allrows = np.sort(np.concatenate([res[r][4] for r in range(G)]))
    assert np.array_equal(allrows, np.arange(X.shape[0]))


class _FakeShard:
    """Host stand-in for one shard's Index (the numbering contract of
    rairs_add / rairs_remove_ids: local row r <-> global id r*G + s)."""

    def __init__(self, s, G, n_local):
        self.s, self.G, self.rows = s, G, [r * G + s for r in range(n_local)]
        self.dead = set()
        self.device = torch.device("cpu")

    def add(self, x):
        first = len(self.rows) * self.G + self.s
        self.rows += [(len(self.rows) + j) * self.G + self.s for j in range(x.shape[0])]
        self.kept = getattr(self, "kept", []) + x[:, 0].tolist()
        return first

    def remove_ids(self, ids):
        held = {int(i) for i in ids.tolist() if i >= 0 and i % self.G == self.s and i in self.rows}
        new = held - self.dead
        self.dead |= new
        return len(new)


def _update_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_07183_b200.distributed import ShardedIndex, shard_rows
        n0 = 11                                        # odd: shards start unequal
        local = _FakeShard(rank, world, len(shard_rows(n0, rank, world)))
        sh = ShardedIndex(local, n_total=n0, merge=lambda a, b: (a, b))
        firsts = []
        for size in (5, 4, 7):                         # batch row j carries id n_total + j
            batch = torch.arange(sh.n_total, sh.n_total + size, dtype=torch.float32)[:, None]
            firsts.append(sh.add(batch.repeat(1, 4)))
        removed = sh.remove_ids(torch.tensor([0, 3, 3, 12, 26, 27, 99, -1]))
        out_q.put((rank, firsts, sh.n_total, local.rows, local.kept, removed))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_insert_delete_numbering():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_update_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_rows = []
    for rank, firsts, n_total, rows, kept, removed in res:
        assert firsts == [11, 16, 20] and n_total == 27
        assert rows == list(range(rank, 27, world))    # id-mod-G shard, no gaps
        assert all(int(v) % world == rank for v in kept)  # each rank kept its own ids
        assert removed == 4                            # 0, 3, 12, 26 (3 repeated; 27, 99, -1 absent)
        all_rows += rows
    assert sorted(all_rows) == list(range(27))
