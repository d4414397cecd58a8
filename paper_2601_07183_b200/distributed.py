"""Index sharding over GPUs: one process per GPU, torch.distributed plumbing.

Partition: vector id x lives on shard
x mod G. Each rank builds its shard from the SAME trained centroids/codebook
(rank 0 trains, ``broadcast_trained`` ships them), searches its shard with
the CUDA kernels, and the per-shard top-k lists are exchanged with ONE
all_gather (NCCL over NVLink on B200; gloo in the CPU tests) and merged by
the K7 kernel (rairs_merge_topk): the first k by (distance, id) -- O11.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_rows(n: int, shard_id: int, nshards: int) -> torch.Tensor:
    """Global ids of shard `shard_id`: {x : x mod G == shard_id}, ascending.
    Local row r <-> global id r*G + shard_id."""
    return torch.arange(shard_id, n, nshards, dtype=torch.int64)


def _via_host(t: torch.Tensor, group) -> bool:
    """gloo collectives run on host tensors (device tensors are staged)."""
    return t.is_cuda and dist.get_backend(group) != "nccl"


def broadcast_trained(centroids: torch.Tensor, codebook: torch.Tensor, src: int = 0,
                      group=None) -> Tuple[torch.Tensor, torch.Tensor]:
    for t in (centroids, codebook):
        if _via_host(t, group):
            h = t.cpu()
            dist.broadcast(h, src=src, group=group)
            t.copy_(h)
        else:
            dist.broadcast(t, src=src, group=group)
    return centroids, codebook


def gather_shard_results(ids: torch.Tensor, dists: torch.Tensor,
                         group=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """[nq, k] per rank -> [G, nq, k] on every rank (one all_gather each)."""
    G = dist.get_world_size(group)
    nq, k = ids.shape
    if dist.get_backend(group) == "nccl":
        all_ids = torch.empty((G, nq, k), dtype=ids.dtype, device=ids.device)
        all_d = torch.empty((G, nq, k), dtype=dists.dtype, device=dists.device)
        dist.all_gather_into_tensor(all_ids, ids.contiguous(), group=group)
        dist.all_gather_into_tensor(all_d, dists.contiguous(), group=group)
        return all_ids, all_d
    dev = ids.device
    hi, hd = ids.contiguous().cpu(), dists.contiguous().cpu()   # gloo: host staging
    li = [torch.empty_like(hi) for _ in range(G)]
    ld = [torch.empty_like(hd) for _ in range(G)]
    dist.all_gather(li, hi, group=group)
    dist.all_gather(ld, hd, group=group)
    return torch.stack(li).to(dev), torch.stack(ld).to(dev)


def batch_slice_for_rank(n_total: int, batch: int, shard_id: int, nshards: int) -> slice:
    """Rows of an insert batch that shard `shard_id` keeps: batch row j gets
    global id n_total + j and lives on shard (n_total + j) mod G, so shard s
    takes rows j = (s - n_total) mod G, +G, ... -- which continues its local
    numbering (local row r <-> global id r*G + s) without gaps."""
    start = (shard_id - n_total) % nshards
    return slice(start, batch, nshards)


class ShardedIndex:
    """A RAIRS index sharded over the ranks of a process group."""

    def __init__(self, local_index, group=None,
                 merge: Optional[Callable] = None, n_total: Optional[int] = None):
        self.local = local_index
        self.group = group
        self.n_total = n_total
        if merge is None:
            from .index import merge_topk
            merge = merge_topk
        self.merge = merge

    @staticmethod
    def from_trained(base_local: torch.Tensor, n_total: int, centroids: torch.Tensor,
                     codebook: torch.Tensor, group=None, **kw) -> "ShardedIndex":
        """This rank's shard built from a trained state held by rank 0
        (broadcast first), e.g. an oracle-trained one in the parity tests."""
        from .index import Index
        rank, G = dist.get_rank(group), dist.get_world_size(group)
        cent = centroids.to(base_local.device).contiguous().clone()
        cb = codebook.to(base_local.device).contiguous().clone()
        broadcast_trained(cent, cb, src=0, group=group)
        nlist, M = cent.shape[0], cb.shape[0]
        idx = Index.build(base_local, nlist, M, centroids=cent, codebook=cb,
                          shard_id=rank, nshards=G, **kw)
        return ShardedIndex(idx, group=group, n_total=n_total)

    @staticmethod
    def build(base_local: torch.Tensor, n_total: int, nlist: int, M: int,
              train_base: Optional[torch.Tensor] = None, group=None, **kw) -> "ShardedIndex":
        """base_local: this rank's rows (shard_rows order) on its GPU.
        train_base: rows used for training on rank 0 (defaults to base_local)."""
        from .index import Index, train
        rank, G = dist.get_rank(group), dist.get_world_size(group)
        d = base_local.shape[1]
        dev = base_local.device
        cent = torch.empty((nlist, d), dtype=torch.float32, device=dev)
        cb = torch.empty((M, 16, d // M), dtype=torch.float32, device=dev)
        train_kw = {key: kw[key] for key in ("kmeans_iters", "train_sample", "seed") if key in kw}
        if rank == 0:
            c0, b0 = train(train_base if train_base is not None else base_local, nlist, M, **train_kw)
            cent.copy_(c0)
            cb.copy_(b0)
        broadcast_trained(cent, cb, src=0, group=group)
        idx = Index.build(base_local, nlist, M, centroids=cent, codebook=cb,
                          shard_id=rank, nshards=G, **kw)
        return ShardedIndex(idx, group=group, n_total=n_total)

    def add(self, x_batch: torch.Tensor) -> int:
        """Insert a batch given in full on every rank (global ids n_total ..
        n_total + batch - 1); each rank inserts its id-mod-G rows. Returns the
        first global id of the batch."""
        rank, G = dist.get_rank(self.group), dist.get_world_size(self.group)
        first = self.n_total
        sl = batch_slice_for_rank(first, x_batch.shape[0], rank, G)
        local = x_batch[sl]
        if local.shape[0] > 0:
            got = self.local.add(local)
            if got != first + sl.start:
                raise RuntimeError(f"shard {rank}: local numbering out of step ({got} != {first + sl.start})")
        self.n_total = first + x_batch.shape[0]
        return first

    def remove_ids(self, ids: torch.Tensor) -> int:
        """Delete global ids (the same list on every rank); returns the total
        deleted over all shards (one all_reduce)."""
        n = torch.tensor([self.local.remove_ids(ids)], dtype=torch.int64,
                         device=self.local.device if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(n, group=self.group)
        return int(n.item())

    def search(self, queries: torch.Tensor, k: int, nprobe: int, refine_factor: int = 10):
        ids, dists = self.local.search(queries, k, nprobe, refine_factor)
        return sharded_merge(ids, dists, group=self.group, merge=self.merge)


def sharded_merge(ids: torch.Tensor, dists: torch.Tensor, group=None,
                  merge: Optional[Callable] = None):
    """all_gather per-shard top-k, then merge to the global top-k (O11)."""
    if merge is None:
        from .index import merge_topk
        merge = merge_topk
    all_ids, all_d = gather_shard_results(ids, dists, group=group)
    return merge(all_ids, all_d)
