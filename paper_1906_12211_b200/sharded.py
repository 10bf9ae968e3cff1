"""Data-sharded multi-GPU mode: one process per GPU, each indexing a contiguous
block of rows under the same seed (identical hash functions on every shard), every rank answering
every query with shard-local adaptive stopping, then an NCCL all-gather of the local top-k lists
and the library's merge kernel.  Why the guarantee carries over: a global top-k point of shard s
is a local top-k point of s, returned with probability >= 1 - delta; after the merge every point
ranked above it is a true point above it, so it stays in the global top-k.

Plumbing only (torch.distributed for the collective); the search and the merge are library calls.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import Index, merge_topk


def shard_range(n: int, world: int, rank: int):
    """contiguous row block [lo, hi) of rank `rank` (the first n % world ranks get one extra row)"""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_merge(ids, sims, group=None, merge=None):
    """all-gather the local [nq, k] lists of every rank (NCCL in production; any backend works)
    and merge them (default: the library's k_merge_topk).  Returns (ids, sims) [nq, k]."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return ids, sims
    nq, k = ids.shape
    g_ids = torch.empty((world * nq, k), dtype=ids.dtype, device=ids.device)
    g_sims = torch.empty((world * nq, k), dtype=sims.dtype, device=sims.device)
    dist.all_gather_into_tensor(g_ids, ids.contiguous(), group=group)
    dist.all_gather_into_tensor(g_sims, sims.contiguous(), group=group)
    return (merge or merge_topk)(g_ids.view(world, nq, k), g_sims.view(world, nq, k))


def gather_rows(local, nrows: int, group=None):
    """all-gather row slices [shard_range(nrows, world, r)] of a [rows, w] tensor from every rank into
    the full [nrows, w] tensor (slices padded to equal length for all_gather_into_tensor)"""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    rank = dist.get_rank(group)
    per = shard_range(nrows, world, 0)[1]        # the largest slice
    buf = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    lo, hi = shard_range(nrows, world, rank)
    buf[: hi - lo] = local
    out = torch.empty((world * per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    parts = [out[r * per: r * per + (shard_range(nrows, world, r)[1] - shard_range(nrows, world, r)[0])]
             for r in range(world)]
    return torch.cat(parts).contiguous()


def distributed_query_hashes(hash_slice, queries, group=None):
    """SURVEY 8(e) (identical functions on every shard): rank r hashes only its slice of the queries,
    hash_slice(q_slice) -> (codes [s, reps], sketches [s, M]); the slices are all-gathered so every
    rank holds every query's codes and sketches without hashing them all"""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    nq = queries.shape[0]
    lo, hi = shard_range(nq, world, rank)
    codes, sk = hash_slice(queries[lo:hi])
    return gather_rows(codes, nq, group), gather_rows(sk, nq, group)


class ShardedIndex:
    """Build this rank's shard: `local_data` are rows [row0, row0 + len) of the global dataset."""

    def __init__(self, local_data, row0: int, memory_budget: int, family, seed: int = 1, group=None, **opts):
        self.group = group
        self.row0 = row0
        self.index = Index(local_data, memory_budget, family, seed=seed, id_offset=row0, **opts)

    def prep_reps(self) -> int:
        """repetitions whose codes the distributed preparation computes (all L unless the family
        hashes later repetitions lazily in the kernels: FHT cross-polytope, independent functions)"""
        inf = self.index.info
        lazy = inf["family"] == 1 and inf["strategy"] == 0 and inf["fht_dim"] in (32, 64, 128)
        return min(inf["reps"], 32) if lazy else inf["reps"]

    def search(self, queries, k: int, recall: float, distributed_prep: bool = False, **sopts):
        """-> merged (ids [nq,k], sims [nq,k]) on every rank (CUDA tensors).  distributed_prep: each rank
        hashes 1/world of the queries and the codes and sketches are all-gathered"""
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        if distributed_prep and world > 1:
            reps = self.prep_reps()
            codes, sk = distributed_query_hashes(lambda qs: self.index.hash_queries_reps(qs, reps), queries, self.group)
            sopts = dict(sopts, ext_codes=codes, ext_sketches=sk if self.index.info["sketch_words"] > 0 else None)
        res = self.index.search(queries, k, recall, **sopts)
        m_ids, m_sims = gather_merge(res[0], res[1], self.group)
        return (m_ids, m_sims) + tuple(res[2:])


class ReplicatedIndex:
    """Query-parallel mode (replicas): every rank builds the whole index under the same seed and
    answers its own query batch; no collective on the data path (the queries are independent
    problems, so N ranks are N independent replicas)."""

    def __init__(self, data, memory_budget: int, family, seed: int = 1, **opts):
        self.row0 = 0
        self.index = Index(data, memory_budget, family, seed=seed, **opts)

    def search(self, queries, k: int, recall: float, **sopts):
        return self.index.search(queries, k, recall, **sopts)
