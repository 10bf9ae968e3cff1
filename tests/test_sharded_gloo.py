"""Multi-process (world size 2, gloo, CPU) checks of the sharded mode's host logic: the row
partition, the all-gather layout and id offsets, and that merging the shard-local exact top-k lists
gives the global exact top-k (P15).  The GPU merge kernel itself is covered by
tests/test_gpu_parity.py; here the merge is the test's own reference (numpy lexsort)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1906_12211_b200.sharded import gather_merge, shard_range


def ref_merge(g_ids, g_sims):
    w, nq, k = g_ids.shape
    ids = g_ids.permute(1, 0, 2).reshape(nq, w * k).numpy()
    sims = g_sims.permute(1, 0, 2).reshape(nq, w * k).numpy()
    out_i = np.empty((nq, k), np.int64)
    out_s = np.empty((nq, k), np.float32)
    for q in range(nq):
        valid = ids[q] >= 0
        order = np.lexsort((ids[q][valid], -sims[q][valid]))[:k]
        out_i[q] = ids[q][valid][order]
        out_s[q] = sims[q][valid][order]
    return torch.from_numpy(out_i), torch.from_numpy(out_s)


def _worker(rank, world, port, x, q, k, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(len(x), world, rank)
    bi, bs = O.bruteforce(x[lo:hi], q, k)          # shard-local exact top-k, local ids
    ids = torch.from_numpy(bi + lo)                  # global ids via the shard's id offset
    sims = torch.from_numpy(bs.astype(np.float32))
    mi, ms = gather_merge(ids, sims, merge=ref_merge)
    out[rank] = mi.numpy()
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions_rows():
    for n in (1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_gloo_world2_gather_merge_equals_global_bruteforce():
    rng = np.random.default_rng(3)
    x = O.normalize(rng.standard_normal((2001, 24)))
    q = O.normalize(rng.standard_normal((40, 24)))
    k = 10
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), x, q, k, out), nprocs=2, join=True)
    gi, _ = O.bruteforce(x, q, k)
    assert np.array_equal(out[0], gi) and np.array_equal(out[1], gi)


def _prep_worker(rank, world, port, data, q, out):
    # every rank hashes only its slice of the queries (here with the oracle, CPU) and the
    # slices are all-gathered; the result must equal hashing every query on one rank
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1906_12211_b200.sharded import distributed_query_hashes
    X = O.OracleIndex(data, O.FHTCP, L=6, seed=4, M=3)

    def hash_slice(qs):
        codes, sk = X.hash(qs.numpy())
        return torch.from_numpy(codes.view(np.int32)), torch.from_numpy(sk.view(np.int64))

    codes, sk = distributed_query_hashes(hash_slice, torch.from_numpy(q))
    out[rank] = (codes.numpy().view(np.uint32), sk.numpy().view(np.uint64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("nq", [7, 40])
def test_gloo_world2_distributed_query_hashing(nq):
    rng = np.random.default_rng(5)
    data = rng.standard_normal((500, 20)).astype(np.float32)
    q = rng.standard_normal((nq, 20)).astype(np.float32)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_prep_worker, args=(2, _free_port(), data, q, out), nprocs=2, join=True)
    codes, sk = O.OracleIndex(data, O.FHTCP, L=6, seed=4, M=3).hash(q)
    for r in (0, 1):
        assert np.array_equal(out[r][0], codes) and np.array_equal(out[r][1], sk)
