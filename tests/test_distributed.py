"""Multi-rank host logic of the id-sharded index (paper_2508_17828_b200/
distributed.py) on CPU: world_size 2 over gloo, with the oracle as each
rank's searcher. Checks: shards partition the index and keep list order; a
rank's result equals the reference semantics over its shard's candidate
subsequence; the all-gather + merge equals the global answer where the bound
is sound (gamma = 0, full probing == brute force); counters sum."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_17828_b200.distributed import ShardedIvfIndex, shard_arrays, shard_bounds
from paper_2508_17828_b200.ivf import IvfArrays
from tests import goldens

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def host_index(a):
    from oracle.oracle import HostIndex
    return HostIndex(**{f: getattr(a, f) for f in goldens.FIELDS})


def np_merge(gd, gi, k):
    """Reference merge by (dist, id) for the test (the product merge is the
    device kernel, covered in tests/test_gpu_distributed.py)."""
    d = gd.numpy()
    i = gi.numpy().view(np.uint32)
    w, nq, kk = d.shape
    out_d = np.zeros((nq, k), np.float32)
    out_i = np.zeros((nq, k), np.uint32)
    for q in range(nq):
        cand = sorted(zip(d[:, q].ravel().tolist(), i[:, q].ravel().tolist()))[:k]
        out_d[q] = [c[0] for c in cand]
        out_i[q] = [c[1] for c in cand]
    return torch.from_numpy(out_d), torch.from_numpy(out_i.view(np.int32))


def _worker(rank, port, results):
    from oracle.oracle import COracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        ix, qs, _ = goldens.load("ivf_fixture")
        full = IvfArrays.from_any(ix)
        sh = shard_arrays(full, rank, WORLD)
        hsh = host_index(sh)
        # the oracle needs global ids -> rows: give it the full vectors (ids index them)
        hsh.vectors = np.ascontiguousarray(ix.vectors)
        co = COracle()

        def searcher(q, k, nprobe, gamma):
            ids, d, ct, cdc = co.search_knn(hsh, q.numpy(), k, nprobe, gamma)
            c6 = np.concatenate([ct.astype(np.int64), cdc.astype(np.int64)[:, None]], 1)
            return (torch.from_numpy(ids.view(np.int32)), torch.from_numpy(d), torch.from_numpy(c6))

        s = ShardedIvfIndex(sh, searcher=searcher, merge=np_merge)
        out = {}
        for gamma, k, nprobe in ((0.0, 10, 20), (0.35, 5, 6), (1.0, 10, 20)):
            mi, md, c = s.search_knn(torch.from_numpy(np.ascontiguousarray(qs)), k, nprobe, gamma)
            out[(gamma, k, nprobe)] = (mi.numpy().view(np.uint32), md.numpy(), c.numpy())
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_shards_partition_the_index():
    ix, _, _ = goldens.load("ivf_fixture")
    full = IvfArrays.from_any(ix)
    seen = []
    for r in range(3):
        sh = shard_arrays(full, r, 3)
        lo, hi = shard_bounds(ix.vectors.shape[0], r, 3)
        assert sh.id_base == lo and sh.vectors.shape[0] == hi - lo
        offs = sh.list_offsets
        for l in range(offs.size - 1):
            seg = sh.list_ids[int(offs[l]):int(offs[l + 1])]
            assert (np.diff(seg.astype(np.int64)) > 0).all()
            assert ((seg >= lo) & (seg < hi)).all()
        seen.append(sh.list_ids)
    allids = np.sort(np.concatenate(seen))
    np.testing.assert_array_equal(allids, np.arange(ix.vectors.shape[0]))


def test_two_rank_gloo_search_and_merge():
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(port, results), nprocs=WORLD, join=True)
    from oracle.oracle import COracle
    co = COracle()
    ix, qs, _ = goldens.load("ivf_fixture")
    full = IvfArrays.from_any(ix)
    for key in results[0]:
        gamma, k, nprobe = key
        (i0, d0, c0), (i1, d1, c1) = results[0][key], results[1][key]
        np.testing.assert_array_equal(i0, i1)  # every rank holds the merged answer
        np.testing.assert_array_equal(c0, c1)
        # counters = sum of the per-shard reference runs
        want_c = np.zeros(5, np.int64)
        for r in range(WORLD):
            sh = shard_arrays(full, r, WORLD)
            h = host_index(sh)
            h.vectors = np.ascontiguousarray(ix.vectors)
            want_c += co.search_knn(h, qs, k, nprobe, gamma)[2].sum(0).astype(np.int64)
        np.testing.assert_array_equal(c0, want_c)
        if gamma == 0.0 and nprobe == full.list_offsets.size - 1:
            # sound bound + full probing: the merge is the exact global kNN
            bf_ids, bf_d = co.brute_force_knn(ix.vectors, qs, k)
            np.testing.assert_array_equal(i0, bf_ids)
            np.testing.assert_array_equal(d0, bf_d)


def _replica_worker(rank, port, results):
    from oracle.oracle import COracle
    from paper_2508_17828_b200.distributed import ReplicaIvfIndex
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        ix, qs, _ = goldens.load("ivf_fixture")
        full = IvfArrays.from_any(ix)
        h = host_index(full)
        co = COracle()

        def searcher(q, k, nprobe, gamma):
            ids, d, ct, cdc = co.search_knn(h, q.numpy(), k, nprobe, gamma)
            c6 = np.concatenate([ct.astype(np.int64), cdc.astype(np.int64)[:, None]], 1)
            return (torch.from_numpy(ids.view(np.int32).copy()), torch.from_numpy(d), torch.from_numpy(c6))
        rep = ReplicaIvfIndex(full, searcher=searcher)
        q = torch.from_numpy(qs)
        part = rep.search_knn(q, 10, 5, 0.35)
        ids, d, cts = rep.gather(q.shape[0], part)
        results[rank] = (part[0], part[1], ids.numpy().copy(), d.numpy().copy(), cts.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_replicas_equal_single_run():
    from oracle.oracle import COracle
    ix, qs, _ = goldens.load("ivf_fixture")
    h = host_index(IvfArrays.from_any(ix))
    want_ids, want_d, want_ct, want_cdc = COracle().search_knn(h, qs, 10, 5, 0.35)
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_replica_worker, args=(_free_port(), results), nprocs=WORLD, join=True)
    spans = sorted((results[r][0], results[r][1]) for r in range(WORLD))
    assert spans[0][0] == 0 and spans[-1][1] == len(qs) and spans[0][1] == spans[1][0]
    for r in range(WORLD):
        _, _, ids, d, cts = results[r]
        np.testing.assert_array_equal(ids.view(np.uint32), want_ids)
        np.testing.assert_array_equal(d.view(np.uint32), want_d.view(np.uint32))
        np.testing.assert_array_equal(cts[:, :5], want_ct.astype(np.int64))


def _range_worker(rank, port, results):
    from oracle.oracle import COracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        ix, qs, _ = goldens.load("ivf_fixture")
        full = IvfArrays.from_any(ix)
        sh = shard_arrays(full, rank, WORLD)
        hsh = host_index(sh)
        hsh.vectors = np.ascontiguousarray(ix.vectors)  # global ids index the rows
        co = COracle()

        def rs(q, r, npb, g, cap):
            offs, ids, d, ct, cdc = co.search_range(hsh, q.numpy(), r, npb, g)
            nq = q.shape[0]
            cnt = np.diff(offs.astype(np.int64))
            I = np.zeros((nq, cap), np.int32)
            D = np.zeros((nq, cap), np.float32)
            for i in range(nq):
                I[i, :cnt[i]] = ids[offs[i]:offs[i + 1]].view(np.int32)
                D[i, :cnt[i]] = d[offs[i]:offs[i + 1]]
            c6 = np.concatenate([ct.astype(np.int64), cdc.astype(np.int64)[:, None]], 1)
            return (torch.from_numpy(cnt.astype(np.int32)), torch.from_numpy(I), torch.from_numpy(D),
                    torch.from_numpy(c6))
        shd = ShardedIvfIndex(sh, searcher=lambda *a: None, merge=np_merge)
        offs, ids, d, c = shd.search_range(torch.from_numpy(qs), 3.0, 12, 0.35, range_searcher=rs, cap=512)
        results[rank] = (offs.numpy().copy(), ids.numpy().copy(), d.numpy().copy(), c.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_sharded_range_equals_single_run():
    """Range search is order-free: the merged shards equal the global run."""
    from oracle.oracle import COracle
    ix, qs, _ = goldens.load("ivf_fixture")
    h = host_index(IvfArrays.from_any(ix))
    offs, ids, d, ct, _ = COracle().search_range(h, qs, 3.0, 12, 0.35)
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_range_worker, args=(_free_port(), results), nprocs=WORLD, join=True)
    for r in range(WORLD):
        go, gi, gd, gc = results[r]
        np.testing.assert_array_equal(go, offs.astype(np.int64))
        np.testing.assert_array_equal(gi.astype(np.uint32), ids)
        np.testing.assert_array_equal(gd.view(np.uint32), d.view(np.uint32))
        # evaluated/dc/pruned sum over shards; edc = evaluated for range
        np.testing.assert_array_equal(gc[[0, 2, 3]], ct.sum(0)[[0, 2, 3]].astype(np.int64))
