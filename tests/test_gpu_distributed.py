"""GPU side of the multi-GPU path: the device merge kernel after the
all-gather (trim_merge_topk_device) against a plain sort by (dist, id), and
ShardedIvfIndex (kNN and range) over a 1-rank NCCL group equal to the
single-GPU search."""
import os
import socket

import numpy as np
import pytest

from tests import goldens

pytestmark = pytest.mark.gpu


def test_merge_kernel_matches_sort():
    import torch

    from paper_2508_17828_b200.distributed import merge_topk_device
    rng = np.random.default_rng(3)
    for w, nq, k in ((2, 7, 10), (8, 33, 10), (4, 5, 100), (3, 4, 1)):
        d = rng.integers(0, 50, size=(w, nq, k)).astype(np.float32)  # many ties
        ids = rng.permutation(w * nq * k).reshape(w, nq, k).astype(np.uint32)
        ids[0, 0, -1] = 0xFFFFFFFF  # an invalid entry is ignored
        md, mi = merge_topk_device(torch.from_numpy(d).cuda(), torch.from_numpy(ids.view(np.int32)).cuda(), k)
        md, mi = md.cpu().numpy(), mi.cpu().numpy().view(np.uint32)
        for q in range(nq):
            cand = sorted((float(d[s, q, j]), int(ids[s, q, j])) for s in range(w) for j in range(k)
                          if ids[s, q, j] != 0xFFFFFFFF)[:k]
            assert [c[1] for c in cand] == mi[q].tolist()
            assert [c[0] for c in cand] == md[q].tolist()


def test_sharded_index_one_rank_nccl():
    import torch
    import torch.distributed as dist

    from paper_2508_17828_b200 import ivf as G
    from paper_2508_17828_b200.distributed import ShardedIvfIndex, shard_arrays
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        ix, qs, _ = goldens.load("ivf_d96_m48")
        full = G.IvfArrays.from_any(ix)
        sh = ShardedIvfIndex(shard_arrays(full, 0, 1))
        q = torch.from_numpy(np.ascontiguousarray(qs)).cuda()
        mi, md, c = sh.search_knn(q, 10, 8, 0.8)
        ids, d, ct = G.search_trim_ivf_knn_batch(G.GpuIvfIndex(full), G.PruningProfile.manual(0.8), qs, 10, 8)
        np.testing.assert_array_equal(mi.cpu().numpy().view(np.uint32), ids)
        np.testing.assert_array_equal(md.cpu().numpy().view(np.uint32), d.view(np.uint32))
        np.testing.assert_array_equal(c.cpu().numpy(), ct[:, :5].sum(0).astype(np.int64))
        # range through the padded all-gather + merge (device range API per rank)
        ix2, qs2, _ = goldens.load("ivf_fixture")
        full2 = G.IvfArrays.from_any(ix2)
        sh2 = ShardedIvfIndex(shard_arrays(full2, 0, 1))
        q2 = torch.from_numpy(np.ascontiguousarray(qs2)).cuda()
        r = torch.full((q2.shape[0],), 3.0, dtype=torch.float32, device="cuda")
        offs, rid, rd, rc = sh2.search_range(q2, r, 12, 0.35)
        wo, wi, wd, wct = G.search_trim_ivf_range_batch(G.GpuIvfIndex(full2), G.PruningProfile.manual(0.35), qs2,
                                                        3.0, 12)
        np.testing.assert_array_equal(offs.cpu().numpy(), wo.astype(np.int64))
        np.testing.assert_array_equal(rid.cpu().numpy().astype(np.uint32), wi)
        np.testing.assert_array_equal(rd.cpu().numpy().view(np.uint32), wd.view(np.uint32))
    finally:
        dist.destroy_process_group()
