"""Multi-device indexes behind the C ABI (include/trim_gpu.h trim_shard_mode;
trim_multi.cu), on the one GPU this box has:

  id_shard over devices [0]          the NCCL path: a 1-rank communicator
                                     (broadcast + all-gather + device merge);
                                     one shard = the whole index, so results and
                                     counters equal the single-device call
  id_shard over devices [0, 0, ...]  W shards on cuda:0 (id_base != 0): the
                                     exchange by device copies; equal to W
                                     separate shard indexes merged by
                                     trim_merge_topk_device (whose per-shard
                                     parity with the reference is pinned by
                                     tests/test_gpu_shards.py), counters summed;
                                     gamma = 0 with every list probed = the exact
                                     kNN; range = the single run exactly
  replicas over devices [0, 0, 0]    query slices: every search equals the
                                     single-device call
"""
import os

import numpy as np
import pytest

from tests import goldens

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def _fixture():
    from paper_2508_17828_b200 import ivf as G
    ix, qs, _ = goldens.load("ivf_d96_m48")
    return ix, G.IvfArrays.from_any(ix), np.ascontiguousarray(qs)


def _manual_shards(full, qs, W, k, nprobe, gamma):
    """W single-device shard indexes, each searched, merged on the device."""
    import torch

    from paper_2508_17828_b200 import ivf as G
    from paper_2508_17828_b200.distributed import merge_topk_device, shard_arrays
    ids, dist, cts = [], [], []
    dq = torch.from_numpy(qs).cuda()
    for r in range(W):
        gix = G.GpuIvfIndex(shard_arrays(full, r, W), device=0)
        ct = torch.zeros((qs.shape[0], 6), dtype=torch.int64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        i, d = G.search_trim_ivf_knn_device(gix, G.PruningProfile.manual(gamma), dq, k, nprobe, d_counters=ct,
                                            d_status=st)
        torch.cuda.synchronize()
        ids.append(i)
        dist.append(d)
        cts.append(ct.cpu().numpy())
        gix.close()
    md, mi = merge_topk_device(torch.stack(dist), torch.stack(ids), k)
    c = np.sum(cts, axis=0)
    c[:, 5] = cts[0][:, 5]
    return mi.cpu().numpy().view(np.uint32), md.cpu().numpy(), c.astype(np.uint64)


@pytest.mark.parametrize("W", [2, 3, 4])
def test_id_shard_copies_equal_manual_shards(W):
    from paper_2508_17828_b200 import ivf as G
    ix, full, qs = _fixture()
    g = G.GpuIvfIndex(full, devices=[0] * W, shard_mode="id_shard")
    info = g.info()
    assert info["ndevices"] == W and info["shard_mode"] == 1 and info["nccl"] == 0
    for nprobe, gamma in ((4, 0.8), (8, 0.6), (32, 0.0)):
        ids, dist, ct = G.search_trim_ivf_knn_batch(g, G.PruningProfile.manual(gamma), qs, 10, nprobe)
        w_ids, w_d, w_ct = _manual_shards(full, qs, W, 10, nprobe, gamma)
        np.testing.assert_array_equal(ids, w_ids)
        np.testing.assert_array_equal(_bits(dist), _bits(w_d))
        np.testing.assert_array_equal(ct, w_ct)
    # gamma = 0, every list probed: the exact kNN (the reference's ground_truth_knn)
    from oracle import oracle as O
    if O.ref_available():
        e_ids, e_d = O.RefOracle().ground_truth_knn(ix.vectors, qs, 10)
        ids, dist, _ = G.search_trim_ivf_knn_batch(g, G.PruningProfile.manual(0.0), qs, 10, 32)
        np.testing.assert_array_equal(ids, e_ids)
        np.testing.assert_array_equal(_bits(dist), _bits(e_d))
    g.close()


def test_id_shard_nccl_one_device_equals_single():
    """devices = [0]: the NCCL communicator path at W = 1."""
    import torch

    from paper_2508_17828_b200 import ivf as G
    _, full, qs = _fixture()
    g = G.GpuIvfIndex(full, devices=[0], shard_mode="id_shard")
    assert g.info()["nccl"] == 1
    s = G.GpuIvfIndex(full, device=0)
    for nprobe, gamma in ((8, 0.8), (32, 0.0), (2, 1.0)):
        a = G.search_trim_ivf_knn_batch(g, G.PruningProfile.manual(gamma), qs, 10, nprobe)
        b = G.search_trim_ivf_knn_batch(s, G.PruningProfile.manual(gamma), qs, 10, nprobe)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(_bits(a[1]), _bits(b[1]))
        np.testing.assert_array_equal(a[2], b[2])
    # the device-resident call on a group index (queries / results on the home device)
    dq = torch.from_numpy(qs).cuda()
    ct = torch.zeros((qs.shape[0], 6), dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    i, d = G.search_trim_ivf_knn_device(g, G.PruningProfile.manual(0.8), dq, 10, 8, d_counters=ct, d_status=st)
    b = G.search_trim_ivf_knn_batch(s, G.PruningProfile.manual(0.8), qs, 10, 8)
    np.testing.assert_array_equal(i.cpu().numpy().view(np.uint32), b[0])
    np.testing.assert_array_equal(ct.cpu().numpy().astype(np.uint64), b[2])
    assert int(st.item()) == 0
    g.close()
    s.close()


def test_id_shard_k_exceeds_total_stream():
    """Shards shorter than k are fine while the total stream holds k entries;
    a query whose whole probed stream is shorter than k is the reference's
    invalid_argument (ivf.hpp:289-290)."""
    from paper_2508_17828_b200 import ivf as G
    from paper_2508_17828_b200._lib import InvalidArgument
    _, full, qs = _fixture()
    g = G.GpuIvfIndex(full, devices=[0] * 8, shard_mode="id_shard")
    ids, _, ct = G.search_trim_ivf_knn_batch(g, G.PruningProfile.manual(0.8), qs, 10, 1)
    assert (ct[:, 3] >= 10).all() and (ids != 0xFFFFFFFF).all()
    biggest = int(np.diff(np.asarray(full.list_offsets, np.int64)).max())
    with pytest.raises(InvalidArgument):
        G.search_trim_ivf_knn_batch(g, G.PruningProfile.manual(0.8), qs, biggest + 1, 1)
    with pytest.raises(InvalidArgument):  # the refine pool needs the whole stream on one device
        G.search_baseline_ivfpq_batch(g, qs, 10, 8, 100)
    g.close()


def test_id_shard_range_equals_single():
    """Range search has no running state: the union over the shards is the
    single run (members, distances, counters) — copies (W = 3) and NCCL (W = 1)."""
    from paper_2508_17828_b200 import ivf as G
    ix, qs, _ = goldens.load("ivf_fixture")
    full = G.IvfArrays.from_any(ix)
    s = G.GpuIvfIndex(full, device=0)
    for devs in ([0, 0, 0], [0]):
        g = G.GpuIvfIndex(full, devices=devs, shard_mode="id_shard")
        for r, nprobe, gamma in ((3.0, 12, 0.35), (2.0, 20, 0.0), (4.0, 5, 1.0)):
            a = G.search_trim_ivf_range_batch(g, G.PruningProfile.manual(gamma), qs, r, nprobe)
            b = G.search_trim_ivf_range_batch(s, G.PruningProfile.manual(gamma), qs, r, nprobe)
            np.testing.assert_array_equal(a[0], b[0])
            np.testing.assert_array_equal(a[1], b[1])
            np.testing.assert_array_equal(_bits(a[2]), _bits(b[2]))
            np.testing.assert_array_equal(a[3], b[3])
        g.close()
    s.close()


def test_replicas_equal_single():
    from paper_2508_17828_b200 import ivf as G
    _, full, qs = _fixture()
    s = G.GpuIvfIndex(full, device=0)
    g = G.GpuIvfIndex(full, devices=[0, 0, 0], shard_mode="replicas")
    assert g.info()["ndevices"] == 3 and g.info()["shard_mode"] == 2
    prof = G.PruningProfile.manual(0.8)
    for a, b in ((G.search_trim_ivf_knn_batch(g, prof, qs, 10, 8), G.search_trim_ivf_knn_batch(s, prof, qs, 10, 8)),
                 (G.search_baseline_ivfpq_batch(g, qs, 10, 8, 100), G.search_baseline_ivfpq_batch(s, qs, 10, 8, 100))):
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(_bits(a[1]), _bits(b[1]))
        np.testing.assert_array_equal(a[2], b[2])
    a = G.search_trim_ivf_range_batch(g, prof, qs, 6.0, 8)
    b = G.search_trim_ivf_range_batch(s, prof, qs, 6.0, 8)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    g.close()
    s.close()


def test_id_shard_device_built_index_vs_reference_shards():
    """Device arrays (a 200k x 96, nlist 256 config-2-shaped build) into a
    4-shard index on cuda:0: merged results equal the manual shard merge and,
    at gamma = 0 with every list probed, the reference's exact kNN."""
    import bench

    from paper_2508_17828_b200 import ivf as G
    from paper_2508_17828_b200.builder import to_host
    cfg = dict(bench.CONFIGS["c2"])
    cfg.update(n=200_000, nlist=256, nq=64, nprobe=16)
    arrays, queries = bench.build_workload(cfg, 0, 1, 0)
    g = G.GpuIvfIndex(arrays, devices=[0, 0, 0, 0], shard_mode="id_shard")  # device-memory descriptor
    full = to_host(arrays)
    qs = queries.cpu().numpy()
    ids, dist, ct = G.search_trim_ivf_knn_batch(g, G.PruningProfile.manual(0.8), qs, 10, 16)
    w_ids, w_d, w_ct = _manual_shards(full, qs, 4, 10, 16, 0.8)
    np.testing.assert_array_equal(ids, w_ids)
    np.testing.assert_array_equal(_bits(dist), _bits(w_d))
    np.testing.assert_array_equal(ct, w_ct)
    from oracle import oracle as O
    if O.ref_available():
        e_ids, e_d = O.RefOracle().ground_truth_knn(np.asarray(full.vectors, np.float32), qs, 10)
        ids, dist, _ = G.search_trim_ivf_knn_batch(g, G.PruningProfile.manual(0.0), qs, 10, 256)
        np.testing.assert_array_equal(ids, e_ids)
        np.testing.assert_array_equal(_bits(dist), _bits(e_d))
    g.close()
