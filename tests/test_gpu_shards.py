"""Id-sharded search on one GPU: W shards of one index as
separate device indexes on cuda:0 (id_base != 0 for every shard but the
first), each checked against the reference run over that shard's candidate
subsequence (oracle/_ref), then merged with trim_merge_topk_device and checked
against the global answer (gamma = 0 with full probing: the exact kNN).

Shards whose share of a query's probed lists is shorter than k return their
partial top-k — every entry of the (short) stream, ascending (dist, id),
padded with (+inf, 0xFFFFFFFF) — with status bit 0 set; the merge ignores the
padding, so the merged answer still has k rows when the total stream does."""
import os

import numpy as np
import pytest

from tests import goldens

pytestmark = pytest.mark.gpu
INVALID = 0xFFFFFFFF


def _bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def _ref():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref is not built")
    r = O.RefOracle()
    r.set_threads(os.cpu_count() or 1)
    return r


def _search_shard(gix, q, k, nprobe, gamma):
    import torch

    from paper_2508_17828_b200 import ivf as G
    dq = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    cts = torch.zeros((q.shape[0], 6), dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ids, d = G.search_trim_ivf_knn_device(gix, G.PruningProfile.manual(gamma), dq, k, nprobe, d_counters=cts,
                                          d_status=st)
    torch.cuda.synchronize()
    return ids, d, cts, int(st.item())


def _check_sharded(full, qs, W, k, nprobe, gamma, ref, exact=None):
    """Per-shard parity vs the reference, merge, and (optionally) the exact kNN."""
    import torch

    from oracle.oracle import COracle, HostIndex
    from paper_2508_17828_b200 import ivf as G
    from paper_2508_17828_b200.distributed import merge_topk_device, shard_arrays
    co = COracle()
    vec_all = np.ascontiguousarray(full.vectors, np.float32)
    nq = qs.shape[0]
    g_ids, g_d, tot = [], [], np.zeros(nq, np.int64)
    for r in range(W):
        sh = shard_arrays(full, r, W)
        assert r == 0 or sh.id_base > 0
        gix = G.GpuIvfIndex(sh, device=0)
        ids, d, cts, st = _search_shard(gix, qs, k, nprobe, gamma)
        hi = ids.cpu().numpy().view(np.uint32)
        hd = d.cpu().numpy()
        ct = cts.cpu().numpy().astype(np.uint64)
        total = ct[:, 3].astype(np.int64)
        tot += total
        short = total < k
        assert bool(st & 1) == bool(short.any())
        # the reference over this shard (its VectorDataset is indexed by global id)
        h = HostIndex(dim=sh.dim, m=sh.m, ksub=sh.ksub, sub_dims=sh.sub_dims, centroids=sh.centroids,
                      coarse=sh.coarse, list_offsets=sh.list_offsets, list_ids=sh.list_ids,
                      list_codes=sh.list_codes, list_lx=sh.list_lx, vectors=vec_all)
        full_rows = np.nonzero(~short)[0]
        if full_rows.size:
            s = ref.session(h)
            try:
                w_ids, w_d, w_ct, w_cdc = ref.session_knn(s, qs[full_rows], k, nprobe, gamma)
            finally:
                ref.session_destroy(s)
            np.testing.assert_array_equal(hi[full_rows], w_ids)
            np.testing.assert_array_equal(_bits(hd[full_rows]), _bits(w_d))
            np.testing.assert_array_equal(ct[full_rows, :5], w_ct)
            np.testing.assert_array_equal(ct[full_rows, 5], w_cdc)
        # short streams: every entry is a seed (ivf.hpp:264-271), all evaluated
        for qi in np.nonzero(short)[0]:
            lists = co.probe_order(h, qs[qi], nprobe)
            offs = np.asarray(sh.list_offsets, np.int64)
            ent = np.concatenate([np.arange(offs[l], offs[l + 1]) for l in lists]) if len(lists) else []
            sid = np.asarray(sh.list_ids, np.uint32)[np.asarray(ent, np.int64)]
            sd = np.array([co.euclidean_sq(qs[qi], vec_all[i]) for i in sid], np.float32)
            order = sorted(zip(sd.tolist(), sid.tolist()))
            n = len(order)
            assert n == total[qi] < k
            assert hi[qi, :n].tolist() == [o[1] for o in order]
            assert hd[qi, :n].tolist() == [o[0] for o in order]
            assert (hi[qi, n:] == INVALID).all() and np.isinf(hd[qi, n:]).all()
            assert ct[qi, 0] == n and ct[qi, 2] == 0  # dc = seeds, nothing pruned
        g_ids.append(ids)
        g_d.append(d)
        gix.close()
    md, mi = merge_topk_device(torch.stack(g_d), torch.stack(g_ids), k)
    mi = mi.cpu().numpy().view(np.uint32)
    md = md.cpu().numpy()
    ok = tot >= k
    assert (mi[ok] != INVALID).all()
    if exact is not None:
        e_ids, e_d = exact
        np.testing.assert_array_equal(mi, e_ids)
        np.testing.assert_array_equal(_bits(md), _bits(e_d))
    return mi, md, tot


@pytest.mark.parametrize("W", [2, 4, 8])
def test_shards_of_fixture(W):
    """ivf_d96_m48 (3,000 rows, 32 lists): nprobe 1 leaves many shard streams
    shorter than k = 10; nprobe 32 (every list) at gamma 0 merges to the exact
    kNN (ground_truth_knn of the reference)."""
    from paper_2508_17828_b200 import ivf as G
    ref = _ref()
    ix, qs, _ = goldens.load("ivf_d96_m48")
    full = G.IvfArrays.from_any(ix)
    for nprobe, gamma in ((1, 0.8), (8, 0.8), (8, 0.0)):
        _check_sharded(full, qs, W, 10, nprobe, gamma, ref)
    e_ids, e_d = ref.ground_truth_knn(ix.vectors, qs, 10)
    _check_sharded(full, qs, W, 10, 32, 0.0, ref, exact=(e_ids, e_d))


def test_shards_of_device_built_index():
    """A device-built 200k x 96, nlist 256 index (config-2 shape, 1/50 scale),
    W in {2, 4}: per-shard parity at gamma 0.8 / nprobe 16; gamma 0 with every
    list probed merges to the reference's exact kNN."""
    import bench
    ref = _ref()
    cfg = dict(bench.CONFIGS["c2"])
    cfg.update(n=200_000, nlist=256, nq=64, nprobe=16)
    arrays, queries = bench.build_workload(cfg, 0, 1, 0)
    from paper_2508_17828_b200.builder import to_host
    full = to_host(arrays)
    qs = queries.cpu().numpy()
    e_ids, e_d = ref.ground_truth_knn(np.asarray(full.vectors, np.float32), qs, 10)
    for W in (2, 4):
        _check_sharded(full, qs, W, 10, 16, 0.8, ref)
        _check_sharded(full, qs, W, 10, 256, 0.0, ref, exact=(e_ids, e_d))
