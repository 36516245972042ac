"""Parity at BASELINE.json's full sizes (configs 2 and 4, the bench workloads
built on the device exactly as bench.py builds them): sampled queries through
the C ABI against the C restatement (oracle/trim_oracle.c) on the same index
bytes — ids, fp32 distances and per-query counters bit for bit — plus the
size-independent properties over a whole 1,024-query batch (accounting
identity, rows sorted by (dist, id), distances equal to the exact L2 of the
returned rows)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def _check(cfg_name, gammas, nsample, nprobe_override=None):
    import bench
    import torch
    from oracle.oracle import COracle
    from paper_2508_17828_b200 import ivf as G

    cfg = dict(bench.CONFIGS[cfg_name])
    cfg["nq"] = 1024
    arrays, queries = bench.build_workload(cfg, 0, 1, 0)
    gix = G.GpuIvfIndex(arrays, device=0)
    hix = bench._host_index(arrays)
    co = COracle()
    k, nprobe = cfg["k"], nprobe_override or cfg["nprobe"]
    q = queries.cpu().numpy()
    rows = np.linspace(0, len(q) - 1, nsample).astype(np.int64)
    for g in gammas:
        prof = G.PruningProfile.manual(g)
        ids, dist, ct = G.search_trim_ivf_knn_batch(gix, prof, q, k, nprobe)
        # the whole batch: sizes-independent properties
        assert (ct[:, 0] + ct[:, 2] == ct[:, 3]).all(), "dc + pruned != evaluated"
        d64 = dist.astype(np.float64)
        assert ((d64[:, 1:] > d64[:, :-1]) | ((d64[:, 1:] == d64[:, :-1]) & (ids[:, 1:] > ids[:, :-1]))).all()
        vec = arrays.vectors
        sel = torch.from_numpy(ids[rows].astype(np.int64).ravel()).to(vec.device)
        got_rows = vec[sel].cpu().numpy().reshape(len(rows), k, -1)
        for i, r in enumerate(rows):
            for j in range(k):
                assert co.euclidean_sq(q[r], got_rows[i, j]) == dist[r, j]
        # sampled queries: bit-exact against the oracle on the same bytes
        w_ids, w_d, w_ct, w_cdc = co.search_knn(hix, q[rows], k, nprobe, g)
        np.testing.assert_array_equal(ids[rows], w_ids)
        np.testing.assert_array_equal(_bits(dist[rows]), _bits(w_d))
        np.testing.assert_array_equal(ct[rows][:, :5], w_ct)
        np.testing.assert_array_equal(ct[rows][:, 5], w_cdc)
    del gix
    torch.cuda.empty_cache()


def test_config2_full_size_parity():
    """10M x 96, nlist 4096, nprobe 64, m = 48, k = 10, gamma in {0.6, 0.8, 1.0}."""
    _check("c2", [0.6, 0.8, 1.0], 12)


def test_config4_full_size_parity():
    """1M x 960 uniform + L2-normalised, flat, m = 120, k = 100, gamma in {0.5, 0.9}
    (the 16-warp filter CTA and the tcgen05 distance bounds)."""
    _check("c4", [0.5, 0.9], 4)


def test_config3_full_size_range_parity():
    """10M x 128 flat range search, m = 32, gamma = 0.8 and 0: the bench's
    calibrated radius (pick_radius_for_fraction, mean result ~100), through the
    block-partition path (99.6% of rows pruned as whole blocks) — sampled
    queries bit-exact against the oracle (members, distances, counters)."""
    import bench
    import torch
    from oracle.oracle import COracle
    from paper_2508_17828_b200 import ivf as G

    cfg = dict(bench.CONFIGS["c3"])
    cfg["nq"] = 256
    arrays, queries = bench.build_workload(cfg, 0, 1, 0)
    radius = bench.calibrate_radius(arrays, queries, cfg)
    gix = G.GpuIvfIndex(arrays, device=0)
    hix = bench._host_index(arrays)
    co = COracle()
    q = queries.cpu().numpy()
    rows = np.array([0, 85, 170, 255])
    for g in (0.8, 0.0):
        prof = G.PruningProfile.manual(g)
        offs, ids, dist, ct = G.search_trim_ivf_range_batch(gix, prof, q[rows], radius, 1)
        w_offs, w_ids, w_d, w_ct, w_cdc = co.search_range(hix, q[rows], radius, 1, g)
        np.testing.assert_array_equal(offs, w_offs)
        np.testing.assert_array_equal(ids, w_ids)
        np.testing.assert_array_equal(_bits(dist), _bits(w_d))
        np.testing.assert_array_equal(ct[:, :5], w_ct)
    assert gix.skipped_positions() > 0  # the block partition pruned whole blocks
    del gix
    torch.cuda.empty_cache()
