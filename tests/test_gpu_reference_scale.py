"""Parity at BASELINE.json's full sizes against the REFERENCE ITSELF
(oracle/_ref: the unmodified reference headers compiled in place), on the same
index bytes the GPU searches.

  config 2  10M x 96, nlist 4096, nprobe 64, m 48, k 10: all 10,000 queries,
            gamma in {0.6, 0.8, 1.0}
  config 4  1M x 960 uniform + L2-normalised, flat, m 120, k 100: all 1,000
            queries, gamma in {0.5, 0.7, 0.9}
  config 3  10M x 128 flat range, m 32, the bench's calibrated radius: 1,000
            queries, gamma in {0.8, 0}
  config 5  one 100M x 96 flat shard, m 48, k 10 (the no-flat-bounds branch of
            knn_launch: > 16M rows): 64 queries, gamma 0.8

Every query: ids, fp32 distance bits and the six per-query counters
{dc, edc, pruned, evaluated, hops, coarse_dc} equal to ivf::search_trim_ivf_knn /
search_trim_ivf_range (ivf.hpp:243-347) run per query by the reference. Plus
the size-independent properties over whole batches (accounting identity, rows
sorted by (dist, id), returned distances equal to the exact L2 of the rows).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def _ref():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref (the reference compiled in place) is not built")
    r = O.RefOracle()
    r.set_threads(os.cpu_count() or 1)
    return r


class _Built:
    """A bench workload built on cuda:0, its host copy and a reference session."""

    def __init__(self, cfg_name, nq=None, n=None):
        import bench
        from paper_2508_17828_b200 import ivf as G

        cfg = dict(bench.CONFIGS[cfg_name])
        if nq:
            cfg["nq"] = nq
        if n:
            cfg["n"] = n
        self.cfg = cfg
        self.arrays, queries = bench.build_workload(cfg, 0, 1, 0)
        self.gix = G.GpuIvfIndex(self.arrays, device=0)
        self.hix = bench._host_index(self.arrays)
        self.q = queries.cpu().numpy()
        self.queries = queries
        self.ref = _ref()
        self.sess = self.ref.session(self.hix)

    def close(self):
        import torch
        self.ref.session_destroy(self.sess)
        self.gix.close()
        del self.arrays, self.hix
        torch.cuda.empty_cache()


def _props(b, ids, dist, ct, k, rows):
    """Whole-batch properties + exact distances of sampled rows."""
    import torch
    from oracle.oracle import COracle
    assert (ct[:, 0] + ct[:, 2] == ct[:, 3]).all(), "dc + pruned != evaluated"
    d64 = dist.astype(np.float64)
    assert ((d64[:, 1:] > d64[:, :-1]) | ((d64[:, 1:] == d64[:, :-1]) & (ids[:, 1:] > ids[:, :-1]))).all()
    co = COracle()
    vec = b.arrays.vectors
    sel = torch.from_numpy(ids[rows].astype(np.int64).ravel() - int(b.arrays.id_base)).to(vec.device)
    got = vec[sel].cpu().numpy().reshape(len(rows), k, -1)
    for i, r in enumerate(rows):
        for j in range(k):
            assert co.euclidean_sq(b.q[r], got[i, j]) == dist[r, j]


def _knn_vs_reference(b, gammas, nq):
    from paper_2508_17828_b200 import ivf as G
    k, nprobe = b.cfg["k"], b.cfg["nprobe"]
    q = b.q[:nq]
    for g in gammas:
        ids, dist, ct = G.search_trim_ivf_knn_batch(b.gix, G.PruningProfile.manual(g), q, k, nprobe)
        w_ids, w_d, w_ct, w_cdc = b.ref.session_knn(b.sess, q, k, nprobe, g)
        bad = np.nonzero((ids != w_ids).any(1) | (_bits(dist) != _bits(w_d)).any(1) |
                         (ct[:, :5] != w_ct).any(1) | (ct[:, 5] != w_cdc))[0]
        assert bad.size == 0, (f"gamma={g}: {bad.size} of {nq} queries differ from the reference "
                               f"(first {bad[:5].tolist()})")
        _props(b, ids, dist, ct, k, np.linspace(0, nq - 1, 8).astype(np.int64))


def test_config2_all_queries_vs_reference():
    """Config 2, all 10,000 queries, gamma 0.6 / 0.8 / 1.0 (3 x 10k queries)."""
    b = _Built("c2")
    try:
        assert b.q.shape[0] == 10_000
        _knn_vs_reference(b, [0.6, 0.8, 1.0], 10_000)
    finally:
        b.close()


def test_config4_all_queries_vs_reference():
    """Config 4, all 1,000 queries at gamma 0.5 / 0.7 / 0.9 (the 16-warp CTA and
    the tcgen05 flat distance bounds; nothing is pruned at gamma <= 0.7)."""
    b = _Built("c4")
    try:
        assert b.q.shape[0] == 1000
        _knn_vs_reference(b, [0.5, 0.7, 0.9], 1000)
    finally:
        b.close()


def test_config3_range_vs_reference():
    """Config 3, 1,000 of the 10,000 queries at the calibrated radius (mean
    result ~100 at gamma 0), gamma 0.8 and 0: members, distances, counters."""
    import bench
    from paper_2508_17828_b200 import ivf as G
    b = _Built("c3")
    try:
        radius = bench.calibrate_radius(b.arrays.vectors, b.queries, b.cfg)
        q = b.q[:1000]
        for g in (0.8, 0.0):
            offs, ids, dist, ct = G.search_trim_ivf_range_batch(b.gix, G.PruningProfile.manual(g), q, radius, 1)
            w_offs, w_ids, w_d, w_ct, w_cdc = b.ref.session_range(b.sess, q, radius, 1, g)
            np.testing.assert_array_equal(offs, w_offs)
            np.testing.assert_array_equal(ids, w_ids)
            np.testing.assert_array_equal(_bits(dist), _bits(w_d))
            np.testing.assert_array_equal(ct[:, :5], w_ct)
            np.testing.assert_array_equal(ct[:, 5], w_cdc)
            if g == 0.0:
                assert 20 < float(np.diff(offs).mean()) < 500  # the calibrated ~100
        assert b.gix.skipped_positions() > 0  # the block partition pruned whole blocks
    finally:
        b.close()


def test_config5_shard_vs_reference():
    """One 100M-row shard of config 5 (flat, > 16M rows: no tensor-core
    distance bounds), 64 queries at gamma 0.8."""
    b = _Built("c5", nq=64)
    try:
        _knn_vs_reference(b, [0.8], 64)
    finally:
        b.close()
