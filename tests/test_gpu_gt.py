"""Exact brute-force ground truth on the GPU (trim_ground_truth_knn: tcgen05
distance bounds + exact fp32 re-ranking) against the reference's own
ground_truth_knn (core/ground_truth.hpp:53-113), bit for bit, including the
massive-tie fallback and the reference's argument errors."""
import numpy as np
import pytest

from oracle.oracle import RefOracle, ref_available
from paper_2508_17828_b200 import ivf as G
from tests import goldens

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


def check(gix, x, qs, k):
    want_i, want_d = RefOracle().ground_truth_knn(x, qs, k)
    got_i, got_d = G.ground_truth_knn(gix, qs, k)
    np.testing.assert_array_equal(got_i, want_i)
    np.testing.assert_array_equal(got_d.view(np.uint32), np.asarray(want_d, np.float32).view(np.uint32))


@pytest.mark.parametrize("name", goldens.names())
@pytest.mark.parametrize("k", [1, 10, 100])
def test_gt_matches_reference(name, k):
    ix, qs, _ = goldens.load(name)
    gix = G.GpuIvfIndex(G.IvfArrays.from_any(ix))
    check(gix, np.asarray(ix.vectors, np.float32), qs, k)


def test_gt_ties_fallback():
    # 40 distinct rows repeated 150 times: > 4096 rows tie at the k-th distance
    rng = np.random.default_rng(7)
    base = rng.standard_normal((40, 24)).astype(np.float32)
    x = np.tile(base, (150, 1))
    n = x.shape[0]
    arr = G.IvfArrays(dim=24, m=4, ksub=256, sub_dims=np.full(4, 6, np.uint32),
                      centroids=rng.standard_normal((256, 24)).astype(np.float32), coarse=x.mean(0)[None],
                      list_offsets=np.array([0, n], np.uint64), list_ids=np.arange(n, dtype=np.uint32),
                      list_codes=np.zeros((n, 4), np.uint8), list_lx=np.zeros(n, np.float32), vectors=x)
    gix = G.GpuIvfIndex(arr)
    check(gix, x, np.concatenate([base[:3], rng.standard_normal((3, 24)).astype(np.float32)]), 300)


def test_gt_errors():
    ix, qs, _ = goldens.load("ivf_fixture")
    gix = G.GpuIvfIndex(G.IvfArrays.from_any(ix))
    with pytest.raises(G.InvalidArgument, match="k out of range"):
        G.ground_truth_knn(gix, qs, 0)
    with pytest.raises(G.InvalidArgument, match="k out of range"):
        G.ground_truth_knn(gix, qs, ix.vectors.shape[0] + 1)
