"""Flat kNN over the segmented block stream (trim_knn_seg_plan_kernel +
trim_knn_kernel<SEG>): ivf::search_trim_ivf_knn with nlist = 1
(ivf.hpp:243-304) when the index carries a block partition.

The rows after the first n0 are regrouped by (segment of consecutive ids,
block); blocks whose list-level bound is >= the threshold after n0 rows are
never read and each segment's kept rows are merged back into ascending-id order,
so ids, distance bits and every counter must equal the reference's sequential scan.
The layout is forced on a small clustered index (the default needs >= 256k
rows) with short segments, so a query's kept blocks interleave in id order in
every segment.

Bar: bit-identical to the C oracle (pinned to the reference by
tests/test_oracle.py) and to the in-order GPU scan (TRIM_FLAT_SEGMENTS=0)."""
import numpy as np
import pytest

from oracle.oracle import COracle, RefOracle, make_reference_index, ref_available
from paper_2508_17828_b200 import ivf as G

pytestmark = pytest.mark.gpu
co = COracle()


def assert_bits(a, b):
    np.testing.assert_array_equal(np.asarray(a, np.float32).view(np.uint32),
                                  np.asarray(b, np.float32).view(np.uint32))


@pytest.fixture(scope="module")
def flat():
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    ref = RefOracle()
    centers = ref.make_normal(32, 64, 31)
    base = ref.make_blobs(centers, 70000, 0.3, 32)
    qs = ref.make_blobs(centers, 41, 0.3, 33)
    qs[5] = 40.0  # far from every block: the threshold after n0 rows prunes nothing
    hix = make_reference_index(ref, base, m=32, c=256, iters=8, pq_seed=34, nlist=1, ivf_seed=35)
    return hix, qs


def seg_index(hix, monkeypatch, rows_per_block="16", n0="4000"):
    monkeypatch.setenv("TRIM_FLAT_PARTITION_MIN_ROWS", "1000")
    monkeypatch.setenv("TRIM_SEG_ROWS_PER_BLOCK", rows_per_block)
    monkeypatch.setenv("TRIM_SEG_N0", n0)
    return G.GpuIvfIndex(G.IvfArrays.from_any(hix))  # the layout is built on the first kNN call


def check(got, want):
    np.testing.assert_array_equal(got[0], want[0])
    assert_bits(got[1], want[1])
    np.testing.assert_array_equal(got[2][:, :5], want[2])


@pytest.mark.parametrize("gamma", [0.0, 0.5, 0.8, 1.0])
@pytest.mark.parametrize("k", [1, 10, 100])
def test_segmented_flat_knn_parity(flat, gamma, k, monkeypatch):
    hix, qs = flat
    gix = seg_index(hix, monkeypatch)
    want = co.search_knn(hix, qs, k, 1, gamma)
    gix.skipped_positions(reset=True)
    got = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(gamma), qs, k, 1)
    check(got, want)
    # the block stream really ran: whole blocks were pruned without being read
    assert gix.skipped_positions() > 0


@pytest.mark.parametrize("mode", ["wide_interval", "no_flat_bounds", "force_plain", "long_segments", "big_n0",
                                  "no_rounds", "tiny_n0"])
@pytest.mark.parametrize("gamma", [0.0, 0.8])
def test_segmented_flat_knn_modes(flat, gamma, mode, monkeypatch):
    hix, qs = flat
    kw = {}
    if mode == "wide_interval":  # every member's est interval straddles: the reference-order ADC decides
        monkeypatch.setenv("TRIM_EPS_SCALE", "20000")
    if mode == "no_flat_bounds":
        monkeypatch.setenv("TRIM_FLAT_BOUNDS", "0")
    if mode == "force_plain":  # no plan ever fits: continue rounds, then row order for the rest
        monkeypatch.setenv("TRIM_SEG_FORCE_PLAIN", "1")
    if mode == "long_segments":  # many rows per (segment, block) run
        kw = dict(rows_per_block="128", n0="2000")
    if mode == "no_rounds":  # a plan that does not fit resumes in order at once
        monkeypatch.setenv("TRIM_SEG_ROUNDS", "0")
    if mode == "tiny_n0":  # too few rows in order for a useful threshold: continue rounds, then planned
        kw = dict(rows_per_block="16", n0="300")
    if mode == "big_n0":
        kw = dict(rows_per_block="7", n0="17000")
    gix = seg_index(hix, monkeypatch, **kw)
    want = co.search_knn(hix, qs, 10, 1, gamma)
    got = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(gamma), qs, 10, 1)
    check(got, want)


def test_segmented_flat_knn_large_k(flat, monkeypatch):
    """k > 256 (shared-memory top-k) through the segmented stream."""
    hix, qs = flat
    gix = seg_index(hix, monkeypatch)
    want = co.search_knn(hix, qs[:9], 300, 1, 0.8)
    got = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(0.8), qs[:9], 300, 1)
    check(got, want)


def test_segmented_equals_in_order_scan(flat, monkeypatch):
    hix, qs = flat
    gix = seg_index(hix, monkeypatch)
    a = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(0.8), qs, 10, 1)
    monkeypatch.setenv("TRIM_FLAT_SEGMENTS", "0")
    gix2 = G.GpuIvfIndex(G.IvfArrays.from_any(hix))
    b = G.search_trim_ivf_knn_batch(gix2, G.PruningProfile.manual(0.8), qs, 10, 1)
    np.testing.assert_array_equal(a[0], b[0])
    assert_bits(a[1], b[1])
    np.testing.assert_array_equal(a[2], b[2])
