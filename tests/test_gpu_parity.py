"""GPU parity: the sm_100a path through the C ABI vs the reference.

Bar (BASELINE.json north_star): identical ids, bit-identical
fp32 dist_sq, identical per-query counters {dc, edc, pruned, evaluated, hops}
and coarse_dc. All checks below are exact equality (tolerance 0).

* golden fixtures: outputs of the reference itself (tests/golden/);
* larger seeded cases: the C restatement (oracle/trim_oracle.c), itself
  pinned to the reference by tests/test_oracle.py;
* edge cases mirroring proj/tests/test_ivf.cpp.
"""
import numpy as np
import pytest

from oracle.oracle import COracle, RefOracle, make_reference_index, ref_available
from paper_2508_17828_b200 import ivf as G
from tests import goldens

pytestmark = pytest.mark.gpu
co = COracle()

_IX = {}


def gpu_index(name):
    if name not in _IX:
        ix, qs, cases = goldens.load(name)
        _IX[name] = (G.GpuIvfIndex(G.IvfArrays.from_any(ix)), ix, qs, cases)
    return _IX[name]


def assert_bits(a, b):
    np.testing.assert_array_equal(np.asarray(a, np.float32).view(np.uint32),
                                  np.asarray(b, np.float32).view(np.uint32))


# TRIM_EPS_SCALE widens the any-order ADC interval, so most members are
# decided by the reference-order fallback (adc_serial) instead of the interval
# — the rare path must be exact too.
@pytest.fixture(params=["default", "wide_interval", "no_flat_bounds"])
def filter_mode(request, monkeypatch):
    if request.param == "wide_interval":
        monkeypatch.setenv("TRIM_EPS_SCALE", "20000")
    if request.param == "no_flat_bounds":  # flat kNN without the tensor-core distance bounds
        monkeypatch.setenv("TRIM_FLAT_BOUNDS", "0")
    return request.param


@pytest.mark.parametrize("name,case", goldens.all_cases())
def test_gpu_matches_reference_goldens(name, case, filter_mode):
    gix, ix, qs, cases = gpu_index(name)
    c = cases[case]
    if c["kind"] == "knn":
        ids, dist, ct = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(c["gamma"]), qs,
                                                    c["k"], c["nprobe"])
        np.testing.assert_array_equal(ids, c["ids"])
        assert_bits(dist, c["dist"])
    elif c["kind"] == "range":
        offs, ids, dist, ct = G.search_trim_ivf_range_batch(
            gix, G.PruningProfile.manual(c["gamma"]), qs, c["radius"], c["nprobe"])
        np.testing.assert_array_equal(offs, c["offsets"])
        np.testing.assert_array_equal(ids, c["ids"])
        assert_bits(dist, c["dist"])
    else:
        ids, dist, ct = G.search_baseline_ivfpq_batch(gix, qs, c["k"], c["nprobe"], c["k_prime"])
        np.testing.assert_array_equal(ids, c["ids"])
        assert_bits(dist, c["dist"])
    np.testing.assert_array_equal(ct[:, :5], c["counters"])
    np.testing.assert_array_equal(ct[:, 5], c["coarse_dc"])


@pytest.mark.parametrize("name", goldens.names())
def test_lut_bit_exact(name):
    # pq::build_distance_table (pq.hpp:158-172); test_pq.cpp:210-216 pins
    # exact equality of table entries with euclidean_sq.
    gix, ix, qs, _ = gpu_index(name)
    lut = G.build_distance_table(gix, qs)
    hix = goldens.host_index(ix)
    for i in range(len(qs)):
        assert_bits(lut[i], co.distance_table(hix, qs[i]))


@pytest.mark.parametrize("name", goldens.names())
def test_probe_order_exact(name):
    gix, ix, qs, _ = gpu_index(name)
    hix = goldens.host_index(ix)
    for npb in (1, 3, hix.nlist):
        got = G.probe_order(gix, qs, npb)
        for i in range(len(qs)):
            np.testing.assert_array_equal(got[i], co.probe_order(hix, qs[i], npb))


def test_per_query_signature_matches_batch():
    gix, ix, qs, cases = gpu_index("ivf_fixture")
    prof = G.PruningProfile.manual(0.35)
    ids, dist, ct = G.search_trim_ivf_knn_batch(gix, prof, qs, 10, 5)
    for i in range(3):
        r = G.search_trim_ivf_knn(gix, prof, qs[i], 10, 5)
        np.testing.assert_array_equal(r.ids, ids[i])
        assert r.counters.dc + r.counters.pruned == r.counters.evaluated
        assert r.coarse_dc == gix.nlist


# ------------------------------------------------------------ edge cases
def test_errors_match_reference_semantics():
    gix, ix, qs, _ = gpu_index("ivf_fixture")
    prof = G.PruningProfile.manual(0.35)
    with pytest.raises(G.InvalidArgument, match="k must be positive"):
        G.search_trim_ivf_knn(gix, prof, qs[0], 0, 2)
    with pytest.raises(G.InvalidArgument, match="uncalibrated"):
        G.search_trim_ivf_knn(gix, G.PruningProfile(), qs[0], 5, 2)
    with pytest.raises(G.InvalidArgument, match="k exceeds probed"):
        G.search_trim_ivf_knn(gix, prof, qs[0], 200, 1)
    with pytest.raises(G.InvalidArgument, match="k exceeds probed"):
        G.search_trim_ivf_knn(gix, prof, qs[0], 5, 0)
    with pytest.raises(G.InvalidArgument, match="negative radius"):
        G.search_trim_ivf_range(gix, prof, qs[0], -1.0, 2)
    with pytest.raises(G.InvalidArgument, match="uncalibrated"):
        G.search_trim_ivf_range(gix, G.PruningProfile(), qs[0], 1.0, 2)
    with pytest.raises(G.InvalidArgument, match="k <= k_prime"):
        G.search_baseline_ivfpq(gix, qs[0], 10, 4, 5)
    with pytest.raises(G.InvalidArgument, match="nprobe must be positive"):
        G.search_baseline_ivfpq(gix, qs[0], 10, 0, 50)


def test_radius_zero_off_dataset_is_empty():
    gix, ix, qs, _ = gpu_index("ivf_fixture")
    r = G.search_trim_ivf_range(gix, G.PruningProfile.manual(0.35), qs[0] + 100.0, 0.0, gix.nlist)
    assert r.ids.size == 0


def test_range_members_are_verified_exact():
    # test_ivf.cpp:266-291: returned members satisfy d <= r^2 and dist_sq == euclidean_sq
    gix, ix, qs, _ = gpu_index("ivf_fixture")
    offs, ids, dist, ct = G.search_trim_ivf_range_batch(gix, G.PruningProfile.manual(0.35), qs,
                                                        3.0, 12)
    v = ix.vectors
    for i in range(len(qs)):
        for j in range(int(offs[i]), int(offs[i + 1])):
            d = co.euclidean_sq(qs[i], v[ids[j]])
            assert d <= np.float32(3.0) * np.float32(3.0)
            assert np.float32(d) == dist[j]
    assert (ct[:, 0] + ct[:, 2] == ct[:, 3]).all()


def test_empty_batch_and_empty_lists():
    gix, ix, qs, _ = gpu_index("ivf_fixture")
    ids, dist, ct = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(0.0),
                                                np.zeros((0, gix.dim), np.float32), 5, 2)
    assert ids.shape == (0, 5)
    # index with empty lists interleaved: split list 0 into [empty, list0, empty]
    offs = ix.list_offsets.astype(np.uint64)
    new_offs = np.concatenate([[0], [0], offs[1:2], offs[1:2], offs[2:]]).astype(np.uint64)
    coarse = ix.coarse.reshape(ix.list_offsets.size - 1, ix.dim)
    far = np.full((1, ix.dim), 1e3, np.float32)
    new_coarse = np.concatenate([far, coarse[:1], far, coarse[1:]])
    arr = G.IvfArrays.from_any(ix)
    arr.coarse = new_coarse
    arr.list_offsets = new_offs
    g2 = G.GpuIvfIndex(arr)
    from oracle.oracle import HostIndex
    h2 = HostIndex(**{f: getattr(arr, f) for f in goldens.FIELDS})
    for g in (0.0, 0.5):
        for npb in (1, 5, h2.nlist):
            want = co.search_knn(h2, qs, 3, npb, g) if npb > 1 else None
            if want is None:
                continue
            got = G.search_trim_ivf_knn_batch(g2, G.PruningProfile.manual(g), qs, 3, npb)
            np.testing.assert_array_equal(got[0], want[0])
            np.testing.assert_array_equal(got[2][:, :5], want[2])


def test_singleton_lists_many_segments():
    # nlist = n-ish: every chunk spans > 32 lists (segment-table truncation path)
    gix, ix, qs, _ = gpu_index("ivf_fixture")
    n = ix.vectors.shape[0]
    order = np.argsort(ix.list_ids, kind="stable")
    arr = G.IvfArrays.from_any(ix)
    nl = 500
    # 500 lists of 2 consecutive ids each, coarse = mean of the pair
    ids = np.arange(n, dtype=np.uint32)
    codes = ix.list_codes[order]
    lx = ix.list_lx[order]
    vec = ix.vectors
    arr.list_ids = ids
    arr.list_codes = codes
    arr.list_lx = lx
    arr.list_offsets = (np.arange(nl + 1, dtype=np.uint64) * 2)
    arr.coarse = vec.reshape(nl, 2, ix.dim).mean(1).astype(np.float32)
    g2 = G.GpuIvfIndex(arr)
    from oracle.oracle import HostIndex
    h2 = HostIndex(**{f: getattr(arr, f) for f in goldens.FIELDS})
    for g in (0.0, 0.35, 1.0):
        for npb in (40, 300):
            want = co.search_knn(h2, qs, 10, npb, g)
            got = G.search_trim_ivf_knn_batch(g2, G.PruningProfile.manual(g), qs, 10, npb)
            np.testing.assert_array_equal(got[0], want[0])
            assert_bits(got[1], want[1])
            np.testing.assert_array_equal(got[2][:, :5], want[2])
        want = co.search_range(h2, qs, 3.0, 300, g)
        got = G.search_trim_ivf_range_batch(g2, G.PruningProfile.manual(g), qs, 3.0, 300)
        np.testing.assert_array_equal(got[0], want[0])
        np.testing.assert_array_equal(got[1], want[1])
        np.testing.assert_array_equal(got[3][:, :5], want[3])


# ------------------------------------------------ full config-1 (configs[0])
@pytest.fixture(scope="module")
def config1():
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    ref = RefOracle()
    centers = ref.make_normal(64, 128, 0)
    base = ref.make_blobs(centers, 100000, 0.3, 1)
    qs = ref.make_blobs(centers, 1000, 0.3, 2)
    hix = make_reference_index(ref, base, m=16, c=256, iters=25, pq_seed=3, nlist=1, ivf_seed=4)
    return hix, qs, G.GpuIvfIndex(G.IvfArrays.from_any(hix))


@pytest.mark.parametrize("gamma", [0.0, 0.605, 1.0])
@pytest.mark.parametrize("bounds", ["1", "0"])
def test_config1_full_scale_parity(config1, gamma, bounds, monkeypatch):
    monkeypatch.setenv("TRIM_FLAT_BOUNDS", bounds)
    hix, qs, gix = config1
    want = co.search_knn(hix, qs, 10, 1, gamma)
    got = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(gamma), qs, 10, 1)
    np.testing.assert_array_equal(got[0], want[0])
    assert_bits(got[1], want[1])
    np.testing.assert_array_equal(got[2][:, :5], want[2])
    ct = got[2].sum(0, dtype=np.float64)
    prune = ct[2] / (ct[2] + ct[0])
    if gamma == 0.0:
        assert abs(prune - 0.97871) < 1e-4  # SURVEY.md §6 probe value


# ------------------------------------------- list-level bound (whole-list skips)
@pytest.fixture(scope="module")
def clustered():
    # well-separated blobs, many lists: most probed lists are provably pruned
    # as a whole after the first chunk (trim_kernels.cuh: list_lower_bound)
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    ref = RefOracle()
    centers = ref.make_normal(32, 48, 11)
    base = ref.make_blobs(centers, 60000, 0.3, 12)
    qs = ref.make_blobs(centers, 200, 0.3, 13)
    hix = make_reference_index(ref, base, m=16, c=256, iters=10, pq_seed=14, nlist=64, ivf_seed=15)
    return hix, qs, G.GpuIvfIndex(G.IvfArrays.from_any(hix))


@pytest.mark.parametrize("gamma", [0.0, 0.5, 1.0, 1.5, 2.5])
@pytest.mark.parametrize("k", [10, 100, 250])
@pytest.mark.parametrize("mode", ["default", "wide_interval", "no_skip"])
def test_list_skip_parity(clustered, gamma, k, mode, monkeypatch):
    hix, qs, gix = clustered
    if mode == "wide_interval":
        monkeypatch.setenv("TRIM_EPS_SCALE", "20000")
    if mode == "no_skip":
        monkeypatch.setenv("TRIM_LIST_SKIP", "0")
    gix.skipped_positions(reset=True)
    want = co.search_knn(hix, qs, k, 32, gamma)
    got = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(gamma), qs, k, 32)
    np.testing.assert_array_equal(got[0], want[0])
    assert_bits(got[1], want[1])
    np.testing.assert_array_equal(got[2][:, :5], want[2])
    skipped = gix.skipped_positions()
    assert skipped <= int(want[2][:, 2].sum())  # skipped positions are pruned positions
    if gamma >= 2.0 or mode == "no_skip":
        assert skipped == 0  # no bound for γ(2-γ) <= 0 / disabled
    elif gamma in (0.5, 1.0) and k == 10:
        assert skipped > 0


# ------------------------------------------- k > 256 (shared-memory top-k)
@pytest.mark.parametrize("k", [257, 1000, 4096])
@pytest.mark.parametrize("gamma", [0.0, 0.8])
def test_large_k_vs_reference(clustered, k, gamma):
    """The reference's priority_queue has no cap (ivf.hpp:256-302): k = 257,
    1000 and 4096 run the shared-memory top-k and must equal the reference
    itself (oracle/_ref, per query) — ids, dist bits and counters."""
    hix, qs, gix = clustered
    ref = RefOracle()
    sess = ref.session(hix)
    try:
        want = ref.session_knn(sess, qs[:40], k, 32, gamma)
    finally:
        ref.session_destroy(sess)
    got = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(gamma), qs[:40], k, 32)
    np.testing.assert_array_equal(got[0], want[0])
    assert_bits(got[1], want[1])
    np.testing.assert_array_equal(got[2][:, :5], want[2])
    np.testing.assert_array_equal(got[2][:, 5], want[3])


def test_large_k_flat_and_cap():
    ix, qs, cases = goldens.load("flat_d128_m16")
    if ix is None:
        pytest.skip("no flat fixture")
    gix = G.GpuIvfIndex(G.IvfArrays.from_any(ix))
    hix = goldens.host_index(ix)
    for k in (300, 999):
        want = co.search_knn(hix, qs, k, 1, 0.5)
        got = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(0.5), qs, k, 1)
        np.testing.assert_array_equal(got[0], want[0])
        assert_bits(got[1], want[1])
        np.testing.assert_array_equal(got[2][:, :5], want[2])
    with pytest.raises(G.InvalidArgument):
        G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(0.5), qs, 4097, 1)
