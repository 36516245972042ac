"""CPU: pin the C restatement (oracle/trim_oracle.c) to the reference.

1. Against the golden fixtures that the reference itself produced
   (tests/golden/make_golden.py) — bit-exact ids, dist_sq and counters.
2. Known-answer tests restated from the reference's own tests:
   test_trim.cpp:18-39, 71-74; test_core.cpp:32-44; test_pq.cpp:210-231;
   test_ivf.cpp:171-200, 202-251, 253-264, 266-291.
3. When oracle/_ref/libtrimref.so is present: random cases against the
   reference library directly.
"""
import math

import numpy as np
import pytest

from oracle.oracle import COracle, RefOracle, make_reference_index, ref_available
from tests import goldens

co = COracle()


@pytest.mark.parametrize("name,case", goldens.all_cases())
def test_oracle_matches_reference_goldens(name, case):
    ix, qs, cases = goldens.load(name)
    hix = goldens.host_index(ix)
    c = cases[case]
    if c["kind"] == "knn":
        ids, dist, ct, cdc = co.search_knn(hix, qs, c["k"], c["nprobe"], c["gamma"])
        np.testing.assert_array_equal(ids, c["ids"])
        np.testing.assert_array_equal(dist.view(np.uint32), c["dist"].view(np.uint32))
    elif c["kind"] == "range":
        offs, ids, dist, ct, cdc = co.search_range(hix, qs, c["radius"], c["nprobe"], c["gamma"])
        np.testing.assert_array_equal(offs, c["offsets"])
        np.testing.assert_array_equal(ids, c["ids"])
        np.testing.assert_array_equal(dist.view(np.uint32), c["dist"].view(np.uint32))
    else:
        ids, dist, ct, cdc = co.search_baseline(hix, qs, c["k"], c["nprobe"], c["k_prime"])
        np.testing.assert_array_equal(ids, c["ids"])
        np.testing.assert_array_equal(dist.view(np.uint32), c["dist"].view(np.uint32))
    np.testing.assert_array_equal(ct, c["counters"])
    np.testing.assert_array_equal(cdc, c["coarse_dc"])


def test_golden_accounting_identities():
    # test_ivf.cpp:202-224: dc + pruned == evaluated for every query
    for name in goldens.names():
        _, _, cases = goldens.load(name)
        for c in cases.values():
            ct = c["counters"]
            assert (ct[:, 0] + ct[:, 2] == ct[:, 3]).all()


def test_bound_kats():
    # test_trim.cpp:18-39
    assert co.strict_lb(4.0, 4.0) == 0.0
    assert co.strict_lb(3.0, 0.0) == 9.0
    assert co.strict_lb(5.0, 2.0) == 9.0
    assert co.relaxed_lb(5.0, 2.0, 0.0) == co.strict_lb(5.0, 2.0)
    assert co.relaxed_lb(3.0, 4.0, 1.0) == 25.0
    prev = 0.0
    for i in range(21):
        lb = co.relaxed_lb(3.0, 4.0, np.float32(i * 0.1))
        assert lb >= prev
        prev = lb


def test_relaxed_equals_expanded_cosine_form():
    # test_ivf.cpp:253-264 (in double precision there; fp32 here with 1e-5)
    r = np.random.default_rng(9)
    for _ in range(2000):
        glq, glx = r.uniform(0, 30, 2).astype(np.float32)
        g = np.float32(r.uniform(0, 1.5))
        lhs = co.relaxed_lb(glq, glx, g)
        rhs = float(glq) ** 2 + float(glx) ** 2 - 2 * float(glq) * float(glx) * (1 - float(g))
        assert math.isclose(lhs, rhs, rel_tol=1e-5, abs_tol=1e-3)


def test_euclidean_kats():
    # test_core.cpp:32-44
    a = np.array([1, 2, 3], np.float32)
    assert co.euclidean_sq(a, a) == 0.0
    assert co.euclidean_sq(np.array([0, 0], np.float32), np.array([3, 4], np.float32)) == 25.0
    assert co.euclidean_sq(np.ones(4, np.float32), np.array([2, 3, 4, 5], np.float32)) == 30.0


def test_adc_hand_filled_table():
    # test_pq.cpp:225-231
    t = np.array([[0.0, 4.0], [9.0, 0.0]], np.float32)
    assert co.adc(t, np.array([1, 0], np.uint8)) == 13.0


def test_table_is_plain_distance_for_m1():
    # test_pq.cpp:210-216: m=1 LUT entry == euclidean_sq exactly
    ix, qs, _ = goldens.load("ivf_fixture")
    hix = goldens.host_index(ix)
    cb = hix.centroids.reshape(hix.ksub, hix.dim)  # only valid when m==1; build one
    from oracle.oracle import HostIndex
    one = HostIndex(dim=hix.dim, m=1, ksub=hix.ksub, sub_dims=np.array([hix.dim], np.uint32),
                    centroids=hix.vectors[: hix.ksub].copy(), coarse=hix.coarse,
                    list_offsets=hix.list_offsets, list_ids=hix.list_ids,
                    list_codes=hix.list_codes[:, :1].copy(), list_lx=hix.list_lx,
                    vectors=hix.vectors)
    t = co.distance_table(one, qs[0])
    for c in range(one.ksub):
        assert t[0, c] == co.euclidean_sq(qs[0], one.centroids.reshape(-1, hix.dim)[c])
    del cb


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_vs_reference_random():
    ref = RefOracle()
    for trial, (n, dim, m, c, nlist) in enumerate([(700, 12, 3, 32, 9), (900, 20, 5, 16, 1),
                                                   (600, 9, 4, 64, 30)]):
        rng_seed = 100 + trial
        centers = ref.make_normal(16, dim, rng_seed)
        ds = ref.make_blobs(centers, n, 0.5, rng_seed + 1)
        ix = make_reference_index(ref, ds, m=m, c=c, iters=5, pq_seed=rng_seed + 2, nlist=nlist,
                                  ivf_seed=rng_seed + 3)
        qs = ref.make_normal(15, dim, rng_seed + 4)
        for g in (0.0, 0.45, 0.9):
            for k, npb in ((1, nlist), (7, max(1, nlist // 2))):
                a = ref.search_knn(ix, qs, k, npb, g)
                b = co.search_knn(ix, qs, k, npb, g)
                for x, y in zip(a, b):
                    np.testing.assert_array_equal(x, y)
            a = ref.search_range(ix, qs, 2.5, max(1, nlist // 2), g)
            b = co.search_range(ix, qs, 2.5, max(1, nlist // 2), g)
            for x, y in zip(a, b):
                np.testing.assert_array_equal(x, y)
        a = ref.search_baseline(ix, qs, 5, nlist, 40)
        b = co.search_baseline(ix, qs, 5, nlist, 40)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_landmark_build_matches_reference():
    ref = RefOracle()
    ix, qs, _ = goldens.load("ivf_d96_m48")
    hix = goldens.host_index(ix)
    data = hix.vectors[:500]
    codes_r, lx_r = ref.build_landmarks(data, hix.m, hix.ksub, hix.sub_dims, hix.centroids)
    codes_c, lx_c = co.build_landmarks(hix, data)
    np.testing.assert_array_equal(codes_r, codes_c)
    np.testing.assert_array_equal(lx_r.view(np.uint32), lx_c.view(np.uint32))


def test_error_cases():
    ix, qs, _ = goldens.load("ivf_fixture")
    hix = goldens.host_index(ix)
    with pytest.raises(ValueError):
        co.search_knn(hix, qs[:1], 0, 2, 0.0)
    with pytest.raises(ValueError):
        co.search_knn(hix, qs[:1], 5, 2, -1.0)  # uncalibrated
    with pytest.raises(ValueError):
        co.search_knn(hix, qs[:1], 3000, 1, 0.0)  # k exceeds probed
    with pytest.raises(ValueError):
        co.search_range(hix, qs[:1], -1.0, 2, 0.0)
    with pytest.raises(ValueError):
        co.search_baseline(hix, qs[:1], 10, 4, 5)  # k > k'
