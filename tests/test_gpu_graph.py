"""TRIM filter over an HNSW graph (graph/search.hpp:188-347)
on the GPU through the C ABI, bit-exact against the reference: the golden
fixtures written by the reference (tests/golden/make_golden_graph.py) and,
where oracle/_ref is present, graphs the reference builds here and now."""
import os

import numpy as np
import pytest

from tests import goldens

pytestmark = pytest.mark.gpu

CASES = [(n, c) for n in goldens.graph_names() for c in sorted(goldens.load_graph(n)[2])]


@pytest.fixture(scope="module")
def graphs():
    from paper_2508_17828_b200 import graph as GG
    out = {}
    for n in goldens.graph_names():
        g, qs, cases = goldens.load_graph(n)
        out[n] = (GG.GpuGraph(GG.GraphArrays.from_any(g)), qs, cases)
    return out


def _bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def check_case(G, gg, qs, c):
    from paper_2508_17828_b200.ivf import PruningProfile
    prof = PruningProfile.manual(c["gamma"])
    if c["kind"] == "knn":
        ids, dist, ct = G.search_trim_knn_batch(gg, prof, qs, c["k"], c["ef"])
        assert (ids == c["ids"]).all(), "ids differ from the reference"
        assert (_bits(dist) == _bits(c["dist"])).all(), "dist_sq differ from the reference"
        assert (ct[:, :5] == c["counters"][:, :5]).all(), "counters differ from the reference"
    else:
        offs, ids, dist, ct = G.search_trim_range_batch(gg, prof, qs, c["radius"], c["ef"])
        assert (offs == c["offsets"]).all(), "range result sizes differ"
        assert (ids == c["ids"]).all() and (_bits(dist) == _bits(c["dist"])).all()
        assert (ct[:, :5] == c["counters"][:, :5]).all(), "counters differ from the reference"


@pytest.mark.parametrize("name,case", CASES)
def test_graph_golden(graphs, name, case):
    from paper_2508_17828_b200 import graph as G
    gg, qs, cases = graphs[name]
    check_case(G, gg, qs, cases[case])


def test_graph_search_queue_overflow_rerun(graphs, monkeypatch):
    """A search queue capacity of 16 overflows on every query; the host re-runs
    them with capacity n + 1 and the results stay the reference's."""
    from paper_2508_17828_b200 import graph as G
    monkeypatch.setenv("TRIM_GRAPH_HEAP_CAP", "16")
    gg, qs, cases = graphs["graph_d32_m8"]
    for c in ("knn_k10_ef32_g0.6", "range_r2.3_ef32_g0.8"):
        check_case(G, gg, qs, cases[c])


def test_graph_single_query_facade(graphs):
    from paper_2508_17828_b200 import graph as G
    from paper_2508_17828_b200.ivf import PruningProfile
    gg, qs, cases = graphs["graph_d32_m8"]
    c = cases["knn_k10_ef32_g0.6"]
    r = G.search_trim_knn(gg, PruningProfile.manual(0.6), qs[3], 10, 32)
    assert (r.ids == c["ids"][3]).all()
    assert r.counters.evaluated == c["counters"][3][3] and r.counters.hops == c["counters"][3][4]


@pytest.mark.parametrize("kw", [dict(k=0, ef=8), dict(k=9, ef=8), dict(k=4, ef=2000)])
def test_graph_knn_argument_errors(graphs, kw):
    from paper_2508_17828_b200 import graph as G
    from paper_2508_17828_b200.ivf import InvalidArgument, PruningProfile
    gg, qs, _ = graphs["graph_d32_m8"]
    with pytest.raises(InvalidArgument):
        G.search_trim_knn_batch(gg, PruningProfile.manual(0.5), qs[:2], kw["k"], kw["ef"])


def test_graph_uncalibrated_and_negative_radius(graphs):
    from paper_2508_17828_b200 import graph as G
    from paper_2508_17828_b200.ivf import InvalidArgument, PruningProfile
    gg, qs, _ = graphs["graph_d32_m8"]
    with pytest.raises(InvalidArgument):
        G.search_trim_knn_batch(gg, PruningProfile(), qs[:2], 4, 8)
    with pytest.raises(InvalidArgument):
        G.search_trim_range_batch(gg, PruningProfile.manual(0.5), qs[:2], -1.0, 8)


@pytest.mark.skipif(not os.path.exists(os.path.join(goldens.GOLDEN, "..", "..", "oracle", "_ref", "libtrimref.so")),
                    reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [21, 22])
def test_graph_live_reference(seed):
    """A graph the reference builds now (other seed, shape and M), kNN and range
    at several gammas, against the reference's own searches."""
    from oracle.oracle import RefOracle, make_reference_graph
    from paper_2508_17828_b200 import graph as G
    from paper_2508_17828_b200.ivf import PruningProfile
    ref = RefOracle()
    c = ref.make_normal(24, 48, seed)
    base = ref.make_blobs(c, 2500, 0.35, seed + 1)
    qs = ref.make_blobs(c, 40, 0.35, seed + 2)
    hg = make_reference_graph(ref, base, M=6 + seed % 4, efc=40, graph_seed=seed, m=12, pq_seed=seed)
    gg = G.GpuGraph(G.GraphArrays.from_any(hg))
    for gam in (0.0, 0.7, 1.2):
        want = ref.graph_search(hg, qs, "trim_knn", k=8, ef=40, gamma=gam)
        ids, dist, ct = G.search_trim_knn_batch(gg, PruningProfile.manual(gam), qs, 8, 40)
        assert (ids == want[0]).all() and (_bits(dist) == _bits(want[1])).all()
        assert (ct[:, :5] == want[3][:, :5]).all()
        r = 2.8
        wi, wd, wc, wct = ref.graph_search(hg, qs, "trim_range", ef=24, gamma=gam, radius=r, cap=hg.n)
        offs, rids, rd, rct = G.search_trim_range_batch(gg, PruningProfile.manual(gam), qs, r, 24)
        assert (np.diff(offs.astype(np.int64)) == wc.astype(np.int64)).all()
        for i in range(len(qs)):
            seg = slice(int(offs[i]), int(offs[i + 1]))
            assert (rids[seg] == wi[i, :wc[i]]).all() and (_bits(rd[seg]) == _bits(wd[i, :wc[i]])).all()
        assert (rct[:, :5] == wct[:, :5]).all()


@pytest.mark.skipif(not os.path.exists(os.path.join(goldens.GOLDEN, "..", "..", "oracle", "_ref", "libtrimref.so")),
                    reason="oracle/_ref not built")
def test_graph_gamma0_exhaustive_ef_equals_brute_force():
    """proj/tests/test_graph.cpp:132-159: with gamma = 0 and ef = n, TRIM graph
    kNN returns the brute-force top 10 and range search the brute-force ball
    (here on the GPU; ef = 600 uses the 1,024-slot candidate queue)."""
    from oracle.oracle import COracle, RefOracle, make_reference_graph
    from paper_2508_17828_b200 import graph as G
    from paper_2508_17828_b200.ivf import PruningProfile
    ref, co = RefOracle(), COracle()
    base = ref.make_normal(600, 16, 100)
    qs = ref.make_normal(25, 16, 101)
    # TrimFixture(600, 16, 100, 4, 32) (test_graph.cpp:29-51): M = 8, ef_construction = 100,
    # PQ m = 4 with c = 32 centroids (a ksub < 256 codebook), 8 k-means iterations
    hg = make_reference_graph(ref, base, M=8, efc=100, graph_seed=101, m=4, c=32, iters=8, pq_seed=102)
    gg = G.GpuGraph(G.GraphArrays.from_any(hg))
    zero = PruningProfile.manual(0.0)
    ids, dist, ct = G.search_trim_knn_batch(gg, zero, qs, 10, 600)
    truth_ids, truth_d = co.brute_force_knn(base, qs, 10)
    assert (ids == truth_ids).all()
    radius = 4.2
    offs, rids, rd, rct = G.search_trim_range_batch(gg, zero, qs, radius, 600)
    r2 = np.float32(radius) * np.float32(radius)
    for i in range(len(qs)):
        d = np.array([co.euclidean_sq(qs[i], base[j]) for j in range(len(base))], np.float32)
        want = sorted((float(d[j]), j) for j in range(len(base)) if d[j] <= r2)
        got = rids[int(offs[i]):int(offs[i + 1])]
        assert [j for _, j in want] == got.tolist()
    # and the whole output is the reference's own
    w = ref.graph_search(hg, qs, "trim_knn", k=10, ef=600, gamma=0.0)
    assert (w[0] == ids).all() and (w[3][:, :5] == ct[:, :5]).all()
