"""CPU: the graph golden fixtures are the reference's own outputs (re-run the
reference on the stored bytes where oracle/_ref exists), and the graph C ABI
rejects bad descriptors with the reference's error classes before touching a
GPU."""
import ctypes as C
import os

import numpy as np
import pytest

from tests import goldens

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libtrimref.so")


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", goldens.graph_names())
def test_graph_goldens_match_reference(name):
    from oracle.oracle import RefOracle
    ref = RefOracle()
    g, qs, cases = goldens.load_graph(name)
    hg = goldens.host_graph(g)
    for cname, c in cases.items():
        if c["kind"] == "knn":
            ids, dist, cnt, ct = ref.graph_search(hg, qs, "trim_knn", k=c["k"], ef=c["ef"], gamma=c["gamma"])
            assert (ids == c["ids"]).all() and (dist.view(np.uint32) == c["dist"].view(np.uint32)).all(), cname
        else:
            ids, dist, cnt, ct = ref.graph_search(hg, qs, "trim_range", ef=c["ef"], gamma=c["gamma"],
                                                  radius=float(c["radius"]), cap=hg.n)
            assert (np.concatenate([[0], np.cumsum(cnt)]) == c["offsets"]).all(), cname
        assert (ct == c["counters"]).all(), cname


def test_graph_fixture_shapes():
    for name in goldens.graph_names():
        g, qs, cases = goldens.load_graph(name)
        assert len(g.offsets) == len(g.nbrs) >= 1
        for o, nb in zip(g.offsets, g.nbrs):
            assert o.shape == (g.n + 1,) and int(o[-1]) == nb.size and (nb < g.n).all()
        assert g.codes.shape == (g.n, g.m) and g.lx.shape == (g.n,)
        assert int(g.sub_dims.sum()) == g.dim


def _desc(**kw):
    from paper_2508_17828_b200 import _lib
    d = _lib.TrimGraphDesc()
    d.n, d.dim, d.m, d.ksub, d.levels, d.code_stride = 10, 8, 2, 16, 1, 2
    for k, v in kw.items():
        setattr(d, k, v)
    return d


@pytest.mark.parametrize("kw", [dict(n=0), dict(dim=0), dict(m=0), dict(ksub=300), dict(levels=0)])
def test_graph_create_validation(kw):
    from paper_2508_17828_b200 import _lib
    h = C.c_void_p()
    with pytest.raises(_lib.InvalidArgument):
        _lib.check(_lib.load().trim_graph_create(C.byref(_desc(**kw)), C.byref(h)))


def test_graph_search_argument_errors_without_gpu():
    """Argument errors surface before any device work (graph/search.hpp:193-196)."""
    from paper_2508_17828_b200 import _lib
    lib = _lib.load()
    q = np.zeros(8, np.float32)
    ids = np.zeros(8, np.uint32)
    d = np.zeros(8, np.float32)
    for k, ef, gam in ((0, 8, 0.5), (9, 8, 0.5), (4, 8, -1.0), (4, 2000, 0.5)):
        with pytest.raises(_lib.InvalidArgument):
            _lib.check(lib.trim_graph_search_knn(C.c_void_p(1), q.ctypes.data, 1, k, ef, gam, ids.ctypes.data,
                                                 d.ctypes.data, None))


@pytest.mark.parametrize("name", goldens.graph_names())
def test_graph_c_restatement_matches_goldens(name):
    """The plain-C restatement (oracle/trim_oracle.c, or_graph_search_trim_*)
    reproduces the reference's fixtures bit for bit, counters included."""
    from oracle.oracle import COracle
    co = COracle()
    g, qs, cases = goldens.load_graph(name)
    hg = goldens.host_graph(g)
    for cname, c in cases.items():
        if c["kind"] == "knn":
            ids, dist, ct = co.graph_search(hg, qs, "trim_knn", k=c["k"], ef=c["ef"], gamma=c["gamma"])
            assert (ids == c["ids"]).all() and (dist.view(np.uint32) == c["dist"].view(np.uint32)).all(), cname
        else:
            offs, ids, dist, ct = co.graph_search(hg, qs, "trim_range", ef=c["ef"], gamma=c["gamma"],
                                                  radius=float(c["radius"]))
            assert (offs == c["offsets"]).all() and (ids == c["ids"]).all(), cname
            assert (dist.view(np.uint32) == c["dist"].view(np.uint32)).all(), cname
        assert (ct == c["counters"][:, :5]).all(), cname
