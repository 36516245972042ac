"""The reference's on-disk formats: files written by the
reference's own save() load through paper_2508_17828_b200.formats, and files
written by formats load through the reference's own load(), field for field.
Host-only (no GPU); needs oracle/_ref (the reference compiled in place)."""
import os

import numpy as np
import pytest

from oracle.oracle import HostIndex, ref_available
from paper_2508_17828_b200 import formats as F
from paper_2508_17828_b200._lib import DataError
from paper_2508_17828_b200.ivf import PruningProfile
from tests import goldens

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import RefOracle
    return RefOracle()


@pytest.fixture(params=goldens.names())
def fixture_index(request):
    ix, qs, cases = goldens.load(request.param)
    return goldens.host_index(ix)


def test_ivf_reference_to_ours(ref, fixture_index, tmp_path):
    h = fixture_index
    path = str(tmp_path / "ix.ivf")
    ref.ivf_save(h, path, mse=1.25, seed=7, iters=25)
    arr, cb = F.load_ivf(path, vectors=h.vectors)
    assert (arr.dim, arr.m, arr.ksub) == (h.dim, h.m, h.ksub)
    assert (cb.training_mse, cb.seed, cb.kmeans_iters) == (1.25, 7, 25)
    np.testing.assert_array_equal(arr.sub_dims, h.sub_dims)
    np.testing.assert_array_equal(arr.centroids.view(np.uint32), np.asarray(h.centroids, np.float32).view(np.uint32))
    np.testing.assert_array_equal(arr.coarse.view(np.uint32),
                                  np.asarray(h.coarse, np.float32).reshape(-1).view(np.uint32))
    np.testing.assert_array_equal(arr.list_offsets, h.list_offsets)
    np.testing.assert_array_equal(arr.list_ids, h.list_ids)
    np.testing.assert_array_equal(arr.list_codes, np.asarray(h.list_codes).reshape(-1, h.code_stride)[:, :h.m])
    np.testing.assert_array_equal(arr.list_lx.view(np.uint32), np.asarray(h.list_lx, np.float32).view(np.uint32))


def test_ivf_ours_to_reference(ref, fixture_index, tmp_path):
    h = fixture_index
    from paper_2508_17828_b200.ivf import IvfArrays
    arr = IvfArrays.from_any(h)
    arr.list_codes = np.asarray(h.list_codes).reshape(-1, h.code_stride)[:, :h.m]
    path = str(tmp_path / "ours.ivf")
    F.save_ivf(path, arr, F.Codebook(h.dim, h.m, h.ksub, np.asarray(h.sub_dims, np.uint32),
                                     np.asarray(h.centroids, np.float32), 0.5, 3, 10))
    got = ref.ivf_load(path)
    assert (got["training_mse"], got["seed"], got["iters"]) == (0.5, 3, 10)
    np.testing.assert_array_equal(got["list_offsets"], h.list_offsets)
    np.testing.assert_array_equal(got["list_ids"], h.list_ids)
    np.testing.assert_array_equal(got["list_codes"], arr.list_codes)
    np.testing.assert_array_equal(got["list_lx"].view(np.uint32), np.asarray(h.list_lx, np.float32).view(np.uint32))
    np.testing.assert_array_equal(got["coarse"], np.asarray(h.coarse, np.float32).reshape(-1))
    # and it round-trips through our loader byte for byte
    path2 = str(tmp_path / "ours2.ivf")
    a2, cb2 = F.load_ivf(path)
    F.save_ivf(path2, a2, cb2)
    assert open(path, "rb").read() == open(path2, "rb").read()


def test_landmarks_both_ways(ref, tmp_path):
    rng = np.random.default_rng(0)
    dim, m, c, n = 24, 6, 256, 500
    sub = np.full(m, dim // m, np.uint32)
    cent = rng.standard_normal(c * dim).astype(np.float32)
    codes = rng.integers(0, 256, (n, m)).astype(np.uint8)
    lx = rng.random(n).astype(np.float32)
    p1 = str(tmp_path / "ref.lm")
    ref.landmarks_save(dim, m, c, sub, cent, codes, lx, p1)
    cb, c2, l2 = F.load_landmarks(p1)
    np.testing.assert_array_equal(c2, codes)
    np.testing.assert_array_equal(l2, lx)
    np.testing.assert_array_equal(cb.centroids, cent)
    p2 = str(tmp_path / "ours.lm")
    F.save_landmarks(p2, cb, codes, lx)
    c3, l3 = ref.landmarks_load(p2, n, m)
    np.testing.assert_array_equal(c3, codes)
    np.testing.assert_array_equal(l3, lx)
    flat = F.flat_index(cb, codes, lx, rng.standard_normal((n, dim)).astype(np.float32))
    assert flat.list_offsets.tolist() == [0, n] and flat.list_ids[-1] == n - 1


def test_profile_and_vecs_both_ways(ref, tmp_path):
    p1 = str(tmp_path / "ref.profile")
    ref.profile_save(0.8125, 0.6051234567890123, p1)
    prof = F.load_profile(p1)
    assert prof.p == 0.8125 and prof.gamma == 0.6051234567890123
    p2 = str(tmp_path / "ours.profile")
    F.save_profile(p2, prof)
    assert ref.profile_load(p2) == (0.8125, 0.6051234567890123)
    with open(p2, "a") as f:
        f.write("bogus = 1\n")
    with pytest.raises(DataError, match="unknown profile key"):
        F.load_profile(p2)
    x = np.random.default_rng(1).standard_normal((37, 13)).astype(np.float32)
    v1 = str(tmp_path / "ref.fvecs")
    ref.write_fvecs(x, v1)
    np.testing.assert_array_equal(F.load_vecs(v1), x)
    v2 = str(tmp_path / "ours.fvecs")
    F.write_fvecs(v2, x)
    np.testing.assert_array_equal(ref.load_fvecs(v2, 37, 13), x)
    assert open(v1, "rb").read() == open(v2, "rb").read()


def test_truncated_files_raise_data_error(ref, fixture_index, tmp_path):
    path = str(tmp_path / "t.ivf")
    ref.ivf_save(fixture_index, path)
    raw = open(path, "rb").read()
    open(path, "wb").write(raw[:-3])
    with pytest.raises(DataError, match="truncated"):
        F.load_ivf(path)


@pytest.mark.gpu
def test_reference_files_search_on_gpu(ref, tmp_path):
    """Reference-written index + fvecs -> open_index -> identical search results."""
    from oracle.oracle import COracle
    from paper_2508_17828_b200 import ivf as G
    ix, qs, cases = goldens.load("ivf_fixture")
    h = goldens.host_index(ix)
    ip, vp = str(tmp_path / "a.ivf"), str(tmp_path / "base.fvecs")
    ref.ivf_save(h, ip)
    ref.write_fvecs(np.asarray(h.vectors, np.float32).reshape(-1, h.dim), vp)
    gix = F.open_index(ip, vp)
    prof_path = str(tmp_path / "p.profile")
    ref.profile_save(0.9, 0.35, prof_path)
    prof = F.load_profile(prof_path)
    want = COracle().search_knn(h, qs, 10, 5, prof.gamma)
    got = G.search_trim_ivf_knn_batch(gix, prof, qs, 10, 5)
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(np.asarray(got[1]).view(np.uint32), np.asarray(want[1]).view(np.uint32))
    np.testing.assert_array_equal(got[2][:, :5], want[2])


@pytest.mark.parametrize("name", goldens.graph_names())
def test_graph_file_both_ways(ref, name, tmp_path):
    """GraphIndex::save (graph/hnsw.hpp:37-56) -> formats.load_graph, and
    formats.save_graph -> GraphIndex::load, level for level."""
    g, qs, cases = goldens.load_graph(name)
    hg = goldens.host_graph(g)
    p1 = str(tmp_path / "ref.graph")
    ref.graph_save(hg, p1)
    gf = F.load_graph(p1)
    assert (gf.count, gf.M, gf.entry, gf.ef_construction) == (g.n, g.M, g.entry, g.efc)
    for a, b in zip(gf.offsets, g.offsets):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(gf.nbrs, g.nbrs):
        np.testing.assert_array_equal(a, b)
    p2 = str(tmp_path / "ours.graph")
    F.save_graph(p2, gf)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    back = ref.graph_load(p2, g.n)
    assert back.entry == g.entry and len(back.offsets) == len(g.offsets)
    for a, b in zip(back.nbrs, g.nbrs):
        np.testing.assert_array_equal(a, b)


def test_graph_file_zero_levels(tmp_path):
    p = str(tmp_path / "bad.graph")
    with open(p, "wb") as f:
        np.array([3], "<u8").tofile(f)
        np.array([4, 0, 0, 8], "<u4").tofile(f)
    with pytest.raises(DataError):
        F.load_graph(p)
