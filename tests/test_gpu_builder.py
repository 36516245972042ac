"""GPU: the device-side index build — bit-exact pieces
against the oracle, determinism, and end-to-end search parity on a
device-built index."""
import numpy as np
import pytest

from oracle.oracle import COracle, HostIndex
from tests import goldens

pytestmark = pytest.mark.gpu
co = COracle()


def _torch():
    import torch
    return torch


def test_encode_and_landmark_dist_bit_exact():
    # pq::encode (pq.hpp:116-134) + Γ(l,x) (landmarks.hpp:57-72)
    torch = _torch()
    from paper_2508_17828_b200 import builder as B
    for name in ("ivf_d96_m48", "flat_d128_m16", "flat_d960_m120", "ivf_fixture"):
        ix, qs, _ = goldens.load(name)
        hix = goldens.host_index(ix)
        x = torch.from_numpy(hix.vectors).cuda()
        cent = torch.from_numpy(hix.centroids).cuda()
        codes, lx = B.pq_encode(x, hix.m, hix.ksub, hix.sub_dims, cent)
        want_codes, want_lx = co.build_landmarks(hix, hix.vectors)
        np.testing.assert_array_equal(codes.cpu().numpy(), want_codes)
        np.testing.assert_array_equal(lx.cpu().numpy().view(np.uint32), want_lx.view(np.uint32))


def test_assign_bit_exact_nearest_centroid():
    torch = _torch()
    from paper_2508_17828_b200 import builder as B
    for name in ("ivf_d96_m48", "ivf_fixture"):
        ix, qs, _ = goldens.load(name)
        hix = goldens.host_index(ix)
        coarse = hix.coarse.reshape(hix.nlist, hix.dim)
        a, d = B.assign(torch.from_numpy(hix.vectors).cuda(), torch.from_numpy(coarse).cuda())
        a = a.cpu().numpy()
        for i in range(0, hix.n, 7):
            dd = np.array([co.euclidean_sq(hix.vectors[i], c) for c in coarse], np.float32)
            assert a[i] == int(np.argmin(dd))  # argmin: first minimum = lowest index
            assert d.cpu().numpy()[i] == dd.min()


def test_kmeans_and_build_are_deterministic():
    torch = _torch()
    from paper_2508_17828_b200 import builder as B
    c = B.synth_normal(16, 12, seed=5)
    x = B.synth_blobs(c, 5000, 0.4, seed=6)
    k1 = B.kmeans(x, 40, 6, seed=7)
    k2 = B.kmeans(x, 40, 6, seed=7)
    assert torch.equal(k1, k2)
    assert torch.equal(B.synth_blobs(c, 5000, 0.4, seed=6), x)


def test_synthetic_distribution():
    torch = _torch()
    from paper_2508_17828_b200 import builder as B
    z = B.synth_normal(200_000, 8, seed=11)
    assert abs(float(z.mean())) < 0.01 and abs(float(z.std()) - 1.0) < 0.01
    c = B.synth_normal(4, 8, seed=1)
    x = B.synth_blobs(c, 40_000, 0.3, seed=2)
    # row i belongs to center i % 4 (round-robin, synthetic.hpp:26-27)
    r = (x.view(10_000, 4, 8) - c.view(1, 4, 8))
    assert abs(float(r.std()) - 0.3) < 0.01
    u = B.synth_uniform(1000, 960, seed=3, normalize=True)
    assert torch.allclose(u.norm(dim=1), torch.ones(1000, device=u.device), atol=1e-5)


def test_lists_ascending_ids():
    torch = _torch()
    from paper_2508_17828_b200 import builder as B
    a = torch.randint(0, 37, (10_000,), dtype=torch.int32, device="cuda")
    offs, ids = B.ivf_lists(a, 37)
    offs, ids, a = offs.cpu().numpy(), ids.cpu().numpy(), a.cpu().numpy()
    assert offs[0] == 0 and offs[-1] == 10_000
    for l in range(37):
        seg = ids[offs[l]:offs[l + 1]]
        assert (np.diff(seg) > 0).all()
        assert (a[seg] == l).all()


@pytest.mark.parametrize("nlist,m", [(1, 8), (24, 8), (24, 12)])
def test_device_built_index_search_parity(nlist, m):
    torch = _torch()
    from paper_2508_17828_b200 import builder as B
    from paper_2508_17828_b200 import ivf as G
    c = B.synth_normal(32, 48, seed=21)
    x = B.synth_blobs(c, 20_000, 0.3, seed=22)
    q = B.synth_blobs(c, 64, 0.3, seed=23)
    arr = B.build_ivf(x, B.BuildParams(m=m, ksub=256, pq_iters=6, nlist=nlist, coarse_iters=5))
    gix = G.GpuIvfIndex(arr)
    h = B.to_host(arr)
    hix = HostIndex(**{f: getattr(h, f) for f in goldens.FIELDS})
    qs = q.cpu().numpy()
    npb = max(1, nlist // 3)
    for g in (0.0, 0.6, 1.0):
        want = co.search_knn(hix, qs, 10, npb, g)
        got = G.search_trim_ivf_knn_batch(gix, G.PruningProfile.manual(g), qs, 10, npb)
        np.testing.assert_array_equal(got[0], want[0])
        np.testing.assert_array_equal(got[1].view(np.uint32), want[1].view(np.uint32))
        np.testing.assert_array_equal(got[2][:, :5], want[2])
        # device-resident + preassigned path gives the same
        d_ids, d_dist = G.search_trim_ivf_knn_device(gix, G.PruningProfile.manual(g), q, 10, npb)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(d_ids.cpu().numpy().view(np.uint32), want[0])
    want = co.search_baseline(hix, qs, 10, npb, 200)
    got = G.search_baseline_ivfpq_batch(gix, qs, 10, npb, 200)
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(got[2][:, :5], want[2])


# ------------------------------------------- reference-equal k-means / build
def _ref_or_skip():
    from oracle.oracle import RefOracle, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    return RefOracle()


@pytest.mark.parametrize("n,dim,m,c,iters,seed,sample", [
    (6000, 16, 4, 256, 8, 3, 0),        # default sample (100*c rows, pq.hpp:67-70)
    (3000, 24, 3, 64, 12, 11, 2000),    # explicit sample, fewer centroids
    (800, 8, 1, 200, 5, 1, 0),          # one subspace: plain kmeans over all rows
    (2000, 10, 3, 100, 6, 7, 0),        # uneven split_sub_dims (4, 3, 3)
])
def test_pq_train_equals_reference(n, dim, m, c, iters, seed, sample):
    """pq::train (pq.hpp:65-113) = sampled rows -> per-subspace pq::kmeans
    (k-means++ with std::mt19937_64, Lloyd, empty-cluster repair): the device
    codebook equals the reference's bit for bit on the reference's own rows."""
    torch = _torch()
    ref = _ref_or_skip()
    from paper_2508_17828_b200 import builder as B
    centers = ref.make_normal(12, dim, 5)
    data = ref.make_blobs(centers, n, 0.4, 6)
    sub_r, cent_r = ref.pq_train(data, m, c, iters, seed, sample)
    sub_g, cent_g = B.pq_train(torch.from_numpy(data).cuda(), m, c, iters, seed, sample)
    np.testing.assert_array_equal(sub_g, sub_r)
    np.testing.assert_array_equal(cent_g.cpu().numpy().view(np.uint32), cent_r.view(np.uint32))


@pytest.mark.parametrize("nlist,coarse_iters,ivf_seed", [(16, 10, 4), (64, 6, 9), (1, 3, 2)])
def test_build_ivf_equals_reference(nlist, coarse_iters, ivf_seed):
    """The whole offline pipeline on the device (pq_train -> encode + Γ(l,x)
    -> coarse k-means on the reference's row sample -> lists) reproduces the
    reference's IvfIndex (ivf.hpp:112-154) from the same rows: codebook,
    coarse centroids, list offsets, ids, codes and lx, bit for bit."""
    torch = _torch()
    ref = _ref_or_skip()
    from oracle.oracle import make_reference_index
    from paper_2508_17828_b200 import builder as B
    centers = ref.make_normal(20, 32, 21)
    data = ref.make_blobs(centers, 12000, 0.3, 22)
    want = make_reference_index(ref, data, m=8, c=256, iters=6, pq_seed=3, nlist=nlist, ivf_seed=ivf_seed,
                                coarse_iters=coarse_iters)
    got = B.to_host(B.build_ivf(torch.from_numpy(data).cuda(),
                                B.BuildParams(m=8, ksub=256, pq_iters=6, pq_seed=3, nlist=nlist, ivf_seed=ivf_seed,
                                              coarse_iters=coarse_iters)))
    for f in ("centroids", "coarse", "list_lx"):
        np.testing.assert_array_equal(np.asarray(getattr(got, f), np.float32).ravel().view(np.uint32),
                                      np.asarray(getattr(want, f), np.float32).ravel().view(np.uint32), err_msg=f)
    for f in ("sub_dims", "list_offsets", "list_ids", "list_codes"):
        np.testing.assert_array_equal(np.asarray(getattr(got, f)).ravel(), np.asarray(getattr(want, f)).ravel(),
                                      err_msg=f)
