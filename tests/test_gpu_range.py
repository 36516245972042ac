"""GPU range search (ivf::search_trim_ivf_range, ivf.hpp:308-347) on flat
indexes, where the query-tiled kernel (trim_range_flat_kernel) runs, and
through the device-resident API (trim_search_range_device).

Bar: identical member sets in (dist, id) order, bit-identical distances,
identical per-query counters, against the C oracle (pinned to the reference
by tests/test_oracle.py) and against the one-query kernel
(TRIM_RANGE_TILED=0)."""
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
    centers = ref.make_normal(32, 64, 21)
    base = ref.make_blobs(centers, 70000, 0.3, 22)  # > 2 slices of 32768
    qs = ref.make_blobs(centers, 37, 0.3, 23)        # not a multiple of the query tile
    hix = make_reference_index(ref, base, m=32, c=256, iters=8, pq_seed=24, nlist=1, ivf_seed=25)
    # radii: per query, from ~0 to a few hundred members; one exactly 0
    rng = np.random.default_rng(26)
    rad = rng.uniform(1.0, 3.2, len(qs)).astype(np.float32)
    rad[3] = 0.0
    return hix, qs, rad, G.GpuIvfIndex(G.IvfArrays.from_any(hix))


def check(got, want):
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(got[1], want[1])
    assert_bits(got[2], want[2])
    np.testing.assert_array_equal(got[3][:, :5], want[3])


@pytest.mark.parametrize("gamma", [0.0, 0.5, 0.8, 1.0])
@pytest.mark.parametrize("mode", ["tiled", "one_query", "wide_interval"])
def test_flat_range_parity(flat, gamma, mode, monkeypatch):
    hix, qs, rad, gix = flat
    if mode == "one_query":
        monkeypatch.setenv("TRIM_RANGE_TILED", "0")
    if mode == "wide_interval":
        monkeypatch.setenv("TRIM_EPS_SCALE", "20000")
    want = co.search_range(hix, qs, rad, 1, gamma)
    got = G.search_trim_ivf_range_batch(gix, G.PruningProfile.manual(gamma), qs, rad, 1)
    check(got, want)
    assert int(want[0][-1]) > 0


def test_range_device_api(flat):
    import torch
    hix, qs, rad, gix = flat
    prof = G.PruningProfile.manual(0.5)
    offs, ids, dist, ct = G.search_trim_ivf_range_batch(gix, prof, qs, rad, 1)
    dq = torch.from_numpy(qs).cuda()
    dr = torch.from_numpy(rad).cuda()
    dct = torch.zeros((len(qs), 6), dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    cnt, di, dd = G.search_trim_ivf_range_device(gix, prof, dq, dr, 1, cap=4096, d_counters=dct,
                                                 d_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    cnt, di, dd = cnt.cpu().numpy(), di.cpu().numpy(), dd.cpu().numpy()
    for i in range(len(qs)):
        b, e = int(offs[i]), int(offs[i + 1])
        assert cnt[i] == e - b
        np.testing.assert_array_equal(di[i, :cnt[i]].astype(np.uint32), ids[b:e])
        assert_bits(dd[i, :cnt[i]], dist[b:e])
    np.testing.assert_array_equal(dct.cpu().numpy(), ct.astype(np.int64))
    # a cap below the largest result: status bit 0, true counts, the listed
    # members a sorted subset of the true set
    mx = int(cnt.max())
    st.zero_()
    c2, d2i, _ = G.search_trim_ivf_range_device(gix, prof, dq, dr, 1, cap=max(1, mx // 2), d_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & 1
    np.testing.assert_array_equal(c2.cpu().numpy(), cnt)
    i = int(np.argmax(cnt))
    sub = d2i[i].cpu().numpy().astype(np.uint32)
    assert set(sub.tolist()) <= set(ids[int(offs[i]):int(offs[i + 1])].tolist())
    # negative radius: status bit 1, no members for that query
    dr2 = dr.clone()
    dr2[0] = -1.0
    st.zero_()
    c3, _, _ = G.search_trim_ivf_range_device(gix, prof, dq, dr2, 1, cap=4096, d_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & 2
    assert int(c3[0].item()) == 0


@pytest.mark.parametrize("gamma", [0.0, 0.5, 0.8, 1.0])
def test_flat_range_block_partition(flat, gamma, monkeypatch):
    """Flat range over the block partition (built when the index is first
    searched; forced here for a small index): identical members and counters."""
    hix, qs, rad, _ = flat
    monkeypatch.setenv("TRIM_FLAT_PARTITION_MIN_ROWS", "1000")
    gix = G.GpuIvfIndex(G.IvfArrays.from_any(hix))  # fresh index: the partition is built on this call
    want = co.search_range(hix, qs, rad, 1, gamma)
    got = G.search_trim_ivf_range_batch(gix, G.PruningProfile.manual(gamma), qs, rad, 1)
    check(got, want)
    # the device API over the same partition
    import torch
    cnt, di, dd = G.search_trim_ivf_range_device(gix, G.PruningProfile.manual(gamma), torch.from_numpy(qs).cuda(),
                                                 torch.from_numpy(rad).cuda(), 1, cap=4096)
    cnt = cnt.cpu().numpy()
    np.testing.assert_array_equal(cnt, np.diff(want[0].astype(np.int64)))
