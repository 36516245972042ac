"""GPU probe order (detail_ivf::probe_order, ivf.hpp:173-187) at large nlist.

The tensor-core path (trim_probe_mma.cuh: tf32 tcgen05 distance bounds,
exact reference-order distances for the candidates) must return exactly
the oracle's order — ids sorted by (exact fp32 distance, list id) — for
every query, including ties and degenerate inputs where the candidate set
overflows and the exact-everything fallback runs. TRIM_PROBE_MMA=0 forces
the SIMT kernels for comparison.
"""
import numpy as np
import pytest

from oracle.oracle import COracle, HostIndex
from paper_2508_17828_b200 import ivf as G
from tests import goldens

pytestmark = pytest.mark.gpu
co = COracle()


def probe_index(nlist, dim, seed, coarse=None):
    rng = np.random.default_rng(seed)
    m = 4 if dim % 4 == 0 else 2 if dim % 2 == 0 else 1
    sub = np.full(m, dim // m, np.uint32)
    if coarse is None:
        coarse = rng.standard_normal((nlist, dim)).astype(np.float32)
    n = nlist
    arr = G.IvfArrays(dim=dim, m=m, ksub=256, sub_dims=sub,
                      centroids=rng.standard_normal((256, dim)).astype(np.float32),
                      coarse=coarse, list_offsets=np.arange(nlist + 1, dtype=np.uint64),
                      list_ids=np.arange(n, dtype=np.uint32), list_codes=np.zeros((n, m), np.uint8),
                      list_lx=np.zeros(n, np.float32), vectors=coarse.copy())
    h = HostIndex(**{f: getattr(arr, f) for f in goldens.FIELDS})
    return G.GpuIvfIndex(arr), h


def check(gix, h, qs, nps):
    for npb in nps:
        got = G.probe_order(gix, qs, npb)
        for i in range(len(qs)):
            np.testing.assert_array_equal(got[i], co.probe_order(h, qs[i], npb), err_msg=f"q{i} np{npb}")


@pytest.mark.parametrize("dim", [96, 128, 20, 7])
@pytest.mark.parametrize("mode", ["mma", "simt"])
def test_probe_order_large_nlist(dim, mode, monkeypatch):
    if mode == "simt":
        monkeypatch.setenv("TRIM_PROBE_MMA", "0")
    gix, h = probe_index(1000, dim, 1)
    rng = np.random.default_rng(2)
    qs = rng.standard_normal((300, dim)).astype(np.float32) * 1.5
    qs[:20] = h.coarse.reshape(-1, dim)[:20]  # queries on centroids: d = 0 exactly
    check(gix, h, qs, (1, 64, 256))


def test_probe_order_clustered_scale():
    # centroids in tight clusters far from the origin: large |q||c| against
    # small gaps, the hardest case for the tf32 bound
    rng = np.random.default_rng(3)
    centers = rng.standard_normal((64, 96)).astype(np.float32) * 10
    coarse = (centers[rng.integers(0, 64, 4096)] + 0.05 * rng.standard_normal((4096, 96))).astype(np.float32)
    gix, h = probe_index(4096, 96, 4, coarse)
    qs = (centers[rng.integers(0, 64, 200)] + 0.05 * rng.standard_normal((200, 96))).astype(np.float32)
    check(gix, h, qs, (64, 200))


def test_probe_order_ties_overflow():
    # many identical centroids: > 512 candidates tie, so the select kernel's
    # exact-everything fallback runs; ties must resolve by ascending list id
    rng = np.random.default_rng(5)
    base = rng.standard_normal((8, 32)).astype(np.float32)
    coarse = np.repeat(base, 128, axis=0)  # 1024 lists, 8 distinct points
    gix, h = probe_index(1024, 32, 6, coarse)
    qs = np.concatenate([base, rng.standard_normal((40, 32)).astype(np.float32)])
    check(gix, h, qs, (1, 100, 256))
