"""Generates tests/golden/*.npz from the REFERENCE itself.

Runs the unmodified reference headers (compiled in place into
oracle/_ref/libtrimref.so by oracle/Makefile): its seeded generators
(core/synthetic.hpp), pq::train, trim::build_landmarks, ivf::build_ivf, and
the three searches in ivf/ivf.hpp. Each fixture stores the index arrays (so
the GPU consumes exactly the reference-built bytes) and the reference's
outputs: ids, dist_sq and counters {dc, edc, pruned, evaluated, hops} plus
coarse_dc per query.

    python tests/golden/make_golden.py        # needs /root/reference
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import RefOracle, build, make_reference_index  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, ix, qs, cases, extra=None):
    arrs = dict(dim=ix.dim, m=ix.m, ksub=ix.ksub, sub_dims=ix.sub_dims, centroids=ix.centroids,
                coarse=ix.coarse, list_offsets=ix.list_offsets, list_ids=ix.list_ids,
                list_codes=ix.list_codes, list_lx=ix.list_lx, vectors=ix.vectors, queries=qs)
    for cname, res in cases.items():
        for k, v in res.items():
            arrs[f"{cname}__{k}"] = v
    arrs["cases"] = np.array(sorted(cases.keys()))
    if extra:
        arrs.update(extra)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrs)
    sz = os.path.getsize(os.path.join(OUT, name + ".npz"))
    print(f"{name}: {len(cases)} cases, {sz/1e6:.2f} MB")


def knn(ref, ix, qs, k, nprobe, gamma):
    ids, dist, ct, cdc = ref.search_knn(ix, qs, k, nprobe, gamma)
    return dict(kind=np.array("knn"), k=k, nprobe=nprobe, gamma=gamma, ids=ids, dist=dist,
                counters=ct, coarse_dc=cdc)


def rng_(ref, ix, qs, radius, nprobe, gamma):
    offs, ids, dist, ct, cdc = ref.search_range(ix, qs, radius, nprobe, gamma)
    return dict(kind=np.array("range"), radius=np.float32(radius), nprobe=nprobe, gamma=gamma,
                offsets=offs, ids=ids, dist=dist, counters=ct, coarse_dc=cdc)


def base(ref, ix, qs, k, nprobe, kp):
    ids, dist, ct, cdc = ref.search_baseline(ix, qs, k, nprobe, kp)
    return dict(kind=np.array("baseline"), k=k, nprobe=nprobe, k_prime=kp, ids=ids, dist=dist,
                counters=ct, coarse_dc=cdc)


def main():
    build()
    ref = RefOracle()

    # 1. The reference's own IvfFixture shape (proj/tests/test_ivf.cpp:17-41):
    #    64 blobs, sigma 0.4, m = dim/4, c = 64, 8 k-means iterations.
    seed = 40
    centers = ref.make_normal(64, 16, seed)
    ds = ref.make_blobs(centers, 1000, 0.4, seed + 1)
    ix = make_reference_index(ref, ds, m=4, c=64, iters=8, pq_seed=seed + 2, nlist=20,
                              ivf_seed=seed + 3)
    qs = ref.make_normal(20, 16, 41)
    cases = {}
    for g in (0.0, 0.35, 1.0):
        for k in (1, 10):
            cases[f"knn_full_g{g}_k{k}"] = knn(ref, ix, qs, k, 20, g)
        cases[f"knn_np5_g{g}_k10"] = knn(ref, ix, qs, 10, 5, g)
        cases[f"range_full_g{g}"] = rng_(ref, ix, qs, 3.0, 20, g)
        cases[f"range_np5_g{g}"] = rng_(ref, ix, qs, 3.0, 5, g)
    cases["range_r0"] = rng_(ref, ix, qs, 0.0, 20, 0.35)
    cases["baseline_full_exact"] = base(ref, ix, qs, 10, 20, 1000)
    cases["baseline_np8_kp100"] = base(ref, ix, qs, 10, 8, 100)
    cases["baseline_np12_kp10"] = base(ref, ix, qs, 10, 12, 10)
    cases["knn_k100_np3"] = knn(ref, ix, qs, 100, 3, 0.35)
    save("ivf_fixture", ix, qs, cases)

    # 2. Config-1 shape (BASELINE.json configs[0]) at 3,000 rows: D=128, 64
    #    blobs sigma 0.3, M=16 x 256, flat (nlist=1), k=10.
    centers = ref.make_normal(64, 128, 0)
    ds = ref.make_blobs(centers, 3000, 0.3, 1)
    qs = ref.make_blobs(centers, 40, 0.3, 2)
    ix = make_reference_index(ref, ds, m=16, c=256, iters=25, pq_seed=3, nlist=1, ivf_seed=4)
    r = ref.pick_radius(ds, qs, 20 / 3000, sample_rows=2000, sample_queries=40, seed=1)
    cases = {}
    for g in (0.0, 0.605, 1.0):
        cases[f"knn_g{g}"] = knn(ref, ix, qs, 10, 1, g)
        cases[f"range_g{g}"] = rng_(ref, ix, qs, r, 1, g)
    cases["knn_k64_g0.605"] = knn(ref, ix, qs, 64, 1, 0.605)
    cases["baseline_kp100"] = base(ref, ix, qs, 10, 1, 100)
    save("flat_d128_m16", ix, qs, cases, extra=dict(radius=np.float32(r)))

    # 3. Config-2 shape (IVF, D=96, M=48) at 3,000 rows, nlist=32.
    centers = ref.make_normal(64, 96, 7)
    ds = ref.make_blobs(centers, 3000, 0.3, 8)
    qs = ref.make_blobs(centers, 40, 0.3, 9)
    ix = make_reference_index(ref, ds, m=48, c=256, iters=10, pq_seed=10, nlist=32, ivf_seed=11)
    cases = {}
    for g in (0.6, 0.8, 1.0):
        cases[f"knn_np8_g{g}"] = knn(ref, ix, qs, 10, 8, g)
    cases["knn_np32_g0"] = knn(ref, ix, qs, 10, 32, 0.0)
    cases["range_np8_g0.8"] = rng_(ref, ix, qs, 2.9, 8, 0.8)
    cases["baseline_np8_kp1000"] = base(ref, ix, qs, 10, 8, 1000)
    save("ivf_d96_m48", ix, qs, cases)

    # 4. Config-4 shape: uniform [0,1) then L2-normalised, D=960, M=120, k=100.
    ds = ref.make_uniform(300, 960, 12, True)
    qs = ref.make_uniform(12, 960, 13, True)
    ix = make_reference_index(ref, ds, m=120, c=256, iters=6, pq_seed=14, nlist=1, ivf_seed=15)
    cases = {}
    for g in (0.5, 0.7, 0.9):
        cases[f"knn_g{g}"] = knn(ref, ix, qs, 100, 1, g)
    save("flat_d960_m120", ix, qs, cases)


if __name__ == "__main__":
    main()
