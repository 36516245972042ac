"""Generates tests/golden/graph_*.npz from the REFERENCE itself: seeded data
(core/synthetic.hpp), graph::build_graph (graph/hnsw.hpp:165-268), pq::train +
trim::build_landmarks, and graph::search_trim_knn / search_trim_range
(graph/search.hpp:188-347) run by the unmodified reference headers
(oracle/_ref/libtrimref.so). Each fixture stores the graph (per-level CSR),
the landmark store, the vectors, the queries and the reference's outputs:
ids, dist_sq and counters {dc, edc, pruned, evaluated, hops} per query.

    python tests/golden/make_golden_graph.py      # needs /root/reference
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import RefOracle, build, make_reference_graph  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, g, qs, cases):
    arrs = dict(entry=g.entry, M=g.M, efc=g.efc, ksub=g.ksub, sub_dims=g.sub_dims, centroids=g.centroids,
                codes=g.codes, lx=g.lx, vectors=g.vectors, levels=g.levels, queries=qs)
    for i in range(g.levels):
        arrs[f"offsets_{i}"] = g.offsets[i]
        arrs[f"nbrs_{i}"] = g.nbrs[i]
    for cname, res in cases.items():
        for k, v in res.items():
            arrs[f"{cname}__{k}"] = v
    arrs["cases"] = np.array(sorted(cases.keys()))
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrs)
    print(f"{name}: levels {g.levels}, {len(cases)} cases, {os.path.getsize(os.path.join(OUT, name + '.npz')) / 1e6:.2f} MB")


def knn(ref, g, qs, k, ef, gamma):
    ids, dist, cnt, ct = ref.graph_search(g, qs, "trim_knn", k=k, ef=ef, gamma=gamma)
    return dict(kind=np.array("knn"), k=k, ef=ef, gamma=gamma, ids=ids, dist=dist, counts=cnt, counters=ct)


def rng_(ref, g, qs, radius, ef, gamma):
    cap = g.n
    ids, dist, cnt, ct = ref.graph_search(g, qs, "trim_range", ef=ef, gamma=gamma, radius=radius, cap=cap)
    offs = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64)
    flat_ids = np.concatenate([ids[i, :cnt[i]] for i in range(len(cnt))]).astype(np.uint32)
    flat_d = np.concatenate([dist[i, :cnt[i]] for i in range(len(cnt))]).astype(np.float32)
    return dict(kind=np.array("range"), radius=np.float32(radius), ef=ef, gamma=gamma, offsets=offs,
                ids=flat_ids, dist=flat_d, counters=ct)


def main():
    build()
    ref = RefOracle()
    # d = 32, 16 blobs, M = 8, m = 8 (4-wide subspaces)
    c = ref.make_normal(16, 32, 0)
    base = ref.make_blobs(c, 3000, 0.3, 1)
    qs = ref.make_blobs(c, 48, 0.3, 2)
    g = make_reference_graph(ref, base, M=8, efc=64, graph_seed=5, m=8, pq_seed=3)
    cases = {}
    for gam in (0.0, 0.6, 1.0):
        cases[f"knn_k10_ef32_g{gam}"] = knn(ref, g, qs, 10, 32, gam)
    cases["knn_k1_ef1_g0.8"] = knn(ref, g, qs, 1, 1, 0.8)
    cases["knn_k50_ef64_g0.8"] = knn(ref, g, qs, 50, 64, 0.8)
    cases["knn_k100_ef256_g0.5"] = knn(ref, g, qs, 100, 256, 0.5)
    for gam in (0.0, 0.8):
        cases[f"range_r2.3_ef32_g{gam}"] = rng_(ref, g, qs, 2.3, 32, gam)
    cases["range_r2.6_ef8_g0.8"] = rng_(ref, g, qs, 2.6, 8, 0.8)
    save("graph_d32_m8", g, qs, cases)
    # d = 64, 32 blobs, M = 16, m = 16 (4-wide), a second codebook shape
    c = ref.make_normal(32, 64, 10)
    base = ref.make_blobs(c, 4000, 0.3, 11)
    qs = ref.make_blobs(c, 32, 0.3, 12)
    g = make_reference_graph(ref, base, M=16, efc=80, graph_seed=7, m=16, pq_seed=13)
    cases = {}
    for gam in (0.0, 0.8):
        cases[f"knn_k10_ef48_g{gam}"] = knn(ref, g, qs, 10, 48, gam)
    cases["knn_k32_ef128_g0.9"] = knn(ref, g, qs, 32, 128, 0.9)
    cases["range_r3.2_ef48_g0.8"] = rng_(ref, g, qs, 3.2, 48, 0.8)
    save("graph_d64_m16", g, qs, cases)


if __name__ == "__main__":
    main()
