"""Loader for tests/golden/*.npz (written by tests/golden/make_golden.py from
the reference itself)."""
import glob
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIELDS = ("dim", "m", "ksub", "sub_dims", "centroids", "coarse", "list_offsets", "list_ids",
          "list_codes", "list_lx", "vectors")


def names():
    """IVF / flat fixtures (graph fixtures: graph_names())."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith("graph_"))


def graph_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "graph_*.npz")))


GRAPH_FIELDS = ("entry", "M", "efc", "ksub", "sub_dims", "centroids", "codes", "lx", "vectors")


def load_graph(name):
    """(graph namespace with per-level offsets/nbrs + landmark store, queries, cases)."""
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    g = SimpleNamespace(**{f: (z[f].item() if z[f].ndim == 0 else z[f]) for f in GRAPH_FIELDS})
    lv = int(z["levels"])
    g.offsets = [z[f"offsets_{i}"] for i in range(lv)]
    g.nbrs = [z[f"nbrs_{i}"] for i in range(lv)]
    g.n, g.dim = g.vectors.shape
    g.m = g.codes.shape[1]
    cases = {}
    for c in z["cases"]:
        c = str(c)
        d = {key[len(c) + 2:]: (z[key].item() if z[key].ndim == 0 else z[key])
             for key in z.files if key.startswith(c + "__")}
        d["kind"] = str(d["kind"])
        cases[c] = d
    return g, z["queries"], cases


def host_graph(g):
    from oracle.oracle import HostGraph
    return HostGraph(n=g.n, M=g.M, efc=g.efc, entry=g.entry, offsets=list(g.offsets), nbrs=list(g.nbrs),
                     dim=g.dim, m=g.m, ksub=g.ksub, sub_dims=g.sub_dims, centroids=g.centroids,
                     codes=g.codes, lx=g.lx, vectors=g.vectors)


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    ix = SimpleNamespace(**{f: (z[f].item() if z[f].ndim == 0 else z[f]) for f in FIELDS})
    cases = {}
    for c in z["cases"]:
        c = str(c)
        d = {}
        for key in z.files:
            if key.startswith(c + "__"):
                v = z[key]
                d[key[len(c) + 2:]] = v.item() if v.ndim == 0 else v
        d["kind"] = str(d["kind"])
        cases[c] = d
    return ix, z["queries"], cases


def all_cases():
    out = []
    for n in names():
        ix, qs, cases = load(n)
        for c in sorted(cases):
            out.append((n, c))
    return out


def host_index(ix):
    from oracle.oracle import HostIndex
    return HostIndex(**{f: getattr(ix, f) for f in FIELDS})
