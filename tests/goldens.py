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
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


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
