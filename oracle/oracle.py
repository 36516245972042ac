"""TEST INFRASTRUCTURE ONLY — ctypes wrappers over the two CPU checkers.

* ``C``   : oracle/_build/liboracle.so, the plain-C restatement
            (oracle/trim_oracle.c) of the reference's hot path;
* ``Ref`` : oracle/_ref/libtrimref.so, the unmodified reference headers
            compiled in place (oracle/ref_harness.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline / reference
legs may import this module. The product package never does.

Both take an index as a ``HostIndex`` (numpy arrays in the CSR layout of
oracle/trim_oracle.h) and return numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtrimref.so")

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)


def build(quiet: bool = True) -> None:
    """Build liboracle.so (and libtrimref.so when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclass
class HostIndex:
    """CSR IVF index + vectors (oracle/trim_oracle.h layout)."""

    dim: int
    m: int
    ksub: int
    sub_dims: np.ndarray  # u32[m]
    centroids: np.ndarray  # f32[ksub*dim]
    coarse: np.ndarray  # f32[nlist*dim]
    list_offsets: np.ndarray  # u64[nlist+1]
    list_ids: np.ndarray  # u32[total]
    list_codes: np.ndarray  # u8[total, code_stride]
    list_lx: np.ndarray  # f32[total]
    vectors: np.ndarray  # f32[n, dim]
    sub_offsets: np.ndarray = field(default=None)

    def __post_init__(self):
        self.sub_dims = np.ascontiguousarray(self.sub_dims, dtype=np.uint32)
        self.sub_offsets = np.ascontiguousarray(
            np.concatenate([[0], np.cumsum(self.sub_dims)[:-1]]).astype(np.uint32))
        self.centroids = np.ascontiguousarray(self.centroids, dtype=np.float32).ravel()
        self.coarse = np.ascontiguousarray(self.coarse, dtype=np.float32).ravel()
        self.list_offsets = np.ascontiguousarray(self.list_offsets, dtype=np.uint64)
        self.list_ids = np.ascontiguousarray(self.list_ids, dtype=np.uint32)
        codes = np.asarray(self.list_codes, dtype=np.uint8)
        if codes.ndim == 1:
            codes = codes.reshape(-1, self.m)
        self.list_codes = np.ascontiguousarray(codes)
        self.list_lx = np.ascontiguousarray(self.list_lx, dtype=np.float32)
        self.vectors = np.ascontiguousarray(self.vectors, dtype=np.float32).reshape(-1, self.dim)

    @property
    def nlist(self) -> int:
        return len(self.list_offsets) - 1

    @property
    def n(self) -> int:
        return self.vectors.shape[0]

    @property
    def code_stride(self) -> int:
        return self.list_codes.shape[1] if self.list_codes.size else self.m


# ---------------------------------------------------------------- C restatement
class _OrIndex(C.Structure):
    _fields_ = [
        ("dim", C.c_uint32), ("m", C.c_uint32), ("ksub", C.c_uint32),
        ("sub_dims", _u32p), ("sub_offsets", _u32p), ("centroids", _f32p),
        ("nlist", C.c_uint32), ("coarse", _f32p),
        ("list_offsets", _u64p), ("list_ids", _u32p), ("list_codes", _u8p),
        ("code_stride", C.c_uint32), ("list_lx", _f32p),
        ("n", C.c_uint64), ("vectors", _f32p),
    ]


class _OrGraph(C.Structure):
    _fields_ = [("n", C.c_uint64), ("levels", C.c_uint32), ("entry", C.c_uint32), ("offsets", _u64p),
                ("nbr_base", _u64p), ("nbrs", _u32p)]


class OrCounters(C.Structure):
    _fields_ = [("dc", C.c_uint64), ("edc", C.c_uint64), ("pruned", C.c_uint64),
                ("evaluated", C.c_uint64), ("hops", C.c_uint64)]


def counters_array(cs) -> np.ndarray:
    """(nq, 5) u64 array {dc, edc, pruned, evaluated, hops}."""
    return np.array([[c.dc, c.edc, c.pruned, c.evaluated, c.hops] for c in cs], dtype=np.uint64)


class COracle:
    """The plain-C restatement (oracle/trim_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.or_last_error.restype = C.c_char_p
        L.or_euclidean_sq.restype = C.c_float
        L.or_euclidean_sq.argtypes = [_f32p, _f32p, C.c_size_t]
        L.or_strict_lb.restype = C.c_float
        L.or_strict_lb.argtypes = [C.c_float, C.c_float]
        L.or_relaxed_lb.restype = C.c_float
        L.or_relaxed_lb.argtypes = [C.c_float, C.c_float, C.c_float]
        L.or_adc_lookup.restype = C.c_float
        L.or_adc_lookup.argtypes = [_f32p, C.c_uint32, C.c_uint32, _u8p]
        L.or_build_distance_table.argtypes = [C.POINTER(_OrIndex), _f32p, _f32p]
        L.or_probe_order.restype = C.c_uint32
        L.or_probe_order.argtypes = [C.POINTER(_OrIndex), _f32p, C.c_uint32, _u32p, _u64p]
        L.or_search_trim_knn_batch.argtypes = [
            C.POINTER(_OrIndex), _f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_float,
            _u32p, _f32p, C.POINTER(OrCounters), _u64p, C.c_int]
        L.or_search_trim_range_batch.argtypes = [
            C.POINTER(_OrIndex), _f32p, C.c_uint64, _f32p, C.c_uint32, C.c_float,
            _u64p, C.POINTER(_u32p), C.POINTER(_f32p), C.POINTER(OrCounters), _u64p, C.c_int]
        L.or_search_baseline_ivfpq_batch.argtypes = [
            C.POINTER(_OrIndex), _f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
            _u32p, _f32p, C.POINTER(OrCounters), _u64p, C.c_int]
        L.or_build_landmarks.argtypes = [C.POINTER(_OrIndex), _f32p, C.c_uint64, _u8p,
                                         C.c_uint32, _f32p, C.c_int]
        L.or_brute_force_knn_batch.argtypes = [_f32p, C.c_uint64, C.c_uint32, _f32p,
                                               C.c_uint64, C.c_uint32, _u32p, _f32p, C.c_int]
        L.or_graph_search_trim_knn_batch.argtypes = [
            C.POINTER(_OrGraph), C.POINTER(_OrIndex), _f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_float,
            _u32p, _f32p, C.POINTER(OrCounters), C.c_int]
        L.or_graph_search_trim_range_batch.argtypes = [
            C.POINTER(_OrGraph), C.POINTER(_OrIndex), _f32p, C.c_uint64, _f32p, C.c_uint32, C.c_float,
            _u64p, C.POINTER(_u32p), C.POINTER(_f32p), C.POINTER(OrCounters), C.c_int]
        L.or_free.argtypes = [C.c_void_p]

    def _graph(self, g: "HostGraph"):
        """(_OrGraph, _OrIndex landmark store, keep-alive arrays)."""
        offs = np.ascontiguousarray(np.concatenate([np.asarray(o, np.uint64) for o in g.offsets]))
        sizes = [int(np.asarray(o)[-1]) for o in g.offsets]
        base = np.ascontiguousarray(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64))
        nb = np.ascontiguousarray(np.concatenate([np.asarray(x, np.uint32) for x in g.nbrs]))
        sub = np.ascontiguousarray(g.sub_dims, np.uint32)
        suboff = np.ascontiguousarray(np.concatenate([[0], np.cumsum(sub)[:-1]]).astype(np.uint32))
        cent = np.ascontiguousarray(g.centroids, np.float32).ravel()
        codes = np.ascontiguousarray(g.codes, np.uint8)
        lx = np.ascontiguousarray(g.lx, np.float32)
        vec = np.ascontiguousarray(g.vectors, np.float32)
        og = _OrGraph(g.n, len(g.offsets), g.entry, _ptr(offs, _u64p), _ptr(base, _u64p), _ptr(nb, _u32p))
        lm = _OrIndex(g.dim, g.m, g.ksub, _ptr(sub, _u32p), _ptr(suboff, _u32p), _ptr(cent, _f32p), 0, None,
                      None, None, _ptr(codes, _u8p), codes.shape[1], _ptr(lx, _f32p), g.n, _ptr(vec, _f32p))
        return og, lm, (offs, base, nb, sub, suboff, cent, codes, lx, vec)

    def graph_search(self, g: "HostGraph", qs, kind: str, *, k=0, ef=0, gamma=0.0, radius=0.0, threads=0):
        """C restatement of graph::search_trim_knn ("trim_knn": ids, dist [nq, k]
        padded, counters [nq, 5]) / search_trim_range ("trim_range": offsets,
        ids, dist, counters)."""
        qs = np.ascontiguousarray(qs, np.float32).reshape(-1, g.dim)
        nq = qs.shape[0]
        og, lm, keep = self._graph(g)
        cs = (OrCounters * max(nq, 1))()
        th = threads or os.cpu_count()
        if kind == "trim_knn":
            ids = np.zeros((nq, k), np.uint32)
            dist = np.zeros((nq, k), np.float32)
            rc = self.lib.or_graph_search_trim_knn_batch(C.byref(og), C.byref(lm), _ptr(qs, _f32p), nq, k, ef,
                                                         np.float32(gamma), _ptr(ids, _u32p), _ptr(dist, _f32p),
                                                         cs, th)
            self._err(rc, "graph search_trim_knn")
            return ids, dist, counters_array(cs[:nq])
        rad = np.ascontiguousarray(np.broadcast_to(np.float32(radius), (nq,)), np.float32)
        offs = np.zeros(nq + 1, np.uint64)
        pids, pd = _u32p(), _f32p()
        rc = self.lib.or_graph_search_trim_range_batch(C.byref(og), C.byref(lm), _ptr(qs, _f32p), nq,
                                                       _ptr(rad, _f32p), ef, np.float32(gamma), _ptr(offs, _u64p),
                                                       C.byref(pids), C.byref(pd), cs, th)
        self._err(rc, "graph search_trim_range")
        tot = int(offs[-1])
        ids = np.ctypeslib.as_array(pids, shape=(max(tot, 1),))[:tot].copy()
        dist = np.ctypeslib.as_array(pd, shape=(max(tot, 1),))[:tot].copy()
        self.lib.or_free(C.cast(pids, C.c_void_p))
        self.lib.or_free(C.cast(pd, C.c_void_p))
        return offs, ids, dist, counters_array(cs[:nq])

    def _err(self, rc: int, what: str):
        if rc != 0:
            msg = self.lib.or_last_error().decode()
            if rc == 1:
                raise ValueError(f"{what}: {msg}")
            raise RuntimeError(f"{what} rc={rc}: {msg}")

    @staticmethod
    def _ix(ix: HostIndex) -> _OrIndex:
        return _OrIndex(ix.dim, ix.m, ix.ksub, _ptr(ix.sub_dims, _u32p), _ptr(ix.sub_offsets, _u32p),
                        _ptr(ix.centroids, _f32p), ix.nlist, _ptr(ix.coarse, _f32p),
                        _ptr(ix.list_offsets, _u64p), _ptr(ix.list_ids, _u32p),
                        _ptr(ix.list_codes, _u8p), ix.code_stride, _ptr(ix.list_lx, _f32p),
                        ix.n, _ptr(ix.vectors, _f32p))

    def euclidean_sq(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.or_euclidean_sq(_ptr(a, _f32p), _ptr(b, _f32p), a.size)

    def strict_lb(self, a, b):
        return self.lib.or_strict_lb(a, b)

    def relaxed_lb(self, a, b, g):
        return self.lib.or_relaxed_lb(a, b, g)

    def distance_table(self, ix: HostIndex, q) -> np.ndarray:
        q = np.ascontiguousarray(q, np.float32)
        out = np.empty((ix.m, ix.ksub), np.float32)
        oi = self._ix(ix)
        self.lib.or_build_distance_table(C.byref(oi), _ptr(q, _f32p), _ptr(out, _f32p))
        return out

    def adc(self, table: np.ndarray, code) -> float:
        table = np.ascontiguousarray(table, np.float32)
        code = np.ascontiguousarray(code, np.uint8)
        return self.lib.or_adc_lookup(_ptr(table, _f32p), table.shape[0], table.shape[1],
                                      _ptr(code, _u8p))

    def probe_order(self, ix: HostIndex, q, nprobe: int) -> np.ndarray:
        q = np.ascontiguousarray(q, np.float32)
        out = np.empty(max(ix.nlist, 1), np.uint32)
        cdc = C.c_uint64(0)
        oi = self._ix(ix)
        n = self.lib.or_probe_order(C.byref(oi), _ptr(q, _f32p), nprobe, _ptr(out, _u32p),
                                    C.byref(cdc))
        return out[:n]

    def search_knn(self, ix: HostIndex, qs, k: int, nprobe: int, gamma: float, threads: int = 0):
        qs = np.ascontiguousarray(qs, np.float32).reshape(-1, ix.dim)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dist = np.zeros((nq, k), np.float32)
        cs = (OrCounters * max(nq, 1))()
        cdc = np.zeros(max(nq, 1), np.uint64)
        oi = self._ix(ix)
        rc = self.lib.or_search_trim_knn_batch(C.byref(oi), _ptr(qs, _f32p), nq, k, nprobe,
                                               np.float32(gamma), _ptr(ids, _u32p),
                                               _ptr(dist, _f32p), cs, _ptr(cdc, _u64p),
                                               threads or os.cpu_count())
        self._err(rc, "search_trim_ivf_knn")
        return ids, dist, counters_array(cs[:nq]), cdc[:nq]

    def search_range(self, ix: HostIndex, qs, radius, nprobe: int, gamma: float,
                     threads: int = 0):
        qs = np.ascontiguousarray(qs, np.float32).reshape(-1, ix.dim)
        nq = qs.shape[0]
        rad = np.ascontiguousarray(np.broadcast_to(np.float32(radius), (nq,)), np.float32) \
            if np.ndim(radius) == 0 else np.ascontiguousarray(radius, np.float32)
        offs = np.zeros(nq + 1, np.uint64)
        pids = _u32p()
        pd = _f32p()
        cs = (OrCounters * max(nq, 1))()
        cdc = np.zeros(max(nq, 1), np.uint64)
        oi = self._ix(ix)
        rc = self.lib.or_search_trim_range_batch(C.byref(oi), _ptr(qs, _f32p), nq,
                                                 _ptr(rad, _f32p), nprobe, np.float32(gamma),
                                                 _ptr(offs, _u64p), C.byref(pids), C.byref(pd),
                                                 cs, _ptr(cdc, _u64p), threads or os.cpu_count())
        self._err(rc, "search_trim_ivf_range")
        tot = int(offs[-1])
        ids = np.ctypeslib.as_array(pids, shape=(max(tot, 1),))[:tot].copy()
        dist = np.ctypeslib.as_array(pd, shape=(max(tot, 1),))[:tot].copy()
        self.lib.or_free(C.cast(pids, C.c_void_p))
        self.lib.or_free(C.cast(pd, C.c_void_p))
        return offs, ids, dist, counters_array(cs[:nq]), cdc[:nq]

    def search_baseline(self, ix: HostIndex, qs, k: int, nprobe: int, k_prime: int,
                        threads: int = 0):
        qs = np.ascontiguousarray(qs, np.float32).reshape(-1, ix.dim)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dist = np.zeros((nq, k), np.float32)
        cs = (OrCounters * max(nq, 1))()
        cdc = np.zeros(max(nq, 1), np.uint64)
        oi = self._ix(ix)
        rc = self.lib.or_search_baseline_ivfpq_batch(C.byref(oi), _ptr(qs, _f32p), nq, k, nprobe,
                                                     k_prime, _ptr(ids, _u32p), _ptr(dist, _f32p),
                                                     cs, _ptr(cdc, _u64p),
                                                     threads or os.cpu_count())
        self._err(rc, "search_baseline_ivfpq")
        return ids, dist, counters_array(cs[:nq]), cdc[:nq]

    def build_landmarks(self, ix: HostIndex, data, threads: int = 0):
        data = np.ascontiguousarray(data, np.float32).reshape(-1, ix.dim)
        n = data.shape[0]
        codes = np.zeros((n, ix.m), np.uint8)
        lx = np.zeros(n, np.float32)
        oi = self._ix(ix)
        rc = self.lib.or_build_landmarks(C.byref(oi), _ptr(data, _f32p), n, _ptr(codes, _u8p),
                                         ix.m, _ptr(lx, _f32p), threads or os.cpu_count())
        self._err(rc, "build_landmarks")
        return codes, lx

    def brute_force_knn(self, data, qs, k: int, threads: int = 0):
        data = np.ascontiguousarray(data, np.float32)
        qs = np.ascontiguousarray(qs, np.float32).reshape(-1, data.shape[1])
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dist = np.zeros((nq, k), np.float32)
        rc = self.lib.or_brute_force_knn_batch(_ptr(data, _f32p), data.shape[0], data.shape[1],
                                               _ptr(qs, _f32p), nq, k, _ptr(ids, _u32p),
                                               _ptr(dist, _f32p), threads or os.cpu_count())
        self._err(rc, "brute_force_knn")
        return ids, dist


# ------------------------------------------------------------------- reference
class _FlatIndex(C.Structure):
    _fields_ = [
        ("dim", C.c_uint32), ("m", C.c_uint32), ("c", C.c_uint32), ("sub_dims", _u32p),
        ("centroids", _f32p), ("nlist", C.c_uint32), ("coarse", _f32p),
        ("list_offsets", _u64p), ("list_ids", _u32p), ("list_codes", _u8p),
        ("code_stride", C.c_uint32), ("list_lx", _f32p), ("n", C.c_uint64),
        ("vectors", _f32p),
    ]


class _FlatGraph(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("M", C.c_uint32), ("levels", C.c_uint32), ("entry", C.c_uint32),
        ("efc", C.c_uint32), ("offsets", _u64p), ("nbr_base", _u64p), ("nbrs", _u32p),
    ]


@dataclass
class HostGraph:
    """HNSW GraphIndex (graph/hnsw.hpp:22-35) as per-level CSR arrays, plus the
    LandmarkStore (trim/landmarks.hpp:18-28) and VectorDataset it searches."""

    n: int
    M: int
    efc: int
    entry: int
    offsets: list  # per level: u64[n+1]
    nbrs: list  # per level: u32[offsets[-1]]
    dim: int = 0
    m: int = 0
    ksub: int = 256
    sub_dims: np.ndarray = None  # u32[m]
    centroids: np.ndarray = None  # f32[ksub*dim]
    codes: np.ndarray = None  # u8[n, m]
    lx: np.ndarray = None  # f32[n]
    vectors: np.ndarray = None  # f32[n, dim]

    @property
    def levels(self) -> int:
        return len(self.offsets)

    def flat(self):
        """(_FlatGraph, keep-alive arrays) for the harness."""
        offs = np.ascontiguousarray(np.concatenate([np.asarray(o, np.uint64) for o in self.offsets]))
        sizes = [int(np.asarray(o)[-1]) for o in self.offsets]
        base = np.ascontiguousarray(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64))
        nb = np.ascontiguousarray(np.concatenate([np.asarray(x, np.uint32) for x in self.nbrs]))
        fg = _FlatGraph(self.n, self.M, self.levels, self.entry, self.efc, _ptr(offs, _u64p),
                        _ptr(base, _u64p), _ptr(nb, _u32p))
        return fg, (offs, base, nb)


def ref_available(path: str = REF_SO) -> bool:
    return os.path.exists(path)


class RefOracle:
    """The reference itself (headers compiled in place; oracle/ref_harness.cpp)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: build it with `make -C oracle` where /root/reference exists")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_uint]
        L.ref_make_normal.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, _f32p]
        L.ref_make_blobs.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_float,
                                     C.c_uint64, _f32p]
        L.ref_make_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, _f32p]
        L.ref_pq_train.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_uint32, C.c_uint64, C.c_uint64, _u32p, _f32p, _f64p]
        L.ref_build_landmarks.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                          _u32p, _f32p, _u8p, C.c_uint32, _f32p]
        L.ref_build_ivf.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                    _f32p, _u8p, C.c_uint32, _f32p, C.c_uint32, C.c_uint64,
                                    C.c_uint32, _f32p, _u64p, _u32p, _u8p, _f32p]
        L.ref_search_knn_batch.argtypes = [C.POINTER(_FlatIndex), _f32p, C.c_uint64, C.c_uint32,
                                           C.c_uint32, C.c_double, _u32p, _f32p, _u64p]
        L.ref_search_range_batch.argtypes = [C.POINTER(_FlatIndex), _f32p, C.c_uint64, _f32p,
                                             C.c_uint32, C.c_double, C.c_uint64, _u32p, _f32p,
                                             _u64p, _u64p]
        L.ref_search_baseline_batch.argtypes = [C.POINTER(_FlatIndex), _f32p, C.c_uint64,
                                                C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _f32p,
                                                _u64p]
        cp = C.c_char_p
        L.ref_ivf_save.argtypes = [C.POINTER(_FlatIndex), C.c_double, C.c_uint64, C.c_uint32, cp]
        L.ref_ivf_load_sizes.argtypes = [cp, _u64p, _u64p, _u32p, _u32p, _u64p]
        L.ref_ivf_load.argtypes = [cp, _u32p, _f32p, _f32p, _u64p, _u32p, _u8p, _f32p, _f64p, _u64p, _u32p]
        L.ref_landmarks_save.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _f32p, C.c_uint64,
                                         _u8p, _f32p, cp]
        L.ref_landmarks_load.argtypes = [cp, C.c_uint64, _u8p, _f32p]
        L.ref_profile_save.argtypes = [C.c_double, C.c_double, cp]
        L.ref_profile_load.argtypes = [cp, _f64p, _f64p]
        L.ref_write_fvecs.argtypes = [_f32p, C.c_uint64, C.c_uint32, cp]
        L.ref_load_fvecs.argtypes = [cp, C.c_uint64, C.c_uint32, _f32p]
        L.ref_session_create.restype = C.c_void_p
        L.ref_session_create.argtypes = [C.POINTER(_FlatIndex)]
        L.ref_session_destroy.argtypes = [C.c_void_p]
        L.ref_session_run.argtypes = [C.c_void_p, C.c_int, _f32p, C.c_uint64, C.c_uint32,
                                      C.c_uint32, C.c_double, C.c_double, _f64p, _u64p]
        L.ref_session_knn.argtypes = [C.c_void_p, _f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double,
                                      _u32p, _f32p, _u64p]
        L.ref_session_range.argtypes = [C.c_void_p, _f32p, C.c_uint64, _f32p, C.c_uint32, C.c_double,
                                        C.c_uint64, _u32p, _f32p, _u64p, _u64p]
        L.ref_ground_truth_knn.argtypes = [_f32p, C.c_uint64, C.c_uint32, _f32p, C.c_uint64,
                                           C.c_uint32, _u32p, _f32p]
        L.ref_pick_radius.argtypes = [_f32p, C.c_uint64, C.c_uint32, _f32p, C.c_uint64,
                                      C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, _f32p]
        L.ref_calibrate_empirical.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                              C.c_uint32, _u32p, _f32p, _u8p, C.c_uint32, _f32p,
                                              _f32p, C.c_uint64, C.c_uint64, C.c_uint64,
                                              C.c_uint64, C.c_double, _f64p]
        L.ref_euclidean_sq.restype = C.c_float
        L.ref_euclidean_sq.argtypes = [_f32p, _f32p, C.c_uint64]
        L.ref_strict_lb.argtypes = [C.c_float, C.c_float, _f32p]
        L.ref_relaxed_lb.argtypes = [C.c_float, C.c_float, C.c_float, _f32p]
        L.ref_build_table.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _f32p, _f32p,
                                      _f32p]
        L.ref_adc_lookup.restype = C.c_float
        L.ref_adc_lookup.argtypes = [_f32p, C.c_uint32, C.c_uint32, _u8p]
        L.ref_graph_build.restype = C.c_void_p
        L.ref_graph_build.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_load.restype = C.c_void_p
        L.ref_graph_load.argtypes = [C.c_char_p]
        L.ref_graph_session_create.restype = C.c_void_p
        L.ref_graph_session_create.argtypes = [C.POINTER(_FlatGraph), C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                               _f32p, _u8p, _f32p, _f32p]
        L.ref_graph_session_run.argtypes = [C.c_void_p, C.c_int, _f32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                            C.c_double, C.c_double, _f64p, _u64p]
        L.ref_graph_info.argtypes = [C.c_void_p, _u32p, _u32p, _u64p]
        L.ref_graph_export.argtypes = [C.c_void_p, C.c_uint32, _u64p, _u32p]
        L.ref_graph_save.argtypes = [C.POINTER(_FlatGraph), C.c_char_p]
        L.ref_graph_search_batch.argtypes = [C.POINTER(_FlatGraph), C.c_uint32, C.c_uint32, C.c_uint32,
                                             _u32p, _f32p, _u8p, _f32p, _f32p, _f32p, C.c_uint64,
                                             C.c_int, C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                             C.c_uint64, _u32p, _f32p, _u64p, _u64p]
        self._keep = []

    def _err(self, rc: int, what: str):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            if rc == 1:
                raise ValueError(f"{what}: {msg}")
            raise RuntimeError(f"{what} rc={rc}: {msg}")

    def set_threads(self, t: int):
        self.lib.ref_set_threads(t)

    # -- HNSW graph (graph/hnsw.hpp:165-268) and graph searches (graph/search.hpp) --
    def build_graph(self, data, M, efc, seed) -> HostGraph:
        data = np.ascontiguousarray(data, np.float32)
        n, dim = data.shape
        h = self.lib.ref_graph_build(_ptr(data, _f32p), n, dim, M, efc, seed)
        if not h:
            raise ValueError(f"build_graph: {self.lib.ref_last_error().decode()}")
        g = self._export_graph(h, n)
        g.M, g.efc, g.dim, g.vectors = M, efc, dim, data
        return g

    def graph_load(self, path: str, n: int) -> HostGraph:
        """graph::GraphIndex::load (graph/hnsw.hpp:58-83); graph fields only."""
        h = self.lib.ref_graph_load(path.encode())
        if not h:
            msg = self.lib.ref_last_error().decode()
            raise RuntimeError(f"graph_load: {msg}")
        return self._export_graph(h, n)

    def _export_graph(self, h, n) -> HostGraph:
        try:
            lv, en = C.c_uint32(0), C.c_uint32(0)
            self.lib.ref_graph_info(h, C.byref(lv), C.byref(en), None)
            sizes = np.zeros(lv.value, np.uint64)
            self.lib.ref_graph_info(h, C.byref(lv), C.byref(en), _ptr(sizes, _u64p))
            offs, nbrs = [], []
            for lvl in range(lv.value):
                o = np.zeros(n + 1, np.uint64)
                nb = np.zeros(max(int(sizes[lvl]), 1), np.uint32)
                self.lib.ref_graph_export(h, lvl, _ptr(o, _u64p), _ptr(nb, _u32p))
                offs.append(o)
                nbrs.append(nb[:int(sizes[lvl])])
        finally:
            self.lib.ref_graph_free(h)
        return HostGraph(n=n, M=0, efc=0, entry=en.value, offsets=offs, nbrs=nbrs)

    def graph_session(self, g: HostGraph):
        """Resident reference graph + landmarks + vectors (for timing)."""
        fg, keep = g.flat()
        arrs = [np.ascontiguousarray(g.sub_dims, np.uint32), np.ascontiguousarray(g.centroids, np.float32).ravel(),
                np.ascontiguousarray(g.codes, np.uint8), np.ascontiguousarray(g.lx, np.float32),
                np.ascontiguousarray(g.vectors, np.float32)]
        h = self.lib.ref_graph_session_create(C.byref(fg), g.dim, g.m, g.ksub, _ptr(arrs[0], _u32p),
                                              _ptr(arrs[1], _f32p), _ptr(arrs[2], _u8p), _ptr(arrs[3], _f32p),
                                              _ptr(arrs[4], _f32p))
        if not h:
            raise ValueError(f"graph_session: {self.lib.ref_last_error().decode()}")
        return h

    def graph_session_run(self, sess, kind: str, qs, *, k=0, ef=0, gamma=0.0, radius=0.0):
        """-> (seconds, counters summed over the queries [6])."""
        qs = np.ascontiguousarray(qs, np.float32)
        sec = C.c_double(0)
        ct = np.zeros(6, np.uint64)
        self._err(self.lib.ref_graph_session_run(sess, {"trim_knn": 0, "trim_range": 1}[kind], _ptr(qs, _f32p),
                                                 qs.shape[0], k, ef, gamma, radius, C.byref(sec), _ptr(ct, _u64p)),
                  "graph_session_run")
        return sec.value, ct

    def graph_session_destroy(self, sess):
        self.lib.ref_graph_free(sess)

    def graph_save(self, g: HostGraph, path: str):
        fg, keep = g.flat()
        self._err(self.lib.ref_graph_save(C.byref(fg), path.encode()), "graph_save")

    def graph_search(self, g: HostGraph, qs, kind: str, *, k=0, ef=0, gamma=0.0, radius=0.0, cap=0):
        """kind: "trim_knn" (graph/search.hpp:188-264), "trim_range" (:267-347,
        results truncated at cap per query) or "baseline_knn" (:85-124).
        Returns ids, dist_sq ([nq, k] or [nq, cap]), counts[nq], counters[nq, 6]."""
        qs = np.ascontiguousarray(qs, np.float32)
        nq = qs.shape[0]
        kid = {"trim_knn": 0, "trim_range": 1, "baseline_knn": 2}[kind]
        w = cap if kid == 1 else k
        ids = np.full((nq, max(w, 1)), 0xFFFFFFFF, np.uint32)
        dist = np.full((nq, max(w, 1)), np.inf, np.float32)
        counts = np.zeros(nq, np.uint64)
        ct = np.zeros((nq, 6), np.uint64)
        fg, keep = g.flat()
        sub = np.ascontiguousarray(g.sub_dims, np.uint32)
        cent = np.ascontiguousarray(g.centroids, np.float32).ravel()
        codes = np.ascontiguousarray(g.codes, np.uint8)
        lx = np.ascontiguousarray(g.lx, np.float32)
        vec = np.ascontiguousarray(g.vectors, np.float32)
        rc = self.lib.ref_graph_search_batch(C.byref(fg), g.dim, g.m, g.ksub, _ptr(sub, _u32p),
                                             _ptr(cent, _f32p), _ptr(codes, _u8p), _ptr(lx, _f32p),
                                             _ptr(vec, _f32p), _ptr(qs, _f32p), nq, kid, k, ef, gamma,
                                             radius, cap, _ptr(ids, _u32p), _ptr(dist, _f32p),
                                             _ptr(counts, _u64p), _ptr(ct, _u64p))
        self._err(rc, f"graph {kind}")
        return ids[:, :w], dist[:, :w], counts, ct

    # -- generators (core/synthetic.hpp) --
    def make_normal(self, n, dim, seed) -> np.ndarray:
        out = np.empty((n, dim), np.float32)
        self._err(self.lib.ref_make_normal(n, dim, seed, _ptr(out, _f32p)), "make_normal")
        return out

    def make_blobs(self, centers, n, sigma, seed) -> np.ndarray:
        centers = np.ascontiguousarray(centers, np.float32)
        out = np.empty((n, centers.shape[1]), np.float32)
        self._err(self.lib.ref_make_blobs(_ptr(centers, _f32p), centers.shape[0],
                                          centers.shape[1], n, sigma, seed, _ptr(out, _f32p)),
                  "make_blobs")
        return out

    def make_uniform(self, n, dim, seed, normalize=True) -> np.ndarray:
        out = np.empty((n, dim), np.float32)
        self._err(self.lib.ref_make_uniform(n, dim, seed, int(normalize), _ptr(out, _f32p)),
                  "make_uniform")
        return out

    # -- build pipeline --
    def pq_train(self, data, m, c=256, iters=25, seed=1, train_sample=0):
        data = np.ascontiguousarray(data, np.float32)
        n, dim = data.shape
        sub = np.zeros(m, np.uint32)
        cent = np.zeros(c * dim, np.float32)
        mse = C.c_double(0)
        self._err(self.lib.ref_pq_train(_ptr(data, _f32p), n, dim, m, c, iters, seed,
                                        train_sample, _ptr(sub, _u32p), _ptr(cent, _f32p),
                                        C.byref(mse)), "pq_train")
        return sub, cent

    def build_landmarks(self, data, m, c, sub_dims, centroids):
        data = np.ascontiguousarray(data, np.float32)
        n, dim = data.shape
        sub_dims = np.ascontiguousarray(sub_dims, np.uint32)
        centroids = np.ascontiguousarray(centroids, np.float32)
        codes = np.zeros((n, m), np.uint8)
        lx = np.zeros(n, np.float32)
        self._err(self.lib.ref_build_landmarks(_ptr(data, _f32p), n, dim, m, c,
                                               _ptr(sub_dims, _u32p), _ptr(centroids, _f32p),
                                               _ptr(codes, _u8p), m, _ptr(lx, _f32p)),
                  "build_landmarks")
        return codes, lx

    def build_ivf(self, data, m, c, sub_dims, centroids, codes, lx, nlist, seed,
                  coarse_iters=10) -> HostIndex:
        data = np.ascontiguousarray(data, np.float32)
        n, dim = data.shape
        sub_dims = np.ascontiguousarray(sub_dims, np.uint32)
        centroids = np.ascontiguousarray(centroids, np.float32)
        codes = np.ascontiguousarray(codes, np.uint8)
        lx = np.ascontiguousarray(lx, np.float32)
        coarse = np.zeros((nlist, dim), np.float32)
        offs = np.zeros(nlist + 1, np.uint64)
        ids = np.zeros(n, np.uint32)
        lcodes = np.zeros((n, m), np.uint8)
        llx = np.zeros(n, np.float32)
        self._err(self.lib.ref_build_ivf(_ptr(data, _f32p), n, dim, m, c, _ptr(sub_dims, _u32p),
                                         _ptr(centroids, _f32p), _ptr(codes, _u8p), m,
                                         _ptr(lx, _f32p), nlist, seed, coarse_iters,
                                         _ptr(coarse, _f32p), _ptr(offs, _u64p), _ptr(ids, _u32p),
                                         _ptr(lcodes, _u8p), _ptr(llx, _f32p)), "build_ivf")
        return HostIndex(dim=dim, m=m, ksub=c, sub_dims=sub_dims, centroids=centroids,
                         coarse=coarse, list_offsets=offs, list_ids=ids, list_codes=lcodes,
                         list_lx=llx, vectors=data)

    def _flat(self, ix: HostIndex) -> _FlatIndex:
        return _FlatIndex(ix.dim, ix.m, ix.ksub, _ptr(ix.sub_dims, _u32p),
                          _ptr(ix.centroids, _f32p), ix.nlist, _ptr(ix.coarse, _f32p),
                          _ptr(ix.list_offsets, _u64p), _ptr(ix.list_ids, _u32p),
                          _ptr(ix.list_codes, _u8p), ix.code_stride, _ptr(ix.list_lx, _f32p),
                          ix.n, _ptr(ix.vectors, _f32p))

    # -- on-disk formats (the reference's own save/load) --
    def ivf_save(self, ix: HostIndex, path: str, mse=0.0, seed=0, iters=0):
        fi = self._flat(ix)
        self._err(self.lib.ref_ivf_save(C.byref(fi), mse, seed, iters, path.encode()), "IvfIndex::save")

    def ivf_load(self, path: str) -> dict:
        dim, nlist, tot = C.c_uint64(), C.c_uint64(), C.c_uint64()
        m, c = C.c_uint32(), C.c_uint32()
        self._err(self.lib.ref_ivf_load_sizes(path.encode(), C.byref(dim), C.byref(nlist), C.byref(m),
                                              C.byref(c), C.byref(tot)), "IvfIndex::load")
        d, nl, mm, cc, t = dim.value, nlist.value, m.value, c.value, tot.value
        sub = np.zeros(mm, np.uint32)
        cent = np.zeros(cc * d, np.float32)
        coarse = np.zeros(nl * d, np.float32)
        offs = np.zeros(nl + 1, np.uint64)
        ids = np.zeros(max(t, 1), np.uint32)
        codes = np.zeros(max(t * mm, 1), np.uint8)
        lx = np.zeros(max(t, 1), np.float32)
        mse, seed, iters = C.c_double(), C.c_uint64(), C.c_uint32()
        self._err(self.lib.ref_ivf_load(path.encode(), _ptr(sub, _u32p), _ptr(cent, _f32p), _ptr(coarse, _f32p),
                                        _ptr(offs, _u64p), _ptr(ids, _u32p), _ptr(codes, _u8p), _ptr(lx, _f32p),
                                        C.byref(mse), C.byref(seed), C.byref(iters)), "IvfIndex::load")
        return dict(dim=d, nlist=nl, m=mm, ksub=cc, sub_dims=sub, centroids=cent, coarse=coarse,
                    list_offsets=offs, list_ids=ids[:t], list_codes=codes[:t * mm].reshape(t, mm),
                    list_lx=lx[:t], training_mse=mse.value, seed=seed.value, iters=iters.value)

    def landmarks_save(self, dim, m, c, sub, cent, codes, lx, path: str):
        codes = np.ascontiguousarray(codes, np.uint8)
        lx = np.ascontiguousarray(lx, np.float32)
        self._err(self.lib.ref_landmarks_save(dim, m, c, _ptr(np.ascontiguousarray(sub, np.uint32), _u32p),
                                              _ptr(np.ascontiguousarray(cent, np.float32), _f32p), lx.size,
                                              _ptr(codes, _u8p), _ptr(lx, _f32p), path.encode()),
                  "LandmarkStore::save")

    def landmarks_load(self, path: str, n: int, m: int):
        codes = np.zeros(n * m, np.uint8)
        lx = np.zeros(n, np.float32)
        self._err(self.lib.ref_landmarks_load(path.encode(), n, _ptr(codes, _u8p), _ptr(lx, _f32p)),
                  "LandmarkStore::load")
        return codes.reshape(n, m), lx

    def profile_save(self, p: float, gamma: float, path: str):
        self._err(self.lib.ref_profile_save(p, gamma, path.encode()), "PruningProfile::save")

    def profile_load(self, path: str):
        p, g = C.c_double(), C.c_double()
        self._err(self.lib.ref_profile_load(path.encode(), C.byref(p), C.byref(g)), "PruningProfile::load")
        return p.value, g.value

    def write_fvecs(self, x, path: str):
        x = np.ascontiguousarray(x, np.float32)
        self._err(self.lib.ref_write_fvecs(_ptr(x, _f32p), x.shape[0], x.shape[1], path.encode()),
                  "write_fvecs")

    def load_fvecs(self, path: str, n: int, dim: int):
        out = np.zeros((n, dim), np.float32)
        self._err(self.lib.ref_load_fvecs(path.encode(), n, dim, _ptr(out, _f32p)), "load_vecs")
        return out

    # -- searches (ivf/ivf.hpp) --
    def search_knn(self, ix: HostIndex, qs, k, nprobe, gamma):
        qs = np.ascontiguousarray(qs, np.float32).reshape(-1, ix.dim)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dist = np.zeros((nq, k), np.float32)
        ct = np.zeros((nq, 6), np.uint64)
        fi = self._flat(ix)
        self._err(self.lib.ref_search_knn_batch(C.byref(fi), _ptr(qs, _f32p), nq, k, nprobe,
                                                gamma, _ptr(ids, _u32p), _ptr(dist, _f32p),
                                                _ptr(ct, _u64p)), "search_trim_ivf_knn")
        return ids, dist, ct[:, :5].copy(), ct[:, 5].copy()

    def search_range(self, ix: HostIndex, qs, radius, nprobe, gamma, cap=4096):
        qs = np.ascontiguousarray(qs, np.float32).reshape(-1, ix.dim)
        nq = qs.shape[0]
        rad = np.ascontiguousarray(np.broadcast_to(np.float32(radius), (nq,)), np.float32) \
            if np.ndim(radius) == 0 else np.ascontiguousarray(radius, np.float32)
        ids = np.zeros((nq, cap), np.uint32)
        dist = np.zeros((nq, cap), np.float32)
        cnt = np.zeros(nq, np.uint64)
        ct = np.zeros((nq, 6), np.uint64)
        fi = self._flat(ix)
        self._err(self.lib.ref_search_range_batch(C.byref(fi), _ptr(qs, _f32p), nq,
                                                  _ptr(rad, _f32p), nprobe, gamma, cap,
                                                  _ptr(ids, _u32p), _ptr(dist, _f32p),
                                                  _ptr(cnt, _u64p), _ptr(ct, _u64p)),
                  "search_trim_ivf_range")
        if nq and int(cnt.max()) > cap:
            return self.search_range(ix, qs, rad, nprobe, gamma, cap=int(cnt.max()))
        offs = np.zeros(nq + 1, np.uint64)
        offs[1:] = np.cumsum(cnt)
        oid = np.concatenate([ids[i, :cnt[i]] for i in range(nq)]) if nq else np.zeros(0, np.uint32)
        od = np.concatenate([dist[i, :cnt[i]] for i in range(nq)]) if nq else np.zeros(0, np.float32)
        return offs, oid, od, ct[:, :5].copy(), ct[:, 5].copy()

    def search_baseline(self, ix: HostIndex, qs, k, nprobe, k_prime):
        qs = np.ascontiguousarray(qs, np.float32).reshape(-1, ix.dim)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dist = np.zeros((nq, k), np.float32)
        ct = np.zeros((nq, 6), np.uint64)
        fi = self._flat(ix)
        self._err(self.lib.ref_search_baseline_batch(C.byref(fi), _ptr(qs, _f32p), nq, k, nprobe,
                                                     k_prime, _ptr(ids, _u32p),
                                                     _ptr(dist, _f32p), _ptr(ct, _u64p)),
                  "search_baseline_ivfpq")
        return ids, dist, ct[:, :5].copy(), ct[:, 5].copy()

    def session(self, ix: HostIndex):
        fi = self._flat(ix)
        s = self.lib.ref_session_create(C.byref(fi))
        if not s:
            raise RuntimeError("ref_session_create: " + self.lib.ref_last_error().decode())
        return s

    def session_run(self, s, kind, qs, k, nprobe, gamma, arg=0.0):
        """kind 0 knn / 1 range(arg=radius) / 2 baseline(arg=k'). -> (seconds, counter sums)."""
        qs = np.ascontiguousarray(qs, np.float32)
        sec = C.c_double(0)
        ct = np.zeros(6, np.uint64)
        self._err(self.lib.ref_session_run(s, kind, _ptr(qs, _f32p), qs.shape[0], k, nprobe,
                                           gamma, arg, C.byref(sec), _ptr(ct, _u64p)),
                  "session_run")
        return sec.value, ct

    def session_knn(self, s, qs, k, nprobe, gamma):
        """ivf::search_trim_ivf_knn per query over a session's index ->
        (ids[nq,k] u32, dist[nq,k] f32, counters[nq,5] u64, coarse_dc[nq])."""
        qs = np.ascontiguousarray(qs, np.float32)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dist = np.zeros((nq, k), np.float32)
        ct = np.zeros((nq, 6), np.uint64)
        self._err(self.lib.ref_session_knn(s, _ptr(qs, _f32p), nq, k, nprobe, gamma, _ptr(ids, _u32p),
                                           _ptr(dist, _f32p), _ptr(ct, _u64p)), "search_trim_ivf_knn")
        return ids, dist, ct[:, :5].copy(), ct[:, 5].copy()

    def session_range(self, s, qs, radius, nprobe, gamma, cap=1024):
        """ivf::search_trim_ivf_range per query over a session's index ->
        (offsets[nq+1], ids, dist, counters[nq,5], coarse_dc[nq])."""
        qs = np.ascontiguousarray(qs, np.float32)
        nq = qs.shape[0]
        rad = np.ascontiguousarray(np.broadcast_to(np.float32(radius), (nq,)), np.float32) \
            if np.ndim(radius) == 0 else np.ascontiguousarray(radius, np.float32)
        ids = np.zeros((nq, cap), np.uint32)
        dist = np.zeros((nq, cap), np.float32)
        cnt = np.zeros(nq, np.uint64)
        ct = np.zeros((nq, 6), np.uint64)
        self._err(self.lib.ref_session_range(s, _ptr(qs, _f32p), nq, _ptr(rad, _f32p), nprobe, gamma, cap,
                                             _ptr(ids, _u32p), _ptr(dist, _f32p), _ptr(cnt, _u64p),
                                             _ptr(ct, _u64p)), "search_trim_ivf_range")
        if nq and int(cnt.max()) > cap:
            return self.session_range(s, qs, rad, nprobe, gamma, cap=int(cnt.max()))
        offs = np.zeros(nq + 1, np.uint64)
        offs[1:] = np.cumsum(cnt)
        oid = np.concatenate([ids[i, :cnt[i]] for i in range(nq)]) if nq else np.zeros(0, np.uint32)
        od = np.concatenate([dist[i, :cnt[i]] for i in range(nq)]) if nq else np.zeros(0, np.float32)
        return offs, oid, od, ct[:, :5].copy(), ct[:, 5].copy()

    def session_destroy(self, s):
        self.lib.ref_session_destroy(s)

    def ground_truth_knn(self, data, qs, k):
        data = np.ascontiguousarray(data, np.float32)
        qs = np.ascontiguousarray(qs, np.float32)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dist = np.zeros((nq, k), np.float32)
        self._err(self.lib.ref_ground_truth_knn(_ptr(data, _f32p), data.shape[0], data.shape[1],
                                                _ptr(qs, _f32p), nq, k, _ptr(ids, _u32p),
                                                _ptr(dist, _f32p)), "ground_truth_knn")
        return ids, dist

    def pick_radius(self, data, qs, e_fraction, sample_rows=2000, sample_queries=200, seed=1):
        data = np.ascontiguousarray(data, np.float32)
        qs = np.ascontiguousarray(qs, np.float32)
        r = C.c_float(0)
        self._err(self.lib.ref_pick_radius(_ptr(data, _f32p), data.shape[0], data.shape[1],
                                           _ptr(qs, _f32p), qs.shape[0], e_fraction, sample_rows,
                                           sample_queries, seed, C.byref(r)), "pick_radius")
        return r.value

    def calibrate_empirical(self, data, ix_codes, ix_lx, m, c, sub_dims, centroids, cal_qs,
                            sample_x=1000, queries_per_x=200, seed=1, p=1.0) -> float:
        data = np.ascontiguousarray(data, np.float32)
        codes = np.ascontiguousarray(ix_codes, np.uint8)
        lx = np.ascontiguousarray(ix_lx, np.float32)
        sub_dims = np.ascontiguousarray(sub_dims, np.uint32)
        centroids = np.ascontiguousarray(centroids, np.float32)
        cal_qs = np.ascontiguousarray(cal_qs, np.float32)
        g = C.c_double(0)
        self._err(self.lib.ref_calibrate_empirical(
            _ptr(data, _f32p), data.shape[0], data.shape[1], m, c, _ptr(sub_dims, _u32p),
            _ptr(centroids, _f32p), _ptr(codes, _u8p), codes.shape[1], _ptr(lx, _f32p),
            _ptr(cal_qs, _f32p), cal_qs.shape[0], sample_x, queries_per_x, seed, p,
            C.byref(g)), "calibrate")
        return g.value

    # -- scalar KATs --
    def euclidean_sq(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.ref_euclidean_sq(_ptr(a, _f32p), _ptr(b, _f32p), a.size)

    def strict_lb(self, a, b) -> float:
        out = C.c_float()
        self._err(self.lib.ref_strict_lb(a, b, C.byref(out)), "strict_lb")
        return out.value

    def relaxed_lb(self, a, b, g) -> float:
        out = C.c_float()
        self._err(self.lib.ref_relaxed_lb(a, b, g, C.byref(out)), "relaxed_lb")
        return out.value

    def distance_table(self, ix: HostIndex, q) -> np.ndarray:
        q = np.ascontiguousarray(q, np.float32)
        out = np.empty((ix.m, ix.ksub), np.float32)
        self._err(self.lib.ref_build_table(ix.dim, ix.m, ix.ksub, _ptr(ix.sub_dims, _u32p),
                                           _ptr(ix.centroids, _f32p), _ptr(q, _f32p),
                                           _ptr(out, _f32p)), "build_distance_table")
        return out

    def adc(self, table, code) -> float:
        table = np.ascontiguousarray(table, np.float32)
        code = np.ascontiguousarray(code, np.uint8)
        return self.lib.ref_adc_lookup(_ptr(table, _f32p), table.shape[0], table.shape[1],
                                       _ptr(code, _u8p))


def make_reference_graph(ref: RefOracle, data, *, M=8, efc=64, graph_seed=5, m, c=256, iters=25,
                         pq_seed=1) -> HostGraph:
    """The reference's graph pipeline: build_graph + pq::train + build_landmarks."""
    g = ref.build_graph(data, M, efc, graph_seed)
    sub, cent = ref.pq_train(data, m, c, iters, pq_seed, 0)
    codes, lx = ref.build_landmarks(data, m, c, sub, cent)
    g.m, g.ksub, g.sub_dims, g.centroids, g.codes, g.lx = m, c, sub, cent, codes, lx
    return g


def make_reference_index(ref: RefOracle, data, *, m, c=256, iters=25, pq_seed=1, nlist=1,
                         ivf_seed=4, coarse_iters=10, train_sample=0) -> HostIndex:
    """The reference's offline pipeline: pq::train -> build_landmarks -> build_ivf."""
    sub, cent = ref.pq_train(data, m, c, iters, pq_seed, train_sample)
    codes, lx = ref.build_landmarks(data, m, c, sub, cent)
    return ref.build_ivf(data, m, c, sub, cent, codes, lx, nlist, ivf_seed, coarse_iters)
