"""TRIM filter over an HNSW graph: Python mirror of
trimsearch::graph (proj/include/trimsearch/graph/search.hpp:188-347) over the
C ABI (include/trim_gpu.h, trim_graph_*). No CPU fallback.

    g = GpuGraph(GraphArrays(...))
    res = search_trim_knn(g, PruningProfile.manual(0.8), q, k=10, ef=64)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .ivf import InvalidArgument, PruningProfile, SearchCounters, _addr


@dataclass
class SearchResult:
    """graph::SearchResult (graph/search.hpp:22-26)."""

    ids: np.ndarray
    dist_sq: np.ndarray
    counters: SearchCounters


@dataclass
class GraphArrays:
    """GraphIndex (graph/hnsw.hpp:22-35) as per-level CSR (offsets[l]: u64[n+1],
    nbrs[l]: u32) + LandmarkStore (trim/landmarks.hpp:18-28: codebook, codes
    [n, m] by node id, lx [n]) + the VectorDataset rows [n, dim]."""

    entry: int
    offsets: list
    nbrs: list
    sub_dims: np.ndarray
    centroids: np.ndarray
    codes: np.ndarray
    lx: np.ndarray
    vectors: np.ndarray
    ksub: int = 256
    M: int = 0
    _keep: list = field(default_factory=list, repr=False)

    @classmethod
    def from_any(cls, g) -> "GraphArrays":
        """From any object with the HostGraph fields (oracle.HostGraph, formats)."""
        return cls(entry=int(g.entry), offsets=list(g.offsets), nbrs=list(g.nbrs), sub_dims=g.sub_dims,
                   centroids=g.centroids, codes=g.codes, lx=g.lx, vectors=g.vectors,
                   ksub=int(getattr(g, "ksub", 256)), M=int(getattr(g, "M", 0)))


class GpuGraph:
    """Device-resident graph + landmark store (trim_graph_create)."""

    def __init__(self, a: GraphArrays, device: int = 0):
        lib = _lib.load()
        vec = np.ascontiguousarray(a.vectors, np.float32)
        n, dim = vec.shape
        codes = np.ascontiguousarray(a.codes, np.uint8).reshape(n, -1)
        m = codes.shape[1]
        sub = np.ascontiguousarray(a.sub_dims, np.uint32)
        cent = np.ascontiguousarray(a.centroids, np.float32).ravel()
        lx = np.ascontiguousarray(a.lx, np.float32)
        offs = np.ascontiguousarray(np.concatenate([np.asarray(o, np.uint64) for o in a.offsets]))
        sizes = [int(np.asarray(o)[-1]) for o in a.offsets]
        base = np.ascontiguousarray(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64))
        nbrs = np.ascontiguousarray(np.concatenate([np.asarray(x, np.uint32) for x in a.nbrs]))
        d = _lib.TrimGraphDesc()
        d.n, d.dim, d.m, d.ksub = n, dim, m, a.ksub
        d.sub_dims, d.centroids, d.codes, d.code_stride = _addr(sub), _addr(cent), _addr(codes), m
        d.lx, d.vectors = _addr(lx), _addr(vec)
        d.levels, d.entry = len(a.offsets), a.entry
        d.offsets, d.nbr_base, d.nbrs, d.total_nbrs = _addr(offs), _addr(base), _addr(nbrs), int(nbrs.size)
        d.device, d.memory = device, _lib.TRIM_MEM_HOST
        h = C.c_void_p()
        _lib.check(lib.trim_graph_create(C.byref(d), C.byref(h)), "trim_graph_create")
        self.handle, self.n, self.dim, self.m, self.device = h, n, dim, m, device

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            _lib.load().trim_graph_destroy(h)
            self.handle = None


def _queries(g: GpuGraph, q) -> np.ndarray:
    q = np.ascontiguousarray(q, np.float32)
    if q.ndim == 1:
        q = q.reshape(1, -1)
    if q.shape[1] != g.dim:
        raise InvalidArgument("query dimension mismatch")
    return q


def search_trim_knn_batch(g: GpuGraph, profile: PruningProfile, queries, k: int, ef: int):
    """Batch graph::search_trim_knn. Returns ids [nq, k], dist_sq [nq, k],
    counters [nq, 6] (dc, edc, pruned, evaluated, hops, 0)."""
    q = _queries(g, queries)
    nq = q.shape[0]
    ids = np.zeros((nq, k), np.uint32)
    dist = np.zeros((nq, k), np.float32)
    ct = np.zeros((nq, 6), np.uint64)
    rc = _lib.load().trim_graph_search_knn(g.handle, _addr(q), nq, k, ef, profile.gamma_f32(), _addr(ids),
                                           _addr(dist), _addr(ct))
    _lib.check(rc, "search_trim_knn")
    return ids, dist, ct


def search_trim_knn_device(g: GpuGraph, profile: PruningProfile, d_queries, k: int, ef: int, d_ids=None,
                           d_dist=None, d_counters=None, stream=None):
    """torch.cuda tensors in and out, async on `stream` (default: torch's current)."""
    import torch

    nq = d_queries.shape[0]
    dev = d_queries.device
    d_ids = torch.empty((nq, k), dtype=torch.int32, device=dev) if d_ids is None else d_ids
    d_dist = torch.empty((nq, k), dtype=torch.float32, device=dev) if d_dist is None else d_dist
    d_counters = torch.zeros((nq, 6), dtype=torch.int64, device=dev) if d_counters is None else d_counters
    stream = torch.cuda.current_stream(dev) if stream is None else stream
    sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    rc = _lib.load().trim_graph_search_knn_device(g.handle, C.c_void_p(d_queries.data_ptr()), nq, k, ef,
                                                  profile.gamma_f32(), C.c_void_p(d_ids.data_ptr()),
                                                  C.c_void_p(d_dist.data_ptr()), C.c_void_p(d_counters.data_ptr()),
                                                  C.c_void_p(sh))
    _lib.check(rc, "search_trim_knn")
    return d_ids, d_dist, d_counters


def search_trim_range_batch(g: GpuGraph, profile: PruningProfile, queries, radius, ef: int):
    """Batch graph::search_trim_range. Returns (offsets[nq+1], ids, dist_sq, counters[nq, 6])."""
    q = _queries(g, queries)
    nq = q.shape[0]
    rad = np.ascontiguousarray(np.broadcast_to(np.asarray(radius, np.float32), (nq,)), np.float32)
    offs = np.zeros(nq + 1, np.uint64)
    pids, pd = _lib._u32p(), _lib._f32p()
    ct = np.zeros((nq, 6), np.uint64)
    lib = _lib.load()
    rc = lib.trim_graph_search_range(g.handle, _addr(q), nq, _addr(rad), ef, profile.gamma_f32(), _addr(offs),
                                     C.byref(pids), C.byref(pd), _addr(ct))
    _lib.check(rc, "search_trim_range")
    tot = int(offs[-1])
    try:
        ids = np.ctypeslib.as_array(pids, shape=(max(tot, 1),))[:tot].copy()
        dist = np.ctypeslib.as_array(pd, shape=(max(tot, 1),))[:tot].copy()
    finally:
        lib.trim_free(C.cast(pids, C.c_void_p))
        lib.trim_free(C.cast(pd, C.c_void_p))
    return offs, ids, dist, ct


def _result(ids, dist, ct) -> SearchResult:
    keep = ids != 0xFFFFFFFF
    c = SearchCounters(*(int(x) for x in ct[:5]))
    return SearchResult(ids[keep], dist[keep], c)


def search_trim_knn(g: GpuGraph, profile: PruningProfile, q, k: int, ef: int) -> SearchResult:
    """graph::search_trim_knn (graph/search.hpp:188-264), one query."""
    ids, dist, ct = search_trim_knn_batch(g, profile, q, k, ef)
    return _result(ids[0], dist[0], ct[0])


def search_trim_range(g: GpuGraph, profile: PruningProfile, q, radius: float, ef: int) -> SearchResult:
    """graph::search_trim_range (graph/search.hpp:267-347), one query."""
    offs, ids, dist, ct = search_trim_range_batch(g, profile, q, radius, ef)
    return SearchResult(ids, dist, SearchCounters(*(int(x) for x in ct[0][:5])))
