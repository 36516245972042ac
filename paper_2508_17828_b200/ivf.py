"""Reference-shaped host API over the C ABI.

Mirrors trimsearch::ivf (proj/include/trimsearch/ivf/ivf.hpp) — same function
names, argument meaning and error behaviour — so callers of the reference's
query path switch by changing the import:

    reference (C++)                               here
    ------------------------------------------    ---------------------------------------
    ivf::IvfIndex + VectorDataset (ivf.hpp:37)    GpuIvfIndex(IvfArrays, device=0)
    trim::PruningProfile (calibration.hpp:215)    PruningProfile
    ivf::search_trim_ivf_knn     (ivf.hpp:243)    search_trim_ivf_knn(ix, profile, q, k, nprobe)
    ivf::search_trim_ivf_range   (ivf.hpp:308)    search_trim_ivf_range(ix, profile, q, r, nprobe)
    ivf::search_baseline_ivfpq   (ivf.hpp:193)    search_baseline_ivfpq(ix, q, k, nprobe, k')
    std::invalid_argument                          InvalidArgument (a ValueError)
    DataError                                      DataError

The per-query functions exist for parity with the reference signatures; the
batch functions (``*_batch``) are the production path: one C-ABI call and one
kernel launch per batch.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import DataError, InvalidArgument, CudaError, TrimCounters  # noqa: F401


@dataclass
class SearchCounters:
    """trimsearch::SearchCounters (core/counters.hpp:10-30)."""

    dc: int = 0
    edc: int = 0
    pruned: int = 0
    evaluated: int = 0
    hops: int = 0

    def pruning_ratio(self) -> float:
        denom = self.pruned + self.dc
        return 0.0 if denom == 0 else self.pruned / denom


@dataclass
class IvfResult:
    """ivf::IvfResult (ivf.hpp:164-169)."""

    ids: np.ndarray
    dist_sq: np.ndarray
    counters: SearchCounters
    coarse_dc: int = 0


@dataclass
class PruningProfile:
    """trim::PruningProfile (calibration.hpp:215-232). The search consumes only
    float(gamma) (ivf.hpp:250)."""

    p: float = -1.0
    gamma: float = -1.0
    strategy: str = "none"

    def calibrated(self) -> bool:
        return self.gamma >= 0.0

    @staticmethod
    def manual(gamma_value: float) -> "PruningProfile":
        if gamma_value < 0.0:
            raise InvalidArgument("PruningProfile::manual: gamma must be nonnegative")
        return PruningProfile(gamma=float(gamma_value), strategy="manual")

    def gamma_f32(self) -> float:
        return float(np.float32(self.gamma)) if self.calibrated() else -1.0


@dataclass
class IvfArrays:
    """Host (numpy) or device (torch.cuda) arrays of an IVF index in CSR form
    (include/trim_gpu.h trim_index_desc)."""

    dim: int
    m: int
    ksub: int
    sub_dims: object       # u32[m]
    centroids: object      # f32[ksub*dim]
    coarse: object         # f32[nlist*dim]
    list_offsets: object   # u64[nlist+1]
    list_ids: object       # u32[total]
    list_codes: object     # u8[total, code_stride]
    list_lx: object        # f32[total]
    vectors: object        # f32[n, dim]
    id_base: int = 0

    @staticmethod
    def from_any(obj) -> "IvfArrays":
        """Adopt any object with the same attribute names (e.g. a test fixture)."""
        return IvfArrays(**{f: getattr(obj, f) for f in (
            "dim", "m", "ksub", "sub_dims", "centroids", "coarse", "list_offsets", "list_ids",
            "list_codes", "list_lx", "vectors")}, id_base=getattr(obj, "id_base", 0))


def _is_torch_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


def _addr(x):
    if _is_torch_cuda(x) or hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    return C.c_void_p(x.ctypes.data)


SHARD_MODES = {"single": _lib.TRIM_SHARD_SINGLE, "id_shard": _lib.TRIM_SHARD_ID,
               "replicas": _lib.TRIM_SHARD_REPLICAS}


class GpuIvfIndex:
    """Device-resident copy of an IvfIndex + VectorDataset (trim_index_create).

    ``devices`` + ``shard_mode`` ("id_shard" | "replicas") build one index over
    several devices (include/trim_gpu.h trim_shard_mode; entries may repeat,
    e.g. four shards on cuda:0): ``arrays`` is then the whole index and every
    search returns the merged answer (id_shard: per-part filters, NCCL
    all-gather, device merge; replicas: query slices per device)."""

    def __init__(self, arrays: IvfArrays, device: int = 0, devices=None, shard_mode: str = "single"):
        lib = _lib.load()
        a = arrays
        dev_mem = _is_torch_cuda(a.vectors)
        if dev_mem:
            keep = [a.sub_dims, a.centroids, a.coarse, a.list_offsets, a.list_ids, a.list_codes,
                    a.list_lx, a.vectors]
            codes = a.list_codes
            code_stride = codes.shape[1] if codes.dim() == 2 else a.m
            n = a.vectors.shape[0]
            nlist = a.list_offsets.shape[0] - 1
        else:
            keep = [np.ascontiguousarray(a.sub_dims, np.uint32),
                    np.ascontiguousarray(a.centroids, np.float32).ravel(),
                    np.ascontiguousarray(a.coarse, np.float32).ravel(),
                    np.ascontiguousarray(a.list_offsets, np.uint64),
                    np.ascontiguousarray(a.list_ids, np.uint32),
                    np.ascontiguousarray(a.list_codes, np.uint8),
                    np.ascontiguousarray(a.list_lx, np.float32),
                    np.ascontiguousarray(a.vectors, np.float32).reshape(-1, a.dim)]
            codes = keep[5]
            code_stride = codes.shape[1] if codes.ndim == 2 else a.m
            n = keep[7].shape[0]
            nlist = keep[3].shape[0] - 1
        d = _lib.TrimIndexDesc()
        d.dim, d.m, d.ksub = a.dim, a.m, a.ksub
        d.sub_dims, d.centroids, d.coarse = _addr(keep[0]), _addr(keep[1]), _addr(keep[2])
        d.nlist = nlist
        d.list_offsets, d.list_ids, d.list_codes = _addr(keep[3]), _addr(keep[4]), _addr(keep[5])
        d.code_stride = code_stride
        d.list_lx, d.n, d.vectors = _addr(keep[6]), n, _addr(keep[7])
        d.id_base = a.id_base
        d.device = device
        d.memory = _lib.TRIM_MEM_DEVICE if dev_mem else _lib.TRIM_MEM_HOST
        if shard_mode not in SHARD_MODES:
            raise InvalidArgument(f"shard_mode must be one of {sorted(SHARD_MODES)}")
        if devices is not None and shard_mode != "single":
            devs = np.ascontiguousarray(devices, np.int32)
            keep.append(devs)
            d.devices = C.c_void_p(devs.ctypes.data)
            d.ndevices = len(devs)
            d.shard_mode = SHARD_MODES[shard_mode]
            device = int(devs[0])
        h = C.c_void_p()
        _lib.check(lib.trim_index_create(C.byref(d), C.byref(h)), "trim_index_create")
        self._h = h
        self.dim = a.dim
        self.m = a.m
        self.ksub = a.ksub
        self.nlist = nlist
        self.n = n
        self.device = device
        self.id_base = a.id_base
        self.shard_mode = shard_mode
        self.devices = list(devices) if devices is not None and shard_mode != "single" else [device]

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        inf = _lib.TrimIndexInfo()
        _lib.check(_lib.load().trim_index_get_info(self._h, C.byref(inf)), "trim_index_get_info")
        return {f: getattr(inf, f) for f, _ in _lib.TrimIndexInfo._fields_}

    def skipped_positions(self, reset: bool = False) -> int:
        """Stream positions pruned as whole lists by the kNN kernel's list-level
        bound (trim_index_skip_stats); a diagnostic, results are unaffected."""
        v = C.c_uint64(0)
        _lib.check(_lib.load().trim_index_skip_stats(self._h, C.byref(v), int(reset)), "trim_index_skip_stats")
        return int(v.value)

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().trim_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _queries(ix: GpuIvfIndex, q) -> np.ndarray:
    q = np.ascontiguousarray(q, np.float32)
    if q.ndim == 1:
        q = q.reshape(1, -1)
    if q.shape[1] != ix.dim:
        raise InvalidArgument("query dimension mismatch")
    return q


def _counters(ct) -> list:
    return [SearchCounters(c.dc, c.edc, c.pruned, c.evaluated, c.hops) for c in ct]


# ------------------------------------------------------------------ batches
def search_trim_ivf_knn_batch(ix: GpuIvfIndex, profile: PruningProfile, queries, k: int,
                              nprobe: int):
    """Batch ivf::search_trim_ivf_knn. Returns (ids[nq,k] u32, dist_sq[nq,k] f32,
    counters[nq,6] u64 {dc, edc, pruned, evaluated, hops, coarse_dc})."""
    q = _queries(ix, queries)
    nq = q.shape[0]
    ids = np.zeros((nq, k), np.uint32)
    dist = np.zeros((nq, k), np.float32)
    ct = np.zeros((nq, 6), np.uint64)
    rc = _lib.load().trim_search_knn(ix.handle, _addr(q), nq, k, nprobe,
                                     profile.gamma_f32(), _addr(ids), _addr(dist), _addr(ct))
    _lib.check(rc, "search_trim_ivf_knn")
    return ids, dist, ct


def search_trim_ivf_range_batch(ix: GpuIvfIndex, profile: PruningProfile, queries, radius,
                                nprobe: int):
    """Batch ivf::search_trim_ivf_range. Returns (offsets[nq+1], ids, dist_sq, counters[nq,6])."""
    q = _queries(ix, queries)
    nq = q.shape[0]
    rad = np.ascontiguousarray(np.broadcast_to(np.asarray(radius, np.float32), (nq,)), np.float32)
    offs = np.zeros(nq + 1, np.uint64)
    pids = _lib._u32p()
    pd = _lib._f32p()
    ct = np.zeros((nq, 6), np.uint64)
    lib = _lib.load()
    rc = lib.trim_search_range(ix.handle, _addr(q), nq, _addr(rad), nprobe, profile.gamma_f32(),
                               _addr(offs), C.byref(pids), C.byref(pd), _addr(ct))
    _lib.check(rc, "search_trim_ivf_range")
    tot = int(offs[-1])
    try:
        ids = np.ctypeslib.as_array(pids, shape=(max(tot, 1),))[:tot].copy()
        dist = np.ctypeslib.as_array(pd, shape=(max(tot, 1),))[:tot].copy()
    finally:
        lib.trim_free(C.cast(pids, C.c_void_p))
        lib.trim_free(C.cast(pd, C.c_void_p))
    return offs, ids, dist, ct


def search_baseline_ivfpq_batch(ix: GpuIvfIndex, queries, k: int, nprobe: int, k_prime: int):
    """Batch ivf::search_baseline_ivfpq. Returns (ids, dist_sq, counters[nq,6])."""
    q = _queries(ix, queries)
    nq = q.shape[0]
    ids = np.zeros((nq, k), np.uint32)
    dist = np.zeros((nq, k), np.float32)
    ct = np.zeros((nq, 6), np.uint64)
    rc = _lib.load().trim_search_baseline_ivfpq(ix.handle, _addr(q), nq, k, nprobe, k_prime,
                                                _addr(ids), _addr(dist), _addr(ct))
    _lib.check(rc, "search_baseline_ivfpq")
    return ids, dist, ct


def build_distance_table(ix: GpuIvfIndex, queries) -> np.ndarray:
    """pq::build_distance_table (pq.hpp:158-172), batched: [nq, m, ksub]."""
    q = _queries(ix, queries)
    out = np.zeros((q.shape[0], ix.m, ix.ksub), np.float32)
    _lib.check(_lib.load().trim_build_lut(ix.handle, _addr(q), q.shape[0], _addr(out)),
               "build_distance_table")
    return out


def probe_order(ix: GpuIvfIndex, queries, nprobe: int) -> np.ndarray:
    """detail_ivf::probe_order (ivf.hpp:173-187), batched."""
    q = _queries(ix, queries)
    np_eff = min(nprobe, ix.nlist)
    out = np.zeros((q.shape[0], np_eff), np.uint32)
    _lib.check(_lib.load().trim_probe(ix.handle, _addr(q), q.shape[0], nprobe, _addr(out)),
               "probe_order")
    return out


# ---------------------------------------------------------------- per query
def _result(ids, dist, ct) -> IvfResult:
    c = ct.reshape(-1)
    return IvfResult(ids=ids.reshape(-1), dist_sq=dist.reshape(-1),
                     counters=SearchCounters(int(c[0]), int(c[1]), int(c[2]), int(c[3]), int(c[4])),
                     coarse_dc=int(c[5]))


def search_trim_ivf_knn(ix: GpuIvfIndex, profile: PruningProfile, q, k: int,
                        nprobe: int) -> IvfResult:
    """ivf::search_trim_ivf_knn (ivf.hpp:243-304) for one query."""
    ids, dist, ct = search_trim_ivf_knn_batch(ix, profile, np.asarray(q).reshape(1, -1), k, nprobe)
    return _result(ids, dist, ct)


def search_trim_ivf_range(ix: GpuIvfIndex, profile: PruningProfile, q, radius: float,
                          nprobe: int) -> IvfResult:
    """ivf::search_trim_ivf_range (ivf.hpp:308-347) for one query."""
    offs, ids, dist, ct = search_trim_ivf_range_batch(ix, profile, np.asarray(q).reshape(1, -1),
                                                      radius, nprobe)
    return _result(ids, dist, ct)


def search_baseline_ivfpq(ix: GpuIvfIndex, q, k: int, nprobe: int, k_prime: int) -> IvfResult:
    """ivf::search_baseline_ivfpq (ivf.hpp:193-237) for one query."""
    ids, dist, ct = search_baseline_ivfpq_batch(ix, np.asarray(q).reshape(1, -1), k, nprobe,
                                                k_prime)
    return _result(ids, dist, ct)


# ------------------------------------------------------ device-resident path
def search_trim_ivf_knn_device(ix: GpuIvfIndex, profile: PruningProfile, d_queries, k: int,
                               nprobe: int, d_ids=None, d_dist=None, d_counters=None,
                               d_status=None, stream=None):
    """Inputs and outputs are torch.cuda tensors on the index's device; async on
    `stream` (torch.cuda.Stream or raw handle; default: torch's current stream)."""
    import torch

    nq = d_queries.shape[0]
    dev = d_queries.device
    if d_ids is None:
        d_ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    if d_dist is None:
        d_dist = torch.empty((nq, k), dtype=torch.float32, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    rc = _lib.load().trim_search_knn_device(
        ix.handle, C.c_void_p(d_queries.data_ptr()), nq, k, nprobe, profile.gamma_f32(),
        C.c_void_p(d_ids.data_ptr()), C.c_void_p(d_dist.data_ptr()),
        C.c_void_p(d_counters.data_ptr()) if d_counters is not None else None,
        C.c_void_p(d_status.data_ptr()) if d_status is not None else None, C.c_void_p(sh))
    _lib.check(rc, "search_trim_ivf_knn")
    return d_ids, d_dist


def search_trim_ivf_range_device(ix: GpuIvfIndex, profile: PruningProfile, d_queries, d_radius,
                                 nprobe: int, cap: int = 1024, d_counters=None, d_status=None,
                                 stream=None):
    """ivf::search_trim_ivf_range (ivf.hpp:308-347) on device tensors
    (trim_search_range_device). Returns (counts[nq] int32, ids[nq,cap] int32,
    dist[nq,cap] f32): query i's members are ids[i, :min(counts[i], cap)],
    sorted by (dist, id). Bit 0 of d_status: some query exceeded cap."""
    import torch

    nq = d_queries.shape[0]
    dev = d_queries.device
    counts = torch.zeros(nq, dtype=torch.int32, device=dev)
    ids = torch.empty((nq, cap), dtype=torch.int32, device=dev)
    dist = torch.empty((nq, cap), dtype=torch.float32, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    rc = _lib.load().trim_search_range_device(
        ix.handle, C.c_void_p(d_queries.data_ptr()), nq, C.c_void_p(d_radius.data_ptr()), nprobe,
        profile.gamma_f32(), cap, C.c_void_p(counts.data_ptr()), C.c_void_p(ids.data_ptr()),
        C.c_void_p(dist.data_ptr()),
        C.c_void_p(d_counters.data_ptr()) if d_counters is not None else None,
        C.c_void_p(d_status.data_ptr()) if d_status is not None else None, C.c_void_p(sh))
    _lib.check(rc, "search_trim_ivf_range")
    return counts, ids, dist


def ground_truth_knn(ix: GpuIvfIndex, queries, k: int):
    """core/ground_truth.hpp ground_truth_knn: exact k nearest rows of every
    query, ascending by (dist_sq, id), bit-identical to the reference
    (trim_ground_truth_knn). Returns (ids[nq, k] u32, dist_sq[nq, k] f32)."""
    q = _queries(ix, queries)
    nq = q.shape[0]
    ids = np.zeros((nq, k), np.uint32)
    dist = np.zeros((nq, k), np.float32)
    _lib.check(_lib.load().trim_ground_truth_knn(ix.handle, _addr(q), nq, k, _addr(ids), _addr(dist)),
               "ground_truth_knn")
    return ids, dist
