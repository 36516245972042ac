"""The reference's on-disk artefacts, read and written byte-for-byte
(SURVEY.md §8f.2), so indexes built by the reference's CLI drop into the GPU
path unchanged and indexes built on the GPU (builder.py) can be handed back.

All multi-byte fields are little-endian (core/io_util.hpp:28-83); there are no
magic numbers or padding.

* codebook (pq/pq.hpp:194-233): u32 m, u32 c, u32 dim, u32 sub_dims[m], then
  per subspace j the f32 centroids [c x sub_dims[j]], f64 training_mse,
  u64 seed, u32 kmeans_iters;
* IvfIndex (ivf/ivf.hpp:53-107): u64 dim, u64 nlist, codebook, f32 coarse
  [nlist x dim], u64 offsets[nlist+1], then per entry (lists in order):
  u32 id, u8 code[m], f32 lx;
* LandmarkStore (trim/landmarks.hpp:29-53): codebook, u64 count,
  u8 codes[count x m], f32 lx[count];
* PruningProfile (trim/calibration.hpp:234-288): text, header
  "trimsearch-profile v1", `key = value` lines;
* vecs (core/vecs_io.hpp): repeated [i32 d][d elements] records; .fvecs f32,
  .bvecs u8, .ivecs i32 (elements widened to f32 by load_vecs).

Errors follow the reference: truncated or inconsistent files raise
DataError with the reference's wording.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from ._lib import DataError
from .ivf import IvfArrays, PruningProfile


@dataclass
class Codebook:
    """pq::PqCodebook (pq/pq.hpp:40-54) as flat arrays: subspace j's [c x
    sub_dims[j]] centroids start at c * sum(sub_dims[:j])."""

    dim: int
    m: int
    c: int
    sub_dims: np.ndarray
    centroids: np.ndarray
    training_mse: float = 0.0
    seed: int = 0
    kmeans_iters: int = 0


def _read(f, dtype, count: int, what: str) -> np.ndarray:
    dt = np.dtype(dtype)
    buf = f.read(dt.itemsize * count)
    if len(buf) != dt.itemsize * count:
        raise DataError(f"truncated {what}")
    return np.frombuffer(buf, dtype=dt, count=count).copy()


def _scalar(f, dtype, what: str):
    return _read(f, dtype, 1, what)[0]


def read_codebook(f) -> Codebook:
    """pq::load_codebook (pq/pq.hpp:207-233)."""
    m = int(_scalar(f, "<u4", "codebook m"))
    c = int(_scalar(f, "<u4", "codebook c"))
    dim = int(_scalar(f, "<u4", "codebook dim"))
    sub = _read(f, "<u4", m, "codebook sub_dim").astype(np.uint32)
    if int(sub.sum()) != dim:
        raise DataError("codebook sub_dims do not sum to dim")
    cent = _read(f, "<f4", c * dim, "codebook centroids").astype(np.float32)
    mse = float(_scalar(f, "<f8", "codebook mse"))
    seed = int(_scalar(f, "<u8", "codebook seed"))
    iters = int(_scalar(f, "<u4", "codebook iters"))
    return Codebook(dim, m, c, sub, cent, mse, seed, iters)


def write_codebook(f, cb: Codebook) -> None:
    """pq::save_codebook (pq/pq.hpp:194-205)."""
    np.array([cb.m, cb.c, cb.dim], "<u4").tofile(f)
    np.asarray(cb.sub_dims, "<u4").tofile(f)
    np.asarray(cb.centroids, "<f4").reshape(-1).tofile(f)
    np.array([cb.training_mse], "<f8").tofile(f)
    np.array([cb.seed], "<u8").tofile(f)
    np.array([cb.kmeans_iters], "<u4").tofile(f)


def _entry_dtype(m: int) -> np.dtype:
    return np.dtype([("id", "<u4"), ("code", "u1", (m,)), ("lx", "<f4")])  # packed, 8 + m bytes


def load_ivf(path: str, vectors=None) -> tuple[IvfArrays, Codebook]:
    """ivf::IvfIndex::load (ivf/ivf.hpp:78-107) -> (IvfArrays, Codebook). The
    reference keeps the dataset separately (VectorDataset); pass its rows as
    `vectors` (e.g. load_vecs(base.fvecs)) to get a searchable IvfArrays."""
    with open(path, "rb") as f:
        dim = int(_scalar(f, "<u8", "ivf dim"))
        nlist = int(_scalar(f, "<u8", "ivf nlist"))
        cb = read_codebook(f)
        coarse = _read(f, "<f4", dim * nlist, "ivf centroids").astype(np.float32)
        offs = _read(f, "<u8", nlist + 1, "ivf offsets").astype(np.uint64)
        if nlist and (offs[0] != 0 or np.any(np.diff(offs.astype(np.int64)) < 0)):
            raise DataError("ivf offsets are not monotone")
        total = int(offs[-1]) if nlist else 0
        ent = _read(f, _entry_dtype(cb.m), total, "ivf entry")
    if vectors is None:
        vectors = np.zeros((0, dim), np.float32)
    arr = IvfArrays(dim=dim, m=cb.m, ksub=cb.c, sub_dims=cb.sub_dims, centroids=cb.centroids,
                    coarse=coarse, list_offsets=offs, list_ids=ent["id"].astype(np.uint32),
                    list_codes=np.ascontiguousarray(ent["code"], np.uint8),
                    list_lx=ent["lx"].astype(np.float32),
                    vectors=np.ascontiguousarray(vectors, np.float32).reshape(-1, dim))
    return arr, cb


def save_ivf(path: str, arrays: IvfArrays, codebook: Codebook | None = None) -> None:
    """ivf::IvfIndex::save (ivf/ivf.hpp:53-76) from host or device arrays."""
    from .builder import to_host
    a = to_host(arrays)
    offs = np.asarray(a.list_offsets, np.uint64)
    nlist = offs.size - 1
    cb = codebook or Codebook(a.dim, a.m, a.ksub, np.asarray(a.sub_dims, np.uint32),
                              np.asarray(a.centroids, np.float32))
    total = int(offs[-1])
    ent = np.empty(total, _entry_dtype(a.m))
    ent["id"] = np.asarray(a.list_ids, np.uint32)
    ent["code"] = np.asarray(a.list_codes, np.uint8).reshape(total, -1)[:, :a.m]
    ent["lx"] = np.asarray(a.list_lx, np.float32)
    with open(path, "wb") as f:
        np.array([a.dim, nlist], "<u8").tofile(f)
        write_codebook(f, cb)
        np.asarray(a.coarse, "<f4").reshape(-1).tofile(f)
        offs.astype("<u8").tofile(f)
        ent.tofile(f)


def load_landmarks(path: str) -> tuple[Codebook, np.ndarray, np.ndarray]:
    """trim::LandmarkStore::load (trim/landmarks.hpp:40-53) -> (codebook,
    codes[count, m] u8, lx[count] f32)."""
    with open(path, "rb") as f:
        cb = read_codebook(f)
        n = int(_scalar(f, "<u8", "landmark count"))
        buf = f.read(n * cb.m)
        if len(buf) != n * cb.m:
            raise DataError(f"truncated landmark codes: {path}")
        codes = np.frombuffer(buf, np.uint8).reshape(n, cb.m).copy()
        lx = _read(f, "<f4", n, "landmark distances").astype(np.float32)
    return cb, codes, lx


def save_landmarks(path: str, codebook: Codebook, codes, lx) -> None:
    """trim::LandmarkStore::save (trim/landmarks.hpp:29-38)."""
    codes = np.ascontiguousarray(codes, np.uint8).reshape(-1, codebook.m)
    with open(path, "wb") as f:
        write_codebook(f, codebook)
        np.array([codes.shape[0]], "<u8").tofile(f)
        codes.tofile(f)
        np.asarray(lx, "<f4").tofile(f)


def flat_index(codebook: Codebook, codes, lx, vectors) -> IvfArrays:
    """A flat scan (nlist = 1, the single list holding every id in order, as
    build_ivf(ds, 1, lm, seed) produces, ivf.hpp:112-154) from a landmark store.
    The single coarse centroid only feeds probe_order over one list, so its
    value never changes a result; the data mean is used."""
    x = np.ascontiguousarray(vectors, np.float32).reshape(-1, codebook.dim)
    n = x.shape[0]
    codes = np.ascontiguousarray(codes, np.uint8).reshape(n, codebook.m)
    return IvfArrays(dim=codebook.dim, m=codebook.m, ksub=codebook.c, sub_dims=codebook.sub_dims,
                     centroids=codebook.centroids, coarse=x.mean(0, dtype=np.float64).astype(np.float32),
                     list_offsets=np.array([0, n], np.uint64), list_ids=np.arange(n, dtype=np.uint32),
                     list_codes=codes, list_lx=np.asarray(lx, np.float32), vectors=x)


_VECS = {".fvecs": "<f4", ".bvecs": "u1", ".ivecs": "<i4"}


def load_vecs(path: str, kind: str | None = None, max_rows: int = 0) -> np.ndarray:
    """core/vecs_io.hpp load_vecs: [i32 d][d elements] records, elements
    widened to f32; all records must share d."""
    ext = kind or os.path.splitext(path)[1]
    if ext not in _VECS:
        raise DataError(f"{path}: unknown vecs element kind")
    el = np.dtype(_VECS[ext])
    raw = np.fromfile(path, np.uint8)
    if raw.size < 4:
        raise DataError(f"{path}: empty vecs file (dimension undetermined)")
    d = int(raw[:4].view("<i4")[0])
    if d <= 0:
        raise DataError(f"{path}: record with non-positive dimension")
    rec = 4 + d * el.itemsize
    n = raw.size // rec
    if max_rows:
        n = min(n, max_rows)
    if not max_rows and raw.size % rec:
        raise DataError(f"truncated {ext[1:]} record")
    rows = raw[:n * rec].reshape(n, rec)
    if np.any(rows[:, :4].copy().view("<i4").reshape(-1) != d):
        raise DataError(f"{path}: inconsistent dimension across records")
    return rows[:, 4:].copy().view(el).reshape(n, d).astype(np.float32)


def write_fvecs(path: str, x) -> None:
    """core/vecs_io.hpp write_fvecs."""
    x = np.ascontiguousarray(x, "<f4")
    n, d = x.shape
    rec = np.empty((n, d + 1), "<f4")
    rec[:, 0] = np.array([d], "<i4").view("<f4")[0]
    rec[:, 1:] = x
    rec.tofile(path)


_PROFILE_HEADER = "trimsearch-profile v1"


def load_profile(path: str) -> PruningProfile:
    """trim::PruningProfile::load (trim/calibration.hpp:247-288)."""
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise DataError(f"cannot open for reading: {path}")
    if not lines or lines[0] != _PROFILE_HEADER:
        raise DataError(f"{path}: not a pruning profile file")
    prof = PruningProfile()
    for line in lines[1:]:
        if "=" not in line:
            continue
        key, value = (t.strip(" \t\r") for t in line.split("=", 1))
        if key == "p":
            prof.p = float(value)
        elif key == "gamma":
            prof.gamma = float(value)
        elif key == "strategy":
            prof.strategy = value
        elif key in ("seed", "sample_x", "samples_per_x"):
            int(value)  # parsed by the reference (stoull); not used by the search
        else:
            raise DataError(f"{path}: unknown profile key '{key}'")
    return prof


def save_profile(path: str, prof: PruningProfile) -> None:
    """trim::PruningProfile::save (trim/calibration.hpp:234-245), 17 digits."""
    with open(path, "w") as f:
        f.write(f"{_PROFILE_HEADER}\n")
        f.write(f"p = {prof.p:.17g}\n")
        f.write(f"gamma = {prof.gamma:.17g}\n")
        f.write(f"strategy = {prof.strategy}\n")
        f.write("seed = 0\nsample_x = 0\nsamples_per_x = 0\n")


def open_index(ivf_path: str, vectors_path: str, device: int = 0):
    """A device index straight from the reference's artefacts: an
    IvfIndex::save file plus the base vectors (.fvecs/.bvecs), as the
    reference CLI's `query` subcommand consumes them."""
    from .ivf import GpuIvfIndex
    arr, _ = load_ivf(ivf_path, vectors=load_vecs(vectors_path))
    return GpuIvfIndex(arr, device=device)


@dataclass
class GraphFile:
    """graph::GraphIndex as saved (graph/hnsw.hpp:37-56): per level, the CSR
    offsets (count + 1, u64) and the concatenated neighbour ids (u32)."""

    count: int
    M: int
    entry: int
    ef_construction: int
    offsets: list
    nbrs: list


def load_graph(path: str) -> GraphFile:
    """graph::GraphIndex::load (graph/hnsw.hpp:58-83), the same checks."""
    with open(path, "rb") as f:
        n = int(_scalar(f, "<u8", "graph count"))
        M = int(_scalar(f, "<u4", "graph M"))
        levels = int(_scalar(f, "<u4", "graph levels"))
        entry = int(_scalar(f, "<u4", "graph entry"))
        efc = int(_scalar(f, "<u4", "graph efc"))
        if levels == 0:
            raise DataError(f"{path}: graph with zero levels")
        offs, nbrs = [], []
        for _ in range(levels):
            o = _read(f, "<u8", n + 1, "graph offsets").astype(np.uint64)
            sizes = np.diff(o.astype(np.int64))
            if (sizes < 0).any():  # read_le_array of a negative degree fails in the reference
                raise DataError(f"truncated graph ids: {path}")
            nb = _read(f, "<u4", int(sizes.sum()), "graph ids").astype(np.uint32)
            offs.append(np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64))
            nbrs.append(nb)
    return GraphFile(n, M, entry, efc, offs, nbrs)


def save_graph(path: str, g) -> None:
    """graph::GraphIndex::save (graph/hnsw.hpp:37-56) of any object with count
    (or n), M, entry, ef_construction (or efc), offsets and nbrs per level."""
    n = int(getattr(g, "count", getattr(g, "n", 0)))
    efc = int(getattr(g, "ef_construction", getattr(g, "efc", 0)))
    with open(path, "wb") as f:
        np.array([n], "<u8").tofile(f)
        np.array([g.M, len(g.offsets), g.entry, efc], "<u4").tofile(f)
        for o, nb in zip(g.offsets, g.nbrs):
            np.asarray(o, "<u8").tofile(f)
            np.asarray(nb, "<u4").tofile(f)


def open_graph(graph_path: str, landmarks_path: str, vectors_path: str, device: int = 0):
    """A device graph straight from the reference's artefacts: GraphIndex::save,
    LandmarkStore::save and the base vectors (.fvecs/.bvecs)."""
    from .graph import GpuGraph, GraphArrays
    g = load_graph(graph_path)
    cb, codes, lx = load_landmarks(landmarks_path)
    vec = load_vecs(vectors_path)
    if codes.shape[0] != g.count or vec.shape[0] != g.count:  # search.hpp:198-199
        raise DataError("graph, landmark store and dataset sizes differ")
    return GpuGraph(GraphArrays(entry=g.entry, offsets=g.offsets, nbrs=g.nbrs, sub_dims=cb.sub_dims,
                                centroids=cb.centroids, codes=codes, lx=lx, vectors=vec, ksub=cb.c, M=g.M),
                    device=device)
