"""Device-side index build: the B200 equivalent of the reference's offline
pipeline:

    reference (host threads)                        here (sm_100a kernels)
    make_normal/make_blob_dataset (synthetic.hpp)   synth_normal / synth_blobs
    pq::train            (pq/pq.hpp:65-113)         pq_train
    trim::build_landmarks (landmarks.hpp:57-72)     pq_encode (codes + Γ(l,x), bit-exact)
    ivf::build_ivf       (ivf/ivf.hpp:112-154)      build_ivf

Device memory is torch.cuda tensors (plumbing); every kernel is ours, called
through the C ABI. Synthetic rows come from a counter-based Philox generator,
not libstdc++'s mt19937_64 + normal_distribution, so they are *distributed*
like the reference's generators (same shapes, sigma, round-robin blob
assignment) but not the same bytes; parity is always checked on the bytes the
GPU actually consumes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .ivf import IvfArrays


def _p(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def synth_normal(n: int, dim: int, seed: int, device: int = 0) -> torch.Tensor:
    out = torch.empty((n, dim), dtype=torch.float32, device=f"cuda:{device}")
    _lib.check(_lib.load().trim_synth_normal_device(n, dim, seed, _p(out), device, _stream(out.device)),
               "synth_normal")
    return out


def synth_blobs(centers: torch.Tensor, n: int, sigma: float, seed: int) -> torch.Tensor:
    dev = centers.device
    out = torch.empty((n, centers.shape[1]), dtype=torch.float32, device=dev)
    _lib.check(_lib.load().trim_synth_blobs_device(_p(centers), centers.shape[0], centers.shape[1], n,
                                                   sigma, seed, _p(out), dev.index or 0, _stream(dev)),
               "synth_blobs")
    return out


def synth_uniform(n: int, dim: int, seed: int, normalize: bool = True, device: int = 0) -> torch.Tensor:
    out = torch.empty((n, dim), dtype=torch.float32, device=f"cuda:{device}")
    _lib.check(_lib.load().trim_synth_uniform_device(n, dim, seed, int(normalize), _p(out), device,
                                                     _stream(out.device)), "synth_uniform")
    return out


def sample_rows(n: int, sample_n: int, seed: int) -> np.ndarray:
    """The reference's Fisher-Yates row sample (pq.hpp:72-80, ivf.hpp:121-126)."""
    out = np.zeros(sample_n, np.uint64)
    _lib.check(_lib.load().trim_sample_rows(n, sample_n, seed, C.c_void_p(out.ctypes.data)),
               "sample_rows")
    return out


def assign(x: torch.Tensor, cent: torch.Tensor):
    n, dim = x.shape
    k = cent.shape[0]
    a = torch.empty(n, dtype=torch.int32, device=x.device)
    d = torch.empty(n, dtype=torch.float32, device=x.device)
    _lib.check(_lib.load().trim_assign_device(_p(x), n, dim, _p(cent), k, _p(a), _p(d),
                                              x.device.index or 0, _stream(x.device)),
               "nearest_centroid")
    return a, d


def kmeans(x: torch.Tensor, k: int, iters: int, seed: int) -> torch.Tensor:
    x = x.contiguous()
    n, dim = x.shape
    cent = torch.empty((k, dim), dtype=torch.float32, device=x.device)
    torch.cuda.current_stream(x.device).synchronize()
    _lib.check(_lib.load().trim_kmeans_device(_p(x), n, dim, k, iters, seed, _p(cent),
                                              x.device.index or 0), "kmeans")
    return cent


def pq_train(x: torch.Tensor, m: int, ksub: int = 256, iters: int = 25, seed: int = 1,
             train_sample: int = 0):
    n, dim = x.shape
    sub = np.zeros(m, np.uint32)
    cent = torch.empty(ksub * dim, dtype=torch.float32, device=x.device)
    torch.cuda.current_stream(x.device).synchronize()
    _lib.check(_lib.load().trim_pq_train_device(_p(x), n, dim, m, ksub, iters, seed, train_sample,
                                                C.c_void_p(sub.ctypes.data), _p(cent),
                                                x.device.index or 0), "pq::train")
    return sub, cent


def pq_encode(x: torch.Tensor, m: int, ksub: int, sub_dims: np.ndarray, cent: torch.Tensor):
    n, dim = x.shape
    codes = torch.empty((n, m), dtype=torch.uint8, device=x.device)
    lx = torch.empty(n, dtype=torch.float32, device=x.device)
    sub = np.ascontiguousarray(sub_dims, np.uint32)
    _lib.check(_lib.load().trim_pq_encode_device(_p(x), n, dim, m, ksub, C.c_void_p(sub.ctypes.data),
                                                 _p(cent), _p(codes), m, _p(lx), x.device.index or 0,
                                                 _stream(x.device)), "pq::encode")
    return codes, lx


def ivf_lists(assign_: torch.Tensor, nlist: int):
    n = assign_.shape[0]
    offs = torch.empty(nlist + 1, dtype=torch.int64, device=assign_.device)
    ids = torch.empty(n, dtype=torch.int32, device=assign_.device)
    _lib.check(_lib.load().trim_ivf_lists_device(_p(assign_), n, nlist, _p(offs), _p(ids),
                                                 assign_.device.index or 0, _stream(assign_.device)),
               "build_ivf lists")
    return offs, ids


@dataclass
class BuildParams:
    m: int
    ksub: int = 256
    pq_iters: int = 25
    pq_seed: int = 1
    train_sample: int = 0
    nlist: int = 1
    ivf_seed: int = 4
    coarse_iters: int = 10


def build_ivf(x: torch.Tensor, p: BuildParams) -> IvfArrays:
    """pq::train -> build_landmarks -> build_ivf, all on x's device."""
    n, dim = x.shape
    sub, cent = pq_train(x, p.m, p.ksub, p.pq_iters, p.pq_seed, p.train_sample)
    codes, lx = pq_encode(x, p.m, p.ksub, sub, cent)
    # ivf.hpp:119-131: coarse k-means on min(n, max(nlist, 50*nlist)) sampled rows
    sample_n = min(n, max(p.nlist, 50 * p.nlist))
    rows = sample_rows(n, sample_n, p.ivf_seed ^ 0x94D049BB133111EB)
    sample = x[torch.from_numpy(rows.astype(np.int64)).to(x.device)].contiguous()
    coarse = kmeans(sample, p.nlist, p.coarse_iters, p.ivf_seed)
    del sample
    if p.nlist == 1:
        a = torch.zeros(n, dtype=torch.int32, device=x.device)
    else:
        a, _ = assign(x, coarse)
    offs, ids = ivf_lists(a, p.nlist)
    idl = ids.long()
    return IvfArrays(dim=dim, m=p.m, ksub=p.ksub, sub_dims=torch.from_numpy(sub).to(x.device),
                     centroids=cent, coarse=coarse.reshape(-1), list_offsets=offs,
                     list_ids=ids, list_codes=codes[idl].contiguous(), list_lx=lx[idl].contiguous(),
                     vectors=x)


def to_host(a: IvfArrays) -> IvfArrays:
    """numpy copy (for the oracle / for saving)."""
    def h(t, dt):
        return t.cpu().numpy().view(dt) if isinstance(t, torch.Tensor) else np.asarray(t, dt)
    return IvfArrays(dim=a.dim, m=a.m, ksub=a.ksub, sub_dims=h(a.sub_dims, np.uint32),
                     centroids=h(a.centroids, np.float32), coarse=h(a.coarse, np.float32),
                     list_offsets=h(a.list_offsets, np.uint64), list_ids=h(a.list_ids, np.uint32),
                     list_codes=h(a.list_codes, np.uint8), list_lx=h(a.list_lx, np.float32),
                     vectors=h(a.vectors, np.float32), id_base=a.id_base)


def build_knn_graph(x: torch.Tensor, M: int, n_random: int, m: int, ksub: int = 256, pq_iters: int = 25,
                    pq_seed: int = 1, seed: int = 0):
    """A single-level search graph for the graph filter benchmark (the HNSW
    builder, graph/hnsw.hpp:165-268, is a sequential host loop and not on the
    hot path): node i's list = its M exact nearest rows (trim_ground_truth_knn,
    itself excluded) followed by n_random seeded random rows (long-range links);
    entry 0. Landmarks: pq::train + encode on the device. Returns GraphArrays
    (host numpy)."""
    from .ivf import GpuIvfIndex

    arrays = build_ivf(x, BuildParams(m=m, ksub=ksub, pq_iters=pq_iters, pq_seed=pq_seed, nlist=1))
    gix = GpuIvfIndex(arrays, device=x.device.index or 0)
    return knn_graph_from_flat(arrays, gix, M, n_random, seed)


def knn_graph_from_flat(arrays: IvfArrays, gix, M: int, n_random: int, seed: int = 0):
    """build_knn_graph over a flat index already on the device (list entry e =
    row e): the landmark store is the index's codes / Γ(l,x)."""
    from .graph import GraphArrays
    from .ivf import ground_truth_knn

    x = arrays.vectors
    n, dim = x.shape
    m = arrays.m
    xh = x.cpu().numpy()
    nbr = np.empty((n, M + 1), np.uint32)
    for b0 in range(0, n, 65536):
        nbr[b0:b0 + 65536] = ground_truth_knn(gix, xh[b0:b0 + 65536], M + 1)[0]
    self_ = nbr == np.arange(n, dtype=np.uint32)[:, None]
    # drop the row itself (or, with exact duplicates ahead of it, the last entry)
    drop = np.where(self_.any(1), self_.argmax(1), M)
    keep = np.ones_like(nbr, dtype=bool)
    keep[np.arange(n), drop] = False
    knn = nbr[keep].reshape(n, M)
    rng = np.random.default_rng(seed)
    rnd = rng.integers(0, n - 1, size=(n, n_random), dtype=np.uint32)
    rnd = rnd + (rnd >= np.arange(n, dtype=np.uint32)[:, None])  # never the row itself
    lists = np.concatenate([knn, rnd.astype(np.uint32)], 1)
    # dedupe each list, first occurrence kept
    srt = np.sort(lists, 1)
    dup_any = (srt[:, 1:] == srt[:, :-1]).any(1)
    sizes = np.full(n, lists.shape[1], np.uint64)
    flat = lists.reshape(-1)
    if dup_any.any():
        parts = []
        for i in range(n):
            li = lists[i]
            if dup_any[i]:
                _, first = np.unique(li, return_index=True)
                li = li[np.sort(first)]
                sizes[i] = li.size
            parts.append(li)
        flat = np.concatenate(parts)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    h = to_host(arrays)
    return GraphArrays(entry=0, offsets=[offs], nbrs=[flat.astype(np.uint32)], sub_dims=h.sub_dims,
                       centroids=h.centroids, codes=np.ascontiguousarray(h.list_codes[:, :m]), lx=h.list_lx,
                       vectors=xh, ksub=h.ksub, M=M)
