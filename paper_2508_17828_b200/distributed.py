"""Multi-GPU: the index sharded by vector id, one process per GPU.

SURVEY.md §8e. Rank r of W holds ids [r*N/W, (r+1)*N/W): for every inverted
list, the contiguous sub-range of that list whose ids fall in the shard (lists
hold ascending ids, ivf.hpp:147-152), plus those vector rows. The coarse
quantizer and PQ codebook are replicated, so every rank computes the same
probe order. Each rank runs the fused filter over its sub-stream of every
query (its result, counters and prunes equal the reference run over that
shard's candidate subsequence), then the only collective — an all-gather of
the per-rank top-k (dist_sq, id), k*8 bytes per query per rank — is merged on
the device by (dist_sq, id), the order ScoredId defines
(core/ground_truth.hpp:39-50). Counters are summed with an all-reduce.

A replicas layout (every rank holds the whole index and a slice of the
queries, ReplicaIvfIndex) needs no data-path collective and reproduces the
single run exactly; bench.py --gpus N measures the id-sharded layout with a
full-size shard per GPU (weak scaling) by default and the replicas layout with
--parallel replicas, DESIGN.md §6.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

import numpy as np

from .ivf import IvfArrays


def shard_bounds(n: int, rank: int, world: int):
    """Even id split: rank r owns [lo, hi)."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return lo, hi


def shard_arrays(a: IvfArrays, rank: int, world: int) -> IvfArrays:
    """Host (numpy) id-shard of a full index: per list, the entries with
    lo <= id < hi (a contiguous run, ids ascend within a list), and vector
    rows [lo, hi). Codebook and coarse centroids are shared."""
    offs = np.asarray(a.list_offsets, np.uint64)
    ids = np.asarray(a.list_ids, np.uint32)
    codes = np.asarray(a.list_codes, np.uint8)
    lx = np.asarray(a.list_lx, np.float32)
    vec = np.asarray(a.vectors, np.float32).reshape(-1, a.dim)
    n = vec.shape[0]
    lo, hi = shard_bounds(n, rank, world)
    nlist = offs.size - 1
    keep_ids, keep_codes, keep_lx = [], [], []
    new_offs = np.zeros(nlist + 1, np.uint64)
    for l in range(nlist):
        b, e = int(offs[l]), int(offs[l + 1])
        seg = ids[b:e]
        s0 = b + int(np.searchsorted(seg, lo, side="left"))
        s1 = b + int(np.searchsorted(seg, hi, side="left"))
        keep_ids.append(ids[s0:s1])
        keep_codes.append(codes[s0:s1])
        keep_lx.append(lx[s0:s1])
        new_offs[l + 1] = new_offs[l] + (s1 - s0)
    return IvfArrays(dim=a.dim, m=a.m, ksub=a.ksub, sub_dims=np.asarray(a.sub_dims, np.uint32),
                     centroids=np.asarray(a.centroids, np.float32),
                     coarse=np.asarray(a.coarse, np.float32), list_offsets=new_offs,
                     list_ids=np.concatenate(keep_ids) if keep_ids else ids[:0],
                     list_codes=np.concatenate(keep_codes) if keep_codes else codes[:0],
                     list_lx=np.concatenate(keep_lx) if keep_lx else lx[:0],
                     vectors=vec[lo:hi], id_base=lo)


def merge_topk_device(dist, ids, k: int):
    """Device merge of gathered per-rank top-k: dist/ids [W, nq, k] (torch.cuda)
    -> [nq, k], the k smallest (dist, id) (trim_merge_topk_device)."""
    import torch

    from . import _lib
    w, nq, kk = dist.shape
    out_d = torch.empty((nq, k), dtype=torch.float32, device=dist.device)
    out_i = torch.empty((nq, k), dtype=torch.int32, device=dist.device)
    st = torch.cuda.current_stream(dist.device).cuda_stream
    _lib.check(_lib.load().trim_merge_topk_device(
        C.c_void_p(dist.data_ptr()), C.c_void_p(ids.data_ptr()), w, nq, k, C.c_void_p(out_d.data_ptr()),
        C.c_void_p(out_i.data_ptr()), dist.device.index or 0, C.c_void_p(st)), "merge_topk")
    return out_d, out_i


class ShardedIvfIndex:
    """One rank's shard plus the collective merge.

    searcher(queries, k, nprobe, gamma) -> (ids[nq,k] int32, dist[nq,k] f32,
    counters[nq,6] int64) as torch tensors on the collective's device. The
    default searcher is the GPU path (GpuIvfIndex over `arrays`); tests pass
    the oracle instead to exercise the host logic under gloo.
    merge(dist[W,nq,k], ids[W,nq,k], k) -> (dist, ids); default: the device
    kernel.
    """

    def __init__(self, arrays: IvfArrays, group=None, searcher: Optional[Callable] = None,
                 merge: Optional[Callable] = None, device: Optional[int] = None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.arrays = arrays
        self._merge = merge or merge_topk_device
        if searcher is None:
            from .ivf import GpuIvfIndex, PruningProfile, search_trim_ivf_knn_device
            self.gpu = GpuIvfIndex(arrays, device=device or 0)

            def searcher(q, k, nprobe, gamma):
                import torch
                nq = q.shape[0]
                cts = torch.zeros((nq, 6), dtype=torch.int64, device=q.device)
                st = torch.zeros(1, dtype=torch.int32, device=q.device)
                ids, d = search_trim_ivf_knn_device(self.gpu, PruningProfile.manual(gamma), q, k, nprobe,
                                                    d_counters=cts, d_status=st)
                return ids, d, cts
        self._search = searcher

    def search_range(self, queries, radius, nprobe: int, gamma: float, range_searcher: Optional[Callable] = None,
                     cap: int = 4096):
        """Global range result: range search has no running
        state (ivf.hpp:323-340), so the union of the shards' member sets is
        exactly the single run's. Each rank's members (sorted slots) go through
        an all-gather of the counts, then a padded all-gather of (dist, id)
        keys, merged per query by (dist, id) (ivf.hpp:341).
        range_searcher(queries, radius, nprobe, gamma, cap) -> (counts[nq],
        ids[nq, cap], dist[nq, cap], counters[nq, 6]); default: the GPU path.
        Returns (offsets[nq+1], ids, dist, summed counters[5])."""
        import torch
        import torch.distributed as dist

        if range_searcher is None:
            from .ivf import PruningProfile, search_trim_ivf_range_device

            def range_searcher(q, r, npb, g, c):
                cts = torch.zeros((q.shape[0], 6), dtype=torch.int64, device=q.device)
                st = torch.zeros(1, dtype=torch.int32, device=q.device)
                cnt, ids, d = search_trim_ivf_range_device(self.gpu, PruningProfile.manual(g), q, r, npb, cap=c,
                                                           d_counters=cts, d_status=st)
                return cnt, ids, d, cts
        cnt, ids, d, cts = range_searcher(queries, radius, nprobe, gamma, cap)
        nq = cnt.shape[0]
        dev = cnt.device
        mx = cnt.max().reshape(1).to(torch.int64) if nq else torch.zeros(1, dtype=torch.int64, device=dev)
        # the largest member count over every rank; a rank whose result outgrew
        # `cap` finds out together with all the others (no rank raises alone and
        # leaves the rest waiting in a collective), and every rank re-runs with
        # the exact size
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=self.group)
        if int(mx.item()) > cap:
            return self.search_range(queries, radius, nprobe, gamma, range_searcher, cap=int(mx.item()))
        w = max(1, int(mx.item()))
        # (dist bits << 32 | id) sorts like (dist, id) for non-negative dist; padding sorts last
        keys = torch.full((nq, w), -1, dtype=torch.int64, device=dev)
        if nq:
            j = torch.arange(w, device=dev).unsqueeze(0)
            valid = j < cnt.unsqueeze(1).to(torch.int64)
            kd = d[:, :w].contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            ki = ids[:, :w].to(torch.int64) & 0xFFFFFFFF
            keys = torch.where(valid, (kd << 32) | ki, keys)
        gk = torch.empty((self.world * nq, w), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(gk, keys.contiguous(), group=self.group)
        gk = gk.view(self.world, nq, w).permute(1, 0, 2).reshape(nq, self.world * w)
        gk = torch.where(gk < 0, torch.full_like(gk, torch.iinfo(torch.int64).max), gk)
        gk, _ = torch.sort(gk, dim=1)
        gcnt = torch.empty((self.world * nq,), dtype=cnt.dtype, device=dev)
        dist.all_gather_into_tensor(gcnt, cnt.contiguous(), group=self.group)
        tot = gcnt.view(self.world, nq).sum(0).to(torch.int64)
        offs = torch.zeros(nq + 1, dtype=torch.int64, device=dev)
        offs[1:] = torch.cumsum(tot, 0)
        sel = torch.arange(self.world * w, device=dev).unsqueeze(0) < tot.unsqueeze(1)
        flat = gk[sel]
        out_ids = (flat & 0xFFFFFFFF).to(torch.int64)
        out_d = ((flat >> 32) & 0xFFFFFFFF).to(torch.int32).view(torch.float32)
        c = cts[:, :5].sum(0)
        dist.all_reduce(c, group=self.group)
        return offs, out_ids, out_d, c

    def search_knn(self, queries, k: int, nprobe: int, gamma: float):
        """Global top-k over all shards + summed counters {dc, edc, pruned,
        evaluated, hops, coarse_dc (one rank's)}."""
        import torch
        import torch.distributed as dist

        ids, d, cts = self._search(queries, k, nprobe, gamma)
        nq = ids.shape[0]
        g_ids = torch.empty((self.world * nq, k), dtype=ids.dtype, device=ids.device)
        g_d = torch.empty((self.world * nq, k), dtype=d.dtype, device=d.device)
        dist.all_gather_into_tensor(g_ids, ids.contiguous(), group=self.group)
        dist.all_gather_into_tensor(g_d, d.contiguous(), group=self.group)
        md, mi = self._merge(g_d.view(self.world, nq, k), g_ids.view(self.world, nq, k), k)
        # per-query counters summed over the shards. A shard whose share of a
        # query's probed lists is shorter than k returns its partial top-k
        # (padded with sentinels, merged above); the reference's "k exceeds
        # probed vectors" (ivf.hpp:289-290) is decided on the total stream
        # length, identically on every rank
        cts = cts.to(torch.int64).contiguous()
        dist.all_reduce(cts, group=self.group)
        if nq and bool((cts[:, 3] < k).any()):
            from ._lib import InvalidArgument
            raise InvalidArgument("search_trim_ivf_knn: k exceeds probed vectors")
        c = cts[:, :5].sum(0)
        return mi, md, c


class ReplicaIvfIndex:
    """Replicas layout: every rank holds the whole index and
    searches its contiguous slice [shard_bounds(nq, rank, world)) of each query
    batch; per-query results and counters are exactly the single run's (each
    query's stream is untouched). No collective on the data path;
    gather() (rank-ordered all-gather) is a convenience for callers that want
    every result on every rank.

    searcher(queries, k, nprobe, gamma) -> (ids, dist, counters) as for
    ShardedIvfIndex; the default is the GPU path over `arrays`."""

    def __init__(self, arrays: IvfArrays, group=None, searcher: Optional[Callable] = None,
                 device: Optional[int] = None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if searcher is None:
            from .ivf import GpuIvfIndex, PruningProfile, search_trim_ivf_knn_device
            self.gpu = GpuIvfIndex(arrays, device=device or 0)

            def searcher(q, k, nprobe, gamma):
                import torch
                cts = torch.zeros((q.shape[0], 6), dtype=torch.int64, device=q.device)
                st = torch.zeros(1, dtype=torch.int32, device=q.device)
                ids, d = search_trim_ivf_knn_device(self.gpu, PruningProfile.manual(gamma), q, k, nprobe,
                                                    d_counters=cts, d_status=st)
                if int(st.item()) & 1:  # each replica is the single run: ivf.hpp:289-290
                    from ._lib import InvalidArgument
                    raise InvalidArgument("search_trim_ivf_knn: k exceeds probed vectors")
                return ids, d, cts
        self._search = searcher

    def bounds(self, nq: int):
        return shard_bounds(nq, self.rank, self.world)

    def search_knn(self, queries, k: int, nprobe: int, gamma: float):
        """This rank's slice: (lo, hi, ids[hi-lo,k], dist, counters[hi-lo,6])."""
        lo, hi = self.bounds(queries.shape[0])
        ids, d, cts = self._search(queries[lo:hi], k, nprobe, gamma)
        return lo, hi, ids, d, cts

    def gather(self, nq: int, part):
        """All ranks' slices in query order (rows padded to the largest slice
        for the all-gather, then trimmed)."""
        import torch
        import torch.distributed as dist

        lo, hi, ids, d, cts = part
        rows = max(shard_bounds(nq, r, self.world)[1] - shard_bounds(nq, r, self.world)[0]
                   for r in range(self.world))
        out = []
        for t in (ids, d, cts):
            pad = torch.zeros((rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            pad[:hi - lo] = t
            g = torch.empty((self.world * rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(g, pad.contiguous(), group=self.group)
            g = g.view(self.world, rows, *t.shape[1:])
            out.append(torch.cat([g[r, :shard_bounds(nq, r, self.world)[1] - shard_bounds(nq, r, self.world)[0]]
                                  for r in range(self.world)]))
        return tuple(out)
