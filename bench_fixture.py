"""bench_fixture.py — the benchmark's synthetic workloads, built with plain
PyTorch ops only (no code from paper_2508_17828_b200, no oracle).

Both bench arms build their index here, so that:
  * the reference arm (`bench.py --impl reference`) never maps the product
    library (libtrim_b200.so) — its process loads only torch and oracle/_ref;
  * both arms search the SAME bytes: every step is deterministic (seeded
    torch.Generator streams, argmin ties to the lowest index, centroid sums
    by a sort + float64 prefix-sum instead of atomics), and `fingerprint()`
    hashes the result into `config.fixture` so the two JSON lines prove it.

The layout is the IvfIndex of the reference (ivf/ivf.hpp:29-51) in CSR form
(include/trim_gpu.h trim_index_desc): PQ codebook (pq/pq.hpp:40-54), codes +
plain Γ(l,x) = |x - decode(code)| (trim/landmarks.hpp:57-72), coarse
quantizer, lists ascending by id (ivf.hpp:147-152). Shapes, mixtures and
sigma follow BASELINE.json's configs; the build algorithm (k-means with
seeded row init, Lloyd, 25 PQ / 10 coarse iterations, coarse sample
max(nlist, 50*nlist) rows as ivf.hpp:119-131) follows the reference's
structure but is not bit-identical to it — parity is always checked on the
bytes both sides consume, never on the build (tests/ pin the build kernels
separately).
"""
from __future__ import annotations

import hashlib
from types import SimpleNamespace

import numpy as np
import torch

CHUNK = 1 << 18


def _gen(dev, seed):
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    return g


def synth_normal(n, dim, seed, dev):
    return torch.randn((n, dim), generator=_gen(dev, seed), device=dev, dtype=torch.float32)


def synth_blobs(centers, n, sigma, seed, row0=0):
    """Row i = centers[(row0 + i) % nc] + sigma * N(0, I) (make_blob_dataset's
    round-robin mixture, core/synthetic.hpp:21-33)."""
    dev = centers.device
    g = _gen(dev, seed)
    out = torch.empty((n, centers.shape[1]), dtype=torch.float32, device=dev)
    nc = centers.shape[0]
    for b in range(0, n, 1 << 22):
        e = min(n, b + (1 << 22))
        idx = (torch.arange(b, e, device=dev) + row0) % nc
        out[b:e] = centers[idx] + sigma * torch.randn((e - b, centers.shape[1]), generator=g, device=dev)
    return out


def synth_uniform(n, dim, seed, dev):
    """uniform [0,1) rows, L2-normalised (dataset.hpp:44-56 normalize_rows)."""
    g = _gen(dev, seed)
    out = torch.empty((n, dim), dtype=torch.float32, device=dev)
    for b in range(0, n, 1 << 20):
        e = min(n, b + (1 << 20))
        x = torch.rand((e - b, dim), generator=g, device=dev)
        out[b:e] = x / x.norm(dim=1, keepdim=True).clamp_min(1e-30)
    return out


def _argmin_rows(x, c, c2=None):
    """Nearest centroid per row (ties to the lowest index), chunked."""
    if c2 is None:
        c2 = (c.double() ** 2).sum(1).float()
    out = torch.empty(x.shape[0], dtype=torch.int64, device=x.device)
    step = max(1, min(CHUNK, (1 << 30) // max(1, c.shape[0])))
    for b in range(0, x.shape[0], step):
        xb = x[b:b + step]
        d = c2.unsqueeze(0) - 2.0 * (xb @ c.t())
        out[b:b + step] = torch.argmin(d, dim=1)
    return out


def _segment_means(x, a, k, old):
    """Mean of the rows of each cluster (sort by cluster + float64 prefix sums:
    deterministic, unlike atomics); an empty cluster keeps its centroid."""
    order = torch.argsort(a, stable=True)
    xs = x[order].double()
    cnt = torch.bincount(a, minlength=k)
    ends = torch.cumsum(cnt, 0)
    cs = torch.cat([torch.zeros((1, x.shape[1]), dtype=torch.float64, device=x.device), torch.cumsum(xs, 0)])
    sums = cs[ends] - cs[ends - cnt]
    mean = (sums / cnt.clamp_min(1).unsqueeze(1).double()).float()
    return torch.where((cnt > 0).unsqueeze(1), mean, old)


def kmeans(x, k, iters, seed):
    """Seeded distinct-row init, then Lloyd steps (pq/kmeans.hpp:102-152 shape)."""
    n = x.shape[0]
    g = _gen(x.device, seed)
    init = torch.randperm(n, generator=g, device=x.device)[:k]
    c = x[init].clone()
    for _ in range(iters):
        a = _argmin_rows(x, c)
        c = _segment_means(x, a, k, c)
    return c


def pq_train(x, m, ksub, iters, seed, sample):
    """Per-subspace k-means on a seeded row sample (pq/pq.hpp:65-113 shape).
    Returns sub_dims (u32[m]) and centroids in the trim_index_desc layout
    (subspace j at ksub*sub_off[j])."""
    n, dim = x.shape
    assert dim % m == 0, "the bench configs split D evenly over m subspaces"
    sd = dim // m
    g = _gen(x.device, seed)
    rows = torch.randperm(n, generator=g, device=x.device)[:min(n, sample)]
    xs = x[rows]
    cent = torch.empty(ksub * dim, dtype=torch.float32, device=x.device)
    for j in range(m):
        cj = kmeans(xs[:, j * sd:(j + 1) * sd].contiguous(), ksub, iters, seed * 1000 + j)
        cent[ksub * j * sd:ksub * (j + 1) * sd] = cj.reshape(-1)
    return np.full(m, sd, np.uint32), cent


def pq_encode(x, m, ksub, cent):
    """Nearest sub-centroid per subspace + Γ(l,x) = |x - decode(code)|."""
    n, dim = x.shape
    sd = dim // m
    C3 = cent.view(m, ksub, sd)
    c2 = (C3 * C3).sum(2)                                   # [m, ksub]
    codes = torch.empty((n, m), dtype=torch.uint8, device=x.device)
    lx = torch.empty(n, dtype=torch.float32, device=x.device)
    step = max(1024, (1 << 29) // (m * ksub))
    ar = torch.arange(m, device=x.device)
    for b in range(0, n, step):
        xb = x[b:b + step].view(-1, m, sd).transpose(0, 1)   # [m, B, sd]
        d = c2.unsqueeze(1) - 2.0 * torch.bmm(xb, C3.transpose(1, 2))  # [m, B, ksub]
        cd = torch.argmin(d, dim=2)                           # [m, B]
        codes[b:b + step] = cd.t().to(torch.uint8)
        dec = C3[ar.unsqueeze(1), cd]                         # [m, B, sd]
        lx[b:b + step] = ((xb - dec) ** 2).sum((0, 2)).sqrt()
    return codes, lx


def build(cfg, rank=0, device=0):
    """The workload of one rank: queries, and the id-shard [rank*n, (rank+1)*n)
    of the index (rank 0 = the whole single-GPU workload). The codebook and the
    coarse quantizer are trained on a seeded sample of rank 0's rows (regenerated
    identically on every rank, no collective) so every shard probes alike.
    Returns a SimpleNamespace with IvfArrays' fields (torch.cuda tensors) and
    `queries`."""
    dev = torch.device(device) if isinstance(device, str) else torch.device(f"cuda:{device}")
    n, dim = cfg["n"], cfg["dim"]
    m, ksub, nlist = cfg["m"], 256, cfg["nlist"]

    def rows_of(r, count):
        if cfg.get("data") == "uniform_normalized":
            return synth_uniform(count, dim, 1 + 7919 * r, dev)
        return synth_blobs(centers, count, cfg["sigma"], 1 + 7919 * r)

    centers = None if cfg.get("data") == "uniform_normalized" else synth_normal(cfg["n_centers"], dim, 0, dev)
    base = rows_of(rank, n)
    if cfg.get("data") == "uniform_normalized":
        queries = synth_uniform(cfg["nq"], dim, 2, dev)
    else:
        queries = synth_blobs(centers, cfg["nq"], cfg["sigma"], 2)
    # training rows: the first rows of rank 0's stream, regenerated by one
    # fixed-shape call on every rank (the same bytes everywhere; a sample from
    # the base distribution, like the reference's training sample)
    n_train = min(n, max(262_144, 50 * nlist))
    train = rows_of(0, n_train)
    sub, cent = pq_train(train, m, ksub, 25, 3, 262_144)
    if nlist > 1:
        coarse = kmeans(train[:min(n_train, max(nlist, 50 * nlist))], nlist, 10, 4)
    else:
        coarse = train.mean(0, keepdim=True)
    del train
    codes, lx = pq_encode(base, m, ksub, cent)
    if nlist > 1:
        a = _argmin_rows(base, coarse)
    else:
        a = torch.zeros(n, dtype=torch.int64, device=dev)
    ids = torch.argsort(a, stable=True)                       # ascending id within a list
    offs = torch.zeros(nlist + 1, dtype=torch.int64, device=dev)
    offs[1:] = torch.cumsum(torch.bincount(a, minlength=nlist), 0)
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)
    return SimpleNamespace(dim=dim, m=m, ksub=ksub, sub_dims=torch.from_numpy(sub.astype(np.int32)).to(dev),
                           centroids=cent, coarse=coarse.reshape(-1).contiguous(), list_offsets=offs,
                           list_ids=(ids + rank * n).to(torch.int32), list_codes=codes[ids].contiguous(),
                           list_lx=lx[ids].contiguous(), vectors=base, id_base=rank * n, queries=queries)


def fingerprint(fx) -> str:
    """A short hash of the fixture's bytes (sampled for the large arrays), so
    the two bench arms can show they searched the same index."""
    h = hashlib.sha1()
    for t in (fx.sub_dims, fx.centroids, fx.coarse, fx.list_offsets, fx.queries):
        h.update(t.detach().contiguous().cpu().numpy().tobytes())
    for t in (fx.list_ids, fx.list_codes, fx.list_lx, fx.vectors):
        flat = t.detach().reshape(-1)
        stride = max(1, flat.numel() // (1 << 20))
        h.update(flat[::stride].contiguous().cpu().numpy().tobytes())
        h.update(str(int(flat.numel())).encode())
    return h.hexdigest()[:16]


def to_host(fx):
    """numpy copies in the oracle's dtypes."""
    def h(t, dt):
        return t.detach().cpu().numpy().view(dt)
    return SimpleNamespace(dim=fx.dim, m=fx.m, ksub=fx.ksub, sub_dims=h(fx.sub_dims, np.uint32),
                           centroids=h(fx.centroids, np.float32), coarse=h(fx.coarse, np.float32),
                           list_offsets=h(fx.list_offsets, np.uint64), list_ids=h(fx.list_ids, np.uint32),
                           list_codes=h(fx.list_codes, np.uint8), list_lx=h(fx.list_lx, np.float32),
                           vectors=h(fx.vectors, np.float32), id_base=fx.id_base)
