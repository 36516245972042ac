"""Same-process A/B of library builds (tools/variant.sh): one bench fixture,
every variant's own index + device search (probe + filter) over the whole
query set on `--streams` streams, CUDA-event timed, repeated interleaved;
checks that every variant returns identical ids, distance bits and counters.
Not a test and not the bench.

    python tests/perf_libs.py --libs base=paper_2508_17828_b200/libtrim_b200.so,v=...so [--config c2]

A variant may carry environment settings read per call by the library:
`name=path@TRIM_FLAT_BOUNDS=0;TRIM_LIST_SKIP=1`.
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
from paper_2508_17828_b200 import _lib as L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--libs", required=True)
    ap.add_argument("--gamma", type=float, default=None)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--streams", type=int, default=3)
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS[a.config])
    if a.nq:
        cfg["nq"] = a.nq
    gamma = a.gamma if a.gamma is not None else cfg["gamma"]
    fx, queries = bench.build_workload(cfg, 0, 1, 0)
    from paper_2508_17828_b200 import ivf as G
    arrays = G.IvfArrays.from_any(fx)
    nq, B, k = cfg["nq"], cfg["batch"], cfg["k"]
    dev = torch.device("cuda:0")
    libs = {}
    envs = {}
    for item in a.libs.split(","):
        name, path = item.split("=", 1)
        path, _, env = path.partition("@")
        envs[name] = dict(kv.split("=", 1) for kv in env.split(";") if kv)
        same = [v for v in libs.values() if v[2] == path]
        if same:  # env-only variant of a library already loaded: share its index
            libs[name] = same[0]
            continue
        lib = C.CDLL(os.path.join(ROOT, path) if not os.path.isabs(path) else path, mode=os.RTLD_LOCAL)
        for fn, (res_t, args_t) in L.SIGNATURES.items():
            f = getattr(lib, fn)
            f.restype, f.argtypes = res_t, args_t
        d = L.TrimIndexDesc()
        keep = [arrays.sub_dims, arrays.centroids, arrays.coarse, arrays.list_offsets, arrays.list_ids,
                arrays.list_codes, arrays.list_lx, arrays.vectors]
        P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        d.dim, d.m, d.ksub = arrays.dim, arrays.m, arrays.ksub
        d.sub_dims, d.centroids, d.coarse = P(keep[0]), P(keep[1]), P(keep[2])
        d.nlist = keep[3].shape[0] - 1
        d.list_offsets, d.list_ids, d.list_codes = P(keep[3]), P(keep[4]), P(keep[5])
        d.code_stride = keep[5].shape[1]
        d.list_lx, d.n, d.vectors = P(keep[6]), keep[7].shape[0], P(keep[7])
        d.id_base, d.device, d.memory = 0, 0, L.TRIM_MEM_DEVICE
        h = C.c_void_p()
        rc = lib.trim_index_create(C.byref(d), C.byref(h))
        assert rc == 0, lib.trim_last_error
        libs[name] = (lib, h, path)
    streams = [torch.cuda.Stream(dev) for _ in range(a.streams)]
    out = {}
    res = {}
    for rep in range(a.reps):
        for name, (lib, h, _) in libs.items():
            for kk in {x for e in envs.values() for x in e}:
                os.environ.pop(kk, None)
            os.environ.update(envs[name])
            ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
            dd = torch.empty((nq, k), dtype=torch.float32, device=dev)
            ct = torch.zeros((nq, 6), dtype=torch.int64, device=dev)
            st = torch.zeros(1, dtype=torch.int32, device=dev)

            def step():
                cur = torch.cuda.current_stream(dev)
                for x in streams:
                    x.wait_stream(cur)
                for i, b0 in enumerate(range(0, nq, B)):
                    nb = min(B, nq - b0)
                    x = streams[i % len(streams)]
                    rc = lib.trim_search_knn_device(
                        h, C.c_void_p(queries.data_ptr() + b0 * cfg["dim"] * 4), C.c_uint64(nb), C.c_uint32(k),
                        C.c_uint32(cfg["nprobe"]), C.c_float(gamma), C.c_void_p(ids.data_ptr() + b0 * k * 4),
                        C.c_void_p(dd.data_ptr() + b0 * k * 4), C.c_void_p(ct.data_ptr() + b0 * 48),
                        C.c_void_p(st.data_ptr()), C.c_void_p(x.cuda_stream))
                    assert rc == 0
                for x in streams:
                    cur.wait_stream(x)
            step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            out.setdefault(name, []).append(ms)
            r = (ids.cpu().numpy(), dd.cpu().numpy().view(np.uint32), ct.cpu().numpy())
            if name not in res:
                res[name] = r
            first = next(iter(res.values()))
            for x, y in zip(first, r):
                assert (x == y).all(), f"variant {name} differs"
    for name, v in out.items():
        print(f"{name:14s} ms/step {min(v):8.3f} (all {', '.join(f'{x:.3f}' for x in v)})  QPS {nq / min(v) * 1e3:,.0f}")
    print("identical results across variants")


if __name__ == "__main__":
    main()
