"""Exploratory timing of the kNN kernel on config-1 data (reference-built).
Not a test and not the bench: prints CUDA-event times per gamma."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle.oracle import COracle, RefOracle, make_reference_index
from paper_2508_17828_b200 import ivf as G

ref = RefOracle()
t = time.time()
centers = ref.make_normal(64, 128, 0)
base = ref.make_blobs(centers, 100000, 0.3, 1)
qs = ref.make_blobs(centers, 1000, 0.3, 2)
hix = make_reference_index(ref, base, m=16, c=256, iters=25, pq_seed=3, nlist=1, ivf_seed=4)
print(f"build {time.time()-t:.1f}s", flush=True)
gix = G.GpuIvfIndex(G.IvfArrays.from_any(hix))
dq = torch.from_numpy(qs).cuda()
for g in (0.0, 0.605, 1.0):
    prof = G.PruningProfile.manual(g)
    for _ in range(3):
        G.search_trim_ivf_knn_device(gix, prof, dq, 10, 1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    R = 10
    for _ in range(R):
        G.search_trim_ivf_knn_device(gix, prof, dq, 10, 1)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / R
    print(f"gamma={g}: {ms:.3f} ms/batch(1000q) -> {1000/ms*1e3:.0f} QPS, "
          f"{1e8/ms*1e3:.3e} cand/s", flush=True)
