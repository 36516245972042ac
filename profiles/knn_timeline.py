"""Per-CTA phase timeline of the kNN filter kernel on the bench workload (c2).

    python profiles/knn_timeline.py [--n N] [--gamma G]

Builds the bench.py workload, runs one batch through
trim_search_knn_preassigned_device with the internal timeline probe enabled
(trim__set_knn_timeline: %globaltimer stamps per CTA) and prints where a
query's time goes: setup (LUT + stream), seeds, chunk 0 + plan, the chunk
pipeline, plus launch-level spans. A diagnostic, not a benchmark.
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# the instrumented build (make -C paper_2508_17828_b200/csrc timeline)
os.environ.setdefault("TRIM_B200_LIB", os.path.join(ROOT, "paper_2508_17828_b200", "libtrim_b200_tl.so"))
import numpy as np
import torch

import bench
from paper_2508_17828_b200 import _lib
from paper_2508_17828_b200 import ivf as G

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--gamma", type=float, default=0.8)
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--out", default="")
ap.add_argument("--config", default="c2")
a = ap.parse_args()
cfg = dict(bench.CONFIGS[a.config])
if a.n:
    cfg["n"] = a.n
cfg["nq"] = a.batch
arrays, queries = bench.build_workload(cfg, 0, 1, 0, False)
gix = G.GpuIvfIndex(arrays, device=0)
lib = _lib.load()
lib.trim__set_knn_timeline.argtypes = [C.c_void_p]
nq, k = a.batch, cfg["k"]
npb = min(cfg["nprobe"], cfg["nlist"])
lists = torch.zeros((nq, npb), dtype=torch.int32, device="cuda")
ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
dist = torch.empty((nq, k), dtype=torch.float32, device="cuda")
cts = torch.zeros((nq, 6), dtype=torch.int64, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
tl = torch.zeros((nq, 32), dtype=torch.int64, device="cuda")
sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: C.c_void_p(t.data_ptr())
_lib.check(lib.trim_probe_device(gix.handle, P(queries), nq, cfg["nprobe"], P(lists), sh), "probe")


def run(timeline):
    lib.trim__set_knn_timeline(C.c_void_p(tl.data_ptr()) if timeline else None)
    _lib.check(lib.trim_search_knn_preassigned_device(gix.handle, P(queries), nq, k, P(lists), npb,
                                                      float(np.float32(a.gamma)), P(ids), P(dist), P(cts),
                                                      P(st), sh), "knn")


for _ in range(3):
    run(False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run(False)
e1.record()
torch.cuda.synchronize()
run(True)
torch.cuda.synchronize()
lib.trim__set_knn_timeline(None)
t = tl.cpu().numpy().astype(np.float64)
c = cts.cpu().numpy()
t0 = t[:, 0].min()
span = (t[:, 4] - t[:, 0]) / 1e3
ph = {
    "setup_us (stream)": (t[:, 1] - t[:, 0]) / 1e3,
    "seeds_us": (t[:, 2] - t[:, 1]) / 1e3,
    "plan_us": (t[:, 3] - t[:, 2]) / 1e3,
    "pipeline_us": (t[:, 4] - t[:, 3]) / 1e3,
    "cta_total_us": span,
}
out = {"launch_ms_events": e0.elapsed_time(e1), "launch_span_us_timeline": (t[:, 4].max() - t0) / 1e3,
       "chunks_mean": float(t[:, 5].mean()), "members_mean": float(t[:, 7].mean()),
       "evaluated_mean": float(c[:, 3].mean())}
for name, v in ph.items():
    out[name] = {"mean": float(v.mean()), "p50": float(np.median(v)), "p90": float(np.percentile(v, 90)),
                 "max": float(v.max())}
GHZ = 1.965e3  # cycles per us at the B200 boost clock
for i, name in ((8, "replay_wait_full_us"), (9, "replay_busy_us"), (10, "w0_lut_us"), (11, "w0_plan_wait_us"),
                (12, "w0_ring_wait_us"), (13, "w0_adc_us"), (14, "w0_l2_us"), (15, "w0_pipeline_us")):
    v = t[:, i] / GHZ
    out[name] = {"mean": float(v.mean()), "p50": float(np.median(v))}
# every worker: ring waits and busy (ADC + exact L2) time (imbalance across workers)
out["worker_ring_wait_us"] = [float((t[:, 16 + w] / GHZ).mean()) for w in range(7)]
out["worker_busy_us"] = [float((t[:, 23 + w] / GHZ).mean()) for w in range(7)]
# per-chunk pipeline cost
pc = ph["pipeline_us"] / np.maximum(1, t[:, 5])
out["pipeline_us_per_chunk"] = {"mean": float(pc.mean()), "p50": float(np.median(pc))}
# concurrency: CTAs resident over time
starts = (t[:, 0] - t0) / 1e3
ends = (t[:, 4] - t0) / 1e3
grid = np.linspace(0, ends.max(), 50)
out["resident_ctas_profile"] = [int(((starts <= x) & (ends > x)).sum()) for x in grid[::5]]
txt = json.dumps(out, indent=1)
print(txt)
if a.out:
    open(a.out, "w").write(txt)
