"""Exploratory A/B timing of trim_knn_kernel knobs (environment variables read
per call, e.g. TRIM_LIST_SKIP, TRIM_FLAT_BOUNDS) on one config, with a check
that every variant returns the same ids, distances and counters. Not a test
and not the bench.

    python tests/perf_modes.py [--config c2] [--variants "A=1|A=2,B=0"] [--gammas 0.8]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
from paper_2508_17828_b200 import ivf as G


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--variants", default="TRIM_LIST_SKIP=1")
    ap.add_argument("--gammas", default="0.8")
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--streams", type=int, default=3)
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS[a.config])
    if a.nq:
        cfg["nq"] = a.nq
    arrays, queries = bench.build_workload(cfg, 0, 1, 0)
    B, k = cfg["batch"], cfg["k"]
    ref = {}
    gix = G.GpuIvfIndex(arrays, device=0)
    sts = [torch.cuda.Stream() for _ in range(a.streams)]
    for rep in range(2):
        for g in [float(x) for x in a.gammas.split(",")]:
            prof = G.PruningProfile.manual(g)
            for var in a.variants.split("|"):
                for kv in var.split(","):
                    kk, vv = kv.split("=")
                    os.environ[kk] = vv

                def run():
                    outs = []
                    cur = torch.cuda.current_stream()
                    for x in sts:
                        x.wait_stream(cur)
                    for i, b0 in enumerate(range(0, cfg["nq"], B)):
                        qb = queries[b0:b0 + B]
                        x = sts[i % len(sts)]
                        with torch.cuda.stream(x):
                            ct = torch.zeros((qb.shape[0], 6), dtype=torch.int64, device=qb.device)
                            outs.append(G.search_trim_ivf_knn_device(gix, prof, qb, k, cfg["nprobe"],
                                                                     d_counters=ct, stream=x) + (ct,))
                    for x in sts:
                        cur.wait_stream(x)
                    return outs

                run()
                torch.cuda.synchronize()
                best = 1e9
                for _ in range(a.reps):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    outs = run()
                    e.record()
                    torch.cuda.synchronize()
                    best = min(best, s.elapsed_time(e))
                cat = [torch.cat([o[i] for o in outs]).cpu().numpy() for i in range(3)]
                ev_n = int(cat[2][:, 3].sum())
                same = ""
                if g in ref:
                    same = "same" if all((x.view(np.uint32) if x.dtype == np.float32 else x).tobytes()
                                         == (y.view(np.uint32) if y.dtype == np.float32 else y).tobytes()
                                         for x, y in zip(cat, ref[g])) else "DIFFERENT"
                else:
                    ref[g] = cat
                print(f"[{rep}] gamma={g} {var}: {best:.3f} ms / {cfg['nq']} q -> "
                      f"{ev_n / best * 1e3:.3e} cand/s, {cfg['nq'] / best * 1e3:.0f} QPS {same}", flush=True)


if __name__ == "__main__":
    main()
