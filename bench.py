#!/usr/bin/env python
"""bench.py — TRIM candidate filter on B200 (BASELINE.json metric).

Default workload: BASELINE.json configs[1] ("IVFPQ refinement with TRIM"):
10M fp32 vectors, D=96, 1,024-component Gaussian mixture (sigma 0.3), IVF
nlist=4,096 / nprobe=64, PQ M=48x256, 10,000 queries in batches of 1,024,
k=10, gamma swept over {0.6, 0.8, 1.0} (headline 0.8). Synthetic, seeded,
generated and indexed on the device (paper_2508_17828_b200/builder.py).

A *step* = the hot path over the whole 10,000-query set (10 batches of
1,024): probe_order + the fused ADC/bound/prune/exact-L2/top-k kernel.
`value` = candidates filtered per second over all ranks (a candidate is one
SearchCounters.evaluated event, ivf.hpp:260), inputs resident in HBM,
device-timed with CUDA events. `e2e` = the same metric through the C-ABI
host call (trim_search_knn) from pinned host buffers, copies included.

    python bench.py                               # N=1, config 2
    torchrun --nproc-per-node N bench.py --gpus N # id-sharded, weak scaling
    python bench.py --impl reference              # the reference CPU path
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1] — the bench workload
    "c2": dict(workload="ivfpq_trim_knn_10M_d96_nlist4096_nprobe64", n=10_000_000, dim=96,
               n_centers=1024, sigma=0.3, nq=10_000, batch=1024, m=48, nlist=4096, nprobe=64,
               k=10, gammas=[0.6, 0.8, 1.0], gamma=0.8, baseline_kprime=1000),
    # BASELINE.json configs[2]: flat range search, one calibrated radius
    "c3": dict(kind="range", workload="flat_trim_range_10M_d128", n=10_000_000, dim=128,
               n_centers=256, sigma=0.3, nq=10_000, batch=1024, m=32, nlist=1, nprobe=1, k=0,
               gammas=[0.0, 0.8], gamma=0.8, result_size=100),
    # BASELINE.json configs[3]: high-dimensional stress, flat kNN, uniform + L2-normalised
    "c4": dict(workload="flat_trim_knn_1M_d960_k100", n=1_000_000, dim=960, data="uniform_normalized",
               n_centers=0, sigma=0.0, nq=1000, batch=1000, m=120, nlist=1, nprobe=1, k=100,
               gammas=[0.5, 0.7, 0.9], gamma=0.9),
    # BASELINE.json configs[4]: billion-scale sharded flat scan, 100M rows per GPU (weak
    # scaling: --gpus 8 is the 800M configuration), batches of 2048
    "c5": dict(workload="flat_trim_knn_100M_per_gpu_d96", n=100_000_000, dim=96, n_centers=4096, sigma=0.3,
               nq=10_000, batch=2048, m=48, nlist=1, nprobe=1, k=10, gammas=[0.8], gamma=0.8),
    # the TRIM filter over a search graph (graph/search.hpp:188-264) on
    # config-1 data; level 0 = 32 exact nearest rows + 8 random long-range links per node
    "g1": dict(kind="graph", workload="graph_trim_knn_100k_d128_deg40", n=100_000, dim=128, n_centers=64,
               sigma=0.3, nq=10_000, batch=2048, m=16, nlist=1, nprobe=1, k=10, ef=64, M=32, n_random=8,
               gammas=[0.0, 1.0], gamma=0.8),
    # BASELINE.json configs[0] (CPU-runnable reference case; parity + extra line)
    "c1": dict(workload="flat_trim_knn_100k_d128", n=100_000, dim=128, n_centers=64, sigma=0.3,
               nq=1000, batch=1000, m=16, nlist=1, nprobe=1, k=10, gammas=[0.0, 0.605, 1.0],
               gamma=0.0),
}


def metric_name(cfg):
    what = "range filter, flat" if cfg.get("kind") == "range" else "kNN filter"
    return f"candidates filtered/sec (TRIM {what}; QPS, %HBM roofline, prune ratio alongside)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- plumbing
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML every
    10 ms; nvidia-smi as a fallback)."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm = []
        self.max_sm = None
        self.reasons = set()
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nv = None

    def _sample_nvml(self):
        nv = self._nv
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        for b, name in self.REASONS.items():
            if bits & b:
                self.reasons.add(name)

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,"
                              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        self.sm.append(float(out[0]))
        self.max_sm = float(out[1])
        for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"],
                           out[2:]):
            if v.strip().lower() == "active":
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                (self._sample_nvml if self._nv else self._sample_smi)()
            except Exception:
                pass
            self._stop.wait(0.01 if self._nv else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_sm,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self._nv else "nvidia-smi"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload: str):
    """Per-launch DRAM bytes of the filter kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    return j.get(workload)


# ------------------------------------------------------------------- data
def build_workload(cfg, rank: int, world: int, device: int, sharded: bool = False):
    """Seeded synthetic data + index on the device. Rank r holds the id-shard
    [r*n, (r+1)*n) (weak scaling); codebook and coarse quantizer are trained
    on rank 0 and broadcast so every shard probes identically."""
    import torch

    from paper_2508_17828_b200 import builder as B
    from paper_2508_17828_b200.ivf import IvfArrays

    dev = torch.device(f"cuda:{device}")
    torch.cuda.set_device(dev)
    t0 = time.time()
    if cfg.get("data") == "uniform_normalized":  # dataset.hpp:44-56 normalize_rows
        base = B.synth_uniform(cfg["n"], cfg["dim"], seed=1 + 7919 * rank, device=device)
        queries = B.synth_uniform(cfg["nq"], cfg["dim"], seed=2, device=device)
    else:
        centers = B.synth_normal(cfg["n_centers"], cfg["dim"], seed=0, device=device)
        base = B.synth_blobs(centers, cfg["n"], cfg["sigma"], seed=1 + 7919 * rank)
        queries = B.synth_blobs(centers, cfg["nq"], cfg["sigma"], seed=2)
    p = B.BuildParams(m=cfg["m"], nlist=cfg["nlist"], pq_seed=3, ivf_seed=4)
    if not sharded:
        arrays = B.build_ivf(base, p)
    else:
        import torch.distributed as dist
        if rank == 0:
            sub, cent = B.pq_train(base, p.m, p.ksub, p.pq_iters, p.pq_seed, p.train_sample)
            n = base.shape[0]
            sn = min(n, max(p.nlist, 50 * p.nlist))
            rows = B.sample_rows(n, sn, p.ivf_seed ^ 0x94D049BB133111EB)
            coarse = B.kmeans(base[torch.from_numpy(rows.astype(np.int64)).to(dev)].contiguous(),
                              p.nlist, p.coarse_iters, p.ivf_seed)
            sub_t = torch.from_numpy(sub.astype(np.int32)).to(dev)
        else:
            cent = torch.empty(p.ksub * cfg["dim"], dtype=torch.float32, device=dev)
            coarse = torch.empty((p.nlist, cfg["dim"]), dtype=torch.float32, device=dev)
            sub_t = torch.empty(p.m, dtype=torch.int32, device=dev)
        for t in (cent, coarse, sub_t):
            dist.broadcast(t, 0)
        sub = sub_t.cpu().numpy().astype(np.uint32)
        codes, lx = B.pq_encode(base, p.m, p.ksub, sub, cent)
        a = B.assign(base, coarse)[0] if p.nlist > 1 else torch.zeros(base.shape[0], dtype=torch.int32, device=dev)
        offs, ids = B.ivf_lists(a, p.nlist)
        idl = ids.long()
        arrays = IvfArrays(dim=cfg["dim"], m=p.m, ksub=p.ksub, sub_dims=sub_t, centroids=cent,
                           coarse=coarse.reshape(-1), list_offsets=offs,
                           list_ids=(ids + rank * cfg["n"]).to(torch.int32),
                           list_codes=codes[idl].contiguous(), list_lx=lx[idl].contiguous(),
                           vectors=base, id_base=rank * cfg["n"])
    torch.cuda.synchronize()
    log(f"[rank {rank}] built {cfg['workload']} shard in {time.time() - t0:.1f}s")
    return arrays, queries


# ------------------------------------------------------------ our GPU arm
def run_ours(args, cfg):
    import torch

    from paper_2508_17828_b200 import _lib
    from paper_2508_17828_b200 import ivf as G

    import torch.distributed as dist

    world, rank, local = dist_env()
    replicas = world > 1 and args.parallel == "replicas"
    sharded = (world > 1 and not replicas) or args.force_shard
    if sharded or replicas:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    arrays, queries = build_workload(cfg, 0 if replicas else rank, 1 if replicas else world, local, sharded)
    gix = G.GpuIvfIndex(arrays, device=local)
    q_lo, q_hi = 0, cfg["nq"]
    if replicas:  # every rank: the whole index, a contiguous slice of the queries
        from paper_2508_17828_b200.distributed import shard_bounds
        q_lo, q_hi = shard_bounds(cfg["nq"], rank, world)
    lib = _lib.load()
    import ctypes as C

    nq, B, k = cfg["nq"], cfg["batch"], cfg["k"]
    np_eff = min(cfg["nprobe"], cfg["nlist"])
    stream = torch.cuda.current_stream(dev)
    sh = C.c_void_p(stream.cuda_stream)
    # consecutive batches alternate between streams so one batch's probe and
    # filter fill the SMs left idle by the previous batch's last wave
    streams = [stream] + [torch.cuda.Stream(dev) for _ in range(max(1, args.streams) - 1)]
    shs = [C.c_void_p(x.cuda_stream) for x in streams]
    lists = torch.empty((nq, np_eff), dtype=torch.int32, device=dev)
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    cts = torch.zeros((nq, 6), dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    batches = [(b, min(B, q_hi - b)) for b in range(q_lo, q_hi, B)]
    if sharded:
        g_ids = torch.empty((world * nq, k), dtype=torch.int32, device=dev)
        g_d = torch.empty((world * nq, k), dtype=torch.float32, device=dev)
        m_ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
        m_d = torch.empty((nq, k), dtype=torch.float32, device=dev)

    def p(t, off=0):
        return C.c_void_p(t.data_ptr() + off)

    n_probe_k = C.c_uint32(0)
    _lib.check(lib.trim_probe_launches(gix.handle, cfg["nprobe"], C.byref(n_probe_k)), "probe_launches")

    def step(gamma, filt_events=None):
        launches = 0
        fork = torch.cuda.Event()
        fork.record(stream)
        for x in streams[1:]:
            x.wait_event(fork)
        for i, (b0, nb) in enumerate(batches):
            st_, sh_ = streams[i % len(streams)], shs[i % len(streams)]
            qoff = b0 * cfg["dim"] * 4
            _lib.check(lib.trim_probe_device(gix.handle, p(queries, qoff), nb, cfg["nprobe"],
                                             p(lists, b0 * np_eff * 4), sh_), "probe")
            launches += n_probe_k.value
            if filt_events is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(st_)
            _lib.check(lib.trim_search_knn_preassigned_device(
                gix.handle, p(queries, qoff), nb, k, p(lists, b0 * np_eff * 4), np_eff,
                float(np.float32(gamma)), p(ids, b0 * k * 4), p(dists, b0 * k * 4),
                p(cts, b0 * 48), p(status), sh_), "knn")
            # the filter kernel, plus trim_knn_setup_kernel (seeds + plan) on IVF indexes
            launches += 1 + (1 if cfg["nlist"] > 1 and os.environ.get("TRIM_KNN_SETUP") != "0" else 0)
            if filt_events is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(st_)
                filt_events.append((e0, e1))
        for x in streams[1:]:
            j = torch.cuda.Event()
            j.record(x)
            stream.wait_event(j)
        if sharded:
            dist.all_gather_into_tensor(g_ids, ids)
            dist.all_gather_into_tensor(g_d, dists)
            _lib.check(lib.trim_merge_topk_device(p(g_d), p(g_ids), world, nq, k, p(m_d), p(m_ids),
                                                  local, sh), "merge")
            launches += 1
        return launches

    def timed(gamma, steps, warmup, clocks=None):
        for _ in range(warmup):
            step(gamma)
        torch.cuda.synchronize()
        if sharded or replicas:
            dist.barrier()
        torch.cuda.synchronize()
        ev = []
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        launches = 0
        ctx = clocks if clocks is not None else _Null()
        with ctx:
            s0.record(stream)
            for _ in range(steps):
                launches += step(gamma, ev)
            s1.record(stream)
            torch.cuda.synchronize()
        if sharded or replicas:
            dist.barrier()
        torch.cuda.synchronize()
        ms = s0.elapsed_time(s1)
        # time with at least one filter kernel in flight (launches may overlap
        # across the two streams): union of the per-launch [start, end] intervals
        iv = sorted((s0.elapsed_time(a), s0.elapsed_time(b)) for a, b in ev)
        filt_ms, cur = 0.0, None
        for a, b in iv:
            if cur is None or a > cur[1]:
                if cur is not None:
                    filt_ms += cur[1] - cur[0]
                cur = [a, b]
            else:
                cur[1] = max(cur[1], b)
        if cur is not None:
            filt_ms += cur[1] - cur[0]
        ct = cts[q_lo:q_hi].sum(0).cpu().numpy()  # identical every step
        if sharded or replicas:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            ctt = torch.from_numpy(ct.astype(np.int64)).to(dev)
            dist.all_reduce(ctt)
            ct = ctt.cpu().numpy()
        return ms, filt_ms, len(ev), ct, launches

    gammas = cfg["gammas"] if not args.gamma else [args.gamma]
    head = args.gamma if args.gamma else cfg["gamma"]
    sweep = {}
    for g in gammas:
        if g == head:
            continue
        ms, fms, nl, ct, _ = timed(g, max(1, min(2, args.steps)), 1)
        sweep[str(g)] = dict(ms_per_step=ms / max(1, min(2, args.steps)),
                             cand_per_s=float(ct[3]) * max(1, min(2, args.steps)) / (ms / 1e3),
                             qps=nq * max(1, min(2, args.steps)) / (ms / 1e3),
                             prune_ratio=float(ct[2] / max(1, ct[2] + ct[0])))
        if rank == 0:
            sweep[str(g)][f"recall@{k}"] = recall(gix, queries, ids, k, args.recall_q, world)
    clk = ClockSampler(local)
    for _ in range(args.warmup):
        step(head)
    gix.skipped_positions(reset=True)  # (synchronises; outside the timed region)
    ms, fms, nl, ct, launches = timed(head, args.steps, 0, clk)
    skipped = gix.skipped_positions() / args.steps  # list-level bound, per step (this rank)
    evaluated, dc = float(ct[3]), float(ct[0])
    total_cand = evaluated * args.steps
    value = total_cand / (ms / 1e3)
    qps = nq * args.steps / (ms / 1e3)
    out = dict(metric=metric_name(cfg),
               value=value, unit="candidates/s", n_gpus=world, steps=args.steps,
               warmup=args.warmup, ms_per_step=ms / args.steps, higher_is_better=True,
               scaling="strong" if replicas else "weak", vs_baseline=None, dtype="f32 (u8 PQ codes)",
               data="synthetic")
    out["config"] = dict(workload=cfg["workload"], n_per_gpu=cfg["n"], dim=cfg["dim"],
                         queries=nq, batch=B, m=cfg["m"], nlist=cfg["nlist"],
                         nprobe=cfg["nprobe"], k=k, gamma=head,
                         parallelism=(f"replicas x{world}" if replicas else f"id-shard x{world}")
                         if (world > 1 or sharded) else "single",
                         l2="index > L2 (no flush needed)" if cfg["n"] * cfg["dim"] * 4 > 126e6
                         else "index fits L2; reported as-is",
                         data_gen=("device Philox uniform [0,1) + L2-normalised rows, seeds base=1 queries=2" if cfg.get("data") == "uniform_normalized" else "device Philox blobs, seeds centers=0 base=1 queries=2"))
    out["qps"] = qps
    out["prune_ratio"] = float(ct[2] / max(1, ct[2] + ct[0]))
    out["candidates_per_query"] = evaluated / (nq * (world if False else 1))
    # roofline of the dominant kernel (the fused filter), per launch
    peak, peak_src = measured_peaks()
    m, D = cfg["m"], cfg["dim"]
    s_frac = dc / max(1.0, evaluated)
    bytes_per_cand = m + 4 + s_frac * (4 * D + 4)
    # positions pruned as whole lists by the list-level bound never read their
    # code/lx: the kernel's algorithmic bytes count only the positions it scans
    skipped_all = skipped * (world if world > 1 else 1)
    scanned = evaluated - skipped_all
    flat_bounds = cfg["nlist"] == 1 and cfg["n"] <= (16 << 20) and os.environ.get("TRIM_FLAT_BOUNDS") != "0"
    if flat_bounds:
        # flat scans read D~[q][row] (4 B) for evaluated candidates; exact rows only
        # for the few members that can enter the top-k (not counted)
        alg_bytes_step = scanned * (m + 4) + dc * 4
    else:
        alg_bytes_step = scanned * (m + 4) + dc * (4 * D + 4)
    per_launch_bytes = alg_bytes_step / max(1, nl // args.steps) / (world if world > 1 else 1)
    avg_launch_ms = fms / max(1, nl)  # filter-busy time per launch (overlap-aware)
    achieved = per_launch_bytes / (avg_launch_ms / 1e3) / 1e9
    tr = ncu_traffic(cfg["workload"])
    out["roofline"] = dict(bound="hbm", achieved=achieved, peak=peak, unit="GB/s",
                           frac=achieved / peak, traffic=tr, kernel="trim_knn_kernel",
                           bytes_per_candidate=bytes_per_cand, peak_source=peak_src,
                           filter_share_of_step=fms / ms,
                           list_skip_fraction=skipped_all / max(1.0, evaluated),
                           flat_distance_bounds=flat_bounds,
                           stream_equivalent_GBps=(evaluated * (m + 4) + dc * (4 * D + 4))
                           / max(1, nl // args.steps) / (world if world > 1 else 1)
                           / (avg_launch_ms / 1e3) / 1e9)
    out["gpu_launches"] = launches
    out["clocks"] = clk.summary()
    out["sweep"] = sweep
    if rank == 0:
        out[f"recall@{k}"] = recall(gix, queries, ids, k, args.recall_q, world)
    # e2e through the C-ABI host call with pinned host buffers
    out["e2e"] = e2e(gix, queries, cfg, head, args, world, rank)
    if cfg.get("baseline_kprime") and rank == 0 and world == 1:
        out["baseline_ivfpq"] = baseline_line(gix, arrays, queries, cfg, args)
    if rank == 0 and world == 1 and not args.skip_cpu:
        out["cpu_baseline"] = cpu_baseline(arrays, queries, cfg, head, args)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if sharded:
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def recall(gix, queries, ids, k, nsample, world):
    """bench::recall_at_k (bench/metrics.hpp:14-24), averaged over `nsample`
    queries, against the exact ground truth computed on the GPU bit-identically
    to core/ground_truth.hpp (trim_ground_truth_knn). Informational; the local
    shard's results at N > 1 are not comparable (None)."""
    if world > 1 or nsample <= 0:
        return None
    if gix.n > (16 << 20):  # the exact GT kernel holds nq x n bounds: not at 100M rows
        return None
    from paper_2508_17828_b200 import ivf as G
    q = queries[:nsample].cpu().numpy()
    gt, _ = G.ground_truth_knn(gix, q, k)
    got = ids[:nsample].cpu().numpy().view(np.uint32)
    hits = sum(len(set(gt[i].tolist()) & set(got[i, :k].tolist())) for i in range(len(gt)))
    return hits / (k * len(gt))


def e2e(gix, queries, cfg, gamma, args, world, rank):
    import torch

    from paper_2508_17828_b200 import ivf as G
    nq, B, k = cfg["nq"], cfg["batch"], cfg["k"]
    hq = queries.cpu().pin_memory()
    hqn = hq.numpy()
    prof = G.PruningProfile.manual(gamma)
    steps = max(1, min(args.steps, 3))

    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max(1, args.streams))  # client threads: one stream each in the C ABI

    # results land in pinned host buffers (a serving client's staging memory)
    from paper_2508_17828_b200 import _lib
    import ctypes as C
    lib = _lib.load()
    h_ids = torch.empty((nq, k), dtype=torch.int32).pin_memory().numpy()
    h_d = torch.empty((nq, k), dtype=torch.float32).pin_memory().numpy()
    h_ct = torch.empty((nq, 6), dtype=torch.int64).pin_memory().numpy()

    def one(b):
        nb = min(B, nq - b)
        _lib.check(lib.trim_search_knn(gix.handle, C.c_void_p(hqn[b:].ctypes.data), nb, k, cfg["nprobe"],
                                       prof.gamma_f32(), C.c_void_p(h_ids[b:].ctypes.data),
                                       C.c_void_p(h_d[b:].ctypes.data), C.c_void_p(h_ct[b:].ctypes.data)),
                   "search_trim_ivf_knn")
        return int(h_ct[b:b + nb, 3].sum())

    def once():
        return sum(pool.map(one, range(0, nq, B)))

    once()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cand = 0
    for _ in range(steps):
        cand += once()
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    return dict(value=cand / sec, unit="candidates/s", qps=nq * steps / sec,
                h2d_bytes_per_step=nq * cfg["dim"] * 4,
                d2h_bytes_per_step=nq * k * 8 + nq * 48 + 4 * len(range(0, nq, B)),
                api=f"trim_search_knn (C ABI, host buffers; pinned queries and results; {max(1, args.streams)} client threads)",
                shard_local=world > 1)


def baseline_line(gix, arrays, queries, cfg, args):
    """Config 2's comparison point: ivf::search_baseline_ivfpq (ivf.hpp:193-237,
    ADC for every probed entry, refine pool k') through the C-ABI host call,
    all queries, two client threads; QPS and recall@k alongside TRIM's."""
    import torch
    from concurrent.futures import ThreadPoolExecutor

    from paper_2508_17828_b200 import ivf as G
    nq, B, k, kp = cfg["nq"], cfg["batch"], cfg["k"], cfg["baseline_kprime"]
    hq = queries.cpu().numpy()
    pool = ThreadPoolExecutor(max(1, args.streams))
    res = {}

    def one(b):
        ids, _, ct = G.search_baseline_ivfpq_batch(gix, hq[b:b + B], k, cfg["nprobe"], kp)
        res[b] = ids
        return int(ct[:, 3].sum())
    sum(pool.map(one, range(0, min(nq, 2 * B), B)))  # warm-up
    t0 = time.perf_counter()
    ev = sum(pool.map(one, range(0, nq, B)))
    sec = time.perf_counter() - t0
    ids = np.concatenate([res[b] for b in range(0, nq, B)])
    rec = recall(gix, queries, torch.from_numpy(ids.view(np.int32)), k, args.recall_q, 1)
    return dict(k_prime=kp, qps=nq / sec, cand_per_s=ev / sec, **{f"recall@{k}": rec},
                api="trim_search_baseline_ivfpq (C ABI, host buffers)")


def _host_index(arrays):
    from oracle.oracle import HostIndex
    from paper_2508_17828_b200.builder import to_host
    h = to_host(arrays)
    return HostIndex(dim=h.dim, m=h.m, ksub=h.ksub, sub_dims=h.sub_dims, centroids=h.centroids,
                     coarse=h.coarse, list_offsets=h.list_offsets, list_ids=h.list_ids,
                     list_codes=h.list_codes, list_lx=h.list_lx, vectors=h.vectors)


class RefTimer:
    """The reference CPU path (oracle/_ref: the unmodified reference headers
    compiled in place) over query samples, timed like
    bench::detail_sweep::run_queries (sweep.hpp:121-152: steady_clock around a
    parallel_for over queries). Falls back to the C restatement ("port") when
    oracle/_ref is absent. Only bench.py's CPU legs use it."""

    def __init__(self, hix, cfg, gamma, threads):
        from oracle import oracle as O
        self.cfg, self.gamma, self.threads = cfg, gamma, threads
        if O.ref_available():
            self.kind = "reference"
            self.ref = O.RefOracle()
            self.ref.set_threads(threads)
            self.sess = self.ref.session(hix)
        else:
            self.kind = "port"
            self.co = O.COracle()
            self.hix = hix

    def run(self, qsub):
        """-> (seconds, evaluated, dc, pruned) for one parallel batch."""
        rng = self.cfg.get("kind") == "range"
        if self.kind == "reference":
            sec, ct = self.ref.session_run(self.sess, 1 if rng else 0, qsub, self.cfg["k"], self.cfg["nprobe"],
                                           self.gamma, arg=self.cfg.get("radius", 0.0))
            return sec, int(ct[3]), int(ct[0]), int(ct[2])
        t0 = time.perf_counter()
        if rng:
            _, _, _, ct, _ = self.co.search_range(self.hix, qsub, self.cfg["radius"], self.cfg["nprobe"],
                                                  self.gamma, threads=self.threads)
        else:
            _, _, ct, _ = self.co.search_knn(self.hix, qsub, self.cfg["k"], self.cfg["nprobe"], self.gamma,
                                             threads=self.threads)
        return time.perf_counter() - t0, int(ct[:, 3].sum()), int(ct[:, 0].sum()), int(ct[:, 2].sum())

    def close(self):
        if self.kind == "reference":
            self.ref.session_destroy(self.sess)

    def calibrate(self, qs):
        n0 = min(len(qs), max(4 * self.threads, 64))
        sec, *_ = self.run(qs[:n0])
        return n0 / max(sec, 1e-9)  # queries/s


def cpu_baseline(arrays, queries, cfg, gamma, args):
    t0 = time.time()
    hix = _host_index(arrays)
    qs = queries.cpu().numpy()
    log(f"host copy for the CPU baseline: {time.time() - t0:.1f}s")
    threads = os.cpu_count() or 1
    rt = RefTimer(hix, cfg, gamma, threads)
    qps = rt.calibrate(qs)
    n = int(min(len(qs), max(4 * threads, args.cpu_seconds * qps)))
    sec, ev, dc, pr = rt.run(qs[:n])
    rt.close()
    return dict(value=ev / sec, unit="candidates/s", cores=threads, kind=rt.kind,
                sample=f"first {n} of {len(qs)} queries of {cfg['workload']} at gamma={gamma}, "
                       f"{threads} threads, {sec:.1f}s",
                qps=n / sec, prune_ratio=pr / max(1, pr + dc))


# ------------------------------------------------------ config 3: range
def calibrate_radius(arrays, queries, cfg):
    """bench::pick_radius_for_fraction (bench/radius.hpp:20-55): the
    e_fraction = result_size/N quantile (EmpiricalCdf: linear between order
    statistics) of pooled query-to-row distances over 20,000 sampled rows x 200
    sampled queries (the reference's Fisher-Yates sampler, seeds 1 and 2).
    Distances by torch.cdist (a workload parameter, not a parity value)."""
    import torch

    from paper_2508_17828_b200 import builder as B
    x = arrays.vectors
    rows = torch.from_numpy(B.sample_rows(x.shape[0], min(20000, x.shape[0]), 1).astype(np.int64)).to(x.device)
    qi = torch.from_numpy(B.sample_rows(queries.shape[0], min(200, queries.shape[0]), 2).astype(np.int64)).to(x.device)
    d = torch.cdist(queries[qi].double(), x[rows].double()).reshape(-1)
    d, _ = torch.sort(d)
    p = cfg["result_size"] / x.shape[0]
    pos = p * (d.numel() - 1)
    lo = int(pos)
    if lo + 1 >= d.numel():
        return float(d[-1])
    return float(d[lo] + (pos - lo) * (d[lo + 1] - d[lo]))


def run_ours_range(args, cfg):
    import ctypes as C

    import torch

    from paper_2508_17828_b200 import _lib
    from paper_2508_17828_b200 import ivf as G

    world, rank, local = dist_env()
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    arrays, queries = build_workload(cfg, rank, world, local, False)
    gix = G.GpuIvfIndex(arrays, device=local)
    lib = _lib.load()
    radius = calibrate_radius(arrays, queries, cfg)
    cfg["radius"] = radius
    nq, B, cap = cfg["nq"], cfg["batch"], 4096
    d_rad = torch.full((nq,), radius, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    streams = [stream] + [torch.cuda.Stream(dev) for _ in range(max(1, args.streams) - 1)]
    shs = [C.c_void_p(x.cuda_stream) for x in streams]
    counts = torch.zeros(nq, dtype=torch.int32, device=dev)
    ids = torch.empty((nq, cap), dtype=torch.int32, device=dev)
    dist = torch.empty((nq, cap), dtype=torch.float32, device=dev)
    cts = torch.zeros((nq, 6), dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    batches = [(b, min(B, nq - b)) for b in range(0, nq, B)]
    P = lambda t, off=0: C.c_void_p(t.data_ptr() + off)

    def step(gamma, ev=None):
        fork = torch.cuda.Event()
        fork.record(stream)
        for x in streams[1:]:
            x.wait_event(fork)
        for i, (b0, nb) in enumerate(batches):
            st_, sh_ = streams[i % len(streams)], shs[i % len(streams)]
            if ev is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(st_)
            _lib.check(lib.trim_search_range_device(
                gix.handle, P(queries, b0 * cfg["dim"] * 4), nb, P(d_rad, b0 * 4), cfg["nprobe"],
                float(np.float32(gamma)), cap, P(counts, b0 * 4), P(ids, b0 * cap * 4), P(dist, b0 * cap * 4),
                P(cts, b0 * 48), P(status), sh_), "range")
            if ev is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(st_)
                ev.append((e0, e1))
        for x in streams[1:]:
            j = torch.cuda.Event()
            j.record(x)
            stream.wait_event(j)
        return len(batches) * 6  # r2, range, seg, cub (2 kernels), finish

    def timed(gamma, steps, warmup, clocks=None):
        for _ in range(warmup):
            step(gamma)
        torch.cuda.synchronize()
        ev = []
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        launches = 0
        with (clocks if clocks is not None else _Null()):
            s0.record(stream)
            for _ in range(steps):
                launches += step(gamma, ev)
            s1.record(stream)
            torch.cuda.synchronize()
        ms = s0.elapsed_time(s1)
        iv = sorted((s0.elapsed_time(a), s0.elapsed_time(b)) for a, b in ev)
        busy, cur = 0.0, None
        for a, b in iv:
            if cur is None or a > cur[1]:
                if cur is not None:
                    busy += cur[1] - cur[0]
                cur = [a, b]
            else:
                cur[1] = max(cur[1], b)
        if cur is not None:
            busy += cur[1] - cur[0]
        return ms, busy, len(ev), cts.sum(0).cpu().numpy(), launches

    head = args.gamma if args.gamma is not None else cfg["gamma"]
    # size the per-query result slots: the largest result set over the gammas run
    gams = [head] if args.gamma is not None else cfg["gammas"]
    mx = 0
    for g in set(gams) | {head}:
        status.zero_()
        step(g)
        torch.cuda.synchronize()
        mx = max(mx, int(counts.max()))
    if mx > cap:
        cap = (mx * 5 // 4 + 127) // 128 * 128
        ids = torch.empty((nq, cap), dtype=torch.int32, device=dev)
        dist = torch.empty((nq, cap), dtype=torch.float32, device=dev)
    status.zero_()
    sweep = {}
    for g in gams:
        if g == head:
            continue
        ms, _, _, ct, _ = timed(g, 1, 1)
        sweep[str(g)] = dict(ms_per_step=ms, cand_per_s=float(ct[3]) / (ms / 1e3), qps=nq / (ms / 1e3),
                             prune_ratio=float(ct[2] / max(1, ct[2] + ct[0])),
                             mean_result_size=float(counts.double().mean()))
    clk = ClockSampler(local)
    for _ in range(args.warmup):
        step(head)
    gix.skipped_positions(reset=True)  # (synchronises; outside the timed region)
    ms, busy, nl, ct, launches = timed(head, args.steps, 0, clk)
    skipped = gix.skipped_positions() / args.steps  # rows pruned as whole blocks, per step
    assert int(status.item()) & 1 == 0, "range result larger than cap"
    evaluated, dc = float(ct[3]), float(ct[0])
    value = evaluated * args.steps / (ms / 1e3)
    out = dict(metric=metric_name(cfg),
               value=value, unit="candidates/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
               ms_per_step=ms / args.steps, higher_is_better=True, scaling="weak", vs_baseline=None,
               dtype="f32 (u8 PQ codes)", data="synthetic")
    out["config"] = dict(workload=cfg["workload"], n_per_gpu=cfg["n"], dim=cfg["dim"], queries=nq, batch=B,
                         m=cfg["m"], nlist=1, gamma=head, radius=radius,
                         radius_rule="pick_radius_for_fraction(100/N, 20000 rows, 200 queries)",
                         parallelism="single", l2="index > L2 (no flush needed)",
                         data_gen=("device Philox uniform [0,1) + L2-normalised rows, seeds base=1 queries=2" if cfg.get("data") == "uniform_normalized" else "device Philox blobs, seeds centers=0 base=1 queries=2"))
    out["qps"] = nq * args.steps / (ms / 1e3)
    out["prune_ratio"] = float(ct[2] / max(1, ct[2] + ct[0]))
    out["mean_result_size"] = float(counts.double().mean())
    qt = gix.info()["range_query_tile"]
    peak, peak_src = measured_peaks()
    m, D = cfg["m"], cfg["dim"]
    if skipped > 0:  # block partition: only the kept blocks' rows are scanned (codes + lx)
        qt = 1
        alg = (evaluated - skipped) * (m + 4) + dc * (4 * D + 4)
    else:  # the query-tiled flat scan streams codes + lx once per query tile
        alg = (nq + qt - 1) // qt * cfg["n"] * (m + 4) + dc * (4 * D + 4)
    achieved = alg / (busy / args.steps / 1e3) / 1e9
    out["roofline"] = dict(bound="hbm", achieved=achieved, peak=peak, unit="GB/s", frac=achieved / peak,
                           traffic=ncu_traffic(cfg["workload"]),
                           kernel="trim_range_kernel (block partition)" if skipped > 0 else "trim_range_flat_kernel",
                           bytes_per_step=alg, query_tile=qt, peak_source=peak_src,
                           block_skip_fraction=skipped / max(1.0, evaluated),
                           pair_equivalent_GBps=(evaluated * (m + 4) + dc * (4 * D + 4)) / (busy / args.steps / 1e3) / 1e9)
    out["gpu_launches"] = launches
    out["clocks"] = clk.summary()
    out["sweep"] = sweep
    # e2e: the host C-ABI call per batch from two client threads
    hq = queries.cpu().pin_memory().numpy()
    prof = G.PruningProfile.manual(head)
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max(1, args.streams))

    def one(b):
        offs, _, _, c = G.search_trim_ivf_range_batch(gix, prof, hq[b:b + B], radius, 1)
        return int(c[:, 3].sum()), int(offs[-1])

    def once():
        r = list(pool.map(one, range(0, nq, B)))
        return sum(x[0] for x in r), sum(x[1] for x in r)
    once()
    t0 = time.perf_counter()
    reps = max(1, min(args.steps, 2))
    tot = 0
    for _ in range(reps):
        c, nres = once()
        tot += c
    sec = time.perf_counter() - t0
    out["e2e"] = dict(value=tot / sec, unit="candidates/s", qps=nq * reps / sec,
                      h2d_bytes_per_step=nq * D * 4 + nq * 4,
                      d2h_bytes_per_step=nres * 8 + (nq + 1) * 8 + nq * 48,
                      api=f"trim_search_range (C ABI, host buffers; {max(1, args.streams)} client threads)")
    if rank == 0 and not args.skip_cpu:
        out["cpu_baseline"] = cpu_baseline(arrays, queries, cfg, head, args)
    print(json.dumps(out), flush=True)


# ------------------------------------------------------ graph filter (g1)
def build_graph_workload(cfg, device):
    """Config-1 data on the device, a flat index (landmarks: pq::train +
    encode), and the kNN + random-link graph over it (builder.build_knn_graph)."""
    import torch

    from paper_2508_17828_b200 import builder as B
    from paper_2508_17828_b200.ivf import GpuIvfIndex
    t0 = time.time()
    centers = B.synth_normal(cfg["n_centers"], cfg["dim"], seed=0, device=device)
    base = B.synth_blobs(centers, cfg["n"], cfg["sigma"], seed=1)
    queries = B.synth_blobs(centers, cfg["nq"], cfg["sigma"], seed=2)
    arrays = B.build_ivf(base, B.BuildParams(m=cfg["m"], nlist=1, pq_seed=3))
    gix = GpuIvfIndex(arrays, device=device)
    ga = B.knn_graph_from_flat(arrays, gix, cfg["M"], cfg["n_random"], seed=5)
    torch.cuda.synchronize()
    log(f"built {cfg['workload']} in {time.time() - t0:.1f}s")
    return arrays, gix, ga, queries


def _host_graph(ga):
    from oracle.oracle import HostGraph
    n, dim = ga.vectors.shape
    return HostGraph(n=n, M=ga.M, efc=0, entry=ga.entry, offsets=ga.offsets, nbrs=ga.nbrs, dim=dim,
                     m=ga.codes.shape[1], ksub=ga.ksub, sub_dims=ga.sub_dims, centroids=ga.centroids,
                     codes=ga.codes, lx=ga.lx, vectors=ga.vectors)


def graph_cpu_timer(ga, cfg, gamma, qs, budget_s, threads):
    """The reference's graph::search_trim_knn (oracle/_ref, unmodified headers)
    over a bounded query sample with all host threads, timed like run_queries
    (sweep.hpp:121-152). -> (seconds, queries, counters[6])."""
    from oracle import oracle as O
    ref = O.RefOracle()
    ref.set_threads(threads)
    sess = ref.graph_session(_host_graph(ga))
    try:
        n0 = min(len(qs), max(4 * threads, 64))
        sec, _ = ref.graph_session_run(sess, "trim_knn", qs[:n0], k=cfg["k"], ef=cfg["ef"], gamma=gamma)
        n = int(min(len(qs), max(4 * threads, budget_s * n0 / max(sec, 1e-9))))
        sec, ct = ref.graph_session_run(sess, "trim_knn", qs[:n], k=cfg["k"], ef=cfg["ef"], gamma=gamma)
    finally:
        ref.graph_session_destroy(sess)
    return sec, n, ct


def run_ours_graph(args, cfg):
    import torch

    from paper_2508_17828_b200 import graph as GG
    from paper_2508_17828_b200.graph import GpuGraph
    from paper_2508_17828_b200.ivf import PruningProfile

    world, rank, local = dist_env()
    if world > 1:  # replicas: the graph is small; every rank searches a slice of the queries
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch.distributed as dist
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    arrays, gix, ga, queries = build_graph_workload(cfg, local)
    gg = GpuGraph(ga, device=local)
    nq, B, k, ef = cfg["nq"], cfg["batch"], cfg["k"], cfg["ef"]
    q_lo, q_hi = 0, nq
    if world > 1:
        from paper_2508_17828_b200.distributed import shard_bounds
        q_lo, q_hi = shard_bounds(nq, rank, world)
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    cts = torch.zeros((nq, 6), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    streams = [stream] + [torch.cuda.Stream(dev) for _ in range(max(1, args.streams) - 1)]
    batches = [(b, min(B, q_hi - b)) for b in range(q_lo, q_hi, B)]

    def step(gamma, ev=None):
        prof = PruningProfile.manual(gamma)
        fork = torch.cuda.Event()
        fork.record(stream)
        for x in streams[1:]:
            x.wait_event(fork)
        for i, (b0, nb) in enumerate(batches):
            st_ = streams[i % len(streams)]
            if ev is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(st_)
            GG.search_trim_knn_device(gg, prof, queries[b0:b0 + nb], k, ef, ids[b0:b0 + nb], dists[b0:b0 + nb],
                                      cts[b0:b0 + nb], stream=st_)
            if ev is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(st_)
                ev.append((e0, e1))
        for x in streams[1:]:
            j = torch.cuda.Event()
            j.record(x)
            stream.wait_event(j)
        return len(batches)

    def timed(gamma, steps, warmup, clocks=None):
        for _ in range(warmup):
            step(gamma)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev = []
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches = 0
        with (clocks if clocks is not None else _Null()):
            s0.record(stream)
            for _ in range(steps):
                launches += step(gamma, ev)
            s1.record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = s0.elapsed_time(s1)
        iv = sorted((s0.elapsed_time(a), s0.elapsed_time(b)) for a, b in ev)
        busy, cur = 0.0, None
        for a, b in iv:
            if cur is None or a > cur[1]:
                if cur is not None:
                    busy += cur[1] - cur[0]
                cur = [a, b]
            else:
                cur[1] = max(cur[1], b)
        if cur is not None:
            busy += cur[1] - cur[0]
        ct = cts[q_lo:q_hi].sum(0).cpu().numpy()
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            ctt = torch.from_numpy(ct.astype(np.int64)).to(dev)
            dist.all_reduce(ctt)
            ct = ctt.cpu().numpy()
        return ms, busy, len(ev), ct, launches

    def rec(nsample):
        if world > 1 or nsample <= 0:
            return None
        from paper_2508_17828_b200 import ivf as G
        gt, _ = G.ground_truth_knn(gix, queries[:nsample].cpu().numpy(), k)
        got = ids[:nsample].cpu().numpy().view(np.uint32)
        return sum(len(set(gt[i].tolist()) & set(got[i].tolist())) for i in range(len(gt))) / (k * len(gt))

    head = args.gamma if args.gamma else cfg["gamma"]
    sweep = {}
    for g in ([] if args.gamma else cfg["gammas"]):
        ms, _, _, ct, _ = timed(g, 1, 1)
        sweep[str(g)] = dict(ms_per_step=ms, cand_per_s=float(ct[3]) / (ms / 1e3), qps=(q_hi - q_lo) * world / (ms / 1e3),
                             prune_ratio=float(ct[2] / max(1, ct[2] + ct[0])), hops_per_query=float(ct[4]) / nq,
                             **{f"recall@{k}": rec(args.recall_q)})
    clk = ClockSampler(local)
    ms, busy, nl, ct, launches = timed(head, args.steps, args.warmup, clk)
    evaluated, dc = float(ct[3]), float(ct[0])
    value = evaluated * args.steps / (ms / 1e3)
    m, D = cfg["m"], cfg["dim"]
    s_frac = dc / max(1.0, evaluated)
    bpc = m + 4 + 4 + s_frac * 4 * D  # code + Γ(l,x) + neighbour id + exact rows
    per_launch = evaluated * bpc / max(1, nl // args.steps) / world
    achieved = per_launch / (busy / max(1, nl) / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    out = dict(metric="candidates filtered/sec (TRIM graph filter, graph/search.hpp:188-264; QPS, prune ratio alongside)",
               value=value, unit="candidates/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
               ms_per_step=ms / args.steps, higher_is_better=True, scaling="strong" if world > 1 else "weak",
               vs_baseline=None, dtype="f32 (u8 PQ codes)", data="synthetic",
               config=dict(workload=cfg["workload"], n=cfg["n"], dim=D, queries=nq, batch=B, m=m, k=k, ef=ef,
                           degree=cfg["M"] + cfg["n_random"], levels=1, gamma=head,
                           parallelism=f"replicas x{world}" if world > 1 else "single",
                           l2="graph + vectors + codes (~60 MB) fit L2; reported as-is",
                           data_gen="device Philox blobs (config-1 shape), seeds centers=0 base=1 queries=2; "
                                    "graph = 32 exact NN (trim_ground_truth_knn) + 8 seeded random links"),
               qps=(q_hi - q_lo) * world * args.steps / (ms / 1e3),
               prune_ratio=float(ct[2] / max(1, ct[2] + ct[0])), hops_per_query=float(ct[4]) / nq,
               candidates_per_query=evaluated / nq)
    out["roofline"] = dict(bound="hbm", achieved=achieved, peak=peak, unit="GB/s", frac=achieved / peak,
                           traffic=ncu_traffic(cfg["workload"]), kernel="trim_graph_kernel",
                           bytes_per_candidate=bpc, peak_source=peak_src, filter_share_of_step=busy / ms,
                           note="one warp per query walks the graph: latency-bound (dependent hops), not "
                                "bandwidth-bound")
    out["gpu_launches"] = launches
    out["clocks"] = clk.summary()
    out["sweep"] = sweep
    out[f"recall@{k}"] = rec(args.recall_q)
    if rank == 0:
        # e2e: the C-ABI host call (pinned host queries in, results + counters out)
        hq = queries[q_lo:q_hi].cpu().pin_memory().numpy()
        from concurrent.futures import ThreadPoolExecutor
        pool = ThreadPoolExecutor(max(1, args.streams))
        prof = PruningProfile.manual(head)

        from paper_2508_17828_b200 import _lib
        import ctypes as C
        lib = _lib.load()
        nh = len(hq)
        h_ids = torch.empty((nh, k), dtype=torch.int32).pin_memory().numpy()
        h_d = torch.empty((nh, k), dtype=torch.float32).pin_memory().numpy()
        h_ct = torch.empty((nh, 6), dtype=torch.int64).pin_memory().numpy()

        def one(b):  # pinned queries in, pinned results out (the serving client's staging memory)
            nb = min(B, nh - b)
            _lib.check(lib.trim_graph_search_knn(gg.handle, C.c_void_p(hq[b:].ctypes.data), nb, k, ef,
                                                 prof.gamma_f32(), C.c_void_p(h_ids[b:].ctypes.data),
                                                 C.c_void_p(h_d[b:].ctypes.data), C.c_void_p(h_ct[b:].ctypes.data)),
                       "search_trim_knn")
            return int(h_ct[b:b + nb, 3].sum())
        sum(pool.map(one, range(0, len(hq), B)))
        t0 = time.perf_counter()
        cand = sum(pool.map(one, range(0, len(hq), B)))
        sec = time.perf_counter() - t0
        out["e2e"] = dict(value=cand / sec, unit="candidates/s", qps=len(hq) / sec,
                          h2d_bytes_per_step=len(hq) * D * 4, d2h_bytes_per_step=len(hq) * (k * 8 + 48),
                          api=f"trim_graph_search_knn (C ABI, pinned host queries and results; {max(1, args.streams)} client threads)")
        if world == 1 and not args.skip_cpu:
            threads = os.cpu_count() or 1
            sec, n, cct = graph_cpu_timer(ga, cfg, head, queries.cpu().numpy(), args.cpu_seconds, threads)
            out["cpu_baseline"] = dict(value=float(cct[3]) / sec, unit="candidates/s", cores=threads, kind="reference",
                                       sample=f"first {n} of {nq} queries of {cfg['workload']} at gamma={head}, "
                                              f"{threads} threads, {sec:.1f}s",
                                       qps=n / sec, prune_ratio=float(cct[2] / max(1, cct[2] + cct[0])))
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference_graph(args, cfg):
    world, rank, local = dist_env()
    if rank != 0:
        return
    import torch
    torch.cuda.set_device(local)
    arrays, gix, ga, queries = build_graph_workload(cfg, local)
    head = args.gamma if args.gamma else cfg["gamma"]
    threads = os.cpu_count() or 1
    qs = queries.cpu().numpy()
    per = max(1.0, args.cpu_seconds / max(1, args.steps + args.warmup))
    secs, evs, nqs = 0.0, 0, 0
    for i in range(args.warmup + args.steps):
        sec, n, ct = graph_cpu_timer(ga, cfg, head, np.roll(qs, -i * 97, 0), per, threads)
        if i >= args.warmup:
            secs, evs, nqs = secs + sec, evs + int(ct[3]), nqs + n
    value = evs / secs
    out = dict(metric="candidates filtered/sec (TRIM graph filter, graph/search.hpp:188-264; QPS, prune ratio alongside)",
               value=value, unit="candidates/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
               ms_per_step=secs * 1e3 / args.steps, higher_is_better=True, scaling="weak", vs_baseline=None,
               dtype="f32 (u8 PQ codes)", data="synthetic", impl="reference",
               config=dict(workload=cfg["workload"], n=cfg["n"], dim=cfg["dim"], queries=cfg["nq"], m=cfg["m"],
                           k=cfg["k"], ef=cfg["ef"], gamma=head),
               qps=nqs / secs,
               cpu_baseline=dict(value=value, unit="candidates/s", cores=threads, kind="reference",
                                 sample=f"~{nqs // max(1, args.steps)} queries per step of {cfg['workload']}, "
                                        f"{threads} threads"),
               e2e=dict(value=value, unit="candidates/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(out), flush=True)


# ------------------------------------------------------ reference CPU arm
def run_reference(args, cfg):
    world, rank, local = dist_env()
    if rank != 0:
        return
    import torch
    torch.cuda.set_device(local)
    arrays, queries = build_workload(cfg, 0, 1, local)
    hix = _host_index(arrays)
    qs = queries.cpu().numpy()
    arrays_r = arrays
    threads = os.cpu_count() or 1
    head = args.gamma if args.gamma else cfg["gamma"]
    if cfg.get("kind") == "range":
        import torch as _t
        cfg["radius"] = calibrate_radius(arrays_r, queries, cfg)
    rt = RefTimer(hix, cfg, head, threads)
    qps = rt.calibrate(qs)
    per_step_s = max(1.0, args.cpu_seconds / max(1, args.steps + args.warmup))
    nstep = int(min(len(qs), max(4 * threads, per_step_s * qps)))
    secs, evs = 0.0, 0
    for i in range(args.warmup + args.steps):
        start = (i * nstep) % len(qs)
        sub = qs[start:start + nstep]
        if len(sub) < nstep:
            sub = np.concatenate([sub, qs[:nstep - len(sub)]])
        sec, ev, _, _ = rt.run(sub)
        if i >= args.warmup:
            secs += sec
            evs += ev
    rt.close()
    value = evs / secs
    out = dict(metric=metric_name(cfg),
               value=value, unit="candidates/s", n_gpus=world, steps=args.steps,
               warmup=args.warmup, ms_per_step=secs * 1e3 / args.steps, higher_is_better=True,
               scaling="weak", vs_baseline=None, dtype="f32 (u8 PQ codes)", data="synthetic",
               impl="reference",
               config=dict(workload=cfg["workload"], n_per_gpu=cfg["n"], dim=cfg["dim"],
                           queries=cfg["nq"], m=cfg["m"], nlist=cfg["nlist"],
                           nprobe=cfg["nprobe"], k=cfg["k"], gamma=head),
               qps=nstep * args.steps / secs,
               cpu_baseline=dict(value=value, unit="candidates/s", cores=threads, kind=rt.kind,
                                 sample=f"{nstep} queries per step (of {len(qs)}) of {cfg['workload']}, "
                                        f"{threads} threads"),
               e2e=dict(value=value, unit="candidates/s", h2d_bytes_per_step=0,
                        d2h_bytes_per_step=0))
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--gamma", type=float, default=None)
    ap.add_argument("--n", type=int, default=None, help="override vectors per GPU (dev runs)")
    ap.add_argument("--nq", type=int, default=None, help="override query count (dev runs)")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--recall-q", type=int, default=200)
    ap.add_argument("--streams", type=int, default=3,
                    help="streams that consecutive batches alternate between (1 = serial)")
    ap.add_argument("--parallel", default="shard", choices=["shard", "replicas"],
                    help="N>1 layout: id-sharded index (weak scaling, all-gather merge) or replicas "
                         "(whole index per GPU, queries partitioned, strong scaling, no collective)")
    ap.add_argument("--force-shard", action="store_true",
                    help="run the id-sharded path (all-gather + device merge) even at N=1")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.n:
        cfg["n"] = args.n
    if args.nq:
        cfg["nq"] = args.nq
    if args.warmup < 3 and args.impl == "ours" and os.environ.get("BENCH_ALLOW_SHORT") != "1":
        log("note: the contract asks for >= 3 warm-up steps")
    if args.impl == "reference":
        run_reference_graph(args, cfg) if cfg.get("kind") == "graph" else run_reference(args, cfg)
    elif cfg.get("kind") == "graph":
        run_ours_graph(args, cfg)
    elif cfg.get("kind") == "range":
        run_ours_range(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
