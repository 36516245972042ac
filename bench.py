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
    what = "range search, flat" if cfg.get("kind") == "range" else "kNN search"
    return f"queries/sec (TRIM {what}; candidates filtered/sec, %HBM roofline, prune ratio alongside)"


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
    """DRAM bytes per launch of the dominant kernel for this workload
    (dram__bytes_read.sum + dram__bytes_write.sum from one `ncu --set full`
    capture of the current kernel build), from profiles/ncu_traffic.json —
    {"dram_bytes_per_launch": B, "source": "<profile file>"} or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    v = j.get(workload)
    if v is None:
        return None
    return v if isinstance(v, dict) else {"dram_bytes_per_launch": v, "source": None}


# ------------------------------------------------------------------- data
def build_workload(cfg, rank: int, world: int, device: int, sharded: bool = False):
    """Seeded synthetic data + index (bench_fixture: plain torch ops, the same
    bytes in both arms). Rank r holds the id-shard [r*n, (r+1)*n) (weak
    scaling); the codebook and coarse quantizer come from the same seeded
    sample of rank 0's rows on every rank, so every shard probes identically.
    Returns (fixture namespace, queries)."""
    import torch

    import bench_fixture as F

    torch.cuda.set_device(device)
    t0 = time.time()
    fx = F.build(cfg, rank if sharded else 0, device)
    log(f"[rank {rank}] built {cfg['workload']} shard in {time.time() - t0:.1f}s")
    return fx, fx.queries


def merged_host_index(parts):
    """The whole index of W id-shards (host numpy; shard p = ids [p*n, (p+1)*n)):
    list l = shard 0's list l, then shard 1's, ... (ids stay ascending inside
    every list, ivf.hpp:147-152)."""
    W = len(parts)
    nlist = len(parts[0].list_offsets) - 1
    sizes = np.stack([np.diff(p.list_offsets.astype(np.int64)) for p in parts])  # [W, nlist]
    offs = np.zeros(nlist + 1, np.uint64)
    offs[1:] = np.cumsum(sizes.sum(0))
    start = offs[:-1].astype(np.int64)[None, :] + np.cumsum(sizes, 0) - sizes  # [W, nlist]
    total = int(offs[-1])
    cs = parts[0].list_codes.shape[1]
    ids = np.empty(total, np.uint32)
    codes = np.empty((total, cs), np.uint8)
    lx = np.empty(total, np.float32)
    for p, s in enumerate(parts):
        po = s.list_offsets.astype(np.int64)
        dest = np.repeat(start[p] - po[:-1], sizes[p]) + np.arange(int(po[-1]), dtype=np.int64)
        ids[dest] = s.list_ids
        codes[dest] = s.list_codes
        lx[dest] = s.list_lx
    from types import SimpleNamespace
    return SimpleNamespace(dim=parts[0].dim, m=parts[0].m, ksub=parts[0].ksub, sub_dims=parts[0].sub_dims,
                           centroids=parts[0].centroids, coarse=parts[0].coarse, list_offsets=offs,
                           list_ids=ids, list_codes=codes, list_lx=lx,
                           vectors=np.concatenate([p.vectors for p in parts]), id_base=0)


def data_gen_note(cfg):
    if cfg.get("data") == "uniform_normalized":
        return "torch Philox uniform [0,1) + L2-normalised rows, seeds base=1+7919*rank queries=2 (bench_fixture.py)"
    return "torch Philox Gaussian blobs, seeds centers=0 base=1+7919*rank queries=2 (bench_fixture.py)"


def config_dict(cfg, head, n_gpus, parallelism, fingerprint, **extra):
    """`config` of the JSON line — built by the same function in both arms."""
    c = dict(workload=cfg["workload"], n_per_gpu=cfg["n"], dim=cfg["dim"], queries=cfg["nq"], batch=cfg["batch"],
             m=cfg["m"], nlist=cfg["nlist"], nprobe=cfg["nprobe"], k=cfg["k"], gamma=head, n_gpus=n_gpus,
             parallelism=parallelism,
             l2=("index > L2 (no flush needed)" if cfg["n"] * cfg["dim"] * 4 > 126e6
                 else "index fits L2; reported as-is"),
             data_gen=data_gen_note(cfg), fixture=fingerprint)
    c.update(extra)
    return c


def parallelism_of(world, mode):
    if mode == "replicas":
        return f"replicas x{world}"
    if mode in ("shard", "group") or world > 1:
        return f"id-shard x{world}"
    return "single"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ------------------------------------------------------------ our GPU arm
def run_ours(args, cfg):
    """Modes: `single` (N=1); `shard` / `replicas` (torchrun, one process per
    GPU, torch.distributed NCCL all-gather + device merge); `group` (one
    process drives N GPUs through ONE multi-device index behind the C ABI:
    trim_index_desc devices[0..N) + TRIM_SHARD_ID, the library's NCCL
    broadcast / filter / all-gather / merge inside every search call)."""
    import torch

    from paper_2508_17828_b200 import _lib
    from paper_2508_17828_b200 import ivf as G

    import torch.distributed as dist
    import bench_fixture as F

    world, rank, local = dist_env()
    if world > 1:
        mode = "replicas" if args.parallel == "replicas" else "shard"
    elif args.gpus > 1 or args.group:
        mode = "group"
    else:
        mode = "shard" if args.force_shard else "single"
    ngpu = args.gpus if mode == "group" else world
    if mode in ("shard", "replicas"):
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    sharded = mode == "shard"
    if mode == "group":
        if torch.cuda.device_count() < ngpu:
            raise SystemExit(f"--gpus {ngpu}: only {torch.cuda.device_count()} CUDA devices visible")
        parts = []
        for r in range(ngpu):
            fx_r, q_r = build_workload(cfg, r, ngpu, r, True)
            if r == 0:
                fx, queries = fx_r, q_r
                fprint = F.fingerprint(fx)
            parts.append(F.to_host(fx_r))
            if r:
                del fx_r, q_r
        torch.cuda.set_device(dev)
        t0 = time.time()
        whole = merged_host_index(parts)
        del parts
        gix = G.GpuIvfIndex(G.IvfArrays.from_any(whole), devices=list(range(ngpu)),
                            shard_mode="replicas" if args.parallel == "replicas" else "id_shard")
        log(f"multi-device index over {ngpu} GPUs in {time.time() - t0:.1f}s ({gix.info()})")
        arrays = whole
    else:
        fx, queries = build_workload(cfg, 0 if mode == "replicas" else rank, world, local, sharded)
        fprint = F.fingerprint(fx)
        arrays = G.IvfArrays.from_any(fx)
        gix = G.GpuIvfIndex(arrays, device=local)
    replicas = mode == "replicas"
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
    setup_k = 1 if cfg["nlist"] > 1 and os.environ.get("TRIM_KNN_SETUP") != "0" else 0
    # flat kNN launches per batch. In-order scan: the filter kernel (+ query tiles, norms and the
    # tcgen05 bounds up to 16M rows). Segmented block stream (>= 64k rows, DESIGN 4.6b; a batch of
    # at most 2,048 queries): the in-order prefix, the block bounds (tcgen05), 1 + 3 plan
    # launches, 3 continue-round launches, the in-order and the table-driven resume
    seg_on = (cfg["nlist"] == 1 and cfg["n"] >= 65536 and cfg["dim"] <= 128
              and os.environ.get("TRIM_FLAT_SEGMENTS") != "0" and os.environ.get("TRIM_FLAT_PARTITION") != "0")
    bounds_k = 3 if cfg["nlist"] == 1 and cfg["n"] <= (16 << 20) and os.environ.get("TRIM_FLAT_BOUNDS") != "0" else 0
    filter_k = (11 if seg_on else 1) + bounds_k

    def step(gamma, filt_events=None):
        launches = 0
        fork = torch.cuda.Event()
        fork.record(stream)
        for x in streams[1:]:
            x.wait_event(fork)
        for i, (b0, nb) in enumerate(batches):
            st_, sh_ = streams[i % len(streams)], shs[i % len(streams)]
            qoff = b0 * cfg["dim"] * 4
            if mode == "group":
                # one C-ABI call: broadcast, every device's probe + filter, all-gather, merge
                if filt_events is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(st_)
                _lib.check(lib.trim_search_knn_device(
                    gix.handle, p(queries, qoff), nb, k, cfg["nprobe"], float(np.float32(gamma)),
                    p(ids, b0 * k * 4), p(dists, b0 * k * 4), p(cts, b0 * 48), p(status), sh_), "knn")
                launches += ngpu * (n_probe_k.value + 1 + setup_k) + 2  # + merge + counters
                if filt_events is not None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(st_)
                    filt_events.append((e0, e1))
                continue
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
            # IVF: trim_knn_setup_kernel (seeds + plan) and the filter kernel's two flavours (with
            # and without early-exit stages, each CTA runs in one of them); flat: filter_k below
            launches += (2 + setup_k) if setup_k else filter_k
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
    skipped = gix.skipped_positions() / args.steps  # list-level bound, per step (this process)
    evaluated, dc = float(ct[3]), float(ct[0])
    total_cand = evaluated * args.steps
    value = total_cand / (ms / 1e3)
    qps = nq * args.steps / (ms / 1e3)
    out = dict(metric=metric_name(cfg),
               value=qps, unit="queries/s", n_gpus=ngpu, steps=args.steps,
               warmup=args.warmup, ms_per_step=ms / args.steps, higher_is_better=True,
               scaling="strong" if replicas else "weak", vs_baseline=None, dtype="f32 (u8 PQ codes)",
               data="synthetic", candidates_per_s=value)
    out["config"] = config_dict(cfg, head, ngpu, parallelism_of(ngpu, mode if ngpu > 1 or sharded else "single"),
                                fprint)
    out["mode"] = {"single": "one process, one GPU", "shard": "torchrun, one process per GPU (id-shard, "
                   "torch.distributed NCCL all-gather + trim_merge_topk_device)",
                   "replicas": "torchrun, one process per GPU (replicas, no collective)",
                   "group": "one process, one multi-device index behind the C ABI (trim_index_desc "
                            "devices[], TRIM_SHARD_ID: NCCL broadcast + all-gather + device merge in "
                            "every trim_search_knn_device call)"}[mode]
    out["prune_ratio"] = float(ct[2] / max(1, ct[2] + ct[0]))
    out["candidates_per_query"] = evaluated / nq
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
    gdiv = ngpu if ngpu > 1 else 1
    per_launch_bytes = alg_bytes_step / max(1, nl // args.steps) / gdiv
    avg_launch_ms = fms / max(1, nl)  # filter-busy time per launch (overlap-aware)
    achieved = per_launch_bytes / (avg_launch_ms / 1e3) / 1e9
    tr = ncu_traffic(cfg["workload"])
    out["roofline"] = dict(bound="hbm", achieved=achieved, peak=peak, unit="GB/s",
                           frac=achieved / peak, traffic=tr.get("dram_bytes_per_launch") if tr else None,
                           traffic_source=tr.get("source") if tr else None,
                           kernel="trim_knn_kernel", scanned_bytes_per_step=alg_bytes_step,
                           bytes_per_candidate=bytes_per_cand, peak_source=peak_src,
                           filter_share_of_step=fms / ms,
                           list_skip_fraction=skipped_all / max(1.0, evaluated),
                           flat_distance_bounds=flat_bounds,
                           # flat indexes: rows skipped as whole blocks by the segmented block stream
                           flat_segments=bool(cfg["nlist"] == 1 and skipped_all > 0),
                           stream_equivalent_GBps=(evaluated * (m + 4) + dc * (4 * D + 4))
                           / max(1, nl // args.steps) / gdiv / (avg_launch_ms / 1e3) / 1e9)
    tp = ncu_traffic("tensor_pipe")  # ncu sm__pipe_tensor_cycles_active of the tcgen05 kernels; none for the LUT
    if tp:
        out["roofline"]["tensor_pipe"] = tp
    if mode == "group":
        out["roofline"]["note"] = ("group mode: one interval per C-ABI call (broadcast + every device's probe "
                                   "and filter + all-gather + merge), per device")
    out["gpu_launches"] = launches
    out["clocks"] = clk.summary()
    out["sweep"] = sweep
    if rank == 0:
        out[f"recall@{k}"] = recall(gix, queries, ids, k, args.recall_q, world if mode != "group" else ngpu)
    # e2e: the public API with host buffers, copies inside the timed region
    if sharded:
        out["e2e"] = e2e_sharded(gix, queries, cfg, head, args, world, rank, local)
    else:
        out["e2e"] = e2e(gix, queries, cfg, head, args, world, rank)
    if mode == "single" and not args.no_group_check and cfg["n"] <= 20_000_000:  # (a second copy of the index)
        # the same workload through the multi-device C-ABI path at one device
        # (trim_index_desc devices = [0], TRIM_SHARD_ID): what `--gpus N` runs
        out["multi_device_abi_1gpu"] = group_check(arrays, queries, cfg, head, args)
    if cfg.get("baseline_kprime") and rank == 0 and world == 1 and mode == "single":
        out["baseline_ivfpq"] = baseline_line(gix, arrays, queries, cfg, args)
    if rank == 0 and world == 1 and not args.skip_cpu:
        out["cpu_baseline"] = cpu_baseline(F.to_host(fx) if mode != "group" else None, queries, cfg, head, args,
                                           fx=fx)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if sharded or replicas:
        dist.destroy_process_group()


def group_check(arrays, queries, cfg, gamma, args):
    """e2e through a one-device TRIM_SHARD_ID index (the multi-device C-ABI
    path: broadcast, filter, all-gather, merge) on the bench workload."""
    import torch

    from paper_2508_17828_b200 import ivf as G
    t0 = time.time()
    gg = G.GpuIvfIndex(arrays, devices=[0], shard_mode="id_shard")
    build_s = time.time() - t0
    try:
        r = e2e(gg, queries, cfg, gamma, args, 1, 0)
    finally:
        gg.close()
        torch.cuda.empty_cache()
    r["index"] = "trim_index_desc devices=[0], shard_mode=TRIM_SHARD_ID"
    r["create_s"] = build_s
    return r


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
    if world > 1 or nsample <= 0 or getattr(gix, "shard_mode", "single") == "id_shard":
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
    """The C-ABI host call trim_search_knn (ivf::search_trim_ivf_knn batched)
    from pinned host queries into pinned host results, `--streams` client
    threads; H2D, search, D2H all inside the timed region. For a multi-device
    index that call also broadcasts, all-gathers and merges."""
    import torch

    from paper_2508_17828_b200 import ivf as G
    nq, B, k = cfg["nq"], cfg["batch"], cfg["k"]
    hq = queries.cpu().pin_memory()
    hqn = hq.numpy()
    prof = G.PruningProfile.manual(gamma)
    steps = max(1, min(args.steps, 3))

    from concurrent.futures import ThreadPoolExecutor

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

    with ThreadPoolExecutor(max(1, args.streams)) as pool:  # client threads: one stream each in the C ABI
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
    return dict(value=nq * steps / sec, unit="queries/s", candidates_per_s=cand / sec,
                h2d_bytes_per_step=nq * cfg["dim"] * 4,
                d2h_bytes_per_step=nq * k * 8 + nq * 48 + 4 * len(range(0, nq, B)),
                api=f"trim_search_knn (C ABI, host buffers; pinned queries and results; {max(1, args.streams)} client threads)")


def e2e_sharded(gix, queries, cfg, gamma, args, world, rank, local):
    """e2e at N ranks, one process per GPU, per step: the query set copied
    from pinned host memory, every batch searched on the local shard
    (trim_search_knn_device, batches alternating over `--streams` streams),
    the local top-k of all batches all-gathered over NCCL, merged on the device
    (trim_merge_topk_device), the counters all-reduced, and the merged rows +
    counters copied back to pinned host memory — the exchange is inside the
    timed region. Wall clock, max over ranks."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2508_17828_b200 import _lib
    lib = _lib.load()
    dev = torch.device(f"cuda:{local}")
    nq, B, k, D = cfg["nq"], cfg["batch"], cfg["k"], cfg["dim"]
    hq = queries.cpu().pin_memory()
    h_ids = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    h_d = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    h_ct = torch.empty((nq, 6), dtype=torch.int64).pin_memory()
    dq = torch.empty((nq, D), dtype=torch.float32, device=dev)
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dd = torch.empty((nq, k), dtype=torch.float32, device=dev)
    ct = torch.zeros((nq, 6), dtype=torch.int64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    g_ids = torch.empty((world * nq, k), dtype=torch.int32, device=dev)
    g_d = torch.empty((world * nq, k), dtype=torch.float32, device=dev)
    m_ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    m_d = torch.empty((nq, k), dtype=torch.float32, device=dev)
    main = torch.cuda.current_stream(dev)
    streams = [main] + [torch.cuda.Stream(dev) for _ in range(max(1, args.streams) - 1)]
    sh = C.c_void_p(main.cuda_stream)
    P = lambda t, off=0: C.c_void_p(t.data_ptr() + off)  # noqa: E731
    steps = max(1, min(args.steps, 3))

    def once():
        dq.copy_(hq, non_blocking=True)
        for x in streams[1:]:
            x.wait_stream(main)
        for i, b in enumerate(range(0, nq, B)):
            nb = min(B, nq - b)
            x = streams[i % len(streams)]
            _lib.check(lib.trim_search_knn_device(gix.handle, P(dq, b * D * 4), nb, k, cfg["nprobe"],
                                                  float(np.float32(gamma)), P(ids, b * k * 4), P(dd, b * k * 4),
                                                  P(ct, b * 48), P(st), C.c_void_p(x.cuda_stream)), "knn")
        for x in streams[1:]:
            main.wait_stream(x)
        dist.all_gather_into_tensor(g_ids, ids)
        dist.all_gather_into_tensor(g_d, dd)
        _lib.check(lib.trim_merge_topk_device(P(g_d), P(g_ids), world, nq, k, P(m_d), P(m_ids), local, sh), "merge")
        dist.all_reduce(ct)
        h_ids.copy_(m_ids, non_blocking=True)
        h_d.copy_(m_d, non_blocking=True)
        h_ct.copy_(ct, non_blocking=True)
        torch.cuda.synchronize()
        return int(h_ct[:, 3].sum())

    once()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cand = 0
    for _ in range(steps):
        cand += once()
    sec = time.perf_counter() - t0
    t = torch.tensor([sec], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t.item())
    return dict(value=nq * steps / sec, unit="queries/s", candidates_per_s=cand / sec,
                h2d_bytes_per_step=nq * D * 4, d2h_bytes_per_step=nq * k * 8 + nq * 48,
                api="per step: pinned H2D of the query set, trim_search_knn_device per batch on the local "
                    "shard, NCCL all-gather (torch.distributed), trim_merge_topk_device, counters all-reduce, "
                    "pinned D2H; wall clock, max over ranks",
                includes_exchange=True)


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


def _host_index(h):
    """oracle HostIndex of a fixture namespace / IvfArrays (host numpy or torch tensors)."""
    from oracle.oracle import HostIndex
    if hasattr(h.vectors, "is_cuda") or hasattr(h.list_ids, "is_cuda"):
        import bench_fixture as F
        h = F.to_host(h)
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

    def set_threads(self, t):
        self.threads = t
        if self.kind == "reference":
            self.ref.set_threads(t)

    def run(self, qsub, kind=None, arg=None):
        """-> (seconds, evaluated, dc, pruned) for one parallel batch. kind:
        0 kNN (default; 1 for range configs), 2 = search_baseline_ivfpq (arg = k')."""
        rng = self.cfg.get("kind") == "range"
        if kind is None:
            kind = 1 if rng else 0
        if arg is None:
            arg = self.cfg.get("radius", 0.0)
        if self.kind == "reference":
            sec, ct = self.ref.session_run(self.sess, kind, qsub, self.cfg["k"], self.cfg["nprobe"],
                                           self.gamma, arg=arg)
            return sec, int(ct[3]), int(ct[0]), int(ct[2])
        t0 = time.perf_counter()
        if kind == 1:
            _, _, _, ct, _ = self.co.search_range(self.hix, qsub, self.cfg["radius"], self.cfg["nprobe"],
                                                  self.gamma, threads=self.threads)
        elif kind == 2:
            _, _, ct = self.co.search_baseline(self.hix, qsub, self.cfg["k"], self.cfg["nprobe"], int(arg),
                                               threads=self.threads)[:3]
        else:
            _, _, ct, _ = self.co.search_knn(self.hix, qsub, self.cfg["k"], self.cfg["nprobe"], self.gamma,
                                             threads=self.threads)
        return time.perf_counter() - t0, int(ct[:, 3].sum()), int(ct[:, 0].sum()), int(ct[:, 2].sum())

    def close(self):
        if self.kind == "reference":
            self.ref.session_destroy(self.sess)

    def calibrate(self, qs, kind=None, arg=None):
        n0 = min(len(qs), max(4 * self.threads, 64 if self.threads > 1 else 8))
        sec, *_ = self.run(qs[:n0], kind, arg)
        return n0 / max(sec, 1e-9)  # queries/s

    def bounded(self, qs, seconds, kind=None, arg=None):
        """A sample sized to ~`seconds` of CPU work -> dict(value, qps, n, sec, prune_ratio)."""
        qps = self.calibrate(qs, kind, arg)
        n = int(min(len(qs), max(4 * self.threads, seconds * qps)))
        sec, ev, dc, pr = self.run(qs[:n], kind, arg)
        return dict(value=ev / sec, qps=n / sec, n=n, sec=sec, prune_ratio=pr / max(1, pr + dc))


def cpu_baseline(hfx, queries, cfg, gamma, args, fx=None):
    """The reference's CPU path on this box's host cores, on bounded samples of
    the same workload: all hardware threads (the reported `value`), one thread
    (the paper's protocol), and for config 2 the IVFPQ baseline
    search_baseline_ivfpq at k' = 1000 (ivf.hpp:193-237)."""
    import bench_fixture as F
    t0 = time.time()
    if hfx is None:
        hfx = F.to_host(fx)
    hix = _host_index(hfx)
    qs = queries.cpu().numpy()
    log(f"host copy for the CPU baseline: {time.time() - t0:.1f}s")
    threads = os.cpu_count() or 1
    rt = RefTimer(hix, cfg, gamma, threads)
    try:
        r = rt.bounded(qs, args.cpu_seconds)
        out = dict(value=r["qps"], unit="queries/s", candidates_per_s=r["value"], cores=threads, kind=rt.kind,
                   sample=f"first {r['n']} of {len(qs)} queries of {cfg['workload']} at gamma={gamma}, "
                          f"{threads} threads, {r['sec']:.1f}s",
                   prune_ratio=r["prune_ratio"], cpu_model=cpu_model(),
                   timing="steady_clock around parallel_for over queries (sweep.hpp:121-152)")
        rt.set_threads(1)
        r1 = rt.bounded(qs, max(2.0, args.cpu_seconds / 3))
        out["single_thread"] = dict(value=r1["qps"], unit="queries/s", candidates_per_s=r1["value"], cores=1,
                                    sample=f"first {r1['n']} queries, 1 thread, {r1['sec']:.1f}s")
        if cfg.get("baseline_kprime"):
            rt.set_threads(threads)
            rb = rt.bounded(qs, max(2.0, args.cpu_seconds / 3), kind=2, arg=float(cfg["baseline_kprime"]))
            out["baseline_ivfpq"] = dict(k_prime=cfg["baseline_kprime"], qps=rb["qps"], cand_per_s=rb["value"],
                                         cores=threads, sample=f"first {rb['n']} queries, {threads} threads, "
                                                               f"{rb['sec']:.1f}s")
    finally:
        rt.close()
    return out


# ------------------------------------------------------ config 3: range
def calibrate_radius(vectors, queries, cfg):
    """bench::pick_radius_for_fraction (bench/radius.hpp:20-55): the
    e_fraction = result_size/N quantile (EmpiricalCdf: linear between order
    statistics) of pooled query-to-row distances over 20,000 sampled rows x 200
    sampled queries (seeded torch.randperm samples, seeds 1 and 2).
    Distances by torch.cdist in float64 (a workload parameter, not a parity value)."""
    import torch

    x = vectors
    g = torch.Generator(device=x.device)
    g.manual_seed(1)
    rows = torch.randperm(x.shape[0], generator=g, device=x.device)[:min(20000, x.shape[0])]
    g.manual_seed(2)
    qi = torch.randperm(queries.shape[0], generator=g, device=x.device)[:min(200, queries.shape[0])]
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

    import bench_fixture as F

    world, rank, local = dist_env()
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    fx, queries = build_workload(cfg, rank, world, local, False)
    fprint = F.fingerprint(fx)
    gix = G.GpuIvfIndex(G.IvfArrays.from_any(fx), device=local)
    lib = _lib.load()
    radius = calibrate_radius(fx.vectors, queries, cfg)
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
               value=nq * args.steps / (ms / 1e3), unit="queries/s", candidates_per_s=value,
               n_gpus=world, steps=args.steps, warmup=args.warmup,
               ms_per_step=ms / args.steps, higher_is_better=True, scaling="weak", vs_baseline=None,
               dtype="f32 (u8 PQ codes)", data="synthetic")
    out["config"] = config_dict(cfg, head, world, parallelism_of(world, "single"), fprint, radius=radius,
                                radius_rule="pick_radius_for_fraction(100/N, 20000 rows, 200 queries)")
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
                           traffic=(ncu_traffic(cfg["workload"]) or {}).get("dram_bytes_per_launch"),
                           traffic_source=(ncu_traffic(cfg["workload"]) or {}).get("source"),
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
    out["e2e"] = dict(value=nq * reps / sec, unit="queries/s", candidates_per_s=tot / sec,
                      h2d_bytes_per_step=nq * D * 4 + nq * 4,
                      d2h_bytes_per_step=nres * 8 + (nq + 1) * 8 + nq * 48,
                      api=f"trim_search_range (C ABI, host buffers; {max(1, args.streams)} client threads)")
    if rank == 0 and not args.skip_cpu:
        out["cpu_baseline"] = cpu_baseline(None, queries, cfg, head, args, fx=fx)
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
                           traffic=(ncu_traffic(cfg["workload"]) or {}).get("dram_bytes_per_launch"),
                           kernel="trim_graph_kernel",
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
    """The reference arm: the unmodified reference (oracle/_ref, its own
    ivf::search_trim_ivf_knn / search_trim_ivf_range, parallel_for over queries
    like run_queries) on this box's host cores, on the same workload bytes as
    our arm (bench_fixture: plain torch; this process never loads
    libtrim_b200.so). Rank 0 only under torchrun."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    import torch

    import bench_fixture as F
    torch.cuda.set_device(local)
    fx, queries = build_workload(cfg, 0, 1, local, False)
    fprint = F.fingerprint(fx)
    ngpu = world if world > 1 else args.gpus
    head = args.gamma if args.gamma else cfg["gamma"]
    extra = {}
    if cfg.get("kind") == "range":
        cfg["radius"] = calibrate_radius(fx.vectors, queries, cfg)
        extra = dict(radius=cfg["radius"], radius_rule="pick_radius_for_fraction(100/N, 20000 rows, 200 queries)")
    mode = "single" if ngpu == 1 else ("replicas" if args.parallel == "replicas" else "shard")
    if cfg.get("kind") == "range":
        mode = "single"
    conf = config_dict(cfg, head, ngpu, parallelism_of(ngpu, mode), fprint, **extra)
    hix = _host_index(F.to_host(fx))
    qs = queries.cpu().numpy()
    del fx, queries
    torch.cuda.empty_cache()
    threads = os.cpu_count() or 1
    rt = RefTimer(hix, cfg, head, threads)
    qps = rt.calibrate(qs)
    per_step_s = max(1.0, args.cpu_seconds / max(1, args.steps + args.warmup))
    nstep = int(min(len(qs), max(4 * threads, per_step_s * qps)))
    secs, evs, dcs, prs = 0.0, 0, 0, 0
    for i in range(args.warmup + args.steps):
        start = (i * nstep) % len(qs)
        sub = qs[start:start + nstep]
        if len(sub) < nstep:
            sub = np.concatenate([sub, qs[:nstep - len(sub)]])
        sec, ev, dc, pr = rt.run(sub)
        if i >= args.warmup:
            secs += sec
            evs += ev
            dcs += dc
            prs += pr
    rt.close()
    value = nstep * args.steps / secs
    out = dict(metric=metric_name(cfg),
               value=value, unit="queries/s", candidates_per_s=evs / secs, n_gpus=ngpu, steps=args.steps,
               warmup=args.warmup, ms_per_step=secs * 1e3 / args.steps, higher_is_better=True,
               scaling="strong" if mode == "replicas" else "weak", vs_baseline=None, dtype="f32 (u8 PQ codes)",
               data="synthetic", impl="reference", config=conf,
               prune_ratio=prs / max(1, prs + dcs),
               cpu_baseline=dict(value=value, unit="queries/s", candidates_per_s=evs / secs, cores=threads,
                                 kind=rt.kind,
                                 sample=f"{nstep} queries per step (of {len(qs)}) of {cfg['workload']}, "
                                        f"{threads} threads" + (" (rank 0's shard)" if ngpu > 1 else ""),
                                 cpu_model=cpu_model()),
               e2e=dict(value=value, unit="queries/s", h2d_bytes_per_step=0,
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
    ap.add_argument("--group", action="store_true",
                    help="one process drives --gpus devices through one multi-device C-ABI index "
                         "(the default when --gpus N > 1 without torchrun)")
    ap.add_argument("--no-group-check", action="store_true",
                    help="skip the N=1 e2e line through the one-device TRIM_SHARD_ID index")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (torchrun --nproc-per-node must "
                         f"equal --gpus)")
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
