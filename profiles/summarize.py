"""Summarise ncu captures into profiles/*.json (run here, on the CPU box).

    python profiles/summarize.py gpurun_out/prof_c2.ncu-rep profiles/r01_c2_knn.json
    python profiles/summarize.py --launches gpurun_out/launches_c2.csv profiles/r01_c2_launches.json

The per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
of the filter kernel is also written to profiles/ncu_traffic.json, which
bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__shared_mem_per_block_dynamic": "dyn_smem_per_block",
    "launch__occupancy_limit_shared_mem": "occupancy_limit_smem_blocks",
    "launch__occupancy_limit_registers": "occupancy_limit_reg_blocks",
    "smsp__inst_executed.sum": "warp_instructions",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
}


def raw(rep):
    if rep.endswith(".csv"):  # already exported on the GPU box (ncu -i ... --page raw --csv)
        text = open(rep).read()
    else:
        text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    h, units, vals = rows[0], rows[1], rows[2:]
    unit = dict(zip(h, units))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9}
    res = []
    for v in vals:
        d = dict(zip(h, v))
        e = {"kernel": d.get("Kernel Name", "")[:120], "grid": d.get("Grid Size"), "block": d.get("Block Size")}
        for m, name in METRICS.items():
            if m in d and d[m] not in ("", "n/a"):
                try:
                    e[name] = float(d[m].replace(",", "")) * scale.get(unit.get(m, ""), 1.0)
                except ValueError:
                    e[name] = d[m]
        stalls = {}
        for k, x in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    if float(x) > 0.05:
                        stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(x)
                except ValueError:
                    pass
        e["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        if "dram_bytes_read" in e:
            e["dram_bytes_total"] = e["dram_bytes_read"] + e.get("dram_bytes_write", 0.0)
        res.append(e)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    out = [{"id": int(r[0]), "kernel": r[4].split("(")[0], "grid": r[8], "ns": float(r[14])} for r in rows]
    tot = sum(x["ns"] for x in out)
    share = {}
    for x in out:
        share[x["kernel"]] = share.get(x["kernel"], 0.0) + x["ns"]
    return {"launches": out, "total_ns": tot, "share": {k: v / tot for k, v in share.items()}}


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        res = launches(sys.argv[2])
        dst = sys.argv[3]
    else:
        res = raw(sys.argv[1])
        dst = sys.argv[2]
        if len(sys.argv) > 3:  # workload key for ncu_traffic.json
            tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
            t = json.load(open(tpath)) if os.path.exists(tpath) else {}
            k = [e for e in res if "knn_kernel" in e["kernel"] or "range" in e["kernel"] or "graph" in e["kernel"]]
            if k and "dram_bytes_total" in k[0]:
                t[sys.argv[3]] = {"dram_bytes_per_launch": k[0]["dram_bytes_total"], "kernel": k[0]["kernel"],
                                  "grid": k[0]["grid"], "duration_ns": k[0].get("duration_ns"),
                                  "source": "profiles/" + os.path.basename(dst)}
                json.dump(t, open(tpath, "w"), indent=1)
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])
