#!/usr/bin/env python
"""Summarises an ncu capture into profiles/ (tracked evidence).

  python tools/ncu_summary.py launches <launches.csv> <out.json>     # launch list -> per-kernel shares
  python tools/ncu_summary.py full <prof.ncu-rep | raw.csv> <out.json> [tag]   # --set full -> key metrics
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr, per = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            rec = dict(zip(hdr, r))
            if rec.get("Metric Name") == "gpu__time_duration.sum":
                per[rec["Kernel Name"]].append(float(rec["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in per.values())
    res = {"source": path, "unit": "ns (cold-cache, serialised; compare shares)", "kernels": [
        {"kernel": k, "launches": len(v), "total_ns": sum(v), "per_launch_ns": v,
         "share": sum(v) / tot} for k, v in sorted(per.items(), key=lambda x: -sum(x[1]))]}
    json.dump(res, open(out, "w"), indent=1)
    for k in res["kernels"]:
        print(f"{k['share']:.4f} {k['launches']:3d} {k['kernel'][:90]}")


def full(path, out, tag=""):
    if path.endswith(".csv"):  # raw page exported on the GPU box (ncu -i rep --page raw --csv)
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {"source": path, "tag": tag, "launches": []}
    for v in rows[2:]:
        rec = {"kernel": v[hdr.index("Kernel Name")]}
        for i, n in enumerate(hdr):
            if n in KEYS or ("stall" in n and n.endswith(".pct") and "ratio" not in n):
                try:
                    rec[n] = [float(v[i].replace(",", "")), units[i]]
                except ValueError:
                    rec[n] = [v[i], units[i]]
        rd = rec.get("dram__bytes_read.sum"), rec.get("dram__bytes_write.sum")
        if all(rd):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rec["dram_bytes_per_launch"] = sum(x[0] * scale[x[1]] for x in rd)
        res["launches"].append(rec)
    if res["launches"]:
        res["dram_bytes_per_launch"] = res["launches"][0].get("dram_bytes_per_launch")
    json.dump(res, open(out, "w"), indent=1)
    for rec in res["launches"]:
        for k, v in rec.items():
            print(k, v)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "")
