"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summarize.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv --tag r2 \
        --workload C4

Writes profiles/ncu_<tag>_full.csv (one row per profiled kernel: duration,
DRAM bytes, throughputs, tensor-pipe activity, registers, occupancy),
profiles/ncu_<tag>_launches.csv (per-kernel mean device time and share of the
step from the gpu__time_duration launch list) and, with --workload,
profiles/ncu_traffic_<workload>.json: DRAM bytes (read + written, each scaled by
its own unit) per launch of each kernel and of each bench stage, keyed by the
workload's shape -- bench.py's roofline.traffic reads it only for that workload.
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = [("attn", "attention"), ("select_kernel", "select"), ("select_thresh", "select"), ("select_shard", "select"),
         ("select_scan", "select"), ("select_postings", "select"), ("prep_kernel", "prep"), ("lut_fma", "prep"),
         ("lut_persist", "prep"), ("qprep", "prep"), ("postings_build", "index"),
         ("encode_cw", "encode"), ("encode_kernel", "encode"), ("keyh", "encode_keyh")]
# prefill (encode_bulk_kernel, prepare_kernel) runs before the timed steps: not a path stage
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def short(name):
    n = name.split("(")[0]
    n = re.sub(r".*::", "", n)
    return n


def stage_of(name):
    for key, st in STAGE:
        if key in name:
            return st
    return None


def full(rep, tag, workload=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m in METRICS if m in hdr}
    ki = hdr.index("Kernel Name")
    res, traffic = [], {}
    for r in rows[2:]:
        d = {"kernel": short(r[ki])}
        for m, i in idx.items():
            v = r[i].replace(",", "")
            try:
                d[m] = float(v)
            except ValueError:
                d[m] = v
        res.append(d)
        if "dram__bytes_read.sum" in d:
            def scaled(m):
                if m not in idx or not isinstance(d.get(m), float):
                    return 0.0
                return d[m] * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[idx[m]], 1)
            rw = scaled("dram__bytes_read.sum") + scaled("dram__bytes_write.sum")
            traffic.setdefault(d["kernel"], []).append(rw)
    path = os.path.join(ROOT, "profiles", f"ncu_{tag}_full.csv")
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["kernel"] + [m for m in METRICS if m in idx])
        w.writeheader()
        for d in res:
            w.writerow(d)
    units_line = {m: units[i] for m, i in idx.items()}
    with open(path.replace(".csv", "_units.json"), "w") as f:
        json.dump(units_line, f, indent=1)
    per_kernel = {k: sum(v) / len(v) for k, v in traffic.items()}
    if workload:
        from synth import CONFIGS  # noqa: E402
        cfg = CONFIGS[workload]
        per_stage = {}
        for k, v in per_kernel.items():
            st = stage_of(k)
            if st:
                per_stage[st] = per_stage.get(st, 0.0) + v
        out = dict(workload=cfg.name, B=cfg.B, N=cfg.N, L=cfg.L, per_launch=dict(per_kernel, **per_stage),
                   _source=f"ncu --set full, {os.path.basename(rep)}: dram__bytes_read.sum + dram__bytes_write.sum "
                           f"per launch (each in its own unit); stages sum their kernels' launches of one step")
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.name}.json"), "w") as f:
            json.dump(out, f, indent=1)
    print(path)


def launches(path_csv, tag):
    rows = list(csv.reader(open(path_csv)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[hi + 1:]:
        n = short(r[ki])
        agg.setdefault(n, []).append(float(r[vi].replace(",", "")))
    # the posting-index rebuild (stage "index") runs once per rebuild period, not per step: no share
    in_step = lambda k: stage_of(k) and stage_of(k) != "index"
    tot = sum(sum(v) for k, v in agg.items() if in_step(k))
    out = os.path.join(ROOT, "profiles", f"ncu_{tag}_launches.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "mean_ns", "share_of_path_time"])
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            w.writerow([k, len(v), sum(v) / len(v), (sum(v) / tot) if in_step(k) and tot else ""])
    print(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r2")
    ap.add_argument("--workload", default=None, help="config name (C2, C4, ...) the capture ran")
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    if a.rep:
        full(a.rep, a.tag, a.workload)
    if a.launches:
        launches(a.launches, a.tag)
