#!/usr/bin/env python
"""Summaries of an `ncu --set full` report for profiles/ (the report itself is not committed).

usage: python profiles/extract_r2.py <report.ncu-rep> <out.json> [--traffic profiles/force_traffic.json]

Per kernel launch: duration, DRAM bytes read / written and the achieved DRAM bandwidth
against the measured HBM peak (MEASURED_PEAKS.json hbm_gbs, 6445 GB/s), FP64-pipe and
issue utilisation, warps active, registers, shared memory and the stall reasons above
0.2 warps per issue.  With --traffic: the mean DRAM bytes of the k_force<0,2,0> launches
(the bench's roofline.traffic) written to that file.
"""
import csv
import io
import json
import os
import subprocess
import sys

HBM_GBS = 6445.0
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6,
         "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0, "%": 1.0, "": 1.0,
         "Kbyte/block": 1e3, "byte/block": 1.0}


def rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    return r[0], r[1], r[2:]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    traffic = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    h, units, data = rows(rep)
    ix = {k: i for i, k in enumerate(h)}

    def val(r, k):
        if k not in ix:
            return None
        try:
            return float(r[ix[k]]) * SCALE.get(units[ix[k]], 1.0)
        except ValueError:
            return None

    res = []
    for r in data:
        name = r[ix["Kernel Name"]]
        dur = val(r, "gpu__time_duration.sum")
        rd, wr = val(r, "dram__bytes_read.sum") or 0.0, val(r, "dram__bytes_write.sum") or 0.0
        stalls = {}
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                v = val(r, k)
                if v and v > 0.2:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        res.append({
            "kernel": name, "grid": val(r, "launch__grid_size"), "block": val(r, "launch__block_size"),
            "duration_us": dur * 1e6 if dur else None,
            "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6,
            "dram_GBs": (rd + wr) / dur / 1e9 if dur else None,
            "dram_frac_of_measured_hbm": (rd + wr) / dur / 1e9 / HBM_GBS if dur else None,
            "fp64_pipe_pct": val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers": val(r, "launch__registers_per_thread"),
            "smem_dynamic_KB": (val(r, "launch__shared_mem_per_block_dynamic") or 0) / 1e3,
            "inst_executed": val(r, "smsp__inst_executed.sum"),
            "threads_per_inst": val(r, "smsp__thread_inst_executed_per_inst_executed.ratio"),
            "smem_ld_bank_conflicts": val(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
            "stalls_per_issue": stalls,
        })
    json.dump({"report": os.path.basename(rep), "hbm_peak_GBs_measured": HBM_GBS, "launches": res}, open(out, "w"),
              indent=1)
    print(f"{len(res)} launches -> {out}")
    if traffic:
        f = [x for x in res if "k_force<0, 2, 0>" in x["kernel"] or "k_force<(bool)0, (int)2, (bool)0>" in x["kernel"]]
        if f:
            t = {"workload": "C2", "kernel": "k_force<0,2,0>",
                 "dram_bytes_per_launch": sum(1e6 * (x["dram_read_MB"] + x["dram_write_MB"]) for x in f) / len(f),
                 "ncu_duration_us_mean": sum(x["duration_us"] for x in f) / len(f), "launches": len(f),
                 "source": os.path.basename(rep)}
            json.dump(t, open(traffic, "w"), indent=1)
            print(json.dumps(t))


if __name__ == "__main__":
    main()
