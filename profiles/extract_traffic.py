#!/usr/bin/env python
"""Write profiles/force_traffic.json from an `ncu --set full` report of bench.py:
mean dram__bytes_read.sum + dram__bytes_write.sum over the captured k_force<0, 2, 0>
launches (the fused force + velocity-Verlet kernel that runs 18 of every 20 steps).

usage: python profiles/extract_traffic.py <report.ncu-rep> <workload> [out.json]
"""
import csv
import io
import json
import os
import subprocess
import sys


def main():
    rep, workload = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(__file__), "force_traffic.json")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    name, rd, wr, dur = (h.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                              "gpu__time_duration.sum"))
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = []
    for r in rows[2:]:
        if "k_force<(bool)0, (int)2" in r[name] or "k_force<0, 2, 0>" in r[name]:
            b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
            vals.append((b, float(r[dur])))
    if not vals:
        raise SystemExit("no k_force<0,2,0> launch in the report")
    res = {"workload": workload, "kernel": "k_force<0,2,0>",
           "dram_bytes_per_launch": sum(v[0] for v in vals) / len(vals),
           "ncu_duration_us_mean": sum(v[1] for v in vals) / len(vals) / (1e3 if units[dur] == "nsecond" else 1),
           "launches": len(vals), "source": os.path.basename(rep)}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
