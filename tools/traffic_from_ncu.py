#!/usr/bin/env python
"""Write profiles/traffic.json from ncu --set full captures of the pass kernel.

usage: python tools/traffic_from_ncu.py TAG [summary-file]
reads gpurun_out/prof_TAG_<variant>.ncu-rep for the four variants."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
BYTES_PER_FVU = {"implicit": 96.0, "explicit": 120.0}
FV = 4032 * 4000


def metrics(rep):
    """Per-pass totals over the kernels of one pass in the capture (the general
    and the all-regular march kernel): DRAM bytes and warp instructions summed,
    serialised durations summed, pipe activities duration-weighted."""
    if rep.endswith(".csv"):                     # raw page exported on the GPU box
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]

    def get(v, name):
        i = h.index(name)
        return float(v[i].replace(",", "")) * UNITS.get(u[i], 1.0)
    tot = {"read": 0.0, "write": 0.0, "us": 0.0, "fp64": 0.0, "issue": 0.0, "inst": 0.0, "kernels": []}
    for v in rows[2:]:
        us = get(v, "gpu__time_duration.sum")
        tot["read"] += get(v, "dram__bytes_read.sum")
        tot["write"] += get(v, "dram__bytes_write.sum")
        tot["inst"] += get(v, "smsp__inst_executed.sum")
        tot["fp64"] += us * get(v, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100.0
        tot["issue"] += us * get(v, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100.0
        tot["us"] += us
        tot["kernels"].append({"name": v[h.index("Kernel Name")][:48], "us": round(us, 1),
                               "grid": int(get(v, "launch__grid_size")),
                               "dram_bytes": int(get(v, "dram__bytes_read.sum") + get(v, "dram__bytes_write.sum")),
                               "warp_inst": int(get(v, "smsp__inst_executed.sum")),
                               "issue_active": round(get(v, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100, 4),
                               "fp64_active": round(get(v, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100, 4)})
    tot["fp64"] /= max(tot["us"], 1e-9)
    tot["issue"] /= max(tot["us"], 1e-9)
    return tot


def main():
    tag = sys.argv[1]
    res = {"_source": f"ncu --set full --clock-control none, the march kernels of one pass (march_fused_kernel; implicit TVD: the general + all-regular kernels, serialised by ncu) after warm-up, C3 4032 x 4000 "
                      f"(16.128 M FVs); dram__bytes_read.sum + dram__bytes_write.sum per launch ({tag}, "
                      f"profiles/{tag}_summary.md)."}
    for var in ("implicit_upwind", "implicit_tvd", "explicit_upwind", "explicit_tvd"):
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_{var}.ncu-rep")
        if not os.path.exists(rep):
            rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_{var}.raw.csv")
        if not os.path.exists(rep):
            continue
        m = metrics(rep)
        res[f"C3_H200_{var}"] = {
            "bytes_per_launch": int(round(m["read"] + m["write"])), "read": int(round(m["read"])),
            "write": int(round(m["write"])), "algorithmic": int(BYTES_PER_FVU[var.split("_")[0]] * FV),
            "ncu_duration_us": round(m["us"], 1), "fp64_pipe_active": round(m["fp64"], 4),
            "issue_active": round(m["issue"], 4), "warp_instructions": int(m["inst"]),
            "thread_instructions_per_fv": round(m["inst"] * 32 / FV, 1), "kernels": m["kernels"]}
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
