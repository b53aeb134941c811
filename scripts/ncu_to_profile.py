#!/usr/bin/env python
"""Write profiles/gather_ncu.json (the roofline 'traffic' source used by
bench.py) and a text summary from one `ncu --set full` capture of the gather
kernel.  Usage: ncu_to_profile.py REPORT.ncu-rep OUT_PREFIX WORKLOAD"""
import csv, io, json, subprocess, sys

rep, prefix, workload = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, u, v = r[0], r[1], r[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}


def num(k, scale=1.0):
    val, unit = d[k]
    x = float(val.replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
            "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0,
            "s": 1.0}.get(unit, 1.0)
    return x * mult * scale


summary = {
    "kernel": d["Kernel Name"][0],
    "workload": workload,
    "report": rep.split("/")[-1],
    "duration_ms": num("gpu__time_duration.sum") * 1e3,
    "dram_read_bytes": num("dram__bytes_read.sum"),
    "dram_write_bytes": num("dram__bytes_write.sum"),
    "l2_hit_rate_pct": float(d["lts__t_sector_hit_rate.pct"][0]),
    "l1_hit_rate_pct": float(d["l1tex__t_sector_hit_rate.pct"][0]),
    "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
    "sm_throughput_pct": float(d["sm__throughput.avg.pct_of_peak_sustained_elapsed"][0]),
    "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
    "registers_per_thread": float(d["launch__registers_per_thread"][0]),
    "instructions": num("smsp__inst_executed.sum"),
    "shared_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "shared_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
}
summary["dram_bytes_per_launch"] = summary["dram_read_bytes"] + summary["dram_write_bytes"]
summary["dram_gbs"] = summary["dram_bytes_per_launch"] / (summary["duration_ms"] / 1e3) / 1e9
json.dump(summary, open(prefix + ".json", "w"), indent=1)
print(json.dumps(summary, indent=1))
