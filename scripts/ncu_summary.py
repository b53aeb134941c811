#!/usr/bin/env python
"""Summarise an ncu report: SOL, occupancy, stalls, instruction mix."""
import csv, subprocess, sys, io, collections

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    rows = []
    for v in r[2:]:
        rows.append({h[i]: (v[i], u[i]) for i in range(len(h))})
    return rows

def main(rep):
    rows = raw(rep)
    for d in rows:
        name = d.get("Kernel Name", ("?",))[0]
        print("kernel:", name[:90])
        keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
                "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
                "sm__warps_active.avg.pct_of_peak_sustained_active",
                "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                "smsp__thread_inst_executed_per_inst_executed.ratio",
                "launch__registers_per_thread", "launch__occupancy_limit_registers",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_local_ld.sum",
                "smsp__sass_inst_executed_op_local_st.sum", "smsp__sass_inst_executed_op_global_ld.sum"]
        for k in keys:
            if k in d:
                print(f"  {k:70s} {d[k][0]:>20s} {d[k][1]}")
        st = {k: float(v[0].replace(',', '')) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v[0].replace(',', '').replace('.', '').isdigit()}
        tot = sum(st.values()) or 1
        print("  stall samples:")
        for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]:
            print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100*v/tot:5.1f}%")

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
