"""Summarise an ncu report (details page) for the kernels in it: key throughput,
occupancy, pipe and stall metrics. Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Theoretical Occupancy", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Dynamic Shared Memory Per Block", "Block Limit Shared Mem", "Block Limit Registers", "Memory Throughput",
        "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
last = None
for row in r[1:]:
    if row[mi] in WANT:
        if row[ii] != last:
            print(f"--- [{row[ii]}] {row[ki][:110]}")
            last = row[ii]
        print(f"    {row[mi]:40s} {row[vi]:>14s} {row[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units = r[0], r[1]
keys = [k for k in h if k.startswith("smsp__average_warp") or k.startswith("smsp__pcsamp_warps_issue_stalled")
        or k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
                 "lts__t_bytes.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                 "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active")]
for row in r[2:]:
    print(f"=== [{row[h.index('ID')]}] {row[h.index('Kernel Name')][:80]}")
    stalls = []
    for k in keys:
        v = row[h.index(k)]
        if k.startswith("smsp__pcsamp_warps_issue_stalled"):
            try:
                stalls.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        else:
            print(f"    {k:75s} {v} {units[h.index(k)]}")
    tot = sum(s for s, _ in stalls) or 1
    for s, k in sorted(stalls, reverse=True)[:8]:
        print(f"    stall {k:60s} {100 * s / tot:5.1f} %")
