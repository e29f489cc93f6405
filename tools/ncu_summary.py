"""Condense an ncu --set full report into the numbers profiles/ records.

    python tools/ncu_summary.py report.ncu-rep > profiles/<name>.md
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


det = page("details")
hdr = det[0]
rows = det[1:]
want = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem",
        "Theoretical Occupancy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Instructions", "Grid Size", "Block Size"]
kname = rows[0][4] if rows else "?"
print(f"# ncu summary: `{kname[:120]}`\n")
print(f"report: `{rep}`\n")
print("| metric | value | unit |\n|---|---|---|")
seen = set()
for r in rows:
    name, unit, val = r[-4], r[-3], r[-2]
    if name in want and name not in seen:
        seen.add(name)
        print(f"| {name} | {val} | {unit} |")
raw = page("raw")
h, v = raw[0], raw[2]
keys = ("dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
print("\n| raw metric | value |\n|---|---|")
for i, name in enumerate(h):
    if name in keys:
        print(f"| {name} | {v[i]} |")
stalls = []
for i, name in enumerate(h):
    if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
        try:
            stalls.append((float(v[i]), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
print("\n| stall reason (warps per issue) | value |\n|---|---|")
for val, name in sorted(stalls, reverse=True)[:8]:
    print(f"| {name} | {val:.2f} |")
