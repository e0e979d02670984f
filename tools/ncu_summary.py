"""Summarise an ncu report (details + raw DRAM bytes) as markdown for
profiles/.   usage: ncu_summary.py report.ncu-rep [title]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
KEEP = ("Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Block Size", "Grid Size", "Cluster Size", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction",
        "No Eligible", "Avg. Active Threads Per Warp", "Executed Instructions", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Max Active Clusters")
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
print(f"### {title}\n")
kernel = None
seen = set()
print("| metric | value | unit |\n|---|---|---|")
for row in csv.reader(io.StringIO(det)):
    if len(row) > 14 and row[0] != "ID":
        kernel = row[4]
        if row[12] in KEEP and row[12] not in seen:
            seen.add(row[12])
            print(f"| {row[12]} | {row[14]} | {row[13]} |")
r = list(csv.reader(io.StringIO(raw)))
if len(r) > 2:
    h, u, v = r[0], r[1], r[2]
    for i, n in enumerate(h):
        if n in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                 "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                 "smsp__issue_active.avg.pct_of_peak_sustained_active"):
            print(f"| {n} | {v[i]} | {u[i]} |")
    # warp-stall reasons, as warps stalled per issued instruction (largest first)
    st = [(n.split("issue_stalled_")[1].replace("_per_issue_active.ratio", ""), float(v[i]))
          for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_")
          and n.endswith("_per_issue_active.ratio") and v[i] not in ("", "n/a")]
    st.sort(key=lambda t: -t[1])
    tot = sum(x for _, x in st) or 1.0
    print("\nStall reasons (share of stalled-warp samples per issue): " +
          ", ".join(f"{n} {100 * x / tot:.0f}%" for n, x in st[:7] if x > 0))
print(f"\nkernel: `{kernel}`\n")
