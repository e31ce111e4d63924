"""Summarise an ncu report: key throughput metrics, instruction mix and the
hottest source lines (needs -lineinfo builds).  Usage:
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [top_n]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issued Warp Per Scheduler", "Achieved Active Warps Per SM",
        "Theoretical Active Warps per SM", "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Avg. Active Threads Per Warp",
        "Dynamic Shared Memory Per Block", "Block Limit Shared Mem", "Block Limit Registers"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
if rows:
    h = rows[0]
    ni, ui, vi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    ki = h.index("Kernel Name")
    seen = set()
    for r in rows[1:]:
        if r[ni] in KEYS and (r[ki], r[ni]) not in seen:
            seen.add((r[ki], r[ni]))
            print(f"{r[ki][:40]:40s} {r[ni]:38s} {r[vi]:>14s} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
if len(rows) > 2:
    h = rows[0]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                 "sm__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
        if name in h:
            i = h.index(name)
            print(f"{name:60s} {rows[2][i]:>16s} {rows[1][i]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
cur = None
lines = []
ops = collections.Counter()
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    ie = 7
    if r[0] and r[2] == "-":
        try:
            lines.append((int(r[ie] or 0), int(r[4] or 0), cur, r[0], r[1][:100]))
        except ValueError:
            pass
    elif not r[0] and r[2].startswith("0x"):
        op = r[3].split()
        if op:
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            try:
                ops[o.split(".")[0]] += int(r[ie] or 0)
            except ValueError:
                pass
tot = sum(x[0] for x in lines) or 1
stot = sum(x[1] for x in lines) or 1
print(f"\nwarp instructions executed: {tot:,}")
print("instruction mix:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in ops.most_common(14)))
print("\nhot source lines (instr %, stall-sample %):")
for x in sorted(lines, reverse=True)[:top]:
    print(f"{x[0] / tot * 100:5.1f}% {x[1] / stot * 100:5.1f}%  {x[2]}:{x[3]}  {x[4]}")
