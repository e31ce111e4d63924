"""Opcode histogram (executed warp instructions per unit) of the SASS that ncu
attributes to a source line range.  Usage:
    python tools/ncu_ops.py REPORT PER_UNIT FILE:LO-HI [top]"""
import csv, io, subprocess, sys
rep, per = sys.argv[1], float(sys.argv[2])
f, rng = sys.argv[3].split(":")
lo, hi = map(int, rng.split("-"))
top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = curf = None
agg, lines = {}, {}
for r in csv.reader(io.StringIO(raw)):
    if r and r[0] == "File Path":
        curf = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        cur = int(r[0])
        continue
    if len(r) > 8 and r[0] == "" and r[2].startswith("0x") and curf == f and cur and lo <= cur <= hi:
        t = r[3].split()
        op = t[1] if t[0].startswith("@") else t[0]
        c = int(r[7] or 0)
        agg[op] = agg.get(op, 0) + c
        lines[cur] = lines.get(cur, 0) + c
print("total per unit:", round(sum(agg.values()) / per, 1))
print([(k, round(v / per, 1)) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]])
print("by line:", [(k, round(v / per, 1)) for k, v in sorted(lines.items(), key=lambda x: -x[1])[:top]])
