"""Top source lines of one ncu report by executed warp instructions (per
agent) with their stall samples; optional line range filter.
Usage: python tools/ncu_top.py <src.csv from --page source --csv --print-source cuda,sass> [agents] [lo-hi] [n]"""
import csv, sys
path = sys.argv[1]
A = float(sys.argv[2]) if len(sys.argv) > 2 else 524288
lo, hi = map(int, sys.argv[3].split("-")) if len(sys.argv) > 3 and sys.argv[3] != "-" else (0, 10**9)
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = []; cur = None; hdr = None
for r in csv.reader(open(path)):
    if r and r[0] in ("File Name", "File Path"):
        cur = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        rows.append((cur, int(r[0]), r[1][:110], dict(zip(hdr[4:], r[4:]))))
f = lambda x: float(x) if x not in ("", None) else 0.0
tot = sum(f(d["Instructions Executed"]) for *_, d in rows)
print(f"total {tot / A:.1f} instr/agent")
sel = [x for x in rows if lo <= x[1] <= hi]
for c, l, s, d in sorted(sel, key=lambda x: -f(x[3]["Instructions Executed"]))[:n]:
    print(f"{f(d['Instructions Executed']) / A:7.1f} {f(d['# Samples']):7.0f} {c}:{l} {s}")
