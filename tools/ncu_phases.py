"""Per-phase instruction counts (per agent) and stall samples of one ncu
report of obs_radial_kernel, by source-line ranges of the CURRENT csrc files.
Usage: python tools/ncu_phases.py <report> [agents]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
agents = float(sys.argv[2]) if len(sys.argv) > 2 else 524288
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
rows = []
for r in csv.reader(io.StringIO(raw)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] in ("Line No", "Function Name"):
        continue
    if len(r) > 8 and r[0] and r[2] == "-":
        try:
            rows.append((cur, int(r[0]), r[1].strip(), int(r[7] or 0), int(r[6] or 0)))
        except ValueError:
            pass
tot = sum(x[3] for x in rows)
smp = sum(x[4] for x in rows)
print(f"total {tot/agents:.0f} instr/agent, {smp} samples")
phases = [a.split("=") for a in sys.argv[3:]]
agg = {}
for f, l, s, c, n in rows:
    key = f
    for name, rng in phases:
        ff, lr = rng.split(":") if ":" in rng else ("ds_obs.cu", rng)
        lo, hi = map(int, lr.split("-"))
        if f == ff and lo <= l <= hi:
            key = name
            break
    a = agg.setdefault(key, [0, 0])
    a[0] += c
    a[1] += n
for k, (c, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{c/agents:8.1f} instr/agent {100*c/tot:5.1f}%  {100*n/smp:5.1f}% samples  {k}")
