"""Per-source-line instruction counts of one ncu report, aggregated over line
ranges given as name=lo-hi (file ds_obs.cu unless file:lo-hi)."""
import csv, io, os, subprocess, sys
rep = sys.argv[1]
per_agent = float(sys.argv[2])
ranges = []
for spec in sys.argv[3:]:
    name, rng = spec.split("=")
    f = os.environ.get("NCU_FILE", "ds_obs.cu")
    if ":" in rng:
        f, rng = rng.split(":")
    lo, hi = rng.split("-")
    ranges.append((name, f, int(lo), int(hi)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
agg = {}
tot = 0
for r in csv.reader(io.StringIO(raw)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] and r[0] != "Line No" and r[2] == "-":
        try:
            ln, c = int(r[0]), int(r[7] or 0)
        except ValueError:
            continue
        tot += c
        key = cur
        for name, f, lo, hi in ranges:
            if f == cur and lo <= ln <= hi:
                key = name
                break
        agg[key] = agg.get(key, 0) + c
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k:28s} {v / tot * 100:5.1f}%  {v / per_agent:8.0f} per unit")
