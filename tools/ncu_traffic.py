"""Update profiles/<round>_traffic.json with dram__bytes_read.sum +
dram__bytes_write.sum of one-launch ncu --set full reports.
Usage: python tools/ncu_traffic.py profiles/r1_traffic.json CONFIG:KERNEL:REPORT ..."""
import csv
import io
import json
import subprocess
import sys


def dram_bytes(rep: str) -> float:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = head.index(k)
        tot += float(vals[i].replace(",", "")) * scale[units[i]]
    return tot


path = sys.argv[1]
try:
    doc = json.load(open(path))
except FileNotFoundError:
    doc = {}
doc["source"] = "ncu --set full --clock-control none, one launch each (dram__bytes_read.sum + dram__bytes_write.sum)"
for spec in sys.argv[2:]:
    cfg, kernel, rep = spec.split(":", 2)
    doc.setdefault(cfg, {})[kernel] = dram_bytes(rep)
json.dump(doc, open(path, "w"), indent=1)
print(json.dumps(doc, indent=1))
