"""Executed exact-test counts of the LiDAR kernel on the C4 workload (needs
the counter build: tools/build_variant.sh lidar_stats -DDS_LIDAR_STATS, run
with DS_LIB_PATH=variants/lidar_stats.so).  Writes profiles/r2_lidar_work.json:
per agent-step box / segment tests, segments fetched, cells examined, and the
FP64 work they amount to with SURVEY §8d's per-test weights (30 FLOP per
ray-box slab test, 11 per ray-segment test), next to the reference's own
candidate work (bench.lidar_flops) for the culling factor."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, lidar_flops, sim_config  # noqa: E402
from paper_2408_01584_b200 import _native as N  # noqa: E402
from paper_2408_01584_b200.engine import SimBatch, random_actions  # noqa: E402
from paper_2408_01584_b200.synthetic import WaymoSpec, generate  # noqa: E402

W, A, P = CONFIGS["c4"][:3]
cfg = sim_config("c4")
raw = generate(WaymoSpec(n_worlds=W, n_agents=A, n_points=P, seed=0))
b = SimBatch.from_raw(raw, cfg, device="cuda:0")
acts = [random_actions(b.n_controlled, cfg, 0, t, "cuda:0") for t in range(8)]
steps = int(os.environ.get("STEPS", "10"))
for t in range(5):                       # the bench's warm-up phase
    b.step(acts[t % 8], auto_reset=True)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
N.lib().ds_debug_lidar_stats(buf)        # clear
for t in range(steps):
    b.step(acts[t % 8], auto_reset=True)
torch.cuda.synchronize()
N.lib().ds_debug_lidar_stats(buf)
rows = buf[0]
per = lambda i: buf[i] / rows
box, seg = per(1), per(3)
ref = lidar_flops(b.packed, cfg.obs.max_range, cfg.obs.n_rays)
out = {"workload": CONFIGS["c4"][6], "steps": steps, "agent_rows": rows,
       "per_agent_step": {"exact_box_tests": box, "exact_segment_tests": seg,
                          "segments_fetched": per(2), "cells_examined": per(4)},
       "flop_weights": {"box_test": 30, "segment_test": 11, "source": "SURVEY.md §8d"},
       "executed_fp64_flop_per_agent_step": 30 * box + 11 * seg,
       "reference_candidate_flop_per_agent_step": ref,
       "culling_factor": ref / max(30 * box + 11 * seg, 1e-9)}
path = os.path.join(ROOT, "profiles", "r2_lidar_work.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
