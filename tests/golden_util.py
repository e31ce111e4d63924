"""Load the committed golden fixtures (tests/golden/*.npz, made from the real
reference by tests/golden/make_golden.py)."""

from __future__ import annotations

import ast
import glob
import hashlib
import os

import numpy as np

from paper_2408_01584_b200.config import ObsConfig, SimConfig
from paper_2408_01584_b200.packing import RawWorlds

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
               if os.path.basename(p) != "decimate.npz")   # (test_decimate.py)


def load(name: str):
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"), allow_pickle=False)
    raw = RawWorlds(names=[str(s) for s in z["raw_names"]],
                    **{f: z["raw_" + f] for f in (
                        "dt", "num_steps", "a_off", "kind", "length", "width", "goal",
                        "force_replay", "controllable", "l_off", "log_x", "log_y", "log_h",
                        "log_vx", "log_vy", "log_valid", "poly_off", "poly_kind",
                        "poly_pt_off", "pt_x", "pt_y")})
    spec = ast.literal_eval(str(z["cfg_json"]))
    cfg = SimConfig(dynamics=spec["dynamics"], collision_behavior=spec["collision_behavior"],
                    init_mode=spec.get("init_mode", "all_valid"), obs=ObsConfig(**spec["obs"]),
                    max_controlled_per_world=spec.get("max_controlled_per_world"))
    return z, raw, cfg


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()
