"""Generate the golden fixtures that pin the oracle (and the GPU path) to the
REAL reference implementation.  Runs only in the build container, where the
reference is importable from /root/reference/pkg/src; the fixtures it writes
(tests/golden/*.npz) are committed and travel to the GPU box.

    python tests/golden/make_golden.py

For each configuration below, the reference's own SimBatch (engine.py:582-677,
numba fast path, as benchmark() times it) is stepped for a full 91-step
episode on Waymo-shaped synthetic scenes with recorded float32-valued actions.
Stored per configuration:
  * the raw scene arrays (so the test does not depend on the generator),
  * the reference World tables (replay tables, controlled ids, road headings)
    that pin the packer,
  * actions, rewards, dones and info flags of every step,
  * the SHA-256 of the float64 observation buffer of every step,
  * full float64 observations at steps 0, 1 and 91, poses of every step,
  * the finished-episode records.
"""

from __future__ import annotations

import hashlib
import zlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)

from drivesim import __file__ as _ref_file  # noqa: E402
from drivesim import _fastpath  # noqa: E402
import drivesim.scenario as rscn  # noqa: E402
from drivesim.engine import SimBatch as RBatch, SimConfig as RCfg  # noqa: E402
from drivesim.observation import ObsConfig as RObs  # noqa: E402

from paper_2408_01584_b200.synthetic import WaymoSpec, generate, to_scenarios  # noqa: E402

CONFIGS = {
    "classic_remove_radial": dict(dynamics="classic", collision_behavior="remove_agent",
                                  obs=dict(mode="radial")),
    "invertible_ignore_radial": dict(dynamics="invertible", collision_behavior="ignore",
                                     obs=dict(mode="radial", radius=30.0, max_agents_obs=8,
                                              max_road_points_obs=20)),
    "classic_end_radial": dict(dynamics="classic", collision_behavior="end_episode",
                               obs=dict(mode="radial")),
    "classic_remove_lidar": dict(dynamics="classic", collision_behavior="remove_agent",
                                 obs=dict(mode="lidar", n_rays=16, max_range=60.0)),
    "classic_ignore_viewcone": dict(dynamics="classic", collision_behavior="ignore",
                                    obs=dict(mode="view_cone", n_rays=12, max_range=70.0),
                                    head=True),
}
FULL_OBS_STEPS = (0, 1, 91)
# ragged batch (tests/ragged.py): hashes only, the GPU compares against the oracle
RAGGED = {"ragged_nontrivial_radial": dict(dynamics="classic", collision_behavior="remove_agent",
                                          init_mode="all_nontrivial", max_controlled_per_world=250,
                                          obs=dict(mode="radial"))}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def make(name: str, spec: dict, n_worlds=3, n_agents=32, n_points=400, seed=21, steps=91,
         raw=None, full_obs=FULL_OBS_STEPS):
    if raw is None:
        raw = generate(WaymoSpec(n_worlds=n_worlds, n_agents=n_agents, n_points=n_points,
                                 seed=seed))
    preps = to_scenarios(raw, rscn)
    obs = RObs(**spec["obs"])
    cfg = RCfg(dynamics=spec["dynamics"], collision_behavior=spec["collision_behavior"],
               init_mode=spec.get("init_mode", "all_valid"), obs=obs,
               max_controlled_per_world=spec.get("max_controlled_per_world"))
    batch = RBatch(preps, cfg)
    n = batch.n_controlled
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    out = {"name": name}
    # raw scene
    for f in ("dt", "num_steps", "a_off", "kind", "length", "width", "goal", "force_replay",
              "controllable", "l_off", "log_x", "log_y", "log_h", "log_vx", "log_vy",
              "log_valid", "poly_off", "poly_kind", "poly_pt_off", "pt_x", "pt_y"):
        out["raw_" + f] = getattr(raw, f)
    out["raw_names"] = np.array(raw.names)
    # reference World tables (pin the packer)
    for w, world in enumerate(batch.worlds):
        out[f"tab{w}_replay_pos"] = world.replay_pos
        out[f"tab{w}_replay_heading"] = world.replay_heading
        out[f"tab{w}_replay_speed"] = world.replay_speed
        out[f"tab{w}_present_log"] = world.present_log
        out[f"tab{w}_controlled_ids"] = world.controlled_ids
        out[f"tab{w}_road_pt_heading"] = world.road_pt_heading
        out[f"tab{w}_circumradius"] = world.circumradius
    acts, rews, dones, infos, hashes, poses = [], [], [], [], [], []
    hashes.append(sha(batch.observations))
    if 0 in full_obs:
        out["obs_0"] = batch.observations.copy()
    head = spec.get("head", False)
    for t in range(1, steps + 1):
        a = np.column_stack([rng.uniform(-4, 4, n), rng.uniform(-0.7, 0.7, n)])
        if head:
            a = np.column_stack([a, rng.uniform(-1.5, 1.5, n)])
        a = a.astype(np.float32)
        o = batch.step(a.astype(np.float64))
        acts.append(a)
        rews.append(o.rewards.copy())
        dones.append(o.dones.copy())
        infos.append(np.stack([o.info[k] for k in ("goal", "veh_collision", "offroad")]))
        hashes.append(sha(o.observations))
        if t in full_obs:
            out[f"obs_{t}"] = o.observations.copy()
        poses.append(np.concatenate([np.stack([w.pos[:, 0], w.pos[:, 1], w.heading, w.speed])
                                     for w in batch.worlds], 1))
    out["actions"] = np.stack(acts)
    out["rewards"] = np.stack(rews)
    out["dones"] = np.stack(dones)
    out["info"] = np.stack(infos)
    out["obs_sha256"] = np.array(hashes)
    out["poses"] = np.stack(poses)
    out["episodes"] = np.array([(e.world_id, e.n_controlled, e.n_goal, e.n_veh_collision,
                                 e.n_offroad) for e in batch.episode_infos], np.int64).reshape(-1, 5)
    out["cfg_json"] = np.array(repr(spec))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {n} rows, {len(out['episodes'])} episodes, "
          f"goal={int(out['info'][:, 0].sum())} coll={int(out['info'][:, 1].sum())} "
          f"off={int(out['info'][:, 2].sum())}")


def main():
    import numba
    assert _fastpath.ENABLED, "the reference's numba fast path must be active"
    with open(os.path.join(HERE, "PROVENANCE.txt"), "w") as f:
        f.write(f"reference: {os.path.dirname(_ref_file)} (numba fast path)\n"
                f"numpy {np.__version__}, numba {numba.__version__}, python {sys.version.split()[0]}\n"
                "generator: paper_2408_01584_b200.synthetic (raw scene arrays stored in each npz)\n")
    for name, spec in CONFIGS.items():
        make(name, spec)
    sys.path.insert(0, os.path.dirname(HERE))
    from ragged import ragged_batch
    for name, spec in RAGGED.items():
        make(name, spec, raw=ragged_batch(seed=5), full_obs=())


if __name__ == "__main__":
    main()
