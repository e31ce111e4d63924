"""Generate the golden fixtures that pin the oracle (and the GPU path) to the
REAL reference implementation.  Runs only in the build container, where the
reference is importable from /root/reference/pkg/src; the fixtures it writes
(tests/golden/*.npz) are committed and travel to the GPU box.

    python tests/golden/make_golden.py [NAME ...]   # default: every fixture

A fixture that already exists is regenerated from ITS OWN stored raw scene
(so re-running reproduces it bit for bit whatever the generator does today);
delete the .npz to draw a fresh scene.

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
sys.path.insert(0, HERE)
from delta_local_shim import install as install_delta_local  # noqa: E402

# (scene, sim config): scene = WaymoSpec kwargs, or ("templates", seeds) for the
# reference's own generate_synthetic templates (synthetic.py:214) run through
# its preprocess (default decimation 0.05, scenario.py:387-411)
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
    # off-lattice scenes (full FP64 coordinates: the float32 copies the GPU
    # culls with carry a rounding error, grid_eps > 0)
    "offlattice_classic_remove_radial": dict(dynamics="classic", collision_behavior="remove_agent",
                                             obs=dict(mode="radial"),
                                             scene=dict(n_worlds=4, n_agents=64, n_points=2000,
                                                        seed=41, quantize=False)),
    "offlattice_invertible_end_radial": dict(dynamics="invertible", collision_behavior="end_episode",
                                             obs=dict(mode="radial", radius=35.0, max_agents_obs=5,
                                                      max_road_points_obs=30),
                                             scene=dict(n_worlds=3, n_agents=40, n_points=900,
                                                        seed=43, quantize=False)),
    "offlattice_classic_remove_lidar": dict(dynamics="classic", collision_behavior="remove_agent",
                                            obs=dict(mode="lidar", n_rays=32, max_range=50.0),
                                            scene=dict(n_worlds=3, n_agents=48, n_points=3000,
                                                       seed=47, quantize=False)),
    # BASELINE config 3 semantics (delta-local dynamics through the reference
    # with tests/golden/delta_local_shim.py, r = 50 m, 128 agents, 10k points),
    # on the benchmark's lattice and off it
    "c3_delta_local_radial": dict(dynamics="delta_local", collision_behavior="ignore",
                                  obs=dict(mode="radial", radius=50.0),
                                  scene=dict(n_worlds=2, n_agents=128, n_points=10000, seed=0),
                                  full_obs=(0, 1, 45, 90)),
    "offlattice_c3_delta_local_radial": dict(dynamics="delta_local", collision_behavior="remove_agent",
                                             obs=dict(mode="radial", radius=50.0),
                                             scene=dict(n_worlds=2, n_agents=128, n_points=10000,
                                                        seed=53, quantize=False),
                                             full_obs=(0, 1, 45, 90)),
    "offlattice_delta_local_viewcone_head": dict(dynamics="delta_local",
                                                 collision_behavior="remove_agent",
                                                 obs=dict(mode="view_cone", n_rays=20, fov=2.2,
                                                          max_range=45.0),
                                                 scene=dict(n_worlds=3, n_agents=40, n_points=1500,
                                                            seed=59, quantize=False),
                                                 head=True),
    # BASELINE config 4 shape: 64-ray LiDAR, 128 agents, 10k points, a full
    # 91-step episode (the reference takes ~0.6 s per world-step here)
    "c4_lidar_full_episode": dict(dynamics="classic", collision_behavior="ignore",
                                  obs=dict(mode="lidar", n_rays=64, max_range=50.0),
                                  scene=dict(n_worlds=2, n_agents=128, n_points=10000, seed=61,
                                             quantize=False),
                                  full_obs=(0, 1, 45, 90)),
    # the reference's own synthetic templates (off-lattice, decimated roads)
    "templates_classic_remove_radial": dict(dynamics="classic", collision_behavior="remove_agent",
                                            obs=dict(mode="radial"), scene=("templates", 4)),
    "templates_invertible_lidar": dict(dynamics="invertible", collision_behavior="ignore",
                                       obs=dict(mode="lidar", n_rays=48, max_range=40.0),
                                       scene=("templates", 3)),
    # the reference's end-to-end acceptance scenario (test_acceptance.py:425-438):
    # straight_road and intersection, 4 agents, seed 0, the default SimConfig
    # with collision ignore, driven by the reference's goal_seek_actions
    # (engine.py:559-574) rounded to float32
    "templates_goal_seek": dict(dynamics="classic", collision_behavior="ignore",
                                init_mode="all_nontrivial", obs=dict(mode="radial"),
                                scene=("acceptance",), policy="goal_seek"),
}
FULL_OBS_STEPS = (0, 1, 91)
# ragged batch (tests/ragged.py): hashes only, the GPU compares against the oracle
RAGGED = {"ragged_nontrivial_radial": dict(dynamics="classic", collision_behavior="remove_agent",
                                          init_mode="all_nontrivial", max_controlled_per_world=250,
                                          obs=dict(mode="radial"))}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


RAW_FIELDS = ("dt", "num_steps", "a_off", "kind", "length", "width", "goal", "force_replay",
              "controllable", "l_off", "log_x", "log_y", "log_h", "log_vx", "log_vy",
              "log_valid", "poly_off", "poly_kind", "poly_pt_off", "pt_x", "pt_y")


def stored_raw(name: str):
    """The raw scene stored in an existing fixture (None if there is none)."""
    path = os.path.join(HERE, f"{name}.npz")
    if not os.path.exists(path):
        return None
    from paper_2408_01584_b200.packing import RawWorlds
    z = np.load(path, allow_pickle=False)
    return RawWorlds(names=[str(s) for s in z["raw_names"]], **{f: z["raw_" + f] for f in RAW_FIELDS})


def template_scene(n_seeds: int):
    """The reference's own templates through its own preprocess."""
    from drivesim.synthetic import TEMPLATES, SyntheticSpec, generate_synthetic
    from paper_2408_01584_b200.packing import raw_from_prepared
    caps = {"straight_road": 24, "intersection": 12, "parking_lot": 25}
    preps = []
    for seed in range(n_seeds):
        for k, tpl in enumerate(TEMPLATES):
            n = min(caps[tpl], 3 + 5 * seed + 2 * k)
            preps.append(rscn.preprocess(generate_synthetic(SyntheticSpec(tpl, n_agents=n, seed=seed))))
    return raw_from_prepared(preps)


def acceptance_scene():
    from drivesim.synthetic import SyntheticSpec, generate_synthetic
    from paper_2408_01584_b200.packing import raw_from_prepared
    return raw_from_prepared([rscn.preprocess(generate_synthetic(SyntheticSpec(t, n_agents=4, seed=0)))
                              for t in ("straight_road", "intersection")])


def draw_actions(spec: dict, n: int, rng, batch=None) -> np.ndarray:
    """float32-valued actions; delta_local: small ego-frame moves plus ~5 %
    of rows far outside delta_bounds (exercises the clip)."""
    if spec.get("policy") == "goal_seek":
        from drivesim.engine import goal_seek_actions
        a = np.vstack([goal_seek_actions(w) for w in batch.worlds])
    elif spec["dynamics"] == "delta_local":
        a = np.column_stack([rng.uniform(-1.0, 1.0, n), rng.uniform(-0.6, 0.6, n),
                             rng.uniform(-0.3, 0.3, n)])
        wild = rng.random(n) < 0.05
        a[wild] = rng.uniform(-9.0, 9.0, (int(wild.sum()), 3))
    else:
        a = np.column_stack([rng.uniform(-4, 4, n), rng.uniform(-0.7, 0.7, n)])
    if spec.get("head", False):
        a = np.column_stack([a, rng.uniform(-1.5, 1.5, n)])
    return a.astype(np.float32)


def make(name: str, spec: dict, n_worlds=3, n_agents=32, n_points=400, seed=21, steps=91,
         raw=None, full_obs=FULL_OBS_STEPS):
    if raw is None:
        raw = stored_raw(name)
    if raw is None:
        scene = spec.get("scene", dict(n_worlds=n_worlds, n_agents=n_agents, n_points=n_points,
                                       seed=seed))
        if isinstance(scene, tuple) and scene[0] == "templates":
            raw = template_scene(scene[1])
        elif isinstance(scene, tuple) and scene[0] == "acceptance":
            raw = acceptance_scene()
        else:
            raw = generate(WaymoSpec(**scene))
    full_obs = spec.get("full_obs", full_obs)
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
    for f in RAW_FIELDS:
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
    for t in range(1, steps + 1):
        a = draw_actions(spec, n, rng, batch)
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
    out["cfg_json"] = np.array(repr({k: v for k, v in spec.items() if k not in ("scene", "full_obs", "policy")}))
    path = os.path.join(HERE, f"{name}.npz")
    if os.path.exists(path):
        old = np.load(path, allow_pickle=False)
        same = all(k in old and np.array_equal(old[k], out[k]) for k in out if k != "name")
        print(f"{name}: {'reproduced bit for bit' if same else 'CHANGED'}")
    np.savez_compressed(path, **out)
    print(f"{name}: {n} rows, {len(out['episodes'])} episodes, "
          f"goal={int(out['info'][:, 0].sum())} coll={int(out['info'][:, 1].sum())} "
          f"off={int(out['info'][:, 2].sum())}")


def main(names=()):
    import numba
    assert _fastpath.ENABLED, "the reference's numba fast path must be active"
    install_delta_local()
    with open(os.path.join(HERE, "PROVENANCE.txt"), "w") as f:
        f.write(f"reference: {os.path.dirname(_ref_file)} (numba fast path)\n"
                f"numpy {np.__version__}, numba {numba.__version__}, python {sys.version.split()[0]}\n"
                "generator: paper_2408_01584_b200.synthetic (raw scene arrays stored in each npz;\n"
                "  re-running make_golden.py regenerates every fixture from its stored scene)\n"
                "templates_*: the reference's drivesim.synthetic.generate_synthetic + preprocess\n"
                "*delta_local*: the reference + tests/golden/delta_local_shim.py\n"
                "decimate.npz: tests/golden/make_golden_decimate.py (reference drivesim.geometry.decimate_polyline)\n")
    for name, spec in CONFIGS.items():
        if not names or name in names:
            make(name, spec)
    sys.path.insert(0, os.path.dirname(HERE))
    from ragged import ragged_batch
    for name, spec in RAGGED.items():
        if not names or name in names:
            make(name, spec, raw=stored_raw(name) or ragged_batch(seed=5), full_obs=())


if __name__ == "__main__":
    main(sys.argv[1:])
