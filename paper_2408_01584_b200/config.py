"""Simulator and observation configuration (the knobs of the batched step).

Mirrors the reference's ``SimConfig`` (pkg/src/drivesim/engine.py:45-107) and
``ObsConfig`` (pkg/src/drivesim/observation.py:51-67) field for field, with the
same defaults, the same ``ValueError`` on unknown models/modes and the same flat
``key = value`` file loader, so a config written for the reference loads here.

One addition: ``dynamics="delta_local"`` (absent from the reference, whose
DYNAMICS_MODELS is ("classic", "invertible") at engine.py:32).  BASELINE config
3 asks for it; its definition lives in DESIGN.md §dynamics and in
``oracle/drivesim_oracle.c`` (parity for it is pinned only to our own oracle).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

DEFAULT_ACCEL_BOUNDS = (-4.0, 4.0)      # dynamics.py:27
DEFAULT_STEER_BOUNDS = (-0.7, 0.7)      # dynamics.py:28
DEFAULT_V_MAX = 100.0                   # dynamics.py:29
# delta_local action bounds (dx, dy in metres per step, dyaw in rad per step).
DEFAULT_DELTA_BOUNDS = ((-6.0, 6.0), (-6.0, 6.0), (-math.pi, math.pi))

DYNAMICS_MODELS = ("classic", "invertible", "delta_local")
COLLISION_BEHAVIORS = ("ignore", "remove_agent", "end_episode")   # engine.py:33
INIT_MODES = ("all_nontrivial", "all_valid")                       # engine.py:34
OBS_MODES = ("radial", "lidar", "view_cone")                       # observation.py:62

OBJECT_KINDS = ("vehicle", "pedestrian", "cyclist")                # scenario.py:32
ROAD_KINDS = ("road_edge", "lane", "road_line", "crosswalk",
              "speed_bump", "stop_sign", "driveway")               # scenario.py:33
PEDESTRIAN = OBJECT_KINDS.index("pedestrian")
ROAD_EDGE = ROAD_KINDS.index("road_edge")

# Flat observation layout (observation.py:39-44).
EGO_WIDTH = 7
PARTNER_WIDTH = 7
ROAD_SLOT_WIDTH = 3 + len(ROAD_KINDS) + 1
RAY_WIDTH = 5
HIT_TYPES = ("agent", "road_edge", "other_road", "none")
MAX_HEAD_ANGLE = 0.5 * math.pi


@dataclass
class ObsConfig:
    mode: str = "radial"            # radial | lidar | view_cone
    radius: float = 50.0
    n_rays: int = 64
    fov: float = 2.0 * math.pi / 3.0
    max_range: float = 100.0
    max_agents_obs: int = 16
    max_road_points_obs: int = 64

    def __post_init__(self):
        if self.mode not in OBS_MODES:
            raise ValueError(f"unknown observation mode {self.mode!r}")
        if self.n_rays < 1:
            raise ValueError("n_rays must be >= 1")
        if not 0.0 < self.fov <= 2.0 * math.pi:
            raise ValueError("fov must be in (0, 2*pi]")
        if self.max_agents_obs < 0 or self.max_road_points_obs < 0:
            raise ValueError("slot caps must be >= 0")


@dataclass
class ObsLayout:
    """Offsets and widths of the blocks of one flat observation row."""

    width: int
    blocks: list

    def offset(self, name: str) -> int:
        for n, off, _ in self.blocks:
            if n == name:
                return off
        raise KeyError(name)


def layout(cfg: ObsConfig) -> ObsLayout:
    """observation.py:84-95: ego, then partners+roads (radial) or rays."""
    blocks = [("ego", 0, EGO_WIDTH)]
    off = EGO_WIDTH
    if cfg.mode == "radial":
        blocks.append(("partners", off, PARTNER_WIDTH * cfg.max_agents_obs))
        off += PARTNER_WIDTH * cfg.max_agents_obs
        blocks.append(("roads", off, ROAD_SLOT_WIDTH * cfg.max_road_points_obs))
        off += ROAD_SLOT_WIDTH * cfg.max_road_points_obs
    else:
        blocks.append(("rays", off, RAY_WIDTH * cfg.n_rays))
        off += RAY_WIDTH * cfg.n_rays
    return ObsLayout(width=off, blocks=blocks)


def obs_width(cfg: ObsConfig) -> int:
    return layout(cfg).width


@dataclass
class SimConfig:
    dynamics: str = "classic"
    obs: ObsConfig = field(default_factory=ObsConfig)
    goal_tolerance: float = 2.0
    collision_behavior: str = "ignore"
    init_mode: str = "all_nontrivial"
    nontrivial_threshold: float = 2.0
    max_controlled_per_world: int | None = None
    seed: int = 0
    accel_bounds: tuple = DEFAULT_ACCEL_BOUNDS
    steer_bounds: tuple = DEFAULT_STEER_BOUNDS
    v_max: float = DEFAULT_V_MAX
    delta_bounds: tuple = DEFAULT_DELTA_BOUNDS

    def __post_init__(self):
        if self.dynamics not in DYNAMICS_MODELS:
            raise ValueError(f"unknown dynamics model {self.dynamics!r}")
        if self.collision_behavior not in COLLISION_BEHAVIORS:
            raise ValueError(f"unknown collision behavior {self.collision_behavior!r}")
        if self.init_mode not in INIT_MODES:
            raise ValueError(f"unknown init mode {self.init_mode!r}")
        if self.goal_tolerance <= 0:
            raise ValueError("goal_tolerance must be > 0")

    @property
    def action_dim(self) -> int:
        """Columns of a continuous action row without head rotation."""
        return 3 if self.dynamics == "delta_local" else 2

    @classmethod
    def from_file(cls, path: str) -> "SimConfig":
        """Flat ``key = value`` file; keys mirror SimConfig/ObsConfig fields
        (engine.py:69-107).  Unknown keys raise KeyError."""
        kv = {}
        with open(path) as f:
            for line in f:
                line = line.split("#", 1)[0].strip()
                if not line:
                    continue
                key, _, value = line.partition("=")
                kv[key.strip()] = value.strip()
        obs_kw = {}
        for name in ("mode", "radius", "n_rays", "fov", "max_range",
                     "max_agents_obs", "max_road_points_obs"):
            if name not in kv:
                continue
            raw = kv.pop(name)
            if name == "mode":
                obs_kw[name] = raw
            elif name in ("n_rays", "max_agents_obs", "max_road_points_obs"):
                obs_kw[name] = int(raw)
            else:
                obs_kw[name] = float(raw)
        cfg = cls()
        for key, raw in kv.items():
            if not hasattr(cfg, key):
                raise KeyError(f"unknown config key {key!r}")
            cur = getattr(cfg, key)
            if key in ("dynamics", "collision_behavior", "init_mode"):
                val = raw
            elif key == "max_controlled_per_world":
                val = None if raw in ("none", "") else int(raw)
            elif key == "delta_bounds":
                nums = [float(v) for v in raw.split(",")]
                val = tuple(zip(nums[0::2], nums[1::2]))
            elif isinstance(cur, tuple):
                val = tuple(float(v) for v in raw.split(","))
            elif isinstance(cur, bool):
                val = raw.lower() in ("1", "true", "yes")
            elif isinstance(cur, int):
                val = int(raw)
            elif isinstance(cur, float):
                val = float(raw)
            else:
                val = raw
            setattr(cfg, key, val)
        cfg.obs = ObsConfig(**obs_kw)
        cfg.__post_init__()
        return cfg
