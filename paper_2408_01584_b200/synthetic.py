"""Waymo-shaped synthetic scenes, generated vectorised.

The reference's own templates (pkg/src/drivesim/synthetic.py) cap at 24/12/25
agents with a handful of road points, so they cannot produce the benchmark
configurations (32-128 agents, 400-10k road points).  This generator follows
the survey's recipe:

* map side L = 40*sqrt(P/100) + 60 m;
* road polylines of 10-60 points at 2 m spacing with a heading random walk
  (sigma 0.05 rad/point), exactly P points per world; kinds lane 40 %,
  road_edge 30 %, road_line 20 %, crosswalk 10 %;
* agents 80 % vehicle (4.6 +- 0.3 x 1.8 m), 10 % pedestrian (0.8 x 0.8),
  10 % cyclist (1.8 x 0.6), uniform in the central L/2 square, heading
  U(-pi, pi], speed U[2, 15] m/s;
* T-step logs from a classic-bicycle rollout with a = 0 and a constant steer
  U(-0.1, 0.1), all valid; goal = final logged position;
* every coordinate quantised to 2^-10 m (lossless in float32) -- or, with
  ``quantize=False``, left at full FP64 resolution (off-lattice: the float32
  copies the kernels cull with carry a non-zero rounding error, as real
  prepared / WOMD inputs do).

A world's content depends only on (seed, global world id), so a world shard
generated on any rank is identical to the same world generated anywhere else.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .config import OBJECT_KINDS, ROAD_KINDS
from .packing import RawWorlds, _offsets

Q = 1.0 / 1024.0
KIND_P = {"lane": 0.4, "road_edge": 0.3, "road_line": 0.2, "crosswalk": 0.1}


@dataclass
class WaymoSpec:
    n_worlds: int
    n_agents: int = 32
    n_points: int = 400
    seed: int = 0
    num_steps: int = 91
    dt: float = 0.1
    world_offset: int = 0       # global id of the first world (sharding)
    map_side: float | None = None
    quantize: bool = True       # False: off-lattice FP64 coordinates

    @property
    def side(self) -> float:
        if self.map_side is not None:
            return self.map_side
        return 40.0 * math.sqrt(self.n_points / 100.0) + 60.0


def _quant(v, on: bool = True):
    return np.round(np.asarray(v) / Q) * Q if on else np.asarray(v, np.float64)


def _world_params(spec: WaymoSpec, wid: int):
    """All random draws of one world, from its own stream (seed, world id)."""
    rng = np.random.default_rng([spec.seed, wid])
    L = spec.side
    A, P = spec.n_agents, spec.n_points
    u = rng.random(A)
    kind = np.where(u < 0.8, 0, np.where(u < 0.9, 1, 2)).astype(np.int8)
    length = np.where(kind == 0, 4.6 + rng.uniform(-0.3, 0.3, A), np.where(kind == 1, 0.8, 1.8))
    width = np.where(kind == 0, 1.8, np.where(kind == 1, 0.8, 0.6))
    q = spec.quantize
    x = _quant(rng.uniform(0.25 * L, 0.75 * L, A), q)
    y = _quant(rng.uniform(0.25 * L, 0.75 * L, A), q)
    h = -rng.uniform(-math.pi, math.pi, A)          # (-pi, pi]
    v = rng.uniform(2.0, 15.0, A)
    steer = rng.uniform(-0.1, 0.1, A)
    # road polylines of 10..60 points summing to exactly P (a short tail is
    # merged into the last polyline)
    lens = rng.integers(10, 61, size=P // 10 + 2)
    cum = np.cumsum(lens)
    m = int(np.searchsorted(cum, P, side="left")) + 1
    lens = lens[:m].copy()
    lens[-1] -= int(cum[m - 1] - P)
    if len(lens) > 1 and lens[-1] < 10:
        lens[-2] += lens[-1]
        lens = lens[:-1]
    R = len(lens)
    ku = rng.random(R)
    cuts = np.cumsum([KIND_P["road_edge"], KIND_P["lane"], KIND_P["road_line"]])
    kinds = np.where(ku < cuts[0], ROAD_KINDS.index("road_edge"),
                     np.where(ku < cuts[1], ROAD_KINDS.index("lane"),
                              np.where(ku < cuts[2], ROAD_KINDS.index("road_line"),
                                       ROAD_KINDS.index("crosswalk")))).astype(np.int8)
    start = rng.uniform(0.0, L, (R, 2))
    h0 = rng.uniform(-math.pi, math.pi, R)
    steps = rng.normal(0.0, 0.05, P)
    poly_of = np.repeat(np.arange(R), lens)
    first = np.concatenate([[0], np.cumsum(lens)[:-1]])
    steps[first] = 0.0
    ang = np.cumsum(steps)
    ang = ang - np.repeat(ang[first], lens) + h0[poly_of]
    dx = 2.0 * np.cos(ang)
    dy = 2.0 * np.sin(ang)
    dx[first] = 0.0
    dy[first] = 0.0
    px = np.cumsum(dx)
    py = np.cumsum(dy)
    px = px - np.repeat(px[first], lens) + start[poly_of, 0]
    py = py - np.repeat(py[first], lens) + start[poly_of, 1]
    return dict(kind=kind, length=length, width=width, x=x, y=y, h=h, v=v, steer=steer,
                lens=lens, pkind=kinds, px=_quant(px, q), py=_quant(py, q))


def generate(spec: WaymoSpec) -> RawWorlds:
    """RawWorlds for worlds [world_offset, world_offset + n_worlds)."""
    parts = [_world_params(spec, spec.world_offset + k) for k in range(spec.n_worlds)]
    W, A, T = spec.n_worlds, spec.n_agents, spec.num_steps
    cat = lambda key: np.concatenate([p[key] for p in parts])
    # classic-bicycle rollout with a = 0 and constant steer, all worlds at once
    length, v, steer = cat("length"), cat("v"), cat("steer")
    cx, cy, ch = cat("x").astype(np.float64), cat("y").astype(np.float64), cat("h")
    beta = np.arctan(0.5 * np.tan(steer))
    turn = v * np.cos(beta) * np.tan(steer) / length * spec.dt
    N = W * A
    lx = np.empty((N, T)); ly = np.empty((N, T)); lh = np.empty((N, T))
    for t in range(T):
        lx[:, t], ly[:, t], lh[:, t] = cx, cy, ch
        cx = cx + v * np.cos(ch + beta) * spec.dt
        cy = cy + v * np.sin(ch + beta) * spec.dt
        ch = np.mod(ch + turn + math.pi, 2 * math.pi) - math.pi
        ch = np.where(ch <= -math.pi, ch + 2 * math.pi, ch)
    lx, ly = _quant(lx, spec.quantize), _quant(ly, spec.quantize)
    vx = v[:, None] * np.cos(lh)
    vy = v[:, None] * np.sin(lh)
    goal = np.stack([lx[:, -1], ly[:, -1]], -1)
    lens = [p["lens"] for p in parts]
    raw = RawWorlds(
        names=[f"waymo-synth-{spec.seed}-{spec.world_offset + k}" for k in range(W)],
        dt=np.full(W, spec.dt), num_steps=np.full(W, T, np.int32),
        a_off=_offsets([A] * W), kind=cat("kind"), length=length, width=cat("width"),
        goal=goal, force_replay=np.zeros(N, bool), controllable=np.zeros(N, bool),
        l_off=_offsets([A * T] * W), log_x=lx.reshape(-1), log_y=ly.reshape(-1),
        log_h=lh.reshape(-1), log_vx=vx.reshape(-1), log_vy=vy.reshape(-1),
        log_valid=np.ones(N * T, bool), poly_off=_offsets([len(l) for l in lens]),
        poly_kind=cat("pkind"), poly_pt_off=_offsets(np.concatenate(lens)), pt_x=cat("px"),
        pt_y=cat("py"))
    # mark_controllable (scenario.py:371-384) with the default 2.0 m threshold;
    # the reference's distance is CPython's math.hypot (pure Python here, so
    # generating a scene never loads the CUDA library)
    d = np.frompyfunc(math.hypot, 2, 1)(lx[:, 0] - goal[:, 0], ly[:, 0] - goal[:, 1])
    raw.controllable = d.astype(np.float64) > 2.0
    return raw


def to_scenarios(raw: RawWorlds, types=None) -> list:
    """Prepared-scenario objects for ``raw`` built with ``types`` (a module
    exposing Vec2/LoggedStep/ObjectLog/RoadElement/Scenario/PreparedScenario/
    PrepStats -- ours by default, or the reference's drivesim.scenario)."""
    if types is None:
        from . import scenario as types
    out = []
    for w in range(raw.n_worlds):
        T = int(raw.num_steps[w])
        objs = []
        for k, g in enumerate(range(raw.a_off[w], raw.a_off[w + 1])):
            base = raw.l_off[w] + k * T
            states = [types.LoggedStep(position=types.Vec2(float(raw.log_x[base + t]),
                                                           float(raw.log_y[base + t])),
                                       heading=float(raw.log_h[base + t]),
                                       velocity=types.Vec2(float(raw.log_vx[base + t]),
                                                           float(raw.log_vy[base + t])),
                                       valid=bool(raw.log_valid[base + t])) for t in range(T)]
            objs.append(types.ObjectLog(id=k, kind=OBJECT_KINDS[raw.kind[g]],
                                        length=float(raw.length[g]), width=float(raw.width[g]),
                                        goal=types.Vec2(float(raw.goal[g, 0]), float(raw.goal[g, 1])),
                                        states=states, force_replay=bool(raw.force_replay[g])))
        roads = []
        for rid, r in enumerate(range(raw.poly_off[w], raw.poly_off[w + 1])):
            pts = [types.Vec2(float(raw.pt_x[q]), float(raw.pt_y[q]))
                   for q in range(raw.poly_pt_off[r], raw.poly_pt_off[r + 1])]
            roads.append(types.RoadElement(id=rid, kind=ROAD_KINDS[raw.poly_kind[r]], geometry=pts))
        s = types.Scenario(name=raw.names[w], timestep=float(raw.dt[w]), num_steps=T,
                           objects=objs, roads=roads)
        ctrl = [bool(c) for c in raw.controllable[raw.a_off[w]:raw.a_off[w + 1]]]
        n_pts = sum(len(r.geometry) for r in roads)
        out.append(types.PreparedScenario(
            base=s, decimated_roads=roads, controllable=ctrl,
            stats=types.PrepStats(len(objs), sum(ctrl), n_pts, n_pts)))
    return out
