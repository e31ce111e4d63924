"""Scenario value types accepted by the batched step.

The batch constructor takes a list of prepared scenarios exactly like the
reference's ``SimBatch(scenarios: list[PreparedScenario], cfg)``
(pkg/src/drivesim/engine.py:591).  These dataclasses mirror the reference's
field names (pkg/src/drivesim/scenario.py:60-121) so that objects produced by
the reference's own ``preprocess``/``load_prepared`` are accepted unchanged
(duck typing); they exist here only so the package runs where the reference is
not installed.

Preprocessing: ``preprocess`` / ``preprocess_many`` decimate
road polylines on the GPU with the reference's exact iterative
smallest-area removal (one warp per polyline, ``ds_decimate_polylines``) and
mark the controllable agents.  JSON schema validation is out of scope.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import NamedTuple

DEFAULT_TIMESTEP = 0.1
DEFAULT_NUM_STEPS = 91


class Vec2(NamedTuple):
    x: float
    y: float


@dataclass
class LoggedStep:
    position: Vec2
    heading: float
    velocity: Vec2
    valid: bool


@dataclass
class ObjectLog:
    id: int
    kind: str
    length: float
    width: float
    goal: Vec2
    states: list
    force_replay: bool = False

    def first_valid(self):
        for i, st in enumerate(self.states):
            if st.valid:
                return i
        return None


@dataclass
class RoadElement:
    id: int
    kind: str
    geometry: list


@dataclass
class Scenario:
    name: str
    timestep: float = DEFAULT_TIMESTEP
    num_steps: int = DEFAULT_NUM_STEPS
    objects: list = field(default_factory=list)
    roads: list = field(default_factory=list)


@dataclass
class PrepStats:
    n_objects: int
    n_controllable: int
    n_road_points_before: int
    n_road_points_after: int


@dataclass
class PreparedScenario:
    base: Scenario
    decimated_roads: list
    controllable: list
    stats: PrepStats


def mark_controllable(s: Scenario, threshold: float) -> list:
    """scenario.py:371-384: valid first state, not force_replay, and strictly
    farther than ``threshold`` from the goal (CPython math.hypot)."""
    mask = []
    for o in s.objects:
        fv = o.first_valid()
        if fv is None or o.force_replay:
            mask.append(False)
            continue
        p = o.states[fv].position
        mask.append(math.hypot(p.x - o.goal.x, p.y - o.goal.y) > threshold)
    return mask


def decimate_keep(x, y, poly_off, threshold: float, skip=None, device=None):
    """Batched decimate_polyline (geometry.py:84-127) on the GPU: keep mask
    (numpy bool [P]) of the points of every polyline [poly_off[p],
    poly_off[p+1]) of the FP64 coordinate arrays x, y; polylines with
    skip[p] are kept whole.  Bit-exact with the reference (same FP64 area
    expression, same removal order)."""
    import ctypes as C

    import numpy as np
    import torch

    from . import _native as N
    dev = torch.device(device if device is not None else "cuda")
    if dev.type != "cuda":
        raise ValueError("decimation runs on a CUDA device only (no CPU fallback)")
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    off = np.ascontiguousarray(poly_off, dtype=np.int64)
    P, n_poly = len(x), len(off) - 1
    if P == 0 or n_poly <= 0:
        return np.ones(P, bool)
    tx = torch.from_numpy(x).to(dev)
    ty = torch.from_numpy(y).to(dev)
    toff = torch.from_numpy(off).to(dev)
    tskip = None
    if skip is not None:
        tskip = torch.from_numpy(np.ascontiguousarray(skip, dtype=np.uint8)).to(dev)
    keep = torch.empty(P, dtype=torch.uint8, device=dev)
    scratch = torch.empty(int(N.lib().ds_decimate_scratch_bytes(P)) // 8 + 1, dtype=torch.float64,
                          device=dev)
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    N.check(N.lib().ds_decimate_polylines(
        tx.data_ptr(), ty.data_ptr(), toff.data_ptr(), n_poly,
        tskip.data_ptr() if tskip is not None else None, float(threshold), keep.data_ptr(),
        scratch.data_ptr(), P, stream), "ds_decimate_polylines")
    return keep.cpu().numpy().astype(bool)


def decimate_polyline(points, area_threshold: float, device=None) -> list:
    """geometry.decimate_polyline (geo:84-127) for one polyline."""
    import numpy as np
    pts = list(points)
    if len(pts) < 3 or area_threshold <= 0.0:
        return pts
    xy = np.array([(float(p[0]), float(p[1])) for p in pts], dtype=np.float64)
    keep = decimate_keep(xy[:, 0], xy[:, 1], [0, len(pts)], area_threshold, device=device)
    return [p for p, k in zip(pts, keep) if k]


def preprocess_many(scenarios: list, decimation_threshold: float = 0.05,
                    controllable_threshold: float = 2.0, device=None) -> list:
    """preprocess (scenario.py:387-411) of many scenarios, every polyline of
    every scenario decimated in one GPU launch.  Stop signs and polylines
    with fewer than 3 points pass through unchanged."""
    import numpy as np
    roads = [(k, r) for k, s in enumerate(scenarios) for r in s.roads]
    counts = np.array([len(r.geometry) for _, r in roads], dtype=np.int64)
    off = np.zeros(len(roads) + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    xy = np.array([(float(p[0]), float(p[1])) for _, r in roads for p in r.geometry],
                  dtype=np.float64).reshape(-1, 2)
    skip = np.array([r.kind == "stop_sign" or len(r.geometry) < 3 for _, r in roads], bool)
    keep = (decimate_keep(xy[:, 0], xy[:, 1], off, decimation_threshold, skip, device)
            if decimation_threshold > 0.0 and len(xy) else np.ones(len(xy), bool))
    out, q = [], 0
    per = [[] for _ in scenarios]
    for (k, r), c in zip(roads, counts):
        geom = [p for p, kk in zip(r.geometry, keep[q:q + c]) if kk]
        per[k].append(RoadElement(id=r.id, kind=r.kind, geometry=geom))
        q += c
    for s, dec in zip(scenarios, per):
        before = sum(len(r.geometry) for r in s.roads)
        after = sum(len(r.geometry) for r in dec)
        ctrl = mark_controllable(s, controllable_threshold)
        out.append(PreparedScenario(base=s, decimated_roads=dec, controllable=ctrl,
                                    stats=PrepStats(len(s.objects), sum(ctrl), before, after)))
    return out


def preprocess(s: Scenario, decimation_threshold: float = 0.05,
               controllable_threshold: float = 2.0, device=None) -> PreparedScenario:
    """scenario.py:387-411: decimate road polylines (GPU) and compute the
    controllable mask; same defaults as the reference."""
    return preprocess_many([s], decimation_threshold, controllable_threshold, device)[0]


def scenario_to_dict(s: Scenario) -> dict:
    """scenario.py:286-305: the scenario JSON document."""
    return {
        "name": s.name, "timestep_s": s.timestep, "num_steps": s.num_steps,
        "objects": [{"id": o.id, "type": o.kind, "length_m": o.length, "width_m": o.width,
                     "goal": [o.goal[0], o.goal[1]], "force_replay": o.force_replay,
                     "states": [{"p": [st.position[0], st.position[1]], "heading": st.heading,
                                 "v": [st.velocity[0], st.velocity[1]], "valid": st.valid}
                                for st in o.states]} for o in s.objects],
        "roads": [{"id": r.id, "type": r.kind, "geometry": [[p[0], p[1]] for p in r.geometry]}
                  for r in s.roads],
    }


def serialize_prepared(p: PreparedScenario) -> str:
    """scenario.py:416-431: scenario JSON plus a "prepared" section."""
    import json
    doc = scenario_to_dict(p.base)
    doc["prepared"] = {
        "roads": [{"id": r.id, "type": r.kind, "geometry": [[q[0], q[1]] for q in r.geometry]}
                  for r in p.decimated_roads],
        "controllable": list(p.controllable),
        "stats": {"n_objects": p.stats.n_objects, "n_controllable": p.stats.n_controllable,
                  "n_road_points_before": p.stats.n_road_points_before,
                  "n_road_points_after": p.stats.n_road_points_after},
    }
    return json.dumps(doc)


def load_prepared(json_text: str, decimation_threshold: float = 0.05,
                  controllable_threshold: float = 2.0) -> PreparedScenario:
    """Reader of the reference's prepared-scenario JSON (scenario.py:434-454:
    scenario fields plus a "prepared" section); plain scenario files are
    preprocessed on the fly with the given thresholds.  No schema validation
    (ingestion is out of scope)."""
    import json
    doc = json.loads(json_text)
    objs = []
    for raw in doc.get("objects", []):
        states = [LoggedStep(position=Vec2(*map(float, st["p"])), heading=float(st["heading"]),
                             velocity=Vec2(*map(float, st["v"])), valid=bool(st.get("valid", True)))
                  for st in raw["states"]]
        if "goal" in raw:
            goal = Vec2(*map(float, raw["goal"]))
        else:
            goal = next(s.position for s in reversed(states) if s.valid)
        objs.append(ObjectLog(id=int(raw["id"]), kind=raw["type"], length=float(raw["length_m"]),
                              width=float(raw["width_m"]), goal=goal, states=states,
                              force_replay=bool(raw.get("force_replay", False))))
    roads = [RoadElement(id=int(r["id"]), kind=r["type"],
                         geometry=[Vec2(float(x), float(y)) for x, y in r["geometry"]])
             for r in doc.get("roads", [])]
    base = Scenario(name=doc["name"], timestep=float(doc.get("timestep_s", DEFAULT_TIMESTEP)),
                    num_steps=int(doc.get("num_steps", DEFAULT_NUM_STEPS)), objects=objs,
                    roads=roads)
    prep = doc.get("prepared")
    if not isinstance(prep, dict):
        return preprocess(base, decimation_threshold, controllable_threshold)
    dec = [RoadElement(id=int(r["id"]), kind=r["type"],
                       geometry=[Vec2(float(x), float(y)) for x, y in r["geometry"]])
           for r in prep["roads"]]
    st = prep["stats"]
    return PreparedScenario(base=base, decimated_roads=dec,
                            controllable=[bool(b) for b in prep["controllable"]],
                            stats=PrepStats(int(st["n_objects"]), int(st["n_controllable"]),
                                            int(st["n_road_points_before"]),
                                            int(st["n_road_points_after"])))
