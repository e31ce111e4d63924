"""Scenario value types accepted by the batched step.

The batch constructor takes a list of prepared scenarios exactly like the
reference's ``SimBatch(scenarios: list[PreparedScenario], cfg)``
(pkg/src/drivesim/engine.py:591).  These dataclasses mirror the reference's
field names (pkg/src/drivesim/scenario.py:60-121) so that objects produced by
the reference's own ``preprocess``/``load_prepared`` are accepted unchanged
(duck typing); they exist here only so the package runs where the reference is
not installed.

Scenario ingestion (JSON parsing, validation, polyline decimation) is out of
scope for the B200 build: ``preprocess`` here supports only
``decimation_threshold == 0`` (the setting every benchmark scene uses).
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


def preprocess(s: Scenario, decimation_threshold: float = 0.0,
               controllable_threshold: float = 2.0) -> PreparedScenario:
    if decimation_threshold > 0.0:
        raise NotImplementedError(
            "polyline decimation is offline preprocessing (out of scope); "
            "prepare scenarios with the reference's preprocess() and pass them in")
    n_pts = sum(len(r.geometry) for r in s.roads)
    roads = [RoadElement(id=r.id, kind=r.kind, geometry=list(r.geometry))
             for r in s.roads]
    ctrl = mark_controllable(s, controllable_threshold)
    return PreparedScenario(base=s, decimated_roads=roads, controllable=ctrl,
                            stats=PrepStats(len(s.objects), sum(ctrl), n_pts, n_pts))


def load_prepared(json_text: str) -> PreparedScenario:
    """Minimal reader of the reference's prepared-scenario JSON
    (scenario.py:418-454: scenario fields plus a "prepared" section); plain
    scenario files are preprocessed with decimation 0.  No schema validation
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
        return preprocess(base)
    dec = [RoadElement(id=int(r["id"]), kind=r["type"],
                       geometry=[Vec2(float(x), float(y)) for x, y in r["geometry"]])
           for r in prep["roads"]]
    st = prep["stats"]
    return PreparedScenario(base=base, decimated_roads=dec,
                            controllable=[bool(b) for b in prep["controllable"]],
                            stats=PrepStats(int(st["n_objects"]), int(st["n_controllable"]),
                                            int(st["n_road_points_before"]),
                                            int(st["n_road_points_after"])))
