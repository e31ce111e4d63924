"""Scripted scenes and a backend-neutral runner for the semantic tests.

The scenes restate the reference's own test scenarios
(pkg/tests/test_engine.py, test_observation.py); the runner drives either the
C oracle (CPU) or the CUDA SimBatch (GPU) through the same calls so one test
body checks both."""

from __future__ import annotations

import math

import numpy as np

from paper_2408_01584_b200 import _native as N
from paper_2408_01584_b200.config import SimConfig
from paper_2408_01584_b200.packing import pack, raw_from_prepared
from paper_2408_01584_b200.scenario import (LoggedStep, ObjectLog, RoadElement, Scenario, Vec2,
                                            preprocess)


def scripted_object(oid, poses, kind="vehicle", goal=None, length=4.0, width=2.0, speed=0.0,
                    force_replay=False, valid=None):
    """ObjectLog from (x, y, heading) poses (test_engine.py:18-32)."""
    states = []
    for t, (x, y, h) in enumerate(poses):
        ok = True if valid is None else valid[t]
        states.append(LoggedStep(position=Vec2(x, y), heading=h,
                                 velocity=Vec2(speed * math.cos(h), speed * math.sin(h)),
                                 valid=ok))
    if goal is None:
        goal = poses[-1][:2]
    return ObjectLog(id=oid, kind=kind, length=length, width=width, goal=Vec2(*goal),
                     states=states, force_replay=force_replay)


def hold(x, y, h, n):
    return [(x, y, h)] * n


def scene(objects, roads=(), num_steps=None, name="scripted"):
    num_steps = num_steps or len(objects[0].states)
    return preprocess(Scenario(name=name, num_steps=num_steps, objects=list(objects),
                               roads=list(roads)), decimation_threshold=0.0)


def obs_agents(agents, roads=(), num_steps=2):
    """test_observation.make_world: (x, y, heading, speed[, kind, L, W, goal])."""
    objects = []
    for i, spec in enumerate(agents):
        x, y, heading, speed = spec[:4]
        kind = spec[4] if len(spec) > 4 else "vehicle"
        length = spec[5] if len(spec) > 5 else 4.0
        width = spec[6] if len(spec) > 6 else 2.0
        goal = spec[7] if len(spec) > 7 else (x + 100.0, y)
        states = [LoggedStep(position=Vec2(x, y), heading=heading,
                             velocity=Vec2(speed * math.cos(heading), speed * math.sin(heading)),
                             valid=True) for _ in range(num_steps)]
        objects.append(ObjectLog(id=i, kind=kind, length=length, width=width, goal=Vec2(*goal),
                                 states=states))
    return scene(objects, roads, num_steps, name="obs-test")


class WorldView:
    def __init__(self, runner, w):
        self.r, self.w = runner, w
        pw = runner.pw
        self.a0, self.a1 = int(pw.a_off[w]), int(pw.a_off[w + 1])
        self.controlled_ids = pw.controlled_ids(w)
        self.n_controlled = len(self.controlled_ids)

    def _arr(self, name):
        return self.r._state(name)[self.a0:self.a1]

    pos = property(lambda s: np.stack([s._arr("x"), s._arr("y")], -1))
    heading = property(lambda s: s._arr("heading"))
    speed = property(lambda s: s._arr("speed"))
    head_angle = property(lambda s: s._arr("head_angle"))
    removed = property(lambda s: (s._arr("flags").astype(np.int64) & N.F_REMOVED) != 0)
    present = property(lambda s: (s._arr("flags").astype(np.int64) & N.F_PRESENT) != 0)
    done = property(lambda s: (s._arr("flags").astype(np.int64) & N.F_DONE) != 0)
    collided_now = property(lambda s: (s._arr("flags").astype(np.int64) & N.F_COLLIDED) != 0)
    offroad_now = property(lambda s: (s._arr("flags").astype(np.int64) & N.F_OFFROAD) != 0)
    t = property(lambda s: int(s.r._state("t")[s.w]))
    episode_over = property(lambda s: bool(s.r._state("episode_over")[s.w]))


class Runner:
    """Same surface over the oracle ("oracle") or the CUDA engine ("gpu")."""

    def __init__(self, prepared, cfg: SimConfig, backend: str):
        self.cfg = cfg
        self.backend = backend
        raw = raw_from_prepared(prepared)
        if backend == "gpu":
            from paper_2408_01584_b200.engine import SimBatch
            self.b = SimBatch.from_raw(raw, cfg, device="cuda:0")
            self.pw = self.b.packed
        else:
            from oracle.oracle import OracleBatch
            self.b = OracleBatch(raw, cfg)
            self.pw = self.b.pw
        self.n_controlled = self.pw.n_controlled

    def _state(self, name):
        if self.backend == "gpu":
            t = {"x": self.b._x, "y": self.b._y, "heading": self.b._h, "speed": self.b._v,
                 "head_angle": self.b._head, "flags": self.b._flags, "t": self.b._t,
                 "episode_over": self.b._over}[name]
            return t.cpu().numpy()
        return getattr(self.b, name)

    def world(self, w=0):
        return WorldView(self, w)

    def step(self, actions):
        if self.backend == "gpu":
            import torch
            act = None if actions is None else torch.as_tensor(np.asarray(actions, np.float32))
            out = self.b.step(act.cuda() if act is not None else None)
            return (out.rewards.cpu().numpy().astype(np.float64), out.dones.cpu().numpy(),
                    {k: v.cpu().numpy() for k, v in out.info.items()})
        _, rew, done, info = self.b.step(
            None if actions is None else np.asarray(actions, np.float32).astype(np.float64))
        return rew.copy(), done.copy(), info

    @property
    def obs(self):
        if self.backend == "gpu":
            return self.b.observations.cpu().numpy().astype(np.float64)
        return self.b.observations.astype(np.float32).astype(np.float64)

    def reset(self, world_ids=None):
        self.b.reset(world_ids)

    def episode_infos(self):
        if self.backend == "gpu":
            return [(e.world_id, e.n_controlled, e.n_goal, e.n_veh_collision, e.n_offroad)
                    for e in self.b.episode_infos]
        return list(self.b.episode_infos)

    def close(self):
        if self.backend == "gpu":
            self.b.close()
