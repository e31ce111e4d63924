"""ctypes driver of the C oracle (drivesim_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs use this module, as the checker / CPU baseline.  It
builds its OWN World.__init__ tables from the raw scene (oracle/tables.py:
numpy + the standard library, no product code, no CUDA library) and keeps
its own FP64 state.  Observations are float64 (the reference's dtype).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .tables import build_tables

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "drivesim_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

_p = C.c_void_p

OR_TABLE_PTRS = ["a_off", "c_off", "r_off", "p_off", "s_off", "num_steps", "dt", "kind",
                 "length", "width", "half_l", "half_w", "circumradius", "goal_x", "goal_y",
                 "sflags", "ctrl_row", "row_agent", "rep_x", "rep_y", "rep_h", "rep_v",
                 "rep_valid", "rep_present", "pt_x", "pt_y", "pt_h", "pt_kind", "seg_ax",
                 "seg_ay", "seg_bx", "seg_by", "seg_kind"]


class OrTables(C.Structure):
    _fields_ = ([("n_worlds", C.c_int32), ("n_agents", C.c_int32), ("n_rows", C.c_int32),
                 ("reserved", C.c_int32)] + [(n, _p) for n in OR_TABLE_PTRS])


class OrConfig(C.Structure):
    _fields_ = [("dynamics", C.c_int32), ("collision_behavior", C.c_int32),
                ("obs_mode", C.c_int32), ("n_rays", C.c_int32),
                ("max_agents_obs", C.c_int32), ("max_road_points_obs", C.c_int32),
                ("obs_width", C.c_int32), ("reserved", C.c_int32),
                ("radius", C.c_double), ("fov", C.c_double), ("max_range", C.c_double),
                ("goal_tolerance", C.c_double), ("accel_lo", C.c_double),
                ("accel_hi", C.c_double), ("steer_lo", C.c_double), ("steer_hi", C.c_double),
                ("v_max", C.c_double), ("delta_lo", C.c_double * 3), ("delta_hi", C.c_double * 3)]


class OrState(C.Structure):
    _fields_ = [(n, _p) for n in ("x", "y", "heading", "speed", "head_angle", "flags", "t",
                                  "episode_over")]


def build(force: bool = False) -> str:
    """gcc the restatement into oracle/liboracle.so (no FMA contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-fopenmp", "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.or_step.argtypes = [C.POINTER(OrTables), C.POINTER(OrConfig), C.POINTER(OrState), _p,
                              C.c_int, _p, _p, _p, _p, _p, _p, C.c_int, C.c_int]
        L.or_reset.argtypes = [C.POINTER(OrTables), C.POINTER(OrConfig), C.POINTER(OrState), _p,
                               _p, _p, _p, _p]
        L.or_observe.argtypes = [C.POINTER(OrTables), C.POINTER(OrConfig), C.POINTER(OrState),
                                 _p, _p]
        for n in ("or_step", "or_reset", "or_observe"):
            getattr(L, n).restype = C.c_int
        L.or_lidar_ties.argtypes = [C.c_int]
        L.or_lidar_ties.restype = C.c_longlong
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(_p) if a is not None else None


# the C-ABI enums (include/drivesim_b200.h), restated
DYN = {"classic": 0, "invertible": 1, "delta_local": 2}
COLL = {"ignore": 0, "remove_agent": 1, "end_episode": 2}
OBS = {"radial": 0, "lidar": 1, "view_cone": 2}


def obs_width(o) -> int:
    """observation.py:84-99: ego 7 + partner slots x 7 + road slots x 11, or ego + rays x 5."""
    if o.mode == "radial":
        return 7 + 7 * o.max_agents_obs + 11 * o.max_road_points_obs
    return 7 + 5 * o.n_rays


class OracleBatch:
    """CPU restatement of SimBatch (float64 everything) over a raw scene batch
    (anything with the RawWorlds attributes)."""

    def __init__(self, raw, cfg, n_threads: int = 0):
        if not hasattr(raw, "log_x"):
            raise TypeError("OracleBatch takes the raw scene batch (it builds its own tables)")
        self.pw = build_tables(raw, cfg)
        self.cfg = cfg
        self.n_threads = n_threads
        pw = self.pw
        self._arrays = {}
        tab = OrTables()
        tab.n_worlds, tab.n_agents, tab.n_rows = pw.n_worlds, pw.n_agents, pw.n_controlled
        for name in OR_TABLE_PTRS:
            arr = np.ascontiguousarray(getattr(pw, name))
            if arr.size == 0:
                arr = np.zeros(1, arr.dtype)
            self._arrays[name] = arr
            setattr(tab, name, arr.ctypes.data)
        self.tab = tab
        c = OrConfig()
        o = cfg.obs
        c.dynamics = DYN[cfg.dynamics]
        c.collision_behavior = COLL[cfg.collision_behavior]
        c.obs_mode = OBS[o.mode]
        c.n_rays, c.max_agents_obs, c.max_road_points_obs = o.n_rays, o.max_agents_obs, \
            o.max_road_points_obs
        c.obs_width = obs_width(o)
        c.radius, c.fov, c.max_range, c.goal_tolerance = o.radius, o.fov, o.max_range, \
            cfg.goal_tolerance
        c.accel_lo, c.accel_hi = cfg.accel_bounds
        c.steer_lo, c.steer_hi = cfg.steer_bounds
        c.v_max = cfg.v_max
        for k in range(3):
            c.delta_lo[k], c.delta_hi[k] = cfg.delta_bounds[k]
        self.ocfg = c
        self.width = c.obs_width
        n, W, nc = pw.n_agents, pw.n_worlds, pw.n_controlled
        self.x = np.zeros(max(n, 1))
        self.y = np.zeros(max(n, 1))
        self.heading = np.zeros(max(n, 1))
        self.speed = np.zeros(max(n, 1))
        self.head_angle = np.zeros(max(n, 1))
        self.flags = np.zeros(max(n, 1), np.uint16)
        self.t = np.zeros(W, np.int32)
        self.episode_over = np.zeros(W, np.uint8)
        st = OrState()
        for name in ("x", "y", "heading", "speed", "head_angle", "flags", "t", "episode_over"):
            setattr(st, name, getattr(self, name).ctypes.data)
        self.st = st
        self.observations = np.zeros((nc, self.width))
        self.rewards = np.zeros(max(nc, 1))[:nc]
        self.dones = np.zeros(max(nc, 1), np.uint8)[:nc]
        self.info = np.zeros((3, max(nc, 1)), np.uint8)
        self.ep = np.zeros((W, 5), np.int32)
        self.episode_infos = []
        self.sel_w = o.max_agents_obs + o.max_road_points_obs
        self.sel_idx = np.zeros((max(nc, 1), max(self.sel_w, 1)), np.int32)
        self.reset()

    def reset(self, world_ids=None):
        mask = None
        if world_ids is not None:
            mask = np.zeros(self.pw.n_worlds, np.uint8)
            mask[list(world_ids)] = 1
        lib().or_reset(C.byref(self.tab), C.byref(self.ocfg), C.byref(self.st), _ptr(mask),
                       _ptr(self.observations), _ptr(self.rewards), _ptr(self.dones),
                       _ptr(self.sel_idx))
        return self.observations

    def step(self, actions, auto_reset: bool = False, with_obs: bool = True):
        act = None
        dim = 0
        if actions is not None:
            act = np.ascontiguousarray(actions, dtype=np.float64)
            if act.shape[0] != self.pw.n_controlled:
                raise ValueError("action row count mismatch")
            dim = act.shape[1]
        lib().or_step(C.byref(self.tab), C.byref(self.ocfg), C.byref(self.st), _ptr(act), dim,
                      _ptr(self.observations) if with_obs else None, _ptr(self.rewards),
                      _ptr(self.dones), _ptr(self.info), _ptr(self.sel_idx) if with_obs else None,
                      _ptr(self.ep), 1 if auto_reset else 0, self.n_threads)
        for w in np.nonzero(self.ep[:, 0])[0]:
            self.episode_infos.append((int(w),) + tuple(int(v) for v in self.ep[w, 1:]))
        return self.observations, self.rewards, self.dones.astype(bool), {
            "goal": self.info[0, :self.pw.n_controlled].astype(bool),
            "veh_collision": self.info[1, :self.pw.n_controlled].astype(bool),
            "offroad": self.info[2, :self.pw.n_controlled].astype(bool)}

    @staticmethod
    def lidar_ties(reset: bool = True) -> int:
        """Exact-distance ties between a road edge and another road kind on a
        ray's nearest segment (the only LiDAR case whose reference answer
        depends on its BVH traversal order, observation.py:261-271) seen by
        this process since the last reset."""
        return int(lib().or_lidar_ties(1 if reset else 0))

    def observe(self):
        lib().or_observe(C.byref(self.tab), C.byref(self.ocfg), C.byref(self.st),
                         _ptr(self.observations), _ptr(self.sel_idx))
        return self.observations
