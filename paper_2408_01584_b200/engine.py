"""Batched multi-world simulation on one B200: the drop-in for the reference's
``SimBatch`` (pkg/src/drivesim/engine.py:582-677).

Every world's state lives in HBM as structure-of-arrays FP64 (packing.py);
``step`` enqueues two kernels on the caller's CUDA stream (the fused world step
and the observation kernel, csrc/) through the C ABI and returns the SAME torch
buffers every call, exactly like the reference returns its reused numpy
buffers (engine.py:648-649).  There is no host synchronisation inside
``step``/``reset``; the only synchronising calls are the explicit readbacks
(``episode_infos``, ``episode_over_host``, ``worlds``).

Documented deviations from the reference surface:
  * observations / rewards are float32 tensors on the device (the reference
    emits float64 numpy); dones / info are torch.bool;
  * actions are consumed as float32 (the oracle sees the same values upcast);
  * ``n_workers`` is accepted and ignored (the GPU replaces the fork pool; one
    process per GPU owns a world shard, see ``parallel.py``).
"""

from __future__ import annotations

import os

import ctypes as C
import math
import time
import warnings
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .config import ObsConfig, SimConfig, obs_width
from .device_layout import DeviceLayout, build_layout
from .packing import PackedWorlds, RawWorlds, pack, raw_from_prepared


class ActionCountMismatch(ValueError):
    pass


class NoControllableAgents(UserWarning):
    pass


@dataclass
class EpisodeInfo:
    scenario: str
    world_id: int
    n_controlled: int
    n_goal: int
    n_veh_collision: int
    n_offroad: int


@dataclass
class Metrics:
    goal_rate: float
    veh_collision_rate: float
    offroad_rate: float
    episodes: int


@dataclass
class StepOutput:
    observations: torch.Tensor  # (n_controlled_total, obs_width) f32, device
    rewards: torch.Tensor       # (n_controlled_total,) f32
    dones: torch.Tensor         # (n_controlled_total,) bool
    info: dict                  # goal / veh_collision / offroad bool tensors


@dataclass
class ThroughputReport:
    worlds: int
    steps: int
    elapsed_s: float
    total_agents: int
    controlled_agents: int
    asps: float = 0.0
    casps: float = 0.0

    def __post_init__(self):
        # engine.py:146-148
        self.asps = self.steps * self.total_agents / self.elapsed_s
        self.casps = self.steps * self.controlled_agents / self.elapsed_s


def compute_metrics(episode_infos: list) -> Metrics:
    """engine.py:151-163."""
    if not episode_infos:
        raise ValueError("no completed episodes")
    total = sum(e.n_controlled for e in episode_infos)
    if total == 0:
        return Metrics(0.0, 0.0, 0.0, len(episode_infos))
    return Metrics(goal_rate=sum(e.n_goal for e in episode_infos) / total,
                   veh_collision_rate=sum(e.n_veh_collision for e in episode_infos) / total,
                   offroad_rate=sum(e.n_offroad for e in episode_infos) / total,
                   episodes=len(episode_infos))


METRICS_CSV_HEADER = "scenario,episode,controlled,goal_rate,veh_collision_rate,offroad_rate"
BENCH_CSV_HEADER = "worlds,steps,total_agents,controlled_agents,elapsed_s,asps,casps"


def metrics_csv_row(e: EpisodeInfo, episode: int) -> str:
    n = max(e.n_controlled, 1)
    return (f"{e.scenario},{episode},{e.n_controlled},"
            f"{e.n_goal / n},{e.n_veh_collision / n},{e.n_offroad / n}")


def bench_csv_row(r: ThroughputReport) -> str:
    return (f"{r.worlds},{r.steps},{r.total_agents},{r.controlled_agents},"
            f"{r.elapsed_s},{r.asps},{r.casps}")


def make_native_config(cfg: SimConfig, grid_cell: float) -> N.DsConfig:
    o = cfg.obs
    c = N.DsConfig()
    c.dynamics = N.DYN[cfg.dynamics]
    c.collision_behavior = N.COLL[cfg.collision_behavior]
    c.obs_mode = N.OBS[o.mode]
    c.n_rays = o.n_rays
    c.max_agents_obs = o.max_agents_obs
    c.max_road_points_obs = o.max_road_points_obs
    c.obs_width = obs_width(o)
    c.radius, c.fov, c.max_range = o.radius, o.fov, o.max_range
    c.goal_tolerance = cfg.goal_tolerance
    c.accel_lo, c.accel_hi = cfg.accel_bounds
    c.steer_lo, c.steer_hi = cfg.steer_bounds
    c.v_max = cfg.v_max
    for k in range(3):
        c.delta_lo[k], c.delta_hi[k] = cfg.delta_bounds[k]
    c.grid_cell = grid_cell
    return c


def default_grid_cell(obs: ObsConfig) -> float:
    """Cell edge of the static road grid (5 m: measured best of 4-8 m at C3 --
    1.38 ms radial observation at 5 m vs 1.40 at 8 m; a radial query disc
    must span at most 32 cell rows, one per lane)."""
    dev = os.environ.get("DS_GRID_CELL")   # dev override (A/B timing of cell sizes)
    if dev:
        return float(dev)
    if obs.mode == "radial":
        return max(5.0, (2.0 * obs.radius + 2.0) / 30.0)
    return 10.0


class AgentIndex(Sequence):
    """SimBatch.agent_index (engine.py:609): the (world, agent) pair of every
    controlled row, in row order -- a lazy, read-only sequence over the packed
    row table (equal to the reference's list of tuples, without building
    n_rows Python tuples for 4096-world batches)."""

    def __init__(self, pw):
        self._world = np.repeat(np.arange(pw.n_worlds, dtype=np.int64), np.diff(pw.c_off))
        self._agent = pw.row_agent.astype(np.int64) - pw.a_off[self._world]

    def __len__(self) -> int:
        return len(self._world)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        return (int(self._world[i]), int(self._agent[i]))

    def __eq__(self, other):
        return list(self) == list(other)

    def __repr__(self) -> str:
        return f"AgentIndex({len(self)} rows)"


class _WorldView:
    """Read-only snapshot view of one world (the attributes tests read from
    reference World objects: t, controlled_ids, replay tables, dt ...)."""

    def __init__(self, batch: "SimBatch", w: int):
        self._b = batch
        self.world_id = w
        pw = batch.packed
        self.name = pw.names[w]
        self.dt = float(pw.dt[w])
        self.num_steps = int(pw.num_steps[w])
        self.n_agents = int(pw.a_off[w + 1] - pw.a_off[w])
        self.controlled_ids = pw.controlled_ids(w)
        self.n_controlled = len(self.controlled_ids)
        self.n_instantiated = int(pw.n_instantiated[w])
        A, T, r0 = self.n_agents, self.num_steps, int(pw.r_off[w])
        sl = slice(r0, r0 + A * T)
        self.replay_pos = np.stack([pw.rep_x[sl].reshape(T, A).T, pw.rep_y[sl].reshape(T, A).T], -1)
        self.replay_heading = pw.rep_h[sl].reshape(T, A).T
        self.replay_speed = pw.rep_v[sl].reshape(T, A).T

    def _agents(self, arr: torch.Tensor) -> np.ndarray:
        pw = self._b.packed
        return arr[int(pw.a_off[self.world_id]):int(pw.a_off[self.world_id + 1])].cpu().numpy()

    @property
    def t(self) -> int:
        return int(self._b._t[self.world_id].item())

    @property
    def episode_over(self) -> bool:
        return bool(self._b._over[self.world_id].item())

    @property
    def pos(self) -> np.ndarray:
        return np.stack([self._agents(self._b._x), self._agents(self._b._y)], -1)

    @property
    def heading(self) -> np.ndarray:
        return self._agents(self._b._h)

    @property
    def speed(self) -> np.ndarray:
        return self._agents(self._b._v)

    @property
    def head_angle(self) -> np.ndarray:
        return self._agents(self._b._head)

    def _flag(self, bit) -> np.ndarray:
        return (self._agents(self._b._flags).astype(np.int64) & bit) != 0

    present = property(lambda s: s._flag(N.F_PRESENT))
    removed = property(lambda s: s._flag(N.F_REMOVED))
    done = property(lambda s: s._flag(N.F_DONE))
    collided_now = property(lambda s: s._flag(N.F_COLLIDED))
    offroad_now = property(lambda s: s._flag(N.F_OFFROAD))
    goal_reached = property(lambda s: s._flag(N.F_GOAL_REACHED))


def _dev(a: np.ndarray, device, dtype=None) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if a.size == 0:   # keep a valid, non-null pointer for empty tables
        a = np.zeros(1, a.dtype)
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device)


class SimBatch:
    """W independent worlds stepped in lockstep on one CUDA device.

    ``SimBatch(scenarios, cfg)`` takes prepared scenarios (ours or the
    reference's objects); ``SimBatch.from_raw(raw, cfg)`` takes a vectorised
    ``RawWorlds`` batch (the synthetic generator's output) without building
    per-object Python lists.
    """

    RING_STEPS = 64   # episode-ring capacity in steps of n_worlds records

    def __init__(self, scenarios: list, cfg: SimConfig, n_workers: int = 1,
                 device=None, grid_cell: float | None = None, _raw: RawWorlds | None = None,
                 _packed: PackedWorlds | None = None):
        if _raw is None and _packed is None:
            if not scenarios:
                raise ValueError("need at least one scenario")
            _raw = raw_from_prepared(scenarios)
        self.cfg = cfg
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.type != "cuda":
            raise ValueError("the B200 SimBatch runs on a CUDA device only (no CPU fallback)")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.packed: PackedWorlds = _packed if _packed is not None else pack(_raw, cfg)
        pw = self.packed
        self.n_worlds = pw.n_worlds
        self.offsets = pw.c_off.copy()
        self.n_controlled = pw.n_controlled
        self.total_agents = int(pw.n_instantiated.sum())
        self.width = obs_width(cfg.obs)
        for w in np.nonzero(np.diff(pw.c_off) == 0)[0]:
            warnings.warn(f"world {w} ({pw.names[w]}): no controllable agents, replay-only",
                          NoControllableAgents)
        self.agent_index = AgentIndex(pw)
        self.grid_cell = grid_cell or default_grid_cell(cfg.obs)
        if cfg.obs.mode == "radial":
            self.grid_cell = max(self.grid_cell, (2.0 * cfg.obs.radius + 2.0) / 30.0)
        self.layout: DeviceLayout = build_layout(pw, self.grid_cell,
                                                  all_segments=cfg.obs.mode != "radial")
        self._upload()
        self._episode_infos: list = []
        # the batch keeps every finished episode (SimBatch.episode_infos,
        # engine.py:614, 647); VecDriveEnv turns this off and hands each
        # step's records out instead (the reference env clears the list every
        # step, env.py:103-104), so a long rollout does not grow host memory
        self.log_episodes = True
        self._by_serial: dict = {}
        self._serial = 0
        self._steps_since_drain = 0
        self._handle = C.c_void_p()
        N.check(N.lib().ds_create(C.byref(self._tables), C.byref(self._cfg_native),
                                  C.byref(self._state), self.device.index,
                                  C.byref(self._handle)), "ds_create")
        self._closed = False
        self.reset()

    @classmethod
    def from_raw(cls, raw: RawWorlds, cfg: SimConfig, device=None,
                 grid_cell: float | None = None) -> "SimBatch":
        return cls([], cfg, device=device, grid_cell=grid_cell, _raw=raw)

    @classmethod
    def from_packed(cls, packed: PackedWorlds, cfg: SimConfig, device=None,
                    grid_cell: float | None = None) -> "SimBatch":
        """A batch over already packed World tables (worldfile.load_packed)."""
        return cls([], cfg, device=device, grid_cell=grid_cell, _packed=packed)

    @classmethod
    def from_file(cls, path: str, cfg: SimConfig, device=None,
                  grid_cell: float | None = None) -> "SimBatch":
        """A batch over a binary world file (worldfile.py): raw scenes are
        packed, packed tables are used as they are."""
        from . import worldfile
        with open(path, "rb") as f:
            hlen = worldfile._PREFIX.unpack(f.read(worldfile._PREFIX.size))[2]
            kind = __import__("json").loads(f.read(hlen))["kind"]
        if kind == "packed":
            return cls.from_packed(worldfile.load_packed(path, cfg), cfg, device, grid_cell)
        return cls.from_raw(worldfile.load_raw(path), cfg, device, grid_cell)

    # -- construction ------------------------------------------------------

    def _upload(self):
        pw, lay, dev = self.packed, self.layout, self.device
        A = np.diff(pw.a_off)
        self.max_agents = int(A.max()) if len(A) else 0
        t = {}
        t["a_off"] = _dev(pw.a_off, dev)
        t["c_off"] = _dev(pw.c_off, dev)
        t["r_off"] = _dev(pw.r_off, dev)
        t["num_steps"] = _dev(pw.num_steps.astype(np.int32), dev)
        t["dt"] = _dev(pw.dt, dev)
        for name in ("kind", "length", "width", "half_l", "half_w", "circumradius", "goal_x",
                     "goal_y", "sflags", "ctrl_row", "row_agent", "rep_x", "rep_y", "rep_h",
                     "rep_v", "rep_valid", "rep_present"):
            t[name] = _dev(getattr(pw, name), dev)
        for name in ("grid_x0", "grid_y0", "grid_nx", "grid_ny", "grid_cell_off",
                     "pt_cell_start", "gpt_x", "gpt_y", "gpt_h", "gpt_kind", "gpt_id",
                     "eseg_cell_start", "eseg_ax", "eseg_ay", "eseg_bx", "eseg_by",
                     "aseg_cell_start", "aseg_ax", "aseg_ay", "aseg_bx", "aseg_by", "aseg_id",
                     "aseg_edge", "gpt_xy", "grid_eps", "eseg_rel"):
            t[name] = _dev(getattr(lay, name), dev)
        # 32-B point records (ds_point_rec) for the observation slot gather
        rec = np.zeros(max(len(lay.gpt_x), 1), dtype=np.dtype(
            [("x", "<f8"), ("y", "<f8"), ("h", "<f8"), ("id", "<i4"), ("kind", "i1"),
             ("pad", "i1", (3,))]))
        if len(lay.gpt_x):
            rec["x"], rec["y"], rec["h"] = lay.gpt_x, lay.gpt_y, lay.gpt_h
            rec["id"], rec["kind"] = lay.gpt_id, lay.gpt_kind
        t["gpt_rec"] = torch.from_numpy(rec.view(np.uint8)).to(dev)
        # 32-B per-agent statics and FP64 edge-segment records (step kernel)
        t["agent_rec"] = _dev(np.stack([pw.half_l, pw.half_w, pw.goal_x, pw.goal_y], 1)
                              .astype(np.float64).reshape(-1), dev)
        t["eseg_rec"] = _dev(np.stack([lay.eseg_ax, lay.eseg_ay, lay.eseg_bx, lay.eseg_by], 1)
                             .astype(np.float64).reshape(-1), dev)
        # 32-B FP64 records of all binned segments (LiDAR / view-cone fetch)
        t["aseg_rec"] = _dev(np.stack([lay.aseg_ax, lay.aseg_ay, lay.aseg_bx, lay.aseg_by], 1)
                             .astype(np.float64).reshape(-1), dev)
        t["p_off"] = _dev(pw.p_off, dev)
        t["s_off"] = _dev(pw.s_off, dev)
        self._t_tensors = t
        tab = N.DsTables()
        tab.n_worlds = pw.n_worlds
        tab.n_agents = pw.n_agents
        tab.n_rows = pw.n_controlled
        tab.max_agents = self.max_agents
        P = np.diff(pw.p_off)
        tab.max_points = int(P.max()) if len(P) else 0
        for name in N.TABLE_PTRS:
            setattr(tab, name, t[name].data_ptr())
        self._tables = tab
        self._cfg_native = make_native_config(self.cfg, self.grid_cell)

        n, W, nc = pw.n_agents, pw.n_worlds, pw.n_controlled
        f64 = dict(dtype=torch.float64, device=dev)
        self._x = torch.zeros(max(n, 1), **f64)
        self._y = torch.zeros(max(n, 1), **f64)
        self._h = torch.zeros(max(n, 1), **f64)
        self._v = torch.zeros(max(n, 1), **f64)
        self._head = torch.zeros(max(n, 1), **f64)
        self._flags = torch.zeros(max(n, 1), dtype=torch.int16, device=dev)
        self._t = torch.zeros(W, dtype=torch.int32, device=dev)
        self._over = torch.zeros(W, dtype=torch.uint8, device=dev)
        self._ring_cap = max(1024, self.RING_STEPS * W)
        self._ring = torch.zeros(self._ring_cap * 6, dtype=torch.int32, device=dev)
        self._ring_head = torch.zeros(1, dtype=torch.int32, device=dev)
        st = N.DsState()
        for name, ten in (("x", self._x), ("y", self._y), ("heading", self._h),
                          ("speed", self._v), ("head_angle", self._head),
                          ("flags", self._flags), ("t", self._t), ("episode_over", self._over),
                          ("ring", self._ring), ("ring_head", self._ring_head)):
            setattr(st, name, ten.data_ptr())
        st.ring_cap = self._ring_cap
        self._hint = torch.zeros((max(n, 1), 4), dtype=torch.float32, device=dev)
        st.obs_hint = self._hint.data_ptr()
        self._status = torch.zeros(1, dtype=torch.int32, device=dev)
        st.status = self._status.data_ptr()
        self._state = st

        # Outputs (reused every call, like the reference's buffers).
        self.observations = torch.zeros((max(nc, 1), self.width), dtype=torch.float32,
                                        device=dev)[:nc]
        self.rewards = torch.zeros(max(nc, 1), dtype=torch.float32, device=dev)[:nc]
        self.dones = torch.zeros(max(nc, 1), dtype=torch.bool, device=dev)[:nc]
        self._info = torch.zeros((3, max(nc, 1)), dtype=torch.bool, device=dev)
        self.info = {k: self._info[i, :nc] for i, k in
                     enumerate(("goal", "veh_collision", "offroad"))}
        self._mask = torch.zeros(W, dtype=torch.uint8, device=dev)

    # -- stepping ----------------------------------------------------------

    def _arg(self, t, dtype, numel: int, name: str, convert: bool = False):
        """A kernel argument tensor checked before its raw pointer is taken:
        on this batch's device, of ``dtype`` (converted when ``convert`` and
        the conversion is exact), contiguous, at least ``numel`` elements.
        Returns the (possibly converted) tensor; the caller keeps it alive."""
        if not torch.is_tensor(t):
            raise TypeError(f"{name}: expected a torch tensor")
        if t.device != self.device:
            raise ValueError(f"{name}: on {t.device}, the batch is on {self.device}")
        if t.dtype != dtype:
            if not convert:
                raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
            t = t.to(dtype)
        if not t.is_contiguous():
            if not convert:
                raise ValueError(f"{name}: must be contiguous")
            t = t.contiguous()
        if t.numel() < numel:
            raise ValueError(f"{name}: {t.numel()} elements, needs {numel}")
        return t

    def _sel_w(self) -> int:
        return self.cfg.obs.max_agents_obs + self.cfg.obs.max_road_points_obs

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _maybe_drain(self):
        if (self._steps_since_drain + 1) * self.n_worlds > self._ring_cap:
            self._drain()

    def step(self, actions, *, sel_idx: torch.Tensor | None = None,
             obs_scale: torch.Tensor | None = None, auto_reset: bool = False,
             action_idx: torch.Tensor | None = None, grid=None, events=None) -> StepOutput:
        """One step of every world; ``actions`` has one row per controlled
        agent (flat over worlds) or is None for expert replay everywhere."""
        self._check_open()
        a = N.DsStepArgs()
        keep = []
        if action_idx is not None:
            idx = torch.as_tensor(action_idx, device=self.device).to(torch.int32).contiguous()
            if idx.shape[0] != self.n_controlled:
                raise ActionCountMismatch(
                    f"expected {self.n_controlled} action rows, got {idx.shape[0]}")
            accel, steer = grid
            accel = self._arg(accel, torch.float64, 1, "grid accel", convert=True)
            steer = self._arg(steer, torch.float64, 1, "grid steer", convert=True)
            keep += [accel, steer]
            a.action_idx = idx.data_ptr()
            a.grid_accel = accel.data_ptr()
            a.grid_steer = steer.data_ptr()
            a.n_accel = accel.numel()
            a.n_steer = steer.numel()
            keep += [idx]
        elif actions is None:
            a.replay = 1
        else:
            act = torch.as_tensor(actions)
            if act.ndim != 2 or act.shape[0] != self.n_controlled:
                n_got = act.shape[0] if act.ndim else 0
                raise ActionCountMismatch(
                    f"expected {self.n_controlled} action rows, got {n_got}")
            act = act.to(device=self.device, dtype=torch.float32).contiguous()
            a.actions = act.data_ptr()
            a.act_dim = act.shape[1]
            keep.append(act)
        if obs_scale is not None:
            obs_scale = self._arg(obs_scale, torch.float32, self.width, "obs_scale", convert=True)
            keep.append(obs_scale)
        if sel_idx is not None:
            sel_idx = self._arg(sel_idx, torch.int32, self.n_controlled * self._sel_w(), "sel_idx")
        self._maybe_drain()
        a.obs = self.observations.data_ptr()
        a.rewards = self.rewards.data_ptr()
        a.dones = self.dones.data_ptr()
        a.info = self._info.data_ptr()
        a.obs_scale = obs_scale.data_ptr() if obs_scale is not None else None
        a.auto_reset = 1 if auto_reset else 0
        a.serial = self._serial
        a.sel_idx = sel_idx.data_ptr() if sel_idx is not None else None
        if events is not None:   # (start, after the world step, after obs): torch.cuda.Event or None
            for k, ev in enumerate(events):
                if ev is not None:
                    a.events[k] = ev.cuda_event
        N.check(N.lib().ds_step(self._handle, C.byref(a), self._stream()), "ds_step")
        self._serial += 1
        self._steps_since_drain += 1
        return StepOutput(self.observations, self.rewards, self.dones, self.info)

    def reset(self, world_ids=None, *, obs_scale: torch.Tensor | None = None,
              sel_idx: torch.Tensor | None = None, world_mask: torch.Tensor | None = None):
        """engine.py:651-663: reset the given worlds (all by default) and
        recompute their observation rows; their rewards/dones rows read 0."""
        self._check_open()
        mask_ptr = None
        if obs_scale is not None:
            obs_scale = self._arg(obs_scale, torch.float32, self.width, "obs_scale", convert=True)
        if sel_idx is not None:
            sel_idx = self._arg(sel_idx, torch.int32, self.n_controlled * self._sel_w(), "sel_idx")
        if world_mask is not None:
            world_mask = self._arg(world_mask, torch.uint8, self.n_worlds, "world_mask",
                                   convert=True)
            mask_ptr = world_mask.data_ptr()
        elif world_ids is not None:
            ids = torch.as_tensor(list(world_ids) if not torch.is_tensor(world_ids) else world_ids,
                                  dtype=torch.int64)
            self._mask.zero_()
            if ids.numel():
                self._mask[ids.to(self.device)] = 1
            mask_ptr = self._mask.data_ptr()
        N.check(N.lib().ds_reset(self._handle, mask_ptr, self.observations.data_ptr(),
                                 self.rewards.data_ptr(), self.dones.data_ptr(),
                                 obs_scale.data_ptr() if obs_scale is not None else None,
                                 sel_idx.data_ptr() if sel_idx is not None else None,
                                 self._stream()), "ds_reset")
        return self.observations

    def set_obs_format(self, dtype=torch.float32, row_stride: int | None = None):
        """Observation buffer format of every later step/reset/observe:
        float32 (default) or bfloat16, rows padded to ``row_stride`` elements
        (pad columns read 0).  ``observations`` stays the [n, width] view of
        the padded buffer; a bf16 buffer padded to a multiple of 8 feeds a
        policy GEMM directly (ds_set_obs_format)."""
        self._check_open()
        code = {torch.float32: N.OBS_F32, torch.bfloat16: N.OBS_BF16}.get(dtype)
        if code is None:
            raise ValueError(f"unsupported observation dtype {dtype}")
        stride = self.width if row_stride is None else int(row_stride)
        N.check(N.lib().ds_set_obs_format(self._handle, code, stride), "ds_set_obs_format")
        nc = self.n_controlled
        self._obs_buf = torch.zeros((max(nc, 1), stride), dtype=dtype, device=self.device)
        self.observations = self._obs_buf[:nc, :self.width]
        return self.observations

    def observe(self, obs_scale=None, sel_idx=None):
        self._check_open()
        if obs_scale is not None:
            obs_scale = self._arg(obs_scale, torch.float32, self.width, "obs_scale", convert=True)
        if sel_idx is not None:
            sel_idx = self._arg(sel_idx, torch.int32, self.n_controlled * self._sel_w(), "sel_idx")
        N.check(N.lib().ds_observe(self._handle, None, self.observations.data_ptr(),
                                   obs_scale.data_ptr() if obs_scale is not None else None,
                                   sel_idx.data_ptr() if sel_idx is not None else None,
                                   self._stream()), "ds_observe")
        return self.observations

    # -- episode records ---------------------------------------------------

    def _drain(self):
        buf = np.zeros((self._ring_cap, 6), np.int32)
        n = C.c_int32(0)
        rc = N.lib().ds_episode_drain(self._handle, buf.ctypes.data_as(C.c_void_p),
                                      self._ring_cap, C.byref(n), self._stream())
        self._steps_since_drain = 0
        recs = buf[:n.value]
        if len(recs):
            recs = recs[np.lexsort((recs[:, 1], recs[:, 0]))]
            names = self.packed.names
            for serial, w, nc, ng, nv, no in recs.tolist():
                e = EpisodeInfo(names[w], w, nc, ng, nv, no)
                if self.log_episodes:
                    self._episode_infos.append(e)
                self._by_serial.setdefault(serial, []).append(e)
        # keep per-step lists only for the recent window (lazy env readers)
        old = [k for k in self._by_serial if k < self._serial - 4 * self.RING_STEPS]
        for k in old:
            del self._by_serial[k]
        N.check(rc, "ds_episode_drain")
        self.check_status()

    def check_status(self):
        """Raise the errors the kernels flagged since the last check (a host
        synchronisation): IndexError for a joint action index outside the
        action grid, as the reference's to_continuous (env.py:111-116)."""
        st = C.c_uint32(0)
        N.check(N.lib().ds_status(self._handle, C.byref(st), 1, self._stream()), "ds_status")
        if st.value & N.STATUS_BAD_ACTION_INDEX:
            raise IndexError("a joint action index was outside the action grid "
                             "(those agents were not advanced)")

    def episodes_of_step(self, serial: int) -> list:
        """Episode records finished during step ``serial`` (synchronises)."""
        self._drain()
        return self._by_serial.pop(serial, [])

    @property
    def episode_infos(self) -> list:
        """Finished-episode records in (step, world) order (synchronises)."""
        self._drain()
        return self._episode_infos

    @property
    def episode_over(self) -> torch.Tensor:
        return self._over.bool()

    def compute_metrics(self) -> Metrics:
        return compute_metrics(self.episode_infos)

    @property
    def worlds(self) -> list:
        return [_WorldView(self, w) for w in range(self.n_worlds)]

    def _slice(self, w: int) -> slice:
        return slice(int(self.offsets[w]), int(self.offsets[w + 1]))

    # -- lifecycle ---------------------------------------------------------

    def _check_open(self):
        if self._closed:
            raise RuntimeError("SimBatch is closed")

    def close(self):
        if not getattr(self, "_closed", True):
            torch.cuda.synchronize(self.device)
            N.lib().ds_destroy(self._handle)
            self._closed = True

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_batch(scenarios: list, cfg: SimConfig, n_workers: int = 1, device=None) -> SimBatch:
    """engine.py:788."""
    return SimBatch(scenarios, cfg, n_workers=n_workers, device=device)


def random_actions(n_rows: int, cfg: SimConfig, seed: int, t: int, device) -> torch.Tensor:
    """Counter-based uniform actions over the config bounds:
    a pure function of (seed, row, t), so shard-invariant."""
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + int(t)) & 0x7FFFFFFFFFFFFFFF)
    cols = cfg.action_dim
    u = torch.rand((n_rows, cols), generator=g, device=device, dtype=torch.float32)
    if cfg.dynamics == "delta_local":
        lo = torch.tensor([b[0] for b in cfg.delta_bounds], device=device, dtype=torch.float32)
        hi = torch.tensor([b[1] for b in cfg.delta_bounds], device=device, dtype=torch.float32)
    else:
        lo = torch.tensor([cfg.accel_bounds[0], cfg.steer_bounds[0]], device=device,
                          dtype=torch.float32)
        hi = torch.tensor([cfg.accel_bounds[1], cfg.steer_bounds[1]], device=device,
                          dtype=torch.float32)
    return lo + (hi - lo) * u


def goal_seek_actions(batch: "SimBatch", out: torch.Tensor | None = None) -> torch.Tensor:
    """goal_seek_actions (engine.py:559-574) for every controlled row of
    ``batch`` from its current device state: float32 [n_controlled, 2]
    (accel, steer) on the device, one ds_goal_seek launch, no host sync."""
    batch._check_open()
    n = batch.n_controlled
    if out is None:
        out = torch.empty((max(n, 1), 2), dtype=torch.float32, device=batch.device)[:n]
    if out.shape != (n, 2) or out.dtype != torch.float32 or not out.is_contiguous() \
            or out.device != batch.device:
        raise ValueError("goal_seek_actions: out must be a contiguous float32 [n, 2] device tensor")
    N.check(N.lib().ds_goal_seek(batch._handle, C.c_void_p(out.data_ptr()), batch._stream()),
            "ds_goal_seek")
    return out


def make_policy(spec: str, cfg: SimConfig, batch: "SimBatch", seed: int = 0):
    """make_policy (engine.py:535-556) over a whole batch: callable(t) ->
    device actions [n_controlled, 2] (or None for replay).  Specs "random"
    (uniform over the bounds, counter-based in (seed, row, t)), "replay",
    "constant[:a:s]", "goal_seek"."""
    n, dev = batch.n_controlled, batch.device
    if spec == "replay":
        return lambda t: None
    if spec == "random":
        return lambda t: random_actions(n, cfg, seed, t, dev)
    if spec.startswith("constant"):
        parts = spec.split(":")
        a = float(parts[1]) if len(parts) > 1 else 0.0
        s = float(parts[2]) if len(parts) > 2 else 0.0
        const = torch.tensor([[a, s]], dtype=torch.float32, device=dev).repeat(n, 1)
        return lambda t: const
    if spec == "goal_seek":
        buf = torch.empty((max(n, 1), 2), dtype=torch.float32, device=dev)[:n]
        return lambda t: goal_seek_actions(batch, buf)
    raise ValueError(f"unknown policy {spec!r}")


def benchmark(scenarios: list, cfg: SimConfig, worlds: int, steps: int, policy: str = "random",
              n_workers=None, seed: int | None = None, device=None) -> ThroughputReport:
    """engine.py:811-857 on the GPU: step ``worlds`` worlds ``steps`` times
    under a trivial policy (make_policy) with observations every step and
    auto-reset; elapsed time from CUDA events (init/upload excluded)."""
    if worlds < 1 or steps < 1:
        raise ValueError("worlds and steps must be >= 1")
    seed = cfg.seed if seed is None else seed
    chosen = [scenarios[w % len(scenarios)] for w in range(worlds)]
    batch = SimBatch(chosen, cfg, device=device)
    dev = batch.device
    pol = make_policy(policy, cfg, batch, seed)
    if policy == "random":       # precomputed: the timed loop holds only the step
        acts = [pol(t) for t in range(min(steps, 8))]
        pol = lambda t: acts[t % len(acts)]   # noqa: E731
    torch.cuda.synchronize(dev)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for t in range(steps):
        batch.step(pol(t), auto_reset=True)
    end.record()
    torch.cuda.synchronize(dev)
    elapsed = start.elapsed_time(end) / 1e3
    rep = ThroughputReport(worlds=worlds, steps=steps, elapsed_s=elapsed,
                           total_agents=batch.total_agents,
                           controlled_agents=batch.n_controlled)
    batch.close()
    return rep


def sample_categorical(logits: torch.Tensor, seed: int, counter: int,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    """One categorical sample per row of ``logits`` ([rows, n], float32 or
    bfloat16, unit column stride, any row stride) by Gumbel-max with noise
    from a counter-based hash of (seed, counter, row, column): the in-loop
    sampler of the device rollout (ds_sample_categorical; the reference
    trainer samples torch.distributions.Categorical, ippo.py:136-142)."""
    if logits.ndim != 2 or logits.stride(1) != 1:
        raise ValueError("logits must be 2-D with unit column stride")
    code = {torch.float32: N.OBS_F32, torch.bfloat16: N.OBS_BF16}.get(logits.dtype)
    if code is None:
        raise ValueError(f"unsupported logits dtype {logits.dtype}")
    rows, n = logits.shape
    if out is None:
        out = torch.empty(rows, dtype=torch.int32, device=logits.device)
    stream = C.c_void_p(torch.cuda.current_stream(logits.device).cuda_stream)
    N.check(N.lib().ds_sample_categorical(C.c_void_p(logits.data_ptr()), code, rows, n,
                                          logits.stride(0), seed & (2**64 - 1),
                                          counter & (2**64 - 1), C.c_void_p(out.data_ptr()),
                                          stream), "ds_sample_categorical")
    return out


@dataclass
class HostStepResult:
    """Host copies of one step's rewards / dones / info (pinned memory,
    reused every ``depth`` steps).  ``wait()`` blocks until they landed."""
    rewards: torch.Tensor
    dones: torch.Tensor
    info: dict
    _event: object

    def wait(self) -> "HostStepResult":
        self._event.synchronize()
        return self


class HostStepper:
    """Stepping from HOST action buffers with the host<->device copies
    overlapped with the kernels (the e2e path of a CPU caller such as the
    reference's trainer loop, ippo.py:173-179, which hands the batch numpy
    actions and reads rewards / dones / info back every step).

    Step t: the actions are staged in pinned memory and copied host->device on
    a copy stream (slot t mod depth); the compute stream waits for that copy,
    runs the world-step kernel, records an event, then the observation
    kernel.  Rewards / dones / info are final once the world-step kernel is
    done, so their device->host copy (a second copy stream) runs while the
    observation kernel is still computing; the next step's world-step kernel
    waits for it before overwriting them.  No host synchronisation per step:
    ``step`` returns a HostStepResult whose ``wait()`` syncs on its copy only.
    Results are identical to ``SimBatch.step`` with the same actions."""

    def __init__(self, batch: SimBatch, act_dim: int | None = None, depth: int = 2,
                 auto_reset: bool = True, obs_scale: torch.Tensor | None = None):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.batch = batch
        dev = batch.device
        n = batch.n_controlled
        self.act_dim = batch.cfg.action_dim if act_dim is None else act_dim
        self.depth, self.auto_reset, self.obs_scale = depth, auto_reset, obs_scale
        self._h2d = torch.cuda.Stream(dev)
        self._d2h = torch.cuda.Stream(dev)
        self._act_dev = [torch.empty((n, self.act_dim), dtype=torch.float32, device=dev)
                         for _ in range(depth)]
        host = lambda shape, dt: [torch.empty(shape, dtype=dt, pin_memory=True)  # noqa: E731
                                  for _ in range(depth)]
        self._act_pin = host((n, self.act_dim), torch.float32)
        self._rew, self._done = host((n,), torch.float32), host((n,), torch.bool)
        self._info = host((3, n), torch.bool)
        main = torch.cuda.current_stream(dev)
        ev = lambda: [torch.cuda.Event() for _ in range(depth)]   # noqa: E731
        self._ev_h2d, self._ev_stepk, self._ev_d2h, self._ev_used = ev(), ev(), ev(), ev()
        for e in self._ev_h2d + self._ev_stepk + self._ev_d2h + self._ev_used:
            e.record(main)    # materialise the CUDA events (ds_step records raw handles)
        self._pending = [False] * depth
        self._t = 0

    def step(self, actions, *, zero_copy: bool = False) -> HostStepResult:
        """actions: host [n_controlled, act_dim] (numpy or CPU tensor).  They
        are staged into an internal pinned buffer, so the caller may reuse
        its own buffer as soon as step() returns.  zero_copy=True (a pinned,
        contiguous float32 tensor only) DMAs straight from the caller's
        buffer instead: the caller must then leave it untouched until this
        step's HostStepResult.wait() returned."""
        b = self.batch
        k = self._t % self.depth
        a = torch.as_tensor(actions)
        if a.device.type != "cpu":
            raise ValueError("HostStepper.step takes host actions; use SimBatch.step for "
                             "device tensors")
        if a.ndim != 2 or a.shape[0] != b.n_controlled:
            raise ActionCountMismatch(
                f"expected {b.n_controlled} action rows, got {a.shape[0] if a.ndim else 0}")
        if a.shape[1] != self.act_dim:
            raise ValueError(f"expected {self.act_dim} action columns, got {a.shape[1]}")
        if self._pending[k]:
            # slot k's previous step: its action copy and result copy are done
            # before the pinned buffers are reused (the caller has had
            # depth - 1 steps to read that result)
            self._ev_d2h[k].synchronize()
        if zero_copy and not (a.dtype == torch.float32 and a.is_contiguous() and a.is_pinned()):
            raise ValueError("zero_copy needs a pinned, contiguous float32 tensor")
        src = a if zero_copy else self._act_pin[k]
        if not zero_copy:
            src.copy_(a)
        main = torch.cuda.current_stream(b.device)
        with torch.cuda.stream(self._h2d):
            # the device slot was last read by step t - depth's kernels
            self._h2d.wait_event(self._ev_used[k])
            self._act_dev[k].copy_(src, non_blocking=True)
            self._ev_h2d[k].record(self._h2d)
        main.wait_event(self._ev_h2d[k])
        if self._t > 0:
            # the previous step's results must be read out before this step's
            # world-step kernel overwrites them
            main.wait_event(self._ev_d2h[(self._t - 1) % self.depth])
        b.step(self._act_dev[k], obs_scale=self.obs_scale, auto_reset=self.auto_reset,
               events=(None, self._ev_stepk[k], None))
        self._ev_used[k].record(main)
        with torch.cuda.stream(self._d2h):
            self._d2h.wait_event(self._ev_stepk[k])
            self._rew[k].copy_(b.rewards, non_blocking=True)
            self._done[k].copy_(b.dones, non_blocking=True)
            self._info[k].copy_(b._info[:, :b.n_controlled], non_blocking=True)
            self._ev_d2h[k].record(self._d2h)
        self._pending[k] = True
        self._t += 1
        info = {key: self._info[k][i] for i, key in enumerate(("goal", "veh_collision", "offroad"))}
        return HostStepResult(self._rew[k], self._done[k], info, self._ev_d2h[k])

    @property
    def h2d_bytes_per_step(self) -> int:
        return self.batch.n_controlled * self.act_dim * 4

    @property
    def d2h_bytes_per_step(self) -> int:
        return self.batch.n_controlled * (4 + 1 + 3)

    def synchronize(self):
        for k in range(self.depth):
            if self._pending[k]:
                self._ev_d2h[k].synchronize()
