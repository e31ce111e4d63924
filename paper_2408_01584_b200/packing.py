"""Scenario batch -> structure-of-arrays world tables.

``RawWorlds`` is a flat, vectorised image of a list of prepared scenarios
(logs + decimated road polylines + controllable mask).  ``pack`` restates the
reference ``World.__init__`` table construction (pkg/src/drivesim/engine.py:
173-314) over the whole batch at once and returns ``PackedWorlds``: the
host-side tables that both the CUDA step (after ``device_layout``) and the CPU
oracle consume.  Everything is in the reference's original agent / road-point /
segment order; spatial binning for the GPU lives in ``device_layout.py``.

Layout conventions (W worlds, N agents, R replay cells, P points, S segments):
  * per-world ranges are CSR offsets: agents ``a_off[W+1]``, controlled rows
    ``c_off[W+1]``, road points ``p_off[W+1]``, segments ``s_off[W+1]``;
  * replay tables are time-major inside each world: cell of (world w, local
    agent i, step t) is ``r_off[w] + t * A_w + i`` so one step of one world is
    one contiguous run (coalesced on the device);
  * controlled agents keep ``controlled_ids`` order (ascending local id), and
    row ``c_off[w] + k`` of every per-agent output belongs to the k-th one
    (engine.py:599-610).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .config import OBJECT_KINDS, ROAD_EDGE, ROAD_KINDS, SimConfig


@dataclass
class RawWorlds:
    """Flat batch of prepared scenarios (inputs of World.__init__)."""

    names: list
    dt: np.ndarray            # f64 [W]      Scenario.timestep
    num_steps: np.ndarray     # i32 [W]      Scenario.num_steps (T_w)
    a_off: np.ndarray         # i64 [W+1]
    kind: np.ndarray          # i8  [N]      index into OBJECT_KINDS
    length: np.ndarray        # f64 [N]
    width: np.ndarray         # f64 [N]
    goal: np.ndarray          # f64 [N,2]
    force_replay: np.ndarray  # bool [N]
    controllable: np.ndarray  # bool [N]     PreparedScenario.controllable
    l_off: np.ndarray         # i64 [W+1]    logs, agent-major: l_off[w] + i*T_w + t
    log_x: np.ndarray         # f64 [L]
    log_y: np.ndarray
    log_h: np.ndarray
    log_vx: np.ndarray
    log_vy: np.ndarray
    log_valid: np.ndarray     # bool [L]
    poly_off: np.ndarray      # i64 [W+1]    road polylines per world
    poly_kind: np.ndarray     # i8  [R]      index into ROAD_KINDS
    poly_pt_off: np.ndarray   # i64 [R+1]    points per polyline (global)
    pt_x: np.ndarray          # f64 [P]
    pt_y: np.ndarray

    @property
    def n_worlds(self) -> int:
        return len(self.names)

    def subset(self, world_ids) -> "RawWorlds":
        """Worlds ``world_ids`` (in that order) as a new RawWorlds."""
        ids = np.asarray(world_ids, dtype=np.int64)
        a_sl = [np.arange(self.a_off[w], self.a_off[w + 1]) for w in ids]
        l_sl = [np.arange(self.l_off[w], self.l_off[w + 1]) for w in ids]
        r_sl = [np.arange(self.poly_off[w], self.poly_off[w + 1]) for w in ids]
        a_idx = np.concatenate(a_sl) if a_sl else np.zeros(0, np.int64)
        l_idx = np.concatenate(l_sl) if l_sl else np.zeros(0, np.int64)
        r_idx = np.concatenate(r_sl) if r_sl else np.zeros(0, np.int64)
        p_sl = [np.arange(self.poly_pt_off[r], self.poly_pt_off[r + 1]) for r in r_idx]
        p_idx = np.concatenate(p_sl) if p_sl else np.zeros(0, np.int64)
        counts_pts = np.array([len(s) for s in p_sl], np.int64)
        return RawWorlds(
            names=[self.names[w] for w in ids], dt=self.dt[ids].copy(),
            num_steps=self.num_steps[ids].copy(),
            a_off=_offsets([len(s) for s in a_sl]), kind=self.kind[a_idx],
            length=self.length[a_idx], width=self.width[a_idx], goal=self.goal[a_idx],
            force_replay=self.force_replay[a_idx], controllable=self.controllable[a_idx],
            l_off=_offsets([len(s) for s in l_sl]), log_x=self.log_x[l_idx],
            log_y=self.log_y[l_idx], log_h=self.log_h[l_idx], log_vx=self.log_vx[l_idx],
            log_vy=self.log_vy[l_idx], log_valid=self.log_valid[l_idx],
            poly_off=_offsets([len(s) for s in r_sl]), poly_kind=self.poly_kind[r_idx],
            poly_pt_off=_offsets(counts_pts), pt_x=self.pt_x[p_idx], pt_y=self.pt_y[p_idx])


def concat_raw(parts: list) -> "RawWorlds":
    """Concatenate RawWorlds batches (world order preserved)."""
    def cat(name):
        return np.concatenate([getattr(p, name) for p in parts])

    def off(name):
        counts = np.concatenate([np.diff(getattr(p, name)) for p in parts])
        return _offsets(counts)
    return RawWorlds(
        names=[n for p in parts for n in p.names], dt=cat("dt"), num_steps=cat("num_steps"),
        a_off=off("a_off"), kind=cat("kind"), length=cat("length"), width=cat("width"),
        goal=np.concatenate([p.goal.reshape(-1, 2) for p in parts]),
        force_replay=cat("force_replay"), controllable=cat("controllable"), l_off=off("l_off"),
        log_x=cat("log_x"), log_y=cat("log_y"), log_h=cat("log_h"), log_vx=cat("log_vx"),
        log_vy=cat("log_vy"), log_valid=cat("log_valid"), poly_off=off("poly_off"),
        poly_kind=cat("poly_kind"), poly_pt_off=off("poly_pt_off"), pt_x=cat("pt_x"),
        pt_y=cat("pt_y"))


def _offsets(counts) -> np.ndarray:
    out = np.zeros(len(counts) + 1, np.int64)
    if len(counts):
        np.cumsum(np.asarray(counts, np.int64), out=out[1:])
    return out


def raw_from_prepared(prepared: list) -> RawWorlds:
    """Flatten prepared scenarios (ours or the reference's, duck-typed)."""
    names, dts, Ts = [], [], []
    a_cnt, kinds, lens, wids, goals, frs, ctrls = [], [], [], [], [], [], []
    l_cnt, lx, ly, lh, lvx, lvy, lv = [], [], [], [], [], [], []
    r_cnt, pkind, pp_cnt, px, py = [], [], [], [], []
    for p in prepared:
        base = p.base
        T = int(base.num_steps)
        names.append(base.name)
        dts.append(float(base.timestep))
        Ts.append(T)
        a_cnt.append(len(base.objects))
        l_cnt.append(len(base.objects) * T)
        for o, c in zip(base.objects, p.controllable):
            kinds.append(OBJECT_KINDS.index(o.kind))
            lens.append(float(o.length))
            wids.append(float(o.width))
            goals.append((float(o.goal.x), float(o.goal.y)))
            frs.append(bool(o.force_replay))
            ctrls.append(bool(c))
            sts = list(o.states[:T])
            if len(sts) < T:   # World.__init__ leaves missing steps zero/invalid
                sts = sts + [None] * (T - len(sts))
            for st in sts:
                if st is None:
                    lx.append(0.0); ly.append(0.0); lh.append(0.0)
                    lvx.append(0.0); lvy.append(0.0); lv.append(False)
                    continue
                lx.append(float(st.position.x)); ly.append(float(st.position.y))
                lh.append(float(st.heading))
                lvx.append(float(st.velocity.x)); lvy.append(float(st.velocity.y))
                lv.append(bool(st.valid))
        r_cnt.append(len(p.decimated_roads))
        for road in p.decimated_roads:
            pkind.append(ROAD_KINDS.index(road.kind))
            pp_cnt.append(len(road.geometry))
            for q in road.geometry:
                px.append(float(q.x)); py.append(float(q.y))
    f64 = lambda v: np.asarray(v, np.float64)
    return RawWorlds(
        names=names, dt=f64(dts), num_steps=np.asarray(Ts, np.int32),
        a_off=_offsets(a_cnt), kind=np.asarray(kinds, np.int8), length=f64(lens),
        width=f64(wids), goal=f64(goals).reshape(-1, 2), force_replay=np.asarray(frs, bool),
        controllable=np.asarray(ctrls, bool), l_off=_offsets(l_cnt), log_x=f64(lx),
        log_y=f64(ly), log_h=f64(lh), log_vx=f64(lvx), log_vy=f64(lvy),
        log_valid=np.asarray(lv, bool), poly_off=_offsets(r_cnt),
        poly_kind=np.asarray(pkind, np.int8), poly_pt_off=_offsets(pp_cnt),
        pt_x=f64(px), pt_y=f64(py))


# Static per-agent flag bits (mirrored in include/drivesim_b200.h).
SF_CONTROLLED = 1
SF_INSTANTIABLE = 2
SF_REPLAY_ONLY = 4
SF_PEDESTRIAN = 8


@dataclass
class PackedWorlds:
    """World.__init__ tables for a whole batch (see module docstring)."""

    names: list
    dt: np.ndarray          # f64 [W]
    num_steps: np.ndarray   # i32 [W]
    a_off: np.ndarray       # i64 [W+1]
    c_off: np.ndarray       # i64 [W+1]
    r_off: np.ndarray       # i64 [W+1]
    p_off: np.ndarray       # i64 [W+1]
    s_off: np.ndarray       # i64 [W+1]
    n_instantiated: np.ndarray  # i64 [W]
    # agents [N]
    kind: np.ndarray
    length: np.ndarray
    width: np.ndarray
    half_l: np.ndarray
    half_w: np.ndarray
    circumradius: np.ndarray
    goal_x: np.ndarray
    goal_y: np.ndarray
    sflags: np.ndarray      # u8 SF_* bits
    ctrl_row: np.ndarray    # i32, -1 if not controlled
    # controlled rows [C]
    row_agent: np.ndarray   # i32 global agent index of each row
    # replay tables [R] (time-major per world)
    rep_x: np.ndarray
    rep_y: np.ndarray
    rep_h: np.ndarray
    rep_v: np.ndarray
    rep_valid: np.ndarray   # u8 log_valid
    rep_present: np.ndarray  # u8 present_log
    # road points [P] (original order)
    pt_x: np.ndarray
    pt_y: np.ndarray
    pt_h: np.ndarray
    pt_kind: np.ndarray     # i8
    # segments [S] (original order)
    seg_ax: np.ndarray
    seg_ay: np.ndarray
    seg_bx: np.ndarray
    seg_by: np.ndarray
    seg_kind: np.ndarray    # i8
    extra: dict = field(default_factory=dict)

    @property
    def n_worlds(self) -> int:
        return len(self.names)

    @property
    def n_agents(self) -> int:
        return int(self.a_off[-1])

    @property
    def n_controlled(self) -> int:
        return int(self.c_off[-1])

    def world_counts(self, off_name: str) -> np.ndarray:
        off = getattr(self, off_name)
        return np.diff(off)

    def controlled_ids(self, w: int) -> np.ndarray:
        rows = np.arange(self.c_off[w], self.c_off[w + 1])
        return self.row_agent[rows].astype(np.int64) - self.a_off[w]


def pack(raw: RawWorlds, cfg: SimConfig) -> PackedWorlds:
    """Restates World.__init__ (engine.py:173-314) for every world at once."""
    W = raw.n_worlds
    A = np.diff(raw.a_off)
    T = raw.num_steps.astype(np.int64)
    if not np.array_equal(np.diff(raw.l_off), A * T):
        raise ValueError("log table size != agents x num_steps")
    N = int(raw.a_off[-1])
    L = len(raw.log_valid)
    world_of_agent = np.repeat(np.arange(W), A)
    T_of_agent = T[world_of_agent]
    local_of_agent = np.arange(N) - np.repeat(raw.a_off[:-1], A)
    agent_start = raw.l_off[:-1][world_of_agent] + local_of_agent * T_of_agent
    start_of_cell = np.repeat(agent_start, T_of_agent)
    loc_t = np.arange(L) - start_of_cell            # step index of each log cell

    # Static agent tables (engine.py:185-194).
    half_l = 0.5 * raw.length
    half_w = 0.5 * raw.width
    circumradius = _native.host_hypot_libm(half_l, half_w)   # np.hypot == glibc

    # Log speed uses CPython's correctly rounded math.hypot (engine.py:205).
    log_speed = _native.host_hypot_cpython(raw.log_vx, raw.log_vy)

    # First valid step per agent (engine.py:207-210).
    big = np.iinfo(np.int64).max
    first_valid = np.full(N, big, np.int64)
    nz = T_of_agent > 0
    if nz.any():
        first_valid[nz] = np.minimum.reduceat(np.where(raw.log_valid, loc_t, big),
                                              agent_start[nz])
    instantiable = first_valid != big
    first_valid = np.where(instantiable, first_valid, T_of_agent)
    fv_cell = np.repeat(first_valid, T_of_agent)

    # Forward-filled replay source cell (engine.py:212-228): before the first
    # valid step use the first valid one; after an invalid step hold the last
    # valid one.  A running max of "index if valid" inside each agent's run.
    marked = np.where(raw.log_valid, np.arange(L), start_of_cell - 1)
    last_valid = np.maximum.accumulate(marked) if L else marked
    src = np.where(loc_t < fv_cell, start_of_cell + np.minimum(fv_cell, np.repeat(T_of_agent, T_of_agent) - 1),
                   last_valid)
    inst_cell = np.repeat(instantiable, T_of_agent)
    src = np.where(inst_cell, src, np.arange(L))      # never-valid agents: raw log
    present_am = inst_cell & (loc_t >= fv_cell)

    # Controlled set (engine.py:233-244).
    valid0 = np.zeros(N, bool)
    has_t = T_of_agent > 0
    valid0[has_t] = raw.log_valid[agent_start[has_t]]
    if cfg.init_mode == "all_valid":
        base_mask = valid0 & ~raw.force_replay
    else:
        base_mask = raw.controllable & valid0
    controlled = base_mask.copy()
    if cfg.max_controlled_per_world is not None:
        cum = np.cumsum(base_mask)
        before = np.concatenate([[0], cum])[raw.a_off[:-1]]
        rank = cum - np.repeat(before, A)               # 1-based rank inside world
        controlled &= rank <= cfg.max_controlled_per_world
    n_ctrl = np.bincount(world_of_agent, weights=controlled, minlength=W).astype(np.int64)
    c_off = _offsets(n_ctrl)
    row_agent = np.nonzero(controlled)[0].astype(np.int32)
    ctrl_row = np.full(N, -1, np.int32)
    ctrl_row[row_agent] = np.arange(len(row_agent), dtype=np.int32)
    replay_only = instantiable & ~controlled
    n_inst = np.bincount(world_of_agent, weights=instantiable, minlength=W).astype(np.int64)
    sflags = (controlled * SF_CONTROLLED + instantiable * SF_INSTANTIABLE
              + replay_only * SF_REPLAY_ONLY
              + (raw.kind == OBJECT_KINDS.index("pedestrian")) * SF_PEDESTRIAN).astype(np.uint8)

    # Agent-major logs -> time-major replay tables per world.
    r_off = raw.l_off.astype(np.int64).copy()
    tm_index = (np.repeat(r_off[:-1][world_of_agent], T_of_agent)
                + loc_t * np.repeat(A[world_of_agent], T_of_agent)
                + np.repeat(local_of_agent, T_of_agent))

    def tm(arr):
        out = np.empty(L, arr.dtype)
        out[tm_index] = arr
        return out

    # Road points and segments (engine.py:251-279).
    pts_per_poly = np.diff(raw.poly_pt_off)
    pt_h = _native.host_road_headings(raw.pt_x, raw.pt_y, raw.poly_pt_off)
    pt_kind = np.repeat(raw.poly_kind, pts_per_poly).astype(np.int8)
    p_off = raw.poly_pt_off[raw.poly_off].astype(np.int64)
    seg_per_poly = np.maximum(pts_per_poly - 1, 0)
    seg_cum = _offsets(seg_per_poly)
    seg_start = (np.repeat(raw.poly_pt_off[:-1], seg_per_poly)
                 + np.arange(seg_cum[-1]) - np.repeat(seg_cum[:-1], seg_per_poly))
    seg_kind = np.repeat(raw.poly_kind, seg_per_poly).astype(np.int8)
    s_off = seg_cum[raw.poly_off].astype(np.int64)

    return PackedWorlds(
        names=list(raw.names), dt=raw.dt.astype(np.float64),
        num_steps=raw.num_steps.astype(np.int32), a_off=raw.a_off.astype(np.int64),
        c_off=c_off, r_off=r_off, p_off=p_off, s_off=s_off, n_instantiated=n_inst,
        kind=raw.kind.astype(np.int8), length=raw.length.astype(np.float64),
        width=raw.width.astype(np.float64), half_l=half_l, half_w=half_w,
        circumradius=circumradius, goal_x=raw.goal[:, 0].copy(), goal_y=raw.goal[:, 1].copy(),
        sflags=sflags, ctrl_row=ctrl_row, row_agent=row_agent,
        rep_x=tm(raw.log_x[src]), rep_y=tm(raw.log_y[src]), rep_h=tm(raw.log_h[src]),
        rep_v=tm(log_speed[src]), rep_valid=tm(raw.log_valid.astype(np.uint8)),
        rep_present=tm(present_am.astype(np.uint8)),
        pt_x=raw.pt_x.astype(np.float64), pt_y=raw.pt_y.astype(np.float64),
        pt_h=pt_h, pt_kind=pt_kind,
        seg_ax=raw.pt_x[seg_start], seg_ay=raw.pt_y[seg_start],
        seg_bx=raw.pt_x[seg_start + 1], seg_by=raw.pt_y[seg_start + 1], seg_kind=seg_kind)


def _check_world_ranges(pw: PackedWorlds) -> None:
    for name in ("a_off", "c_off", "r_off", "p_off", "s_off"):
        off = getattr(pw, name)
        if len(off) != pw.n_worlds + 1 or (np.diff(off) < 0).any():
            raise ValueError(f"bad offsets {name}")


ROAD_EDGE_KIND = ROAD_EDGE
