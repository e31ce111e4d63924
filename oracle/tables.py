"""The oracle's own World.__init__ table builder -- TEST INFRASTRUCTURE.

A plain restatement of the reference's per-world table construction
(/root/reference/pkg/src/drivesim/engine.py:173-314), written independently
of the product packer (paper_2408_01584_b200/packing.py) so that the checker
shares no code with the thing it checks and never loads the CUDA library:
numpy + the Python standard library only.

Input: any object with the ``RawWorlds`` attributes (a flat image of prepared
scenarios: per-world offsets, agent statics, agent-major logs, road
polylines).  Output: ``OracleTables``, the arrays ``drivesim_oracle.c`` reads
(agent statics, time-major replay tables, road points and segments in the
reference's original order).  Functions follow the reference line by line:

  * circumradius = np.hypot(half_l, half_w)                      (eng:185-189)
  * log speed = CPython math.hypot(vx, vy)                       (eng:205)
  * first valid step, forward-filled replay pose, present_log    (eng:207-231)
  * controlled ids: all_valid / all_nontrivial, max per world    (eng:233-244)
  * road point heading = atan2 to the next point, last point uses the
    previous segment, single-point polyline 0                    (eng:251-265)
  * segments between consecutive points of every polyline        (eng:266-275)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PEDESTRIAN = 1        # OBJECT_KINDS.index("pedestrian"), scenario.py:32
SF_CONTROLLED, SF_INSTANTIABLE, SF_REPLAY_ONLY, SF_PEDESTRIAN = 1, 2, 4, 8


def _offsets(counts) -> np.ndarray:
    out = np.zeros(len(counts) + 1, np.int64)
    out[1:] = np.cumsum(np.asarray(counts, np.int64))
    return out


@dataclass
class OracleTables:
    n_worlds: int
    names: list
    dt: np.ndarray
    num_steps: np.ndarray
    a_off: np.ndarray
    c_off: np.ndarray
    r_off: np.ndarray
    p_off: np.ndarray
    s_off: np.ndarray
    n_instantiated: np.ndarray
    kind: np.ndarray
    length: np.ndarray
    width: np.ndarray
    half_l: np.ndarray
    half_w: np.ndarray
    circumradius: np.ndarray
    goal_x: np.ndarray
    goal_y: np.ndarray
    sflags: np.ndarray
    ctrl_row: np.ndarray
    row_agent: np.ndarray
    rep_x: np.ndarray
    rep_y: np.ndarray
    rep_h: np.ndarray
    rep_v: np.ndarray
    rep_valid: np.ndarray
    rep_present: np.ndarray
    pt_x: np.ndarray
    pt_y: np.ndarray
    pt_h: np.ndarray
    pt_kind: np.ndarray
    seg_ax: np.ndarray
    seg_ay: np.ndarray
    seg_bx: np.ndarray
    seg_by: np.ndarray
    seg_kind: np.ndarray

    @property
    def n_agents(self) -> int:
        return int(self.a_off[-1])

    @property
    def n_controlled(self) -> int:
        return int(self.c_off[-1])

    def controlled_ids(self, w: int) -> np.ndarray:
        return self.row_agent[self.c_off[w]:self.c_off[w + 1]].astype(np.int64) - self.a_off[w]


def _world(raw, w: int, cfg) -> dict:
    """engine.py:173-314 for world w."""
    a0, a1 = int(raw.a_off[w]), int(raw.a_off[w + 1])
    n, T = a1 - a0, int(raw.num_steps[w])
    length = np.asarray(raw.length[a0:a1], np.float64)
    width = np.asarray(raw.width[a0:a1], np.float64)
    half_l, half_w = 0.5 * length, 0.5 * width
    lo = int(raw.l_off[w])
    cells = lambda arr: np.asarray(arr[lo:lo + n * T]).reshape(n, T)
    valid = cells(raw.log_valid).astype(bool)
    lx, ly, lh = cells(raw.log_x), cells(raw.log_y), cells(raw.log_h)
    vx, vy = cells(raw.log_vx), cells(raw.log_vy)
    speed = np.array([[math.hypot(vx[i, t], vy[i, t]) for t in range(T)] for i in range(n)],
                     np.float64).reshape(n, T)
    instantiable = valid.any(axis=1)
    first_valid = np.where(instantiable, valid.argmax(axis=1), T)
    # forward fill: step t replays the last valid step <= t, before the first
    # valid step the first valid one; never-valid agents keep the raw log
    src = np.tile(np.arange(T), (n, 1))
    for i in range(n):
        if not instantiable[i]:
            continue
        fv = first_valid[i]
        src[i, :fv] = fv
        for t in range(fv + 1, T):
            if not valid[i, t]:
                src[i, t] = src[i, t - 1]
    take = lambda a: np.take_along_axis(a, src, 1)
    present = instantiable[:, None] & (np.arange(T)[None, :] >= first_valid[:, None])
    valid0 = valid[:, 0] if T else np.zeros(n, bool)
    force = np.asarray(raw.force_replay[a0:a1], bool)
    if cfg.init_mode == "all_valid":
        base_mask = valid0 & ~force
    else:
        base_mask = np.asarray(raw.controllable[a0:a1], bool) & valid0
    ids = np.nonzero(base_mask)[0]
    if cfg.max_controlled_per_world is not None:
        ids = ids[:cfg.max_controlled_per_world]
    controlled = np.zeros(n, bool)
    controlled[ids] = True
    kind = np.asarray(raw.kind[a0:a1], np.int8)
    sflags = (controlled * SF_CONTROLLED + instantiable * SF_INSTANTIABLE
              + (instantiable & ~controlled) * SF_REPLAY_ONLY
              + (kind == PEDESTRIAN) * SF_PEDESTRIAN).astype(np.uint8)
    # roads: points, headings, segments per polyline, original order
    px, py, ph, pk, sax, say, sbx, sby, sk = [], [], [], [], [], [], [], [], []
    for r in range(int(raw.poly_off[w]), int(raw.poly_off[w + 1])):
        q0, q1 = int(raw.poly_pt_off[r]), int(raw.poly_pt_off[r + 1])
        gx = [float(v) for v in raw.pt_x[q0:q1]]
        gy = [float(v) for v in raw.pt_y[q0:q1]]
        m, kd = q1 - q0, int(raw.poly_kind[r])
        for j in range(m):
            px.append(gx[j])
            py.append(gy[j])
            if m == 1:
                ph.append(0.0)
            else:
                nj, cj = (j + 1, j) if j + 1 < m else (j, j - 1)
                ph.append(math.atan2(gy[nj] - gy[cj], gx[nj] - gx[cj]))
            pk.append(kd)
        for j in range(m - 1):
            sax.append(gx[j]); say.append(gy[j]); sbx.append(gx[j + 1]); sby.append(gy[j + 1])
            sk.append(kd)
    tm = lambda a: np.ascontiguousarray(a.T).reshape(-1)       # time-major: t * n + i
    return dict(n=n, T=T, ids=ids, n_inst=int(instantiable.sum()), kind=kind, length=length,
                width=width, half_l=half_l, half_w=half_w, circumradius=np.hypot(half_l, half_w),
                goal=np.asarray(raw.goal[a0:a1], np.float64).reshape(n, 2), sflags=sflags,
                rep_x=tm(take(lx)), rep_y=tm(take(ly)), rep_h=tm(take(lh)), rep_v=tm(take(speed)),
                rep_valid=tm(valid.astype(np.uint8)), rep_present=tm(present.astype(np.uint8)),
                pt_x=px, pt_y=py, pt_h=ph, pt_kind=pk, seg_ax=sax, seg_ay=say, seg_bx=sbx,
                seg_by=sby, seg_kind=sk)


def build_tables(raw, cfg) -> OracleTables:
    W = len(raw.names)
    ws = [_world(raw, w, cfg) for w in range(W)]
    cat = lambda key, dt: (np.concatenate([np.asarray(x[key], dt) for x in ws]) if ws
                           else np.zeros(0, dt))
    a_off = _offsets([x["n"] for x in ws])
    c_off = _offsets([len(x["ids"]) for x in ws])
    row_agent = np.concatenate([a_off[w] + x["ids"] for w, x in enumerate(ws)]).astype(np.int32) \
        if ws else np.zeros(0, np.int32)
    ctrl_row = np.full(int(a_off[-1]), -1, np.int32)
    ctrl_row[row_agent] = np.arange(len(row_agent), dtype=np.int32)
    goal = np.concatenate([x["goal"] for x in ws]) if ws else np.zeros((0, 2))
    return OracleTables(
        n_worlds=W, names=list(raw.names), dt=np.asarray(raw.dt, np.float64),
        num_steps=np.asarray(raw.num_steps, np.int32), a_off=a_off, c_off=c_off,
        r_off=_offsets([x["n"] * x["T"] for x in ws]),
        p_off=_offsets([len(x["pt_x"]) for x in ws]), s_off=_offsets([len(x["seg_ax"]) for x in ws]),
        n_instantiated=np.array([x["n_inst"] for x in ws], np.int64),
        kind=cat("kind", np.int8), length=cat("length", np.float64), width=cat("width", np.float64),
        half_l=cat("half_l", np.float64), half_w=cat("half_w", np.float64),
        circumradius=cat("circumradius", np.float64), goal_x=goal[:, 0].copy(),
        goal_y=goal[:, 1].copy(), sflags=cat("sflags", np.uint8), ctrl_row=ctrl_row,
        row_agent=row_agent, rep_x=cat("rep_x", np.float64), rep_y=cat("rep_y", np.float64),
        rep_h=cat("rep_h", np.float64), rep_v=cat("rep_v", np.float64),
        rep_valid=cat("rep_valid", np.uint8), rep_present=cat("rep_present", np.uint8),
        pt_x=cat("pt_x", np.float64), pt_y=cat("pt_y", np.float64), pt_h=cat("pt_h", np.float64),
        pt_kind=cat("pt_kind", np.int8), seg_ax=cat("seg_ax", np.float64),
        seg_ay=cat("seg_ay", np.float64), seg_bx=cat("seg_bx", np.float64),
        seg_by=cat("seg_by", np.float64), seg_kind=cat("seg_kind", np.int8))
