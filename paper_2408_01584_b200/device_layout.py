"""Per-world uniform grids over the static road geometry (device layout).

The reference prunes with a median-split BVH (broadphase.py:43-281) whose
results are pinned equal to brute force; the B200 layout replaces it with a
static uniform grid per world, built once at batch construction:

* road points are stored cell-major (row-major cells, original index ascending
  inside a cell), so the cells of one cell row that a query disc covers are a
  single contiguous range -> coalesced, L2-resident lane-strided reads;
* road-edge segments (off-road test) and all segments (LiDAR) are binned into
  every cell their AABB touches, with duplicates; a query visits the cells
  overlapping its own AABB and the exact narrow-phase test decides.

All offsets are absolute (into the concatenated arrays of all worlds) so the
device needs no per-world base arithmetic beyond ``grid_cell_off[w]``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import ROAD_EDGE
from .packing import PackedWorlds, _offsets


@dataclass
class DeviceLayout:
    cell: float
    grid_x0: np.ndarray       # f64 [W]
    grid_y0: np.ndarray
    grid_nx: np.ndarray       # i32 [W]
    grid_ny: np.ndarray
    grid_cell_off: np.ndarray # i64 [W+1]  (ncell_w + 1 entries per world)
    pt_cell_start: np.ndarray # i32 [sum(ncell+1)]
    gpt_x: np.ndarray
    gpt_y: np.ndarray
    gpt_h: np.ndarray
    gpt_kind: np.ndarray      # i8
    gpt_id: np.ndarray        # i32 original local index
    eseg_cell_start: np.ndarray
    eseg_ax: np.ndarray
    eseg_ay: np.ndarray
    eseg_bx: np.ndarray
    eseg_by: np.ndarray
    eseg_rel: np.ndarray      # f32 [E, 4] (ax, ay, bx, by) - grid origin (off-road prefilter)
    aseg_cell_start: np.ndarray
    aseg_ax: np.ndarray
    aseg_ay: np.ndarray
    aseg_bx: np.ndarray
    aseg_by: np.ndarray
    aseg_id: np.ndarray
    aseg_edge: np.ndarray
    gpt_xy: np.ndarray        # f32 [P, 2] grid-sorted, relative to (grid_x0, grid_y0)
    grid_eps: np.ndarray      # f64 [W] max |f32 - exact| of those coordinates


def _bin_segments(pw: PackedWorlds, sel: np.ndarray, world_of_seg: np.ndarray,
                  x0, y0, nx, ny, cell_base, n_cells_total, cell):
    """Bin selected segments into every cell of their AABB.  Returns
    (cell_start[n_cells_total], order) where order indexes pw.seg_* arrays."""
    idx = np.nonzero(sel)[0]
    w = world_of_seg[idx]
    lox = np.minimum(pw.seg_ax[idx], pw.seg_bx[idx])
    hix = np.maximum(pw.seg_ax[idx], pw.seg_bx[idx])
    loy = np.minimum(pw.seg_ay[idx], pw.seg_by[idx])
    hiy = np.maximum(pw.seg_ay[idx], pw.seg_by[idx])
    cx0 = np.clip(np.floor((lox - x0[w]) / cell), 0, nx[w] - 1).astype(np.int64)
    cx1 = np.clip(np.floor((hix - x0[w]) / cell), 0, nx[w] - 1).astype(np.int64)
    cy0 = np.clip(np.floor((loy - y0[w]) / cell), 0, ny[w] - 1).astype(np.int64)
    cy1 = np.clip(np.floor((hiy - y0[w]) / cell), 0, ny[w] - 1).astype(np.int64)
    nxs = cx1 - cx0 + 1
    nys = cy1 - cy0 + 1
    cnt = nxs * nys
    rep = np.repeat(np.arange(len(idx)), cnt)
    k = np.arange(cnt.sum()) - np.repeat(_offsets(cnt)[:-1], cnt)
    kx = k % np.repeat(nxs, cnt)
    ky = k // np.repeat(nxs, cnt)
    cells = (cell_base[w[rep]] + (cy0[rep] + ky) * nx[w[rep]] + (cx0[rep] + kx)).astype(np.int64)
    order = np.argsort(cells, kind="stable")      # idx[rep] is already ascending
    cells_sorted = cells[order]
    counts = np.bincount(cells_sorted, minlength=n_cells_total)
    start = np.zeros(n_cells_total + 1, np.int64)
    np.cumsum(counts, out=start[1:])
    return start, idx[rep][order]


def build_layout(pw: PackedWorlds, cell: float = 8.0, all_segments: bool = True) -> DeviceLayout:
    W = pw.n_worlds
    P = np.diff(pw.p_off)
    world_of_pt = np.repeat(np.arange(W), P)
    big = np.inf
    x0 = np.zeros(W)
    y0 = np.zeros(W)
    x1 = np.zeros(W)
    y1 = np.zeros(W)
    has = P > 0
    if has.any():
        starts = pw.p_off[:-1][has]
        x0[has] = np.minimum.reduceat(pw.pt_x, starts)
        y0[has] = np.minimum.reduceat(pw.pt_y, starts)
        x1[has] = np.maximum.reduceat(pw.pt_x, starts)
        y1[has] = np.maximum.reduceat(pw.pt_y, starts)
    nx = (np.floor((x1 - x0) / cell).astype(np.int64) + 1)
    ny = (np.floor((y1 - y0) / cell).astype(np.int64) + 1)
    if (nx * ny > 1 << 26).any():
        raise ValueError("road grid too large; increase grid_cell")
    ncell = nx * ny
    cell_base_ptr = np.zeros(W + 1, np.int64)      # offsets into *_cell_start arrays
    np.cumsum(ncell + 1, out=cell_base_ptr[1:])
    cell_base = np.zeros(W + 1, np.int64)          # offsets of the cells themselves
    np.cumsum(ncell, out=cell_base[1:])
    n_cells_total = int(cell_base[-1])

    # --- road points, cell-major
    local = np.arange(len(world_of_pt)) - np.repeat(pw.p_off[:-1], P)
    w = world_of_pt
    if len(w):
        cx = np.clip(np.floor((pw.pt_x - x0[w]) / cell), 0, nx[w] - 1).astype(np.int64)
        cy = np.clip(np.floor((pw.pt_y - y0[w]) / cell), 0, ny[w] - 1).astype(np.int64)
        gcell = cell_base[w] + cy * nx[w] + cx
    else:
        gcell = np.zeros(0, np.int64)
    order = np.argsort(gcell, kind="stable")   # world-major cells, original order inside
    counts = np.bincount(gcell, minlength=n_cells_total)
    pstart = np.zeros(n_cells_total + 1, np.int64)
    np.cumsum(counts, out=pstart[1:])

    def per_world_ptr(start):
        # expand cell starts to (ncell_w + 1) entries per world
        out = np.empty(int(cell_base_ptr[-1]), np.int64)
        for_w = np.repeat(np.arange(W), ncell + 1)
        k = np.arange(len(out)) - np.repeat(cell_base_ptr[:-1], ncell + 1)
        out[:] = start[cell_base[for_w] + k]
        return out.astype(np.int32)

    # --- segments
    S = np.diff(pw.s_off)
    world_of_seg = np.repeat(np.arange(W), S)
    edge = pw.seg_kind == ROAD_EDGE
    es, eorder = _bin_segments(pw, edge, world_of_seg, x0, y0, nx, ny, cell_base,
                               n_cells_total, cell)
    # all segments (LiDAR / view-cone rays); empty bins when the sensor is radial
    as_, aorder = _bin_segments(pw, np.full(len(world_of_seg), bool(all_segments)), world_of_seg,
                                x0, y0, nx, ny, cell_base, n_cells_total, cell)
    seg_local = np.arange(len(world_of_seg)) - np.repeat(pw.s_off[:-1], S)
    ew = world_of_seg[eorder]
    erel = np.stack([pw.seg_ax[eorder] - x0[ew], pw.seg_ay[eorder] - y0[ew],
                     pw.seg_bx[eorder] - x0[ew], pw.seg_by[eorder] - y0[ew]], -1).astype(np.float32)
    # float2 coordinates relative to the world origin for the shared-memory scan,
    # with the exact per-world rounding bound used by the key error analysis
    ws = world_of_pt[order] if len(order) else np.zeros(0, np.int64)
    relx = pw.pt_x[order] - x0[ws]
    rely = pw.pt_y[order] - y0[ws]
    gxy = np.stack([relx, rely], -1).astype(np.float32)
    err = np.maximum(np.abs(gxy[:, 0].astype(np.float64) - relx),
                     np.abs(gxy[:, 1].astype(np.float64) - rely)) if len(ws) else np.zeros(0)
    eps = np.zeros(W)
    if len(ws) and has.any():
        eps[has] = np.maximum.reduceat(err, pw.p_off[:-1][has])
    return DeviceLayout(
        cell=float(cell), grid_x0=x0.astype(np.float64), grid_y0=y0.astype(np.float64),
        grid_nx=nx.astype(np.int32), grid_ny=ny.astype(np.int32), grid_cell_off=cell_base_ptr,
        pt_cell_start=per_world_ptr(pstart), gpt_x=pw.pt_x[order], gpt_y=pw.pt_y[order],
        gpt_h=pw.pt_h[order], gpt_kind=pw.pt_kind[order].astype(np.int8),
        gpt_id=local[order].astype(np.int32),
        eseg_cell_start=per_world_ptr(es), eseg_ax=pw.seg_ax[eorder], eseg_ay=pw.seg_ay[eorder],
        eseg_bx=pw.seg_bx[eorder], eseg_by=pw.seg_by[eorder],
        eseg_rel=np.ascontiguousarray(erel.reshape(-1, 4)),
        aseg_cell_start=per_world_ptr(as_), aseg_ax=pw.seg_ax[aorder], aseg_ay=pw.seg_ay[aorder],
        aseg_bx=pw.seg_bx[aorder], aseg_by=pw.seg_by[aorder],
        aseg_id=seg_local[aorder].astype(np.int32), aseg_edge=edge[aorder].astype(np.uint8),
        gpt_xy=np.ascontiguousarray(gxy), grid_eps=eps)
