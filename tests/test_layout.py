"""Device layout invariants: the uniform grids are exact supersets of what
the kernels query (every point in its cell, every segment in every cell its
AABB touches), and the float2 rounding bound is what the key analysis uses."""

import numpy as np
import pytest

from paper_2408_01584_b200.config import ROAD_EDGE, SimConfig
from paper_2408_01584_b200.device_layout import build_layout
from paper_2408_01584_b200.packing import pack
from paper_2408_01584_b200.synthetic import WaymoSpec, generate


def _pw(quantize=True):
    raw = generate(WaymoSpec(n_worlds=3, n_agents=16, n_points=900, seed=4, quantize=quantize))
    return pack(raw, SimConfig(init_mode="all_valid"))


def test_points_sorted_into_their_cells():
    pw = _pw()
    lay = build_layout(pw, 8.0)
    for w in range(pw.n_worlds):
        nx, ny = int(lay.grid_nx[w]), int(lay.grid_ny[w])
        cs = lay.pt_cell_start[lay.grid_cell_off[w]:lay.grid_cell_off[w + 1]]
        assert len(cs) == nx * ny + 1 and (np.diff(cs) >= 0).all()
        assert cs[0] == pw.p_off[w] and cs[-1] == pw.p_off[w + 1]
        for c in range(nx * ny):
            s = slice(cs[c], cs[c + 1])
            ix = np.floor((lay.gpt_x[s] - lay.grid_x0[w]) / 8.0).clip(0, nx - 1)
            iy = np.floor((lay.gpt_y[s] - lay.grid_y0[w]) / 8.0).clip(0, ny - 1)
            assert ((iy * nx + ix) == c).all()
            ids = lay.gpt_id[s]
            assert (np.diff(ids) > 0).all()           # original order inside a cell
    # a permutation of every world's points
    for w in range(pw.n_worlds):
        p0, p1 = pw.p_off[w], pw.p_off[w + 1]
        assert sorted(lay.gpt_id[p0:p1]) == list(range(p1 - p0))
        assert np.array_equal(lay.gpt_x[p0:p1], pw.pt_x[p0:p1][lay.gpt_id[p0:p1]])


def test_edge_segments_binned_into_every_touched_cell():
    pw = _pw()
    lay = build_layout(pw, 8.0)
    for w in range(pw.n_worlds):
        nx = int(lay.grid_nx[w])
        base = lay.grid_cell_off[w]
        s0, s1 = pw.s_off[w], pw.s_off[w + 1]
        edges = [k for k in range(s0, s1) if pw.seg_kind[k] == ROAD_EDGE]
        cs = lay.eseg_cell_start[base:lay.grid_cell_off[w + 1]]
        for k in edges[:200]:
            lo = np.floor((min(pw.seg_ax[k], pw.seg_bx[k]) - lay.grid_x0[w]) / 8.0)
            hi = np.floor((max(pw.seg_ax[k], pw.seg_bx[k]) - lay.grid_x0[w]) / 8.0)
            ylo = np.floor((min(pw.seg_ay[k], pw.seg_by[k]) - lay.grid_y0[w]) / 8.0)
            yhi = np.floor((max(pw.seg_ay[k], pw.seg_by[k]) - lay.grid_y0[w]) / 8.0)
            for iy in range(int(ylo), int(yhi) + 1):
                for ix in range(int(lo), int(hi) + 1):
                    c = iy * nx + ix
                    sl = slice(cs[c], cs[c + 1])
                    assert (np.isclose(lay.eseg_ax[sl], pw.seg_ax[k]) &
                            np.isclose(lay.eseg_by[sl], pw.seg_by[k])).any()


@pytest.mark.parametrize("quantize", [True, False])
def test_float2_rounding_bound(quantize):
    pw = _pw(quantize)
    lay = build_layout(pw, 8.0)
    for w in range(pw.n_worlds):
        p0, p1 = pw.p_off[w], pw.p_off[w + 1]
        ex = np.abs(lay.gpt_xy[p0:p1, 0].astype(np.float64) - (lay.gpt_x[p0:p1] - lay.grid_x0[w]))
        ey = np.abs(lay.gpt_xy[p0:p1, 1].astype(np.float64) - (lay.gpt_y[p0:p1] - lay.grid_y0[w]))
        assert max(ex.max(), ey.max()) == lay.grid_eps[w]
    if quantize:   # quantised synthetic coordinates are exact in float32
        assert (lay.grid_eps == 0).all()
    else:          # off-lattice: the key bound's eps_p term is live
        assert (lay.grid_eps > 0).all() and (lay.grid_eps < 1e-4).all()
