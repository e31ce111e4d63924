"""Off-road knife edges: road-edge segments placed at tiny gaps from (and
touching, crossing, grazing) rotated vehicle boxes far from the origin.  The
step kernel decides off-road behind float prefilters (grid-relative AABB and
a separating-axis filter) whose margins must only ever keep a segment the
exact FP64 slab test (_fastpath.seg_box_hits, fp:55-90) could hit; the flags
must equal the oracle's bit for bit in every world."""

import math

import numpy as np
import pytest

from paper_2408_01584_b200.config import SimConfig
from paper_2408_01584_b200.scenario import RoadElement, Vec2
from scenes import Runner, hold, scene, scripted_object


def _worlds(seed=0, n=240):
    rng = np.random.default_rng(seed)
    gaps = [0.0, 1e-12, 1e-9, 1e-7, 1e-6, 1e-5, 1e-4, 5e-4, 1e-3, 1e-2]
    out = []
    for w in range(n):
        # far from the origin: float copies carry real rounding
        cx, cy = rng.uniform(200.0, 3000.0, 2) * rng.choice([-1.0, 1.0], 2)
        h = float(rng.uniform(-math.pi, math.pi))
        L, W = float(rng.uniform(3.5, 5.5)), float(rng.uniform(1.6, 2.2))
        c, s = math.cos(h), math.sin(h)
        gap = gaps[w % len(gaps)] * (1.0 if rng.random() < 0.5 else -1.0)
        case = w % 4
        if case == 0:       # parallel to the long side, lateral offset W/2 + gap
            off, half, along = W / 2 + gap, float(rng.uniform(0.5, 60.0)), float(rng.uniform(-3, 3))
            p0 = (along - half, off)
            p1 = (along + half, off)
        elif case == 1:     # parallel to the short side
            off, half, along = L / 2 + gap, float(rng.uniform(0.5, 60.0)), float(rng.uniform(-1, 1))
            p0 = (off, along - half)
            p1 = (off, along + half)
        elif case == 2:     # through the corner's diagonal neighbourhood
            ang = float(rng.uniform(0, 2 * math.pi))
            d = (L / 2 + gap, W / 2 + gap)
            p0 = (d[0] + 2.0 * math.cos(ang), d[1] + 2.0 * math.sin(ang))
            p1 = (d[0] - 0.5 * math.cos(ang), d[1] - 0.5 * math.sin(ang))
        else:               # a long segment grazing the box (tangent-ish)
            ang = float(rng.uniform(0, math.pi))
            nrm = (-math.sin(ang), math.cos(ang))
            reach = abs(L / 2 * nrm[0]) + abs(W / 2 * nrm[1]) + gap
            mid = (reach * nrm[0], reach * nrm[1])
            p0 = (mid[0] - 150.0 * math.cos(ang), mid[1] - 150.0 * math.sin(ang))
            p1 = (mid[0] + 150.0 * math.cos(ang), mid[1] + 150.0 * math.sin(ang))
        to_world = lambda p: Vec2(cx + p[0] * c - p[1] * s, cy + p[0] * s + p[1] * c)
        edge = RoadElement(id=0, kind="road_edge", geometry=[to_world(p0), to_world(p1)])
        veh = scripted_object(0, hold(cx, cy, h, 3), goal=(cx + 500.0, cy), length=L, width=W)
        out.append(scene([veh], [edge], name=f"knife-{w}"))
    return out


def _offroad(backend, worlds):
    r = Runner(worlds, SimConfig(), backend)
    _, _, info = r.step(np.zeros((r.n_controlled, 2)))
    r.close()
    return info["offroad"].astype(bool)


def test_knife_edge_scenes_exercise_both_outcomes():
    got = _offroad("oracle", _worlds())
    assert got.any() and not got.all()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1])
def test_offroad_knife_edges_match_oracle(seed):
    worlds = _worlds(seed)
    ref = _offroad("oracle", worlds)
    got = _offroad("gpu", worlds)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"off-road flags differ in worlds {bad[:10]} (oracle {ref[bad[:10]]})"
