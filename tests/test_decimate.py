"""Polyline decimation (preprocess): the oracle restatement
pinned to golden vectors from the real reference, the GPU kernel pinned to
both (bit-exact keep masks), and the prepared-scenario file format."""

import os

import numpy as np
import pytest

from oracle.decimate import decimate_keep, decimate_keep_batch

HERE = os.path.dirname(os.path.abspath(__file__))


def golden():
    g = np.load(os.path.join(HERE, "golden", "decimate.npz"))
    return g["x"], g["y"], g["off"], g["threshold"], g["keep"]


def test_oracle_matches_reference_golden():
    x, y, off, thr, keep = golden()
    for p in range(len(off) - 1):
        a, b = off[p], off[p + 1]
        got = decimate_keep(list(zip(x[a:b].tolist(), y[a:b].tolist())), float(thr[p]))
        assert np.array_equal(got, keep[a:b]), p


def test_oracle_reference_unit_cases():
    # test_geometry.py:24-47
    assert decimate_keep([(0, 0), (1, 0), (2, 0)], 0.01).tolist() == [True, False, True]
    assert decimate_keep([(0, 0), (1, 0.5), (2, 0), (3, 0.5), (4, 0)], 0.6).tolist() == \
        [True, False, False, True, True]


def test_prepared_round_trip():
    from paper_2408_01584_b200.scenario import (LoggedStep, ObjectLog, PrepStats,
                                                PreparedScenario, RoadElement, Scenario,
                                                Vec2, load_prepared, serialize_prepared)
    st = [LoggedStep(Vec2(1.0, 2.0), 0.5, Vec2(3.0, 0.0), True)] * 3
    s = Scenario(name="rt", num_steps=3,
                 objects=[ObjectLog(0, "vehicle", 4.5, 1.8, Vec2(9.0, 2.0), st)],
                 roads=[RoadElement(7, "road_edge", [Vec2(0.0, 0.0), Vec2(5.0, 0.25)])])
    p = PreparedScenario(base=s, decimated_roads=s.roads, controllable=[True],
                         stats=PrepStats(1, 1, 2, 2))
    q = load_prepared(serialize_prepared(p))
    assert q.base.name == "rt" and q.controllable == [True]
    assert [tuple(v) for v in q.decimated_roads[0].geometry] == [(0.0, 0.0), (5.0, 0.25)]
    assert q.stats == p.stats
    assert q.base.objects[0].goal == (9.0, 2.0)


@pytest.mark.gpu
def test_gpu_decimation_matches_reference_golden():
    from paper_2408_01584_b200.scenario import decimate_keep as gpu_keep
    x, y, off, thr, keep = golden()
    for t in np.unique(thr):
        sel = np.nonzero(thr == t)[0]
        counts = off[sel + 1] - off[sel]
        sub_off = np.concatenate([[0], np.cumsum(counts)])
        idx = np.concatenate([np.arange(off[p], off[p + 1]) for p in sel])
        got = gpu_keep(x[idx], y[idx], sub_off, float(t), device="cuda:0")
        assert np.array_equal(got, keep[idx]), t


@pytest.mark.gpu
def test_gpu_decimation_large_batch_matches_oracle():
    from paper_2408_01584_b200.scenario import decimate_keep as gpu_keep
    rng = np.random.default_rng(3)
    lens = rng.integers(1, 400, 1500)
    lens[:5] = [1, 2, 3, 1000, 3000]
    off = np.concatenate([[0], np.cumsum(lens)])
    steps = rng.normal(0, 1, (off[-1], 2)) * np.repeat(rng.uniform(0.01, 2, len(lens)), lens)[:, None]
    xy = np.cumsum(steps, axis=0)
    xy = np.round(xy * 64) / 64          # lattice-ish values: plenty of exact area ties
    skip = rng.random(len(lens)) < 0.1
    for t in (0.05, 0.5, 3.0):
        want = decimate_keep_batch(xy[:, 0], xy[:, 1], off, t, skip)
        got = gpu_keep(xy[:, 0], xy[:, 1], off, t, skip, device="cuda:0")
        assert np.array_equal(got, want), t
        assert got[off[:-1]].all() and got[off[1:] - 1].all()   # endpoints kept


@pytest.mark.gpu
def test_preprocess_many_equals_per_scenario():
    from paper_2408_01584_b200.scenario import decimate_polyline, preprocess, preprocess_many
    from paper_2408_01584_b200.synthetic import WaymoSpec, generate, to_scenarios
    raw = generate(WaymoSpec(n_worlds=3, n_agents=8, n_points=300, seed=4, num_steps=5))
    scen = [p.base for p in to_scenarios(raw)]
    many = preprocess_many(scen, 0.05, device="cuda:0")
    for s, m in zip(scen, many):
        one = preprocess(s, device="cuda:0")           # reference default threshold 0.05
        assert [r.geometry for r in one.decimated_roads] == [r.geometry for r in m.decimated_roads]
        assert one.stats == m.stats and one.controllable == m.controllable
        for r0, r1 in zip(s.roads, m.decimated_roads):
            pts = [(p[0], p[1]) for p in r0.geometry]
            k = decimate_keep(pts, 0.05)
            assert [tuple(p) for p in r1.geometry] == [p for p, kk in zip(pts, k) if kk]
            assert decimate_polyline(r0.geometry, 0.05, device="cuda:0") == r1.geometry
