"""Exactness of the scalar math restatements shared by the device kernels and
the packer (csrc/ds_math.cuh, exported host-side), against the libm / CPython
behaviour the reference runs on."""

import math

import numpy as np

from paper_2408_01584_b200 import _native as N


def _inputs(n=200_000, seed=0):
    rng = np.random.default_rng(seed)
    x = np.concatenate([rng.uniform(-60, 60, n), rng.uniform(-1e-3, 1e-3, n // 10),
                        rng.normal(0, 1e4, n // 10), [0.0, -0.0, 3.0, 1e-300, 1e300, 5e-324]])
    y = np.concatenate([rng.uniform(-60, 60, n), rng.uniform(-60, 60, n // 10),
                        rng.normal(0, 1e-2, n // 10), [4.0, 0.0, 4.0, 1e-300, 1e-300, 1.0]])
    return x, y


def test_hypot_port_equals_glibc_hypot():
    """ds::hypot (device distance) == glibc hypot == numba math.hypot / np.hypot."""
    x, y = _inputs()
    assert np.array_equal(N.host_hypot_port(x, y), N.host_hypot_libm(x, y))
    assert np.array_equal(N.host_hypot_port(x, y), np.hypot(x, y))


def test_cpython_hypot_restatement():
    """World.__init__ log speed uses CPython's math.hypot (engine.py:205)."""
    x, y = _inputs(50_000, 1)
    ref = np.array([math.hypot(a, b) for a, b in zip(x, y)])
    assert np.array_equal(N.host_hypot_cpython(x, y), ref)


def test_wrap_port_matches_python_floor_mod():
    rng = np.random.default_rng(2)
    pi = math.pi
    edges = np.array([0.0, -0.0, pi, -pi, 2 * pi, -2 * pi, 3 * pi, -3 * pi, 7 * pi, -9 * pi])
    x = np.concatenate([rng.uniform(-30, 30, 200_000), edges, np.nextafter(edges, 50),
                        np.nextafter(edges, -50)])
    ref = np.mod(x + pi, 2 * pi) - pi
    ref = np.where(ref <= -pi, ref + 2 * pi, ref)
    got = N.host_wrap_port(x)
    assert np.array_equal(got, ref)
    assert np.array_equal(np.signbit(got), np.signbit(ref))


def test_road_headings_match_math_atan2():
    rng = np.random.default_rng(3)
    pts = rng.uniform(-100, 100, (500, 2))
    off = np.array([0, 1, 5, 7, 40, 500], np.int64)       # includes a 1-point polyline
    got = N.host_road_headings(pts[:, 0], pts[:, 1], off)
    ref = []
    for r in range(len(off) - 1):
        g = pts[off[r]:off[r + 1]]
        for j in range(len(g)):
            if len(g) == 1:
                ref.append(0.0)
                continue
            q = g[j + 1] if j + 1 < len(g) else g[j]
            p = g[j] if j + 1 < len(g) else g[j - 1]
            ref.append(math.atan2(q[1] - p[1], q[0] - p[0]))
    assert np.array_equal(got, np.array(ref))
