"""Golden vectors for polyline decimation from the REAL reference
(drivesim.geometry.decimate_polyline, geometry.py:84-127), mirroring the
reference's own decimation tests (pkg/tests/test_geometry.py:24-92,
test_acceptance.py:113-153).  Runs only in the build container:

    python tests/golden/make_golden_decimate.py   -> tests/golden/decimate.npz
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from drivesim.geometry import Vec2, decimate_polyline  # noqa: E402
from drivesim.synthetic import SyntheticSpec, generate_synthetic  # noqa: E402


def main():
    lines, thresholds = [], []
    # the reference's unit cases
    lines.append([(0, 0), (1, 0), (2, 0)]); thresholds.append(0.01)
    lines.append([(0, 0), (1, 1)]); thresholds.append(1e9)
    lines.append([(0, 0), (1, 0.5), (2, 0), (3, 0.5), (4, 0)]); thresholds.append(0.6)
    rng = np.random.default_rng(0)
    lines.append([tuple(p) for p in rng.normal(size=(40, 2))]); thresholds.append(0.0)
    for seed in range(30):
        r = np.random.default_rng(seed)
        n = int(r.integers(3, 25))
        lines.append([tuple(p) for p in np.cumsum(r.normal(size=(n, 2)), axis=0)])
        thresholds.append(float(r.uniform(0.001, 2.0)))
    r = np.random.default_rng(7)
    lines.append([tuple(p) for p in np.cumsum(r.normal(size=(20, 2)), axis=0)])
    thresholds.append(1.0)
    # acceptance corpus: straight line, template roads, noisy dense lines
    lines.append([(float(x), 0.0) for x in np.linspace(0, 100, 100)]); thresholds.append(0.05)
    for template in ("straight_road", "intersection", "parking_lot"):
        for seed in range(4):
            s = generate_synthetic(SyntheticSpec(template, n_agents=4, seed=seed))
            for road in s.roads:
                lines.append([(p.x, p.y) for p in road.geometry]); thresholds.append(0.05)
    r = np.random.default_rng(103)
    for _ in range(20):
        n = int(r.integers(200, 400))
        xs = np.linspace(0, 100, n)
        ys = r.normal(0, 0.01, n)
        lines.append(list(zip(xs.tolist(), ys.tolist()))); thresholds.append(0.05)
    # exact ties on a lattice (many equal areas)
    for seed in range(6):
        r = np.random.default_rng(500 + seed)
        n = int(r.integers(30, 200))
        pts = np.cumsum(r.integers(-2, 3, size=(n, 2)), axis=0).astype(float)
        lines.append([tuple(p) for p in pts]); thresholds.append(float(r.choice([0.5, 1.0, 2.5])))
    keeps = []
    for pts, t in zip(lines, thresholds):
        v = [Vec2(float(x), float(y)) for x, y in pts]
        out = decimate_polyline(v, t)
        keep, it = np.zeros(len(v), bool), 0
        for k, p in enumerate(v):
            if it < len(out) and out[it] is p:
                keep[k] = True
                it += 1
        assert it == len(out)
        keeps.append(keep)
    off = np.zeros(len(lines) + 1, np.int64)
    np.cumsum([len(l) for l in lines], out=off[1:])
    xy = np.array([p for l in lines for p in l], dtype=np.float64).reshape(-1, 2)
    np.savez_compressed(os.path.join(HERE, "decimate.npz"), x=xy[:, 0], y=xy[:, 1], off=off,
                        threshold=np.array(thresholds), keep=np.concatenate(keeps))
    print(f"{len(lines)} polylines, {len(xy)} points, kept {int(np.concatenate(keeps).sum())}")


if __name__ == "__main__":
    main()
