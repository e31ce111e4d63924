"""TEST INFRASTRUCTURE ONLY (the checker, never the product).

Pure-Python restatement of the reference's polyline decimation, used by
tests/ to check the GPU kernel (csrc/ds_decimate.cu):

  triangle_area      pkg/src/drivesim/geometry.py:79-81
  decimate_polyline  pkg/src/drivesim/geometry.py:84-127 (lazy-deletion heap
                     keyed (area, index, version); ties remove the smaller
                     index)
  preprocess skips   pkg/src/drivesim/scenario.py:396-401 (stop signs and
                     polylines with < 3 points are not decimated)

Pinned against the real reference by tests/golden/decimate.npz
(tests/golden/make_golden_decimate.py).
"""

from __future__ import annotations

import heapq

import numpy as np


def triangle_area(a, b, c) -> float:
    return 0.5 * abs((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]))


def decimate_keep(points, threshold: float) -> np.ndarray:
    """Keep mask of decimate_polyline(points, threshold)."""
    n = len(points)
    keep = np.ones(n, bool)
    if n < 3 or threshold <= 0.0:
        return keep
    prev = list(range(-1, n - 1))
    nxt = list(range(1, n + 1))
    version = [0] * n

    def area_at(i):
        return triangle_area(points[prev[i]], points[i], points[nxt[i]])

    heap = [(area_at(i), i, 0) for i in range(1, n - 1)]
    heapq.heapify(heap)
    while heap:
        a, i, ver = heapq.heappop(heap)
        if not keep[i] or ver != version[i]:
            continue
        if a >= threshold:
            break
        keep[i] = False
        p, q = prev[i], nxt[i]
        nxt[p] = q
        prev[q] = p
        if p > 0:
            version[p] += 1
            heapq.heappush(heap, (area_at(p), p, version[p]))
        if q < n - 1:
            version[q] += 1
            heapq.heappush(heap, (area_at(q), q, version[q]))
    return keep


def decimate_keep_batch(x, y, poly_off, threshold: float, skip=None) -> np.ndarray:
    keep = np.ones(len(x), bool)
    for p in range(len(poly_off) - 1):
        a, b = int(poly_off[p]), int(poly_off[p + 1])
        if skip is not None and skip[p]:
            continue
        pts = list(zip(x[a:b].tolist(), y[a:b].tolist()))
        keep[a:b] = decimate_keep(pts, threshold)
    return keep
