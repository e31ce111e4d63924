"""Heterogeneous ("ragged") batches for parity tests: worlds with different
agent and road-point counts, empty maps, single-point polylines, invalid log
steps (late entry, blink-outs, never valid), forced replay, and agents far
off the map."""

from __future__ import annotations

import numpy as np

from paper_2408_01584_b200.config import ROAD_KINDS
from paper_2408_01584_b200.packing import RawWorlds, concat_raw, _offsets
from paper_2408_01584_b200.synthetic import WaymoSpec, generate


def _single_point_roads(raw: RawWorlds, rng) -> RawWorlds:
    """Split the last point off some polylines as a 1-point stop_sign element
    (World.__init__ gives a single-point polyline heading 0, engine.py:259)."""
    stop = ROAD_KINDS.index("stop_sign")
    kinds, counts, per_world = [], [], []
    for w in range(raw.n_worlds):
        n = 0
        for r in range(raw.poly_off[w], raw.poly_off[w + 1]):
            m = int(raw.poly_pt_off[r + 1] - raw.poly_pt_off[r])
            if m >= 4 and rng.random() < 0.3:
                kinds += [raw.poly_kind[r], stop]
                counts += [m - 1, 1]
                n += 2
            else:
                kinds.append(raw.poly_kind[r])
                counts.append(m)
                n += 1
        per_world.append(n)
    raw.poly_kind = np.asarray(kinds, np.int8)
    raw.poly_pt_off = _offsets(counts)
    raw.poly_off = _offsets(per_world)
    return raw


def ragged_batch(seed: int = 0, num_steps: int = 91, quantize: bool = True) -> RawWorlds:
    rng = np.random.default_rng(seed)
    specs = [(1, 0), (5, 3), (33, 400), (130, 5000), (17, 1), (300, 2500), (64, 64), (2, 900)]
    parts = []
    for k, (A, P) in enumerate(specs):
        if P == 0:
            raw = generate(WaymoSpec(n_worlds=1, n_agents=A, n_points=12, seed=seed,
                                     world_offset=k, num_steps=num_steps, quantize=quantize))
            raw.poly_off = np.zeros(2, np.int64)
            raw.poly_kind = raw.poly_kind[:0]
            raw.poly_pt_off = np.zeros(1, np.int64)
            raw.pt_x = raw.pt_x[:0]
            raw.pt_y = raw.pt_y[:0]
        elif P < 10:
            raw = generate(WaymoSpec(n_worlds=1, n_agents=A, n_points=12, seed=seed,
                                     world_offset=k, num_steps=num_steps, quantize=quantize))
            raw.poly_off = np.array([0, 1], np.int64)
            raw.poly_kind = raw.poly_kind[:1]
            raw.poly_pt_off = np.array([0, P], np.int64)
            raw.pt_x = raw.pt_x[:P].copy()
            raw.pt_y = raw.pt_y[:P].copy()
        else:
            raw = generate(WaymoSpec(n_worlds=1, n_agents=A, n_points=P, seed=seed,
                                     world_offset=k, num_steps=num_steps, quantize=quantize))
        T = num_steps
        valid = raw.log_valid.reshape(A, T)
        for i in range(A):
            u = rng.random()
            if u < 0.08:
                valid[i, :rng.integers(1, T // 2)] = False          # late entry
            elif u < 0.16:
                a = rng.integers(1, T - 5)
                valid[i, a:a + rng.integers(1, 5)] = False           # blink-out
            elif u < 0.19:
                valid[i, :] = False                                  # never valid
        raw.log_valid = valid.reshape(-1)
        raw.force_replay = rng.random(A) < 0.1
        if A > 3:
            far = rng.integers(0, A)                                 # off the map
            lx = raw.log_x.reshape(A, T)
            lx[far] += 5000.0
            raw.log_x = lx.reshape(-1)
        parts.append(raw)
    raw = concat_raw(parts)
    return _single_point_roads(raw, rng)
