"""Multi-GPU data parallelism over worlds.

Worlds are share-nothing (engine.py:4-7), so one process per GPU owns a
contiguous shard of worlds and steps it with no collective on the step path;
the global flat output is the concatenation of the shards in world order,
which matches the reference's ``offsets`` (engine.py:599-601).  The only
collective is the optional episode-statistics reduction (eng:151-163), done
with torch.distributed (NCCL over NVLink on the GPU box, gloo in CPU tests)
off the step stream.
"""

from __future__ import annotations

import numpy as np


def shard_ranges(costs, n_shards: int) -> list:
    """Contiguous [start, stop) world ranges balancing the summed cost
    (e.g. agents + road points per world) over n_shards.  Every shard gets at
    least one world when there are enough worlds."""
    costs = np.asarray(costs, dtype=np.float64)
    W = len(costs)
    if n_shards < 1:
        raise ValueError("n_shards must be >= 1")
    if W == 0:
        return [(0, 0)] * n_shards
    cum = np.concatenate([[0.0], np.cumsum(costs)])
    total = cum[-1]
    bounds = [0]
    for s in range(1, n_shards):
        target = total * s / n_shards
        b = int(np.searchsorted(cum, target, side="left"))
        lo = bounds[-1] + (1 if W - bounds[-1] > n_shards - s else 0)
        hi = W - (n_shards - s)
        bounds.append(int(min(max(b, lo), max(hi, lo))))
    bounds.append(W)
    return [(bounds[i], bounds[i + 1]) for i in range(n_shards)]


def world_costs(raw) -> np.ndarray:
    """Agents + road points per world of a RawWorlds batch."""
    agents = np.diff(raw.a_off)
    pts = raw.poly_pt_off[raw.poly_off[1:]] - raw.poly_pt_off[raw.poly_off[:-1]]
    return agents.astype(np.float64) + pts.astype(np.float64) / 64.0


STAT_FIELDS = ("n_controlled", "n_goal", "n_veh_collision", "n_offroad")


def episode_stats(episode_infos) -> np.ndarray:
    """[episodes, n_controlled, n_goal, n_veh_collision, n_offroad] sums."""
    out = np.zeros(5, np.int64)
    out[0] = len(episode_infos)
    for e in episode_infos:
        out[1] += e.n_controlled
        out[2] += e.n_goal
        out[3] += e.n_veh_collision
        out[4] += e.n_offroad
    return out


def allreduce_episode_stats(local: np.ndarray, device=None) -> np.ndarray:
    """Sum the per-rank statistics over the process group (one small
    all-reduce, off the step path)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(np.asarray(local), dtype=torch.int64)   # copy: all_reduce is in place
    if device is not None:
        t = t.to(device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
    return t.cpu().numpy()


def metrics_from_stats(stats: np.ndarray) -> dict:
    """compute_metrics (engine.py:151-163) from reduced sums."""
    total = int(stats[1])
    if stats[0] == 0:
        raise ValueError("no completed episodes")
    if total == 0:
        return {"goal_rate": 0.0, "veh_collision_rate": 0.0, "offroad_rate": 0.0,
                "episodes": int(stats[0])}
    return {"goal_rate": stats[2] / total, "veh_collision_rate": stats[3] / total,
            "offroad_rate": stats[4] / total, "episodes": int(stats[0])}
