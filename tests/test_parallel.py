"""Multi-process (world_size 2, gloo on CPU) coverage of the world sharding
and the episode-statistics reduction (the only collective)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2408_01584_b200.parallel import (episode_stats, metrics_from_stats, shard_ranges,
                                            world_costs)


def test_shard_ranges_partition_and_balance():
    rng = np.random.default_rng(0)
    for W in (1, 2, 7, 64, 4096):
        for n in (1, 2, 4, 8):
            costs = rng.integers(1, 100, W)
            r = shard_ranges(costs, n)
            assert r[0][0] == 0 and r[-1][1] == W
            assert all(a[1] == b[0] for a, b in zip(r[:-1], r[1:]))
            if W >= n:
                assert all(b > a for a, b in r)
            if W >= 64:
                loads = [costs[a:b].sum() for a, b in r]
                assert max(loads) <= costs.sum() / n + costs.max()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2408_01584_b200.config import SimConfig
    from paper_2408_01584_b200.packing import pack
    from paper_2408_01584_b200.parallel import allreduce_episode_stats
    from paper_2408_01584_b200.synthetic import WaymoSpec, generate
    from oracle.oracle import OracleBatch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W = 6
    ranges = shard_ranges(np.ones(W), world)
    lo, hi = ranges[rank]
    cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent")
    # each rank generates ONLY its own world ids (global seeds) and steps them
    raw = generate(WaymoSpec(n_worlds=hi - lo, n_agents=16, n_points=300, seed=3,
                             world_offset=lo, num_steps=12))
    ora = OracleBatch(raw, cfg)
    rng = np.random.default_rng(100 + lo)
    for _ in range(12):
        ora.step(rng.uniform(-1, 1, (ora.pw.n_controlled, 2)))
    local = np.zeros(5, np.int64)
    local[0] = len(ora.episode_infos)
    for (_, nc, ng, nv, no) in ora.episode_infos:
        local[1:] += (nc, ng, nv, no)
    total = allreduce_episode_stats(local)
    q.put((rank, lo, hi, local.tolist(), total.tolist(),
           [float(v) for v in ora.observations.sum(1)]))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_shards_and_stats():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, l0, t0, o0), (r1, lo1, hi1, l1, t1, o1) = res
    assert (lo0, hi1) == (0, 6) and hi0 == lo1
    assert t0 == t1 == (np.array(l0) + np.array(l1)).tolist()
    assert t0[0] == 6                     # every world finished its 12-step episode
    m = metrics_from_stats(np.array(t0))
    assert 0.0 <= m["goal_rate"] <= 1.0
    # the sharded run equals one unsharded run of all six worlds
    from paper_2408_01584_b200.config import SimConfig
    from paper_2408_01584_b200.packing import pack
    from paper_2408_01584_b200.synthetic import WaymoSpec, generate
    from oracle.oracle import OracleBatch
    cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent")
    parts = []
    for lo, hi in ((lo0, hi0), (lo1, hi1)):
        raw = generate(WaymoSpec(n_worlds=hi - lo, n_agents=16, n_points=300, seed=3,
                                 world_offset=lo, num_steps=12))
        ora = OracleBatch(raw, cfg)
        rng = np.random.default_rng(100 + lo)
        for _ in range(12):
            ora.step(rng.uniform(-1, 1, (ora.pw.n_controlled, 2)))
        parts.extend(ora.observations.sum(1).tolist())
    assert parts == o0 + o1


def test_world_costs_and_stats_helpers():
    from paper_2408_01584_b200.synthetic import WaymoSpec, generate
    raw = generate(WaymoSpec(n_worlds=3, n_agents=8, n_points=128))
    c = world_costs(raw)
    assert c.shape == (3,) and (c == 8 + 128 / 64).all()

    class E:
        def __init__(self, *v):
            self.n_controlled, self.n_goal, self.n_veh_collision, self.n_offroad = v
    s = episode_stats([E(4, 3, 1, 0), E(2, 0, 2, 2)])
    assert s.tolist() == [2, 6, 3, 3, 2]
    m = metrics_from_stats(s)
    assert m["goal_rate"] == 0.5 and m["episodes"] == 2
