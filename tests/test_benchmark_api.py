"""engine.benchmark / ThroughputReport / compute_metrics: the reference's
benchmark surface (engine.py:136-163, 535-556, 811-857) on the GPU batch."""

import math

import pytest

from paper_2408_01584_b200.config import SimConfig
from paper_2408_01584_b200.engine import SimBatch, benchmark, compute_metrics, random_actions
from scenes import hold, scene, scripted_object

pytestmark = pytest.mark.gpu


def _scenarios():
    a = scripted_object(0, hold(0.0, 0.0, 0.0, 91), goal=(60.0, 0.0), speed=5.0)
    b = scripted_object(1, hold(0.0, 20.0, math.pi, 91), goal=(-60.0, 20.0), speed=5.0)
    c = scripted_object(2, hold(30.0, -20.0, 0.5, 91), goal=(90.0, 0.0), speed=3.0)
    return [scene([a, b]), scene([a, b, c])]


@pytest.mark.parametrize("policy", ["random", "constant:1.0:0.1", "replay", "goal_seek"])
def test_benchmark_report(policy):
    cfg = SimConfig(init_mode="all_valid")
    rep = benchmark(_scenarios(), cfg, worlds=6, steps=20, policy=policy, device="cuda:0")
    assert rep.worlds == 6 and rep.steps == 20 and rep.elapsed_s > 0
    assert rep.total_agents == 3 * 2 + 3 * 3          # worlds cycle the scenario list
    assert rep.controlled_agents == rep.total_agents   # all_valid
    assert rep.asps == pytest.approx(rep.steps * rep.total_agents / rep.elapsed_s)
    assert rep.casps == pytest.approx(rep.asps)


def test_benchmark_rejects_bad_arguments():
    cfg = SimConfig(init_mode="all_valid")
    with pytest.raises(ValueError):
        benchmark(_scenarios(), cfg, worlds=0, steps=5, device="cuda:0")
    with pytest.raises(ValueError):
        benchmark(_scenarios(), cfg, worlds=2, steps=5, policy="nonsense", device="cuda:0")


def test_metrics_over_full_episodes():
    cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent")
    b = SimBatch(_scenarios(), cfg, device="cuda:0")
    for t in range(2 * 91):
        b.step(random_actions(b.n_controlled, cfg, 3, t, "cuda:0"), auto_reset=True)
    eps = b.episode_infos
    assert len(eps) == 2 * 2                           # two worlds, two episodes each
    m = compute_metrics(eps)
    n = sum(e.n_controlled for e in eps)
    assert n == 2 * (2 + 3)
    for rate, count in ((m.goal_rate, "n_goal"), (m.veh_collision_rate, "n_veh_collision"),
                        (m.offroad_rate, "n_offroad")):
        assert rate == pytest.approx(sum(getattr(e, count) for e in eps) / n)
    assert b.compute_metrics() == m
    b.close()
