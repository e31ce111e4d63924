"""Throughput benchmark of the B200 batched world step (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
    python bench.py --impl reference ...      # CPU restatement of the reference

A "step" = one SimBatch.step over every world of the rank's shard: dynamics,
replay, collisions, goal/done, and observations for every controlled agent
(two kernels).  Metric: agent-steps/s (ASPS = CASPS, init_mode="all_valid"),
whole job = sum over ranks.  Worlds shard across ranks with no collective on
the step path ("scaling": "weak": each rank owns the configured world count).
The working set (C3: 1.7 GB of observations written per step, 1.4 GB of road
tables) exceeds the 126 MB L2, so no flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (worlds per GPU, agents, road points, dynamics, collision, obs kwargs, workload)
    "c1": (16, 32, 400, "classic", "ignore", {}, "C1 synthetic 16 worlds x 32 agents, 400 pts"),
    "c2": (1024, 64, 2000, "classic", "remove_agent", {},
           "C2 synthetic 1024 worlds x 64 agents, 2k pts, collision+goal"),
    "c3": (4096, 128, 10000, "delta_local", "ignore", {"radius": 50.0},
           "C3 Waymo-shaped 4096 worlds x 128 agents, 10k pts, r=50 m, delta-local"),
    "c4": (4096, 128, 10000, "classic", "ignore", {"mode": "lidar", "n_rays": 64},
           "C4 LiDAR 64 rays, 4096 worlds x 128 agents, 10k pts"),
}
# CPU sample (worlds, steps) per config for the oracle timing legs (~10-30 s of CPU)
CPU_SAMPLE = {"c1": (16, 91), "c2": (64, 10), "c3": (32, 3), "c4": (8, 1)}


def bytes_per_agent_step(cfg_name: str, act_dim: int, width: int, P: int, A: int) -> dict:
    """Algorithmic (compulsory) HBM bytes per agent-step, SURVEY.md §8d:
    actions + FP64 state read/write + static agent fields + obs row (f32) +
    reward/done/info + road tables read once per world-step (x,y f32 +
    heading f32 + kind u8 = 13 B per point, amortised over the A agents)."""
    step_k = 4 * act_dim + 66 + 26 + 8
    obs_k = 4 * width + 13.0 * P / A + 66
    return {"total": step_k + 4 * width + 13.0 * P / A, "step_kernel": step_k, "obs_kernel": obs_k}


def flops_per_agent_step(width_mode: str, P: int, A: int) -> float:
    """Reference linear-scan FP32 work: 5(P + A - 1) + 20*(16+64) + 40."""
    return 5.0 * (P + A - 1) + 20.0 * (16 + 64) + 40.0


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu_index: int):
        self.rows = []
        self.proc = None
        self.gpu = gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 7 for k in range(4)
                          if r[3 + k].lower() == "active"})
        sm_sorted = sorted(sm)
        return {"sm_mhz": sm_sorted[len(sm_sorted) // 2] if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_oracle_rate(cfg_name: str, threads: int, budget_s: float = 20.0):
    """Oracle (C restatement of the reference, bit-exact with it) on host cores:
    a bounded sample of the same workload; returns (ASPS, sample description)."""
    from paper_2408_01584_b200.config import ObsConfig, SimConfig
    from paper_2408_01584_b200.packing import pack
    from paper_2408_01584_b200.synthetic import WaymoSpec, generate
    from oracle.oracle import OracleBatch
    import numpy as np
    W, A, P, dyn, coll, okw, _ = CONFIGS[cfg_name]
    ws, max_steps = CPU_SAMPLE[cfg_name]
    cfg = SimConfig(dynamics=dyn, collision_behavior=coll, init_mode="all_valid",
                    obs=ObsConfig(**okw))
    raw = generate(WaymoSpec(n_worlds=ws, n_agents=A, n_points=P, seed=0))
    ora = OracleBatch(pack(raw, cfg), cfg, n_threads=threads)
    rng = np.random.default_rng(0)
    n = ora.pw.n_controlled
    steps = 0
    t0 = time.perf_counter()
    while True:
        if cfg.dynamics == "delta_local":
            act = rng.uniform(-0.9, 0.9, (n, 3))
        else:
            act = rng.uniform([-4, -0.7], [4, 0.7], (n, 2))
        ora.step(act.astype(np.float32).astype(np.float64), auto_reset=True)
        steps += 1
        el = time.perf_counter() - t0
        if steps >= max_steps or el > budget_s:
            break
    asps = steps * int(ora.pw.n_instantiated.sum()) / el
    return asps, f"{ws} worlds x {A} agents x {steps} steps ({el:.1f} s)"


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from oracle import oracle as _o
    _o.build()
    vals = []
    sample = ""
    for _ in range(args.warmup):
        cpu_oracle_rate(args.config, threads, budget_s=2.0)
    for _ in range(args.steps):
        v, sample = cpu_oracle_rate(args.config, threads, budget_s=10.0)
        vals.append(v)
    value = sum(vals) / len(vals)
    W, A, P, dyn, coll, okw, workload = CONFIGS[args.config]
    line = {"impl": "reference", "metric": "agent_steps_per_sec", "value": value,
            "unit": "agent-steps/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "worlds": W, "agents": A, "road_points": P,
                       "dynamics": dyn, "collision": coll, "obs": okw or {"mode": "radial"}},
            "cpu_baseline": {"value": value, "unit": "agent-steps/s", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "agent-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--worlds", type=int, default=None, help="override worlds per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2408_01584_b200.config import ObsConfig, SimConfig, obs_width
    from paper_2408_01584_b200.engine import SimBatch, random_actions
    from paper_2408_01584_b200.synthetic import WaymoSpec, generate

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    W, A, P, dyn, coll, okw, workload = CONFIGS[args.config]
    if args.worlds:
        W = args.worlds
    cfg = SimConfig(dynamics=dyn, collision_behavior=coll, init_mode="all_valid",
                    obs=ObsConfig(**okw))
    t_gen = time.perf_counter()
    raw = generate(WaymoSpec(n_worlds=W, n_agents=A, n_points=P, seed=0, world_offset=rank * W))
    batch = SimBatch.from_raw(raw, cfg, device=dev)
    t_gen = time.perf_counter() - t_gen
    n = batch.n_controlled
    width = obs_width(cfg.obs)
    acts = [random_actions(n, cfg, 0, t, dev) for t in range(8)]
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    for t in range(args.warmup):
        batch.step(acts[t % 8], auto_reset=True)
    torch.cuda.synchronize(dev)

    # ---- device-resident timed region (inputs already in HBM)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    for e3 in ev:
        for e in e3:
            e.record(stream)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize(dev)
    start.record(stream)
    for t in range(args.steps):
        batch.step(acts[t % 8], auto_reset=True, events=ev[t])
    end.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clocks = sampler.stop()
    ms = start.elapsed_time(end)
    step_ms = sum(e3[0].elapsed_time(e3[1]) for e3 in ev) / args.steps
    obs_ms = sum(e3[1].elapsed_time(e3[2]) for e3 in ev) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    agents_total = batch.total_agents * world
    value = agents_total * args.steps / (ms / 1e3)
    gpu_launches = 2 * args.steps

    # ---- end-to-end through the public API with host buffers: pinned host
    # actions -> device each step, rewards/dones/info -> host each step.
    e2e_steps = args.e2e_steps or args.steps
    host_acts = [a.cpu().pin_memory() for a in acts]
    rew_h = torch.empty(n, dtype=torch.float32).pin_memory()
    done_h = torch.empty(n, dtype=torch.bool).pin_memory()
    info_h = torch.empty((3, n), dtype=torch.bool).pin_memory()
    barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(e2e_steps):
        d_act = host_acts[t % 8].to(dev, non_blocking=True)
        out = batch.step(d_act, auto_reset=True)
        rew_h.copy_(out.rewards, non_blocking=True)
        done_h.copy_(out.dones, non_blocking=True)
        info_h.copy_(batch._info[:, :n], non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = agents_total * e2e_steps / (e2e_ms / 1e3)
    h2d = host_acts[0].numel() * 4
    d2h = n * 4 + n + 3 * n

    # ---- episode statistics (the only collective; off the step path)
    infos = batch.episode_infos
    stats = torch.tensor([sum(e.n_controlled for e in infos), sum(e.n_goal for e in infos),
                          sum(e.n_veh_collision for e in infos), sum(e.n_offroad for e in infos),
                          len(infos)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(stats)

    # ---- roofline of the dominant kernel (observation kernel)
    peak, peak_kind = load_peaks()
    bpa = bytes_per_agent_step(args.config, acts[0].shape[1], width, P, A)
    obs_bytes = bpa["obs_kernel"] * batch.n_controlled
    achieved = obs_bytes / (obs_ms / 1e3) / 1e9
    step_bytes = bpa["total"] * batch.total_agents
    fl = flops_per_agent_step(cfg.obs.mode, P, A)
    hbm_bound = peak * 1e9 / bpa["total"]
    fp32_bound = 74.4e12 / fl
    result = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            try:
                v, sample = cpu_oracle_rate(args.config, threads)
                cpu = {"value": v, "unit": "agent-steps/s", "cores": threads, "kind": "port",
                       "sample": sample}
            except Exception as exc:  # report, never fake
                cpu = {"value": None, "unit": "agent-steps/s", "cores": threads, "kind": "port",
                       "sample": f"failed: {exc}"}
        result = {
            "metric": "agent_steps_per_sec", "value": value, "unit": "agent-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "worlds_per_gpu": W, "agents": A, "road_points": P,
                       "dynamics": dyn, "collision": coll, "obs_mode": cfg.obs.mode,
                       "obs_width": width, "episode_steps": 91, "auto_reset": True,
                       "l2": "working set > L2 (no flush needed)", "parallelism": f"worlds/{world} GPU"},
            "e2e": {"value": e2e_value, "unit": "agent-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": gpu_launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "obs_radial_kernel" if cfg.obs.mode == "radial" else "obs_lidar_kernel",
                         "bytes_per_agent_step": bpa["obs_kernel"], "peak_kind": peak_kind},
            "step_roofline": {"bytes_per_agent_step": bpa["total"], "fp32_flop_per_agent_step": fl,
                              "hbm_bound_asps": hbm_bound, "fp32_bound_asps": fp32_bound,
                              "bound_asps": min(hbm_bound, fp32_bound),
                              "frac": (value / world) / min(hbm_bound, fp32_bound)},
            "kernel_ms": {"step_kernel": step_ms, "obs_kernel": obs_ms},
            "clocks": clocks,
            "cpu_baseline": cpu,
            "episodes": {"count": int(stats[4].item()),
                         "goal_rate": float(stats[1] / max(stats[0].item(), 1)),
                         "veh_collision_rate": float(stats[2] / max(stats[0].item(), 1)),
                         "offroad_rate": float(stats[3] / max(stats[0].item(), 1))},
            "setup_s": t_gen,
        }
        print(json.dumps(result), flush=True)
    batch.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
