"""Throughput benchmark of the B200 batched world step (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
    python bench.py --impl reference ...      # CPU restatement of the reference

A "step" = one SimBatch.step over every world of the rank's shard: dynamics,
replay, collisions, goal/done, and observations for every controlled agent
(two kernels); with auto-reset of finished worlds (the reference benchmark's
semantics, engine.py:794-802).  Config c5 steps the VecDriveEnv with an
in-loop torch policy (the reference trainer's ActorCritic, ippo.py:48-66, in
bf16 on bf16 observations) and the fused device sampler choosing the
discrete actions.  Metric: agent-steps/s (ASPS = CASPS,
init_mode="all_valid"), whole job = sum over ranks.  Worlds shard across ranks
with no collective on the step path ("scaling": "weak": each rank owns the
configured world count; scene seed = global world id).  The working set (C3:
1.7 GB of observations written per step, 0.7 GB of road tables) exceeds the
126 MB L2, so no flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# name: worlds per GPU, agents, road points, dynamics, collision, obs kwargs, workload
CONFIGS = {
    "c1": (16, 32, 400, "classic", "ignore", {}, "C1 synthetic 16 worlds x 32 agents, 400 pts"),
    "c2": (1024, 64, 2000, "classic", "remove_agent", {},
           "C2 synthetic 1024 worlds x 64 agents, 2k pts, collision+goal reward"),
    "c3": (4096, 128, 10000, "delta_local", "ignore", {"radius": 50.0},
           "C3 Waymo-shaped 4096 worlds x 128 agents, 10k pts, r=50 m, delta-local"),
    "c4": (4096, 128, 10000, "classic", "ignore", {"mode": "lidar", "n_rays": 64},
           "C4 LiDAR 64 rays, 4096 worlds x 128 agents, 10k pts"),
    "c5": (1024, 128, 10000, "classic", "remove_agent", {"radius": 50.0},
           "C5 RL rollout: 1024 worlds/GPU (8192 on 8 GPUs) x 128 agents, 10k pts, "
           "VecDriveEnv + in-loop ActorCritic policy"),
}
# CPU sample of the same workload for the oracle legs: worlds stepped per "step"
L2_BYTES = 126 * 1024 * 1024   # B200 L2
CPU_WORLDS = {"c1": 16, "c2": 128, "c3": 64, "c4": 8, "c5": 64}


def bytes_per_agent_step(act_dim: int, width: int, P: int, A: int) -> dict:
    """Algorithmic (compulsory) HBM bytes per agent-step, SURVEY.md §8d:
    actions + FP64 state read/write + static agent fields + reward/done/info
    (step kernel) and the float32 observation row + road tables read once
    per world-step (x, y, heading f32 + kind u8 = 13 B per point, amortised
    over the A agents) + the agent state it reads (observation kernel)."""
    step_k = 4 * act_dim + 66 + 26 + 8
    obs_k = 4 * width + 13.0 * P / A + 66
    return {"total": step_k + 4 * width + 13.0 * P / A, "step_kernel": step_k, "obs_kernel": obs_k}


def radial_flops(P: int, A: int) -> float:
    """Reference linear-scan FP32 work: 5(P + A - 1) + 20*(16+64) + 40."""
    return 5.0 * (P + A - 1) + 20.0 * (16 + 64) + 40.0


def lidar_flops(pw, max_range: float, n_rays: int, worlds: int = 4) -> float:
    """sum over rays of 11 |candidate segments| + 30 |candidate
    boxes| with the reference's own candidate sets (segments whose AABB meets
    the +-max_range box, visible boxes within max_range + circumradius),
    counted exactly on the first worlds of the scene."""
    import numpy as np
    tot, n = 0.0, 0
    for w in range(min(worlds, pw.n_worlds)):
        a0, a1 = pw.a_off[w], pw.a_off[w + 1]
        s0, s1 = pw.s_off[w], pw.s_off[w + 1]
        X = pw.rep_x[pw.r_off[w]:pw.r_off[w] + (a1 - a0)]
        Y = pw.rep_y[pw.r_off[w]:pw.r_off[w] + (a1 - a0)]
        lx = np.minimum(pw.seg_ax[s0:s1], pw.seg_bx[s0:s1])
        hx = np.maximum(pw.seg_ax[s0:s1], pw.seg_bx[s0:s1])
        ly = np.minimum(pw.seg_ay[s0:s1], pw.seg_by[s0:s1])
        hy = np.maximum(pw.seg_ay[s0:s1], pw.seg_by[s0:s1])
        cr = pw.circumradius[a0:a1]
        for i in range(a1 - a0):
            segs = ((lx <= X[i] + max_range) & (hx >= X[i] - max_range) &
                    (ly <= Y[i] + max_range) & (hy >= Y[i] - max_range)).sum()
            d = np.hypot(X - X[i], Y - Y[i])
            boxes = ((d <= max_range + cr).sum() - 1)
            tot += n_rays * (11.0 * segs + 30.0 * boxes)
            n += 1
    return tot / max(n, 1)


class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms through NVML during the
    timed region (B200_PROFILING.md clocks line; the timed regions here are
    tens of milliseconds, too short for nvidia-smi -lms)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu_index: int):
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.REASONS:
                    if r & getattr(nv, attr):
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.005)

    def start(self):
        if self.nv is not None:
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()

    def stop(self) -> dict:
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self._stop.set()
        self.thread.join(timeout=2)
        sm = sorted(self.samples)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(sm)}


def load_traffic(config: str, kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/r1_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as f:
            return json.load(f)[config][kernel]
    except Exception:
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def sim_config(name):
    from paper_2408_01584_b200.config import ObsConfig, SimConfig
    W, A, P, dyn, coll, okw, _ = CONFIGS[name]
    return SimConfig(dynamics=dyn, collision_behavior=coll, init_mode="all_valid",
                     obs=ObsConfig(**okw))


class CpuSample:
    """The C oracle (restatement of the reference, bit-exact with it on the
    golden fixtures) stepping a bounded sample of the same workload on the
    host cores (OpenMP over worlds).  For c5 the reference trainer's policy
    runs on the CPU too."""

    def __init__(self, name: str, threads: int):
        import numpy as np
        from oracle.oracle import OracleBatch, build
        from paper_2408_01584_b200.packing import pack
        from paper_2408_01584_b200.synthetic import WaymoSpec, generate
        build()
        W, A, P = CONFIGS[name][:3]
        self.name, self.threads = name, threads
        self.cfg = sim_config(name)
        ws = min(CPU_WORLDS[name], W)
        raw = generate(WaymoSpec(n_worlds=ws, n_agents=A, n_points=P, seed=0))
        self.ora = OracleBatch(pack(raw, self.cfg), self.cfg, n_threads=threads)
        self.agents = int(self.ora.pw.n_instantiated.sum())
        self.rng = np.random.default_rng(0)
        self.desc = f"{ws} worlds x {A} agents"
        self.policy = None
        if name == "c5":
            import torch
            torch.set_num_threads(threads)
            from paper_2408_01584_b200.policy import ActorCritic
            from paper_2408_01584_b200.env import ActionGrid, obs_scale
            self.policy = ActorCritic(self.ora.width, 91)
            self.scale = torch.tensor(obs_scale(self.cfg), dtype=torch.float32)
            g = ActionGrid()
            self.accels = np.array(g.accelerations)
            self.steers = np.array(g.steerings)

    def step(self):
        import numpy as np
        n = self.ora.pw.n_controlled
        if self.policy is not None:
            import torch
            with torch.inference_mode():
                obs = torch.from_numpy(self.ora.observations).float() / self.scale
                logits, _ = self.policy(obs)
                idx = torch.distributions.Categorical(logits=logits).sample().numpy()
            act = np.column_stack([self.accels[idx // 13], self.steers[idx % 13]])
        elif self.cfg.dynamics == "delta_local":
            lo = np.array([b[0] for b in self.cfg.delta_bounds])
            hi = np.array([b[1] for b in self.cfg.delta_bounds])
            act = self.rng.uniform(lo, hi, (n, 3))
        else:
            act = self.rng.uniform([-4, -0.7], [4, 0.7], (n, 2))
        self.ora.step(act.astype(np.float32).astype(np.float64), auto_reset=True)

    def rate(self, steps: int, warmup: int = 1, budget_s: float = 30.0, min_s: float = 0.0):
        """At least `steps` steps (and at least min_s seconds of them), at
        most budget_s seconds."""
        for _ in range(warmup):
            self.step()
        t0 = time.perf_counter()
        k = 0
        while k < steps or time.perf_counter() - t0 < min_s:
            self.step()
            k += 1
            if time.perf_counter() - t0 > budget_s:
                break
        el = time.perf_counter() - t0
        return self.agents * k / el, f"{self.desc} x {k} steps ({el:.1f} s)"


def bench_config(name: str, W: int, W_total: int, world: int,
                 l2: str = "working set > L2 (no flush needed)") -> dict:
    """The `config` object of a bench line (both arms print the same one)."""
    from paper_2408_01584_b200.config import obs_width
    _, A, P, dyn, coll, okw, workload = CONFIGS[name]
    cfg = sim_config(name)
    return {"workload": workload, "worlds_per_gpu": W, "worlds_total": W_total,
            "agents": A, "road_points": P, "dynamics": dyn, "collision": coll,
            "obs_mode": cfg.obs.mode, "obs_width": obs_width(cfg.obs), "episode_steps": 91,
            "auto_reset": True, "l2": l2,
            "parallelism": f"world shards x {world} GPU (no step collective)"}


def run_reference(args, rank):
    """--impl reference: the reference's CPU path (oracle port) on the host
    cores, rank 0 only, one bounded-sample step per timed step."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    cs = CpuSample(args.config, threads)
    value, sample = cs.rate(args.steps, warmup=args.warmup, budget_s=120.0)
    W = args.worlds or CONFIGS[args.config][0]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    W_total = W if args.strong else W * world
    if args.strong:
        W = -(-W // world)
    line = {"impl": "reference", "metric": "agent_steps_per_sec", "value": value,
            "unit": "agent-steps/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.config, W, W_total, world),
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
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: the config's worlds split over the ranks "
                         "(default weak: the config's worlds on every rank)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2408_01584_b200.config import obs_width
    from paper_2408_01584_b200.engine import SimBatch, random_actions
    from paper_2408_01584_b200.synthetic import WaymoSpec, generate

    # DS_BENCH_SHARE_GPU=1 (test only): ranks share the visible GPUs over gloo,
    # to exercise the N > 1 path on a one-GPU box; never used for bench lines
    share = os.environ.get("DS_BENCH_SHARE_GPU") == "1"
    gpu = local_rank % torch.cuda.device_count() if share else local_rank
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    W, A, P, dyn, coll, okw, workload = CONFIGS[args.config]
    if args.worlds:
        W = args.worlds
    W_total = W * world
    w_off = rank * W
    if args.strong:
        import numpy as np
        from paper_2408_01584_b200.parallel import shard_ranges
        W_total = W
        lo, hi = shard_ranges(np.ones(W), world)[rank]
        W, w_off = hi - lo, lo
    cfg = sim_config(args.config)
    width = obs_width(cfg.obs)
    t_setup = time.perf_counter()
    raw = generate(WaymoSpec(n_worlds=W, n_agents=A, n_points=P, seed=0, world_offset=w_off))
    rl = args.config == "c5"
    if rl:
        from paper_2408_01584_b200.engine import sample_categorical
        from paper_2408_01584_b200.env import EnvConfig, VecDriveEnv
        from paper_2408_01584_b200.policy import ActorCritic
        # rollout formats: bf16 observations in rows padded to 8 (the policy
        # GEMM's input, no cast), a bf16 policy with 16-B aligned operands,
        # one fused sampler launch per step
        env = VecDriveEnv(EnvConfig(raw=raw, sim=cfg, device=str(dev), obs_dtype="bfloat16"))
        batch = env.batch
        policy = ActorCritic(width, env.n_actions, pad_to=8).to(dev).to(torch.bfloat16)
        obs0 = env.reset()
    else:
        batch = SimBatch.from_raw(raw, cfg, device=dev)
        acts = [random_actions(batch.n_controlled, cfg, 0, t, dev) for t in range(8)]
    t_setup = time.perf_counter() - t_setup
    n = batch.n_controlled
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    state = {"obs": obs0} if rl else {}

    def one_step(t, events=None):
        if rl:
            with torch.inference_mode():
                logits, value = policy(state["obs"])
                idx = sample_categorical(logits, seed=1234 + rank, counter=t)
            obs, rew, done, infos = env.step(idx)
            state["obs"] = obs
            return rew
        return batch.step(acts[t % 8], auto_reset=True, events=events).rewards

    def restart():
        # every timed leg covers the same episode phase (steps W .. W+K after
        # a reset): work per step changes over an episode (remove_agent)
        if rl:
            state["obs"] = env.reset()
        else:
            batch.reset()
        torch.cuda.synchronize(dev)

    restart()
    for t in range(args.warmup):
        one_step(t)
    torch.cuda.synchronize(dev)

    # ---- device-resident timed region (inputs already in HBM); the
    # per-kernel split comes from a separate pass after it (no event records
    # inside the timed steps)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    # small working sets (C1, C2 at a few worlds) would stay L2-resident across
    # steps: flush L2 (write 2x its size) before every timed step and time the
    # steps individually instead
    ws = torch.cuda.memory_allocated(dev)
    flush_l2 = ws < L2_BYTES * 2
    l2_note = (f"L2 flushed before each timed step (working set {ws / 1e6:.0f} MB)" if flush_l2
               else f"working set {ws / 1e6:.0f} MB > 2x L2 (no flush needed)")
    flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush_l2 else None
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.05)
    barrier()
    torch.cuda.synchronize(dev)
    start.record(stream)
    for t in range(args.steps):
        if flush_l2:
            flush_buf.fill_(float(t))
            step_ev[t][0].record(stream)
        one_step(t)
        if flush_l2:
            step_ev[t][1].record(stream)
    end.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clocks = sampler.stop()
    ms = start.elapsed_time(end)
    if flush_l2:
        ms = sum(a.elapsed_time(b) for a, b in step_ev)
    kernel_ms = None
    if not rl:
        # per-kernel split (CUDA events on the launching stream around each
        # kernel) over a further pass of the same steps, L2 flushed likewise
        n_ev = min(args.steps, 10)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_ev)]
        for e3 in ev:           # materialise the CUDA events (ds_step records raw handles)
            for e in e3:
                e.record(stream)
        restart()
        for t in range(args.warmup):
            one_step(t)
        for t in range(n_ev):
            if flush_l2:
                flush_buf.fill_(float(t))
            one_step(t, events=ev[t])
        torch.cuda.synchronize(dev)
        kernel_ms = {"step_kernel": sum(e[0].elapsed_time(e[1]) for e in ev) / n_ev,
                     "obs_kernel": sum(e[1].elapsed_time(e[2]) for e in ev) / n_ev}
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    # units all ranks processed: every rank's agents (allreduce of the counts)
    agents_total = batch.total_agents
    if world > 1:
        ta = torch.tensor([float(agents_total)], device=dev)
        dist.all_reduce(ta)
        agents_total = int(ta.item())
    value = agents_total * args.steps / (ms / 1e3)

    # ---- end to end through the public API with host buffers: every step
    # copies its inputs from pinned host memory to the device and its result
    # back (c1-c4: actions in, rewards/dones/info out through HostStepper,
    # whose copies overlap the kernels; c5: the policy samples the actions on
    # the device, the step's reward sum comes back).
    if rl:
        rsum_h = torch.empty(1, dtype=torch.float32).pin_memory()
        h2d, d2h = 0, 4
    else:
        from paper_2408_01584_b200.engine import HostStepper
        stepper = HostStepper(batch, act_dim=acts[0].shape[1])
        host_acts = [a.cpu().pin_memory() for a in acts]
        h2d, d2h = stepper.h2d_bytes_per_step, stepper.d2h_bytes_per_step
    def e2e_step(t):
        if rl:
            rew = one_step(t)
            rsum_h.copy_(rew.sum().reshape(1), non_blocking=True)
        else:
            stepper.step(host_acts[t % 8])

    restart()
    for t in range(args.warmup):          # untimed warm-up of this leg's own ops
        e2e_step(t)
    barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if not rl:
        stepper._h2d.wait_event(e0)        # the first action copy is inside the region
    for t in range(args.steps):
        e2e_step(t)
    if not rl:
        stream.wait_stream(stepper._d2h)   # the last result copy is inside the region
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = agents_total * args.steps / (e2e_ms / 1e3)

    # ---- episode statistics: the only collective, off the step path
    from paper_2408_01584_b200.parallel import allreduce_episode_stats, episode_stats
    stats = allreduce_episode_stats(episode_stats(batch.episode_infos), device=dev)

    # ---- roofline of the dominant kernel (the observation kernel)
    peak, peak_kind = load_peaks()
    act_dim = 1 if rl else acts[0].shape[1]
    bpa = bytes_per_agent_step(act_dim, width, P, A)
    fl = radial_flops(P, A) if cfg.obs.mode == "radial" else \
        lidar_flops(batch.packed, cfg.obs.max_range, cfg.obs.n_rays)
    hbm_bound = peak * 1e9 / bpa["total"]
    fp32_bound = 74.4e12 / fl
    roofline = None
    if kernel_ms is not None:
        achieved = bpa["obs_kernel"] * batch.n_controlled / (kernel_ms["obs_kernel"] / 1e3) / 1e9
        kname = "obs_radial_kernel" if cfg.obs.mode == "radial" else "obs_lidar_kernel"
        tr = load_traffic(args.config, kname) if (args.worlds or W) == CONFIGS[args.config][0] else None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": tr / 1e9 if tr else None,
                    "traffic_unit": "GB per launch (ncu dram__bytes_read+write)",
                    "algorithmic_gb_per_launch": bpa["obs_kernel"] * batch.n_controlled / 1e9,
                    "kernel": kname,
                    "bytes_per_agent_step": bpa["obs_kernel"], "peak_kind": peak_kind}
    if rank == 0:
        cpu = None
        # the CPU baseline leg runs at N = 1 only (rank 0); N > 1 lines reuse it
        if not args.no_cpu_baseline and world == 1:
            threads = os.cpu_count() or 1
            try:
                v, sample = CpuSample(args.config, threads).rate(91, warmup=1, budget_s=20.0,
                                                                  min_s=10.0)
                cpu = {"value": v, "unit": "agent-steps/s", "cores": threads, "kind": "port",
                       "sample": sample}
            except Exception as exc:   # report, never fake
                cpu = {"value": None, "unit": "agent-steps/s", "cores": threads, "kind": "port",
                       "sample": f"failed: {exc!r}"}
        total = max(int(stats[1]), 1)
        result = {
            "metric": "agent_steps_per_sec", "value": value, "unit": "agent-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.config, W, W_total, world, l2_note),
            "e2e": {"value": e2e_value, "unit": "agent-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": (2 * args.steps) if not rl else 3 * args.steps,
            "roofline": roofline,
            "step_roofline": {"bytes_per_agent_step": bpa["total"],
                              "fp32_flop_per_agent_step": fl, "hbm_bound_asps": hbm_bound,
                              "fp32_bound_asps": fp32_bound,
                              "bound_asps": min(hbm_bound, fp32_bound),
                              "frac": (value / world) / min(hbm_bound, fp32_bound)},
            "kernel_ms": kernel_ms,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "episodes": {"count": int(stats[0]), "goal_rate": stats[2] / total,
                         "veh_collision_rate": stats[3] / total, "offroad_rate": stats[4] / total},
            "setup_s": t_setup,
        }
        print(json.dumps(result), flush=True)
    batch.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
