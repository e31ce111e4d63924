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
with no collective on the step path (scene seed = global world id): at N = 1
the config's worlds; at N > 1 the main line is STRONG scaling (the config's
worlds split into contiguous shards) plus a "weak" sub-object (the config's
worlds on every rank), BASELINE.md §3.4.  `--gpus N` outside torchrun
launches the N ranks itself.  Rank 0 at N = 1 also steps one full episode of
the benched batch against the C oracle on the host cores: the line's
"parity" verdict and its "cpu_baseline".  The working set (C3:
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


TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r2_traffic.json")
FP_PEAKS_FILE = os.path.join(ROOT, "profiles", "r2_fp_peaks.json")
LIDAR_WORK_FILE = os.path.join(ROOT, "profiles", "r2_lidar_work.json")


def load_json(path: str):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def load_traffic(config: str, kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/r2_traffic.json, tools/ncu_traffic.py), or None."""
    try:
        return load_json(TRAFFIC_FILE)[config][kernel]
    except Exception:
        return None


def fp_peaks() -> tuple:
    """(FP32, FP64) FMA peaks in FLOP/s and their source: measured on a B200
    by tools/fp_peak.cu (profiles/r2_fp_peaks.json), else derived from the SM
    count and clock (148 SMs x 128 / 64 lanes x 2 x 1.965 GHz)."""
    p = load_json(FP_PEAKS_FILE)
    if p and p.get("fp32_tflops") and p.get("fp64_tflops"):
        return p["fp32_tflops"] * 1e12, p["fp64_tflops"] * 1e12, "measured (tools/fp_peak.cu)"
    return 74.4e12, 37.2e12, "derived (148 SMs x lanes x 2 x 1.965 GHz)"


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
    golden fixtures; its own table builder, no product code) stepping a
    bounded sample of the same workload on the host cores (OpenMP over
    worlds).  For c5 the reference trainer's policy runs on the CPU too."""

    def __init__(self, name: str, threads: int):
        import numpy as np
        from oracle.oracle import OracleBatch, build
        from paper_2408_01584_b200.synthetic import WaymoSpec, generate
        build()
        W, A, P = CONFIGS[name][:3]
        self.name, self.threads = name, threads
        self.cfg = sim_config(name)
        ws = min(CPU_WORLDS[name], W)
        raw = generate(WaymoSpec(n_worlds=ws, n_agents=A, n_points=P, seed=0))
        self.ora = OracleBatch(raw, self.cfg, n_threads=threads)
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


def leg_worlds(args, world: int, rank: int):
    """(worlds on this rank, global id of its first world, worlds in the job)
    of the main line: N = 1 the config's worlds; N > 1 STRONG scaling, the
    config's worlds split into contiguous shards."""
    total = args.worlds or CONFIGS[args.config][0]
    if world == 1:
        return total, 0, total
    import numpy as np
    from paper_2408_01584_b200.parallel import shard_ranges
    lo, hi = shard_ranges(np.ones(total), world)[rank]
    return hi - lo, lo, total


def bench_config(name: str, W: int, W_total: int, world: int, scaling: str) -> dict:
    """The `config` object of a bench line (both arms print the same one)."""
    from paper_2408_01584_b200.config import obs_width
    _, A, P, dyn, coll, okw, workload = CONFIGS[name]
    cfg = sim_config(name)
    return {"workload": workload, "worlds_per_gpu": W, "worlds_total": W_total,
            "agents": A, "road_points": P, "dynamics": dyn, "collision": coll,
            "obs_mode": cfg.obs.mode, "obs_width": obs_width(cfg.obs), "episode_steps": 91,
            "auto_reset": True,
            "parallelism": f"world shards x {world} GPU (no step collective), {scaling} scaling"}


def run_reference(args, rank):
    """--impl reference: the reference's CPU path (oracle port) on the host
    cores, rank 0 only, one bounded-sample step per timed step."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    cs = CpuSample(args.config, threads)
    value, sample = cs.rate(args.steps, warmup=args.warmup, budget_s=120.0)
    world = args.gpus
    W, _, W_total = leg_worlds(args, world, 0)
    scaling = "strong" if world > 1 else "weak"
    line = {"impl": "reference", "metric": "agent_steps_per_sec", "value": value,
            "unit": "agent-steps/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.config, W, W_total, world, scaling),
            "cpu_baseline": {"value": value, "unit": "agent-steps/s", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "agent-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def parity_check(batch, raw, cfg, dev, n_worlds: int, steps: int, threads: int) -> tuple:
    """The bench's own parity verdict and CPU baseline in one pass: a full
    episode of the benched batch (reset, `steps` steps of the bench's device
    actions, no auto-reset) against the C oracle stepping the first
    `n_worlds` worlds with the same actions on the host cores.  Flags
    (rewards, dones, goal / collision / off-road) and the partner / road-point
    selection indices must be bit-exact, float32 observations within
    2 ulp + 1e-6 of the FP64 oracle, FP64 poses within 1e-9 m / 1e-12 rad.
    Returns (parity dict, cpu_baseline dict)."""
    import numpy as np
    import torch
    from oracle.oracle import OracleBatch, build
    from paper_2408_01584_b200.engine import random_actions
    build()
    nw = min(n_worlds, batch.n_worlds)
    OracleBatch.lidar_ties()
    ora = OracleBatch(raw.subset(range(nw)), cfg, n_threads=threads)
    rows = int(batch.offsets[nw])
    n_ag = int(batch.packed.a_off[nw])
    if ora.pw.n_controlled != rows or ora.pw.n_agents != n_ag:
        raise RuntimeError("oracle and batch disagree on the controlled rows")
    radial = cfg.obs.mode == "radial"
    sel_w = cfg.obs.max_agents_obs + cfg.obs.max_road_points_obs
    sel = torch.full((batch.n_controlled, sel_w), -7, dtype=torch.int32, device=dev) if radial else None
    batch.reset(sel_idx=sel)
    res = {"worlds": nw, "rows": rows, "steps": steps, "flag_mismatches": 0, "sel_mismatches": 0,
           "obs_out_of_tol": 0, "max_obs_err": 0.0,
           "tolerance": "flags/indices bit-exact; obs 2 f32 ulp + 1e-6; poses 1e-9 m, 1e-12 rad"}

    def compare(o_obs, o_rew, o_done, o_info, flags=True):
        got = batch.observations[:rows].cpu().numpy().astype(np.float64)
        ref = o_obs.astype(np.float32)
        err = np.abs(got - ref.astype(np.float64))
        tol = 2.0 * np.spacing(np.abs(ref)).astype(np.float64) + 1e-6
        res["obs_out_of_tol"] += int((err > tol).sum())
        res["max_obs_err"] = max(res["max_obs_err"], float(err.max()) if err.size else 0.0)
        if flags:
            bad = (batch.rewards[:rows].cpu().numpy() != o_rew.astype(np.float32)) | \
                  (batch.dones[:rows].cpu().numpy() != o_done)
            info = batch._info[:, :rows].cpu().numpy()
            for k, key in enumerate(("goal", "veh_collision", "offroad")):
                bad |= info[k] != o_info[key]
            res["flag_mismatches"] += int(bad.sum())
        if radial:
            res["sel_mismatches"] += int((sel[:rows].cpu().numpy() != ora.sel_idx[:rows]).any(1).sum())

    # after reset only the observations / selections are outputs (engine.py:651-663)
    compare(ora.observations, None, None, None, flags=False)
    cpu_s = 0.0
    for t in range(1, steps + 1):
        act = random_actions(batch.n_controlled, cfg, 0, t, dev)
        batch.step(act, sel_idx=sel)
        a_h = act[:rows].cpu().numpy().astype(np.float64)
        t0 = time.perf_counter()
        o = ora.step(a_h)
        cpu_s += time.perf_counter() - t0
        compare(*o)
    x, y, h = (v[:n_ag].cpu().numpy() for v in (batch._x, batch._y, batch._h))
    res["max_pose_err_m"] = float(max(np.abs(x - ora.x[:n_ag]).max(), np.abs(y - ora.y[:n_ag]).max()))
    dh = np.abs(np.mod(h - ora.heading[:n_ag] + np.pi, 2 * np.pi) - np.pi)
    res["max_heading_err_rad"] = float(dh.max())
    res["state_flag_mismatches"] = int((batch._flags[:n_ag].cpu().numpy().astype(np.uint16)
                                        != ora.flags[:n_ag]).sum())
    if not radial:
        # edge / non-edge exact-distance ties met by the oracle's rays: the
        # one LiDAR case whose reference answer follows its BVH order
        res["lidar_edge_ties"] = OracleBatch.lidar_ties()
    res["ok"] = (res["flag_mismatches"] == 0 and res["sel_mismatches"] == 0
                 and res["obs_out_of_tol"] == 0 and res["state_flag_mismatches"] == 0
                 and res["max_pose_err_m"] <= 1e-9 and res["max_heading_err_rad"] <= 1e-12)
    agents = int(ora.pw.n_instantiated.sum())
    cpu = {"value": agents * steps / cpu_s, "unit": "agent-steps/s", "cores": threads,
           "kind": "port", "sample": f"the parity episode: {nw} worlds x {agents // max(nw, 1)} agents "
                                     f"x {steps} steps ({cpu_s:.1f} s)"}
    return res, cpu


class Leg:
    """One benched batch (a rank's shard) and its step function."""

    def __init__(self, args, W: int, w_off: int, rank: int, dev):
        import torch
        from paper_2408_01584_b200.config import obs_width
        from paper_2408_01584_b200.engine import SimBatch, random_actions
        from paper_2408_01584_b200.synthetic import WaymoSpec, generate
        _, A, P, dyn, coll, okw, workload = CONFIGS[args.config]
        self.cfg = cfg = sim_config(args.config)
        self.width = obs_width(cfg.obs)
        self.P, self.A, self.W = P, A, W
        self.dev = dev
        t0 = time.perf_counter()
        self.raw = generate(WaymoSpec(n_worlds=W, n_agents=A, n_points=P, seed=0, world_offset=w_off))
        self.rl = args.config == "c5"
        if self.rl:
            from paper_2408_01584_b200.env import EnvConfig, VecDriveEnv
            from paper_2408_01584_b200.policy import ActorCritic
            # rollout formats: bf16 observations in rows padded to 8 (the policy
            # GEMM's input, no cast), a bf16 policy with 16-B aligned operands,
            # one fused sampler launch per step
            self.env = VecDriveEnv(EnvConfig(raw=self.raw, sim=cfg, device=str(dev),
                                             obs_dtype="bfloat16"))
            self.batch = self.env.batch
            self.batch.log_episodes = True    # the line's episode statistics
            self.policy = ActorCritic(self.width, self.env.n_actions, pad_to=8).to(dev).to(torch.bfloat16)
            self.obs = self.env.reset()
        else:
            self.batch = SimBatch.from_raw(self.raw, cfg, device=dev)
            self.acts = [random_actions(self.batch.n_controlled, cfg, 0, t, dev) for t in range(8)]
        self.setup_s = time.perf_counter() - t0
        self.rank = rank

    def step(self, t, events=None):
        import torch
        if self.rl:
            from paper_2408_01584_b200.engine import sample_categorical
            with torch.inference_mode():
                logits, value = self.policy(self.obs)
                idx = sample_categorical(logits, seed=1234 + self.rank, counter=t)
            obs, rew, done, infos = self.env.step(idx)
            self.obs = obs
            return rew
        return self.batch.step(self.acts[t % 8], auto_reset=True, events=events).rewards

    def restart(self):
        """Every timed leg covers the same episode phase (steps W .. W+K after
        a reset): work per step changes over an episode (remove_agent)."""
        import torch
        if self.rl:
            self.obs = self.env.reset()
        else:
            self.batch.reset()
        torch.cuda.synchronize(self.dev)


def time_leg(leg: Leg, args, world: int, barrier, local_rank: int) -> dict:
    """Device-timed steps (inputs resident in HBM), the per-kernel split and
    the end-to-end leg through the public API with host buffers."""
    import torch
    import torch.distributed as dist
    dev = leg.dev
    stream = torch.cuda.current_stream(dev)
    leg.restart()
    for t in range(args.warmup):
        leg.step(t)
    torch.cuda.synchronize(dev)
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
        leg.step(t)
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
    if not leg.rl:
        # per-kernel split (CUDA events on the launching stream around each
        # kernel) over a further pass of the same steps, L2 flushed likewise
        n_ev = min(args.steps, 10)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_ev)]
        for e3 in ev:           # materialise the CUDA events (ds_step records raw handles)
            for e in e3:
                e.record(stream)
        leg.restart()
        for t in range(args.warmup):
            leg.step(t)
        for t in range(n_ev):
            if flush_l2:
                flush_buf.fill_(float(t))
            leg.step(t, events=ev[t])
        torch.cuda.synchronize(dev)
        kernel_ms = {"step_kernel": sum(e[0].elapsed_time(e[1]) for e in ev) / n_ev,
                     "obs_kernel": sum(e[1].elapsed_time(e[2]) for e in ev) / n_ev}
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    # units all ranks processed: every rank's agents (allreduce of the counts)
    agents_total = leg.batch.total_agents
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
    if leg.rl:
        rsum_h = torch.empty(1, dtype=torch.float32).pin_memory()
        h2d, d2h = 0, 4
    else:
        from paper_2408_01584_b200.engine import HostStepper
        stepper = HostStepper(leg.batch, act_dim=leg.acts[0].shape[1])
        host_acts = [a.cpu().pin_memory() for a in leg.acts]
        h2d, d2h = stepper.h2d_bytes_per_step, stepper.d2h_bytes_per_step

    def e2e_step(t):
        if leg.rl:
            rew = leg.step(t)
            rsum_h.copy_(rew.sum().reshape(1), non_blocking=True)
        else:
            # the actions already live in pinned host buffers (8, reused every
            # 8 steps, long after their DMA): copied straight from them
            stepper.step(host_acts[t % 8], zero_copy=True)

    leg.restart()
    for t in range(args.warmup):          # untimed warm-up of this leg's own ops
        e2e_step(t)
    barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if not leg.rl:
        stepper._h2d.wait_event(e0)        # the first action copy is inside the region
    for t in range(args.steps):
        e2e_step(t)
    if not leg.rl:
        stream.wait_stream(stepper._d2h)   # the last result copy is inside the region
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    return {"value": value, "ms": ms, "kernel_ms": kernel_ms, "clocks": clocks, "l2": l2_note,
            "agents_total": agents_total,
            "e2e": {"value": agents_total * args.steps / (e2e_ms / 1e3), "unit": "agent-steps/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}}


def self_launch(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one process per
    GPU) with torch.distributed.run on 127.0.0.1 and return their exit code."""
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def launch_check(world: int, rank: int):
    """--launch-check: each rank joins a gloo group and rank 0 prints how
    many ranks answered (the CPU test of the self-launch path)."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.ones(1)
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"launch_check": True, "world_size": world, "ranks_answered": int(t.item())}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--worlds", type=int, default=None,
                    help="override the config's world count (N > 1: the total for strong "
                         "scaling, per GPU for the weak sub-line)")
    ap.add_argument("--no-cpu-baseline", action="store_true",
                    help="skip the parity episode against the oracle (and its CPU timing)")
    ap.add_argument("--no-weak", action="store_true", help="N > 1: skip the weak-scaling sub-line")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.launch_check:
        launch_check(world, rank)
        return

    import torch
    import torch.distributed as dist

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

    def barrier():
        if world > 1:
            dist.barrier()

    W, w_off, W_total = leg_worlds(args, world, rank)
    scaling = "strong" if world > 1 else "weak"
    leg = Leg(args, W, w_off, rank, dev)
    main_leg = time_leg(leg, args, world, barrier, local_rank)
    cfg, width, P, A = leg.cfg, leg.width, leg.P, leg.A

    # ---- episode statistics: the only collective, off the step path
    from paper_2408_01584_b200.parallel import allreduce_episode_stats, episode_stats
    stats = allreduce_episode_stats(episode_stats(leg.batch.episode_infos), device=dev)

    # ---- roofline of the dominant kernel (the observation kernel)
    peak, peak_kind = load_peaks()
    act_dim = 1 if leg.rl else leg.acts[0].shape[1]
    bpa = bytes_per_agent_step(act_dim, width, P, A)
    fl = radial_flops(P, A) if cfg.obs.mode == "radial" else \
        lidar_flops(leg.batch.packed, cfg.obs.max_range, cfg.obs.n_rays)
    hbm_bound = peak * 1e9 / bpa["total"]
    fp32_peak, fp64_peak, fp_kind = fp_peaks()
    fp32_bound = fp32_peak / fl
    roofline = None
    kernel_ms = main_leg["kernel_ms"]
    if kernel_ms is not None:
        n = leg.batch.n_controlled
        achieved = bpa["obs_kernel"] * n / (kernel_ms["obs_kernel"] / 1e3) / 1e9
        kname = "obs_radial_kernel" if cfg.obs.mode == "radial" else "obs_lidar_kernel"
        tr = load_traffic(args.config, kname) if (W == CONFIGS[args.config][0]) else None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": tr / 1e9 if tr else None,
                    "traffic_unit": "GB per launch (ncu dram__bytes_read+write)",
                    "algorithmic_gb_per_launch": bpa["obs_kernel"] * n / 1e9,
                    "kernel": kname,
                    "bytes_per_agent_step": bpa["obs_kernel"], "peak_kind": peak_kind}
        if cfg.obs.mode != "radial":
            # the LiDAR kernel's executed FP64 work: exact box / segment tests
            # counted by the counter build on this workload (tools/lidar_work.py)
            lw = load_json(LIDAR_WORK_FILE)
            if lw and W == CONFIGS[args.config][0]:
                flop = lw["executed_fp64_flop_per_agent_step"]
                ach = flop * n / (kernel_ms["obs_kernel"] / 1e3)
                roofline["fp64_executed"] = {
                    "flop_per_agent_step": flop, "tests_per_agent_step": lw["per_agent_step"],
                    "achieved_tflops": ach / 1e12, "peak_tflops": fp64_peak / 1e12,
                    "frac": ach / fp64_peak, "peak_kind": fp_kind,
                    "reference_candidate_flop_per_agent_step":
                        lw["reference_candidate_flop_per_agent_step"],
                    "note": "neither HBM nor FP64 bound: issue/latency bound on the culling "
                            "and pair flattening (see DESIGN.md §4)"}

    # ---- parity episode against the oracle (rank 0, N = 1): the line's
    # parity verdict and its CPU baseline
    parity, cpu = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        try:
            if leg.rl:
                cpu_v, sample = CpuSample(args.config, threads).rate(91, warmup=1, budget_s=20.0,
                                                                     min_s=10.0)
                cpu = {"value": cpu_v, "unit": "agent-steps/s", "cores": threads, "kind": "port",
                       "sample": sample}
                parity = {"skipped": "c5 steps the same simulator as c3 (policy-chosen actions); "
                                     "parity is checked on the c1-c4 lines"}
            else:
                parity, cpu = parity_check(leg.batch, leg.raw, cfg, dev, CPU_WORLDS[args.config],
                                           91, threads)
        except Exception as exc:   # report, never fake
            cpu = {"value": None, "unit": "agent-steps/s", "cores": threads, "kind": "port",
                   "sample": f"failed: {exc!r}"}
            parity = {"ok": False, "error": repr(exc)}

    # ---- N > 1: the weak-scaling sub-line (the config's worlds on EVERY rank)
    weak = None
    if world > 1 and not args.no_weak:
        Ww = args.worlds or CONFIGS[args.config][0]
        leg.batch.close()
        wleg = Leg(args, Ww, rank * Ww, rank, dev)
        r = time_leg(wleg, args, world, barrier, local_rank)
        weak = {"value": r["value"], "ms_per_step": r["ms"] / args.steps, "scaling": "weak",
                "worlds_per_gpu": Ww, "worlds_total": Ww * world, "e2e": r["e2e"],
                "kernel_ms": r["kernel_ms"], "clocks": r["clocks"]}
        wleg.batch.close()
    if rank == 0:
        total = max(int(stats[1]), 1)
        result = {
            "metric": "agent_steps_per_sec", "value": main_leg["value"], "unit": "agent-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": main_leg["ms"] / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.config, W, W_total, world, scaling),
            "l2": main_leg["l2"],
            "e2e": main_leg["e2e"],
            "gpu_launches": (2 * args.steps) if not leg.rl else 3 * args.steps,
            "roofline": roofline,
            "step_roofline": {"bytes_per_agent_step": bpa["total"],
                              "fp32_flop_per_agent_step": fl, "hbm_bound_asps": hbm_bound,
                              "fp32_bound_asps": fp32_bound, "fp32_peak_kind": fp_kind,
                              "bound_asps": min(hbm_bound, fp32_bound),
                              "frac": (main_leg["value"] / world) / min(hbm_bound, fp32_bound)},
            "kernel_ms": kernel_ms,
            "clocks": main_leg["clocks"],
            "cpu_baseline": cpu,
            "parity": parity,
            "weak": weak,
            "episodes": {"count": int(stats[0]), "goal_rate": stats[2] / total,
                         "veh_collision_rate": stats[3] / total, "offroad_rate": stats[4] / total},
            "setup_s": leg.setup_s,
        }
        print(json.dumps(result), flush=True)
    if weak is None:
        leg.batch.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
