"""Diagnose the c5 loop: CPU enqueue time vs device time per step."""
import time
import torch
import bench
from paper_2408_01584_b200.config import obs_width
from paper_2408_01584_b200.engine import sample_categorical
from paper_2408_01584_b200.env import EnvConfig, VecDriveEnv
from paper_2408_01584_b200.policy import ActorCritic
from paper_2408_01584_b200.synthetic import WaymoSpec, generate

dev = torch.device("cuda", 0)
cfg = bench.sim_config("c5")
raw = generate(WaymoSpec(n_worlds=1024, n_agents=128, n_points=10000, seed=0))
env = VecDriveEnv(EnvConfig(raw=raw, sim=cfg, device="cuda:0", obs_dtype="bfloat16"))
policy = ActorCritic(obs_width(cfg.obs), 91, pad_to=8).to(dev).to(torch.bfloat16)
obs = env.reset()
rs = torch.empty(1, dtype=torch.float32).pin_memory()


def run(k, copy, label):
    global obs
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for t in range(k):
        with torch.inference_mode():
            logits, _ = policy(obs)
            idx = sample_categorical(logits, 1, t)
        obs, rew, done, infos = env.step(idx)
        if copy:
            rs.copy_(rew.sum().reshape(1), non_blocking=True)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label}: enqueue {1e3*(t1-t0)/k:.3f} ms/step, device {e0.elapsed_time(e1)/k:.3f} ms/step, wall {1e3*(t2-t0)/k:.3f}")


for _ in range(2):
    run(20, False, "no copy")
    run(20, True, "copy")
