"""Shared parity helpers: run the CUDA batch and the C oracle in lock step
and compare every output (tests only)."""

from __future__ import annotations

import math

import numpy as np

F32_ULPS = 2
OBS_ABS = 1e-6     # absolute floor of the FP32 observation tolerance
POS_TOL = 1e-9     # metres, free-run pose tolerance after a full episode
ANG_TOL = 1e-12    # radians


def obs_tolerance(ref64: np.ndarray) -> np.ndarray:
    r32 = np.abs(ref64).astype(np.float32)
    return F32_ULPS * np.spacing(r32).astype(np.float64) + OBS_ABS


def actions_for(cfg, n_rows: int, rng: np.random.Generator, head: bool = False) -> np.ndarray:
    """Uniform actions over the config bounds, float32 (what the GPU consumes)."""
    if cfg.dynamics == "delta_local":
        lo = np.array([b[0] for b in cfg.delta_bounds])
        hi = np.array([b[1] for b in cfg.delta_bounds])
        # small local moves so agents stay on the map
        lo, hi = lo * 0.15, hi * 0.15
    else:
        lo = np.array([cfg.accel_bounds[0], cfg.steer_bounds[0]])
        hi = np.array([cfg.accel_bounds[1], cfg.steer_bounds[1]])
    a = rng.uniform(lo, hi, (n_rows, len(lo)))
    if head:
        a = np.concatenate([a, rng.uniform(-1.0, 1.0, (n_rows, 1))], 1)
    return a.astype(np.float32)


def wrap_diff(a, b):
    d = np.mod(a - b + math.pi, 2 * math.pi) - math.pi
    return np.abs(d)


class Mismatch(AssertionError):
    pass


def compare_step(t, gpu, ora, gpu_sel=None, ora_sel=None, check_obs=True):
    """gpu: dict of numpy arrays (obs f32, rewards, dones, info[3]); ora: oracle outputs."""
    o_obs, o_rew, o_done, o_info = ora
    msgs = []
    if not np.array_equal(gpu["dones"], o_done):
        msgs.append(f"t={t}: dones differ at rows {np.nonzero(gpu['dones'] != o_done)[0][:10]}")
    if not np.array_equal(gpu["rewards"], o_rew.astype(np.float32)):
        msgs.append(f"t={t}: rewards differ at rows "
                    f"{np.nonzero(gpu['rewards'] != o_rew.astype(np.float32))[0][:10]}")
    for k, key in enumerate(("goal", "veh_collision", "offroad")):
        if not np.array_equal(gpu["info"][k], o_info[key]):
            msgs.append(f"t={t}: info[{key}] differs at rows "
                        f"{np.nonzero(gpu['info'][k] != o_info[key])[0][:10]}")
    if gpu_sel is not None and not np.array_equal(gpu_sel, ora_sel):
        rows = np.nonzero((gpu_sel != ora_sel).any(1))[0]
        msgs.append(f"t={t}: selection indices differ in {len(rows)} rows, first {rows[:5]}")
    if check_obs:
        err = np.abs(gpu["obs"].astype(np.float64) - o_obs.astype(np.float32).astype(np.float64))
        bad = err > obs_tolerance(o_obs)
        if bad.any():
            r, c = np.argwhere(bad)[0]
            msgs.append(f"t={t}: {bad.sum()} obs entries out of tolerance, first row {r} col {c}: "
                        f"gpu {gpu['obs'][r, c]!r} oracle {o_obs[r, c]!r}")
    if msgs:
        raise Mismatch("\n".join(msgs))
