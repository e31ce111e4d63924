"""B200-native batched world step of GPUDrive (arXiv 2408.01584).

Drop-in for the reference's ``SimBatch`` / ``VecDriveEnv`` hot path; the step
runs in hand-written sm_100a CUDA (csrc/) behind a C ABI
(include/drivesim_b200.h).  See DESIGN.md.
"""

from .config import (EGO_WIDTH, PARTNER_WIDTH, RAY_WIDTH, ROAD_SLOT_WIDTH, ObsConfig,
                     ObsLayout, SimConfig, layout, obs_width)

__all__ = ["SimConfig", "ObsConfig", "ObsLayout", "layout", "obs_width", "EGO_WIDTH",
           "PARTNER_WIDTH", "ROAD_SLOT_WIDTH", "RAY_WIDTH", "SimBatch", "init_batch",
           "benchmark", "make_policy", "goal_seek_actions", "VecDriveEnv", "EnvConfig",
           "HostStepper"]


def __getattr__(name):
    # engine/env import torch; keep `import paper_2408_01584_b200` light.
    if name in ("SimBatch", "init_batch", "benchmark", "StepOutput", "EpisodeInfo", "Metrics",
                "ThroughputReport", "compute_metrics", "ActionCountMismatch", "HostStepper",
                "HostStepResult", "make_policy", "goal_seek_actions"):
        from . import engine
        return getattr(engine, name)
    if name in ("VecDriveEnv", "EnvConfig", "ActionGrid"):
        from . import env
        return getattr(env, name)
    raise AttributeError(name)
