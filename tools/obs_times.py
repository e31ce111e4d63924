"""Dev: CTA timeline of the radial observation kernel at C3 (needs a build with
-DDS_OBS_TIMES: tools/build_variant.sh times -DDS_OBS_TIMES, then
DS_LIB_PATH=variants/times.so python tools/obs_times.py).  Splits the SMs'
warp-slot time into prologue, row loop, CTA tail (warps done, CTA still
resident) and gaps between CTAs."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from bench import sim_config
from paper_2408_01584_b200.engine import SimBatch, random_actions
from paper_2408_01584_b200.synthetic import WaymoSpec, generate
from paper_2408_01584_b200 import _native as N

W = 37
nw = int(os.environ.get("NW", "4096"))
cfg = sim_config("c3")
raw = generate(WaymoSpec(n_worlds=nw, n_agents=128, n_points=10000, seed=0))
b = SimBatch.from_raw(raw, cfg, device="cuda:0")
for t in range(12):
    b.step(random_actions(b.n_controlled, cfg, 0, t, "cuda:0"), auto_reset=True)
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * (8192 * W))()
N.lib().ds_debug_obs_times(out)
a = np.frombuffer(out, dtype=np.uint64).reshape(8192, W)[:nw].astype(np.int64)
sm, t0, t1, ends = a[:, 0], a[:, 1], a[:, 2], a[:, 3:35]
tend = ends.max(1)
base = t0.min()
span = tend.max() - base
pro = (t1 - t0).astype(np.float64)
loop = (ends - t1[:, None]).clip(0).sum(1).astype(np.float64)
tail = (tend[:, None] - ends).sum(1).astype(np.float64)
nsm = len(np.unique(sm))
slots = 32.0 * span * nsm
gap = slots - 32 * pro.sum() - loop.sum() - tail.sum()
print(f"worlds {nw} SMs {nsm} kernel span {span / 1e3:.1f} us, CTA mean {np.mean(tend - t0) / 1e3:.2f} us")
print(f"prologue mean {pro.mean() / 1e3:.2f} us: thread 0 staged at {np.mean(a[:, 35] - t0) / 1e3:.2f}, "
      f"barrier passed at {np.mean(a[:, 36] - t0) / 1e3:.2f}")
for k, v in [("prologue", 32 * pro.sum()), ("row loop", loop.sum()), ("CTA tail", tail.sum()), ("between CTAs / kernel tail", gap)]:
    print(f"  {k:28s} {100 * v / slots:5.1f} % of warp-slot time")
last = np.sort(tend - base)
print("last CTA ends at", last[-1] / 1e3, "us; 95% of CTAs done by", last[int(0.95 * nw)] / 1e3, "us")
