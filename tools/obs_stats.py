"""Dev: counts of the radial selection's fallback paths (needs a stats build)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.getcwd())
from bench import sim_config
from paper_2408_01584_b200.engine import SimBatch, random_actions
from paper_2408_01584_b200.synthetic import WaymoSpec, generate
from paper_2408_01584_b200 import _native as N
cfg = sim_config("c3")
raw = generate(WaymoSpec(n_worlds=256, n_agents=128, n_points=10000, seed=0))
b = SimBatch.from_raw(raw, cfg, device="cuda:0")
for t in range(30):
    b.step(random_actions(b.n_controlled, cfg, 0, t, "cuda:0"), auto_reset=True)
torch.cuda.synchronize()
N.lib().ds_debug_obs_stats((ctypes.c_ulonglong * 8)())   # clear
b.step(random_actions(b.n_controlled, cfg, 0, 99, "cuda:0"), auto_reset=True)
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 8)()
N.lib().ds_debug_obs_stats(out)
names = ["rows", "hist_candidates", "narrow_rerun", "serial", "sum_n_g", "flagged_BC", "partner_not_direct", "nbuf>ccap"]
print({n: v for n, v in zip(names, out)}, "rows/step", b.n_controlled)
