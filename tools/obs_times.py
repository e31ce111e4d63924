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

# Row durations of two consecutive steps: does the previous step's duration
# predict this one's, and what would handing rows out longest-first save?
def row_durs():
    buf = (ctypes.c_uint * (8192 * 128))()
    N.lib().ds_debug_obs_row_dur(buf)
    return np.frombuffer(buf, dtype=np.uint32).reshape(8192, 128)[:nw].astype(np.float64)
d1 = row_durs()
b.step(random_actions(b.n_controlled, cfg, 0, 99, "cuda:0"), auto_reset=True)
torch.cuda.synchronize()
d2 = row_durs()
print("row time mean %.2f us, cv %.2f, max/mean %.2f" % (d2.mean() / 1e3, d2.std() / d2.mean(), d2.max() / d2.mean()))
print("corr(prev step, this step) per row: %.3f" % np.corrcoef(d1.ravel(), d2.ravel())[0, 1])
import heapq
def makespan(d, order, nwarp=32):
    fin = [0.0] * nwarp
    h = [(0.0, k) for k in range(nwarp)]
    for r in order:
        t, k = heapq.heappop(h)
        heapq.heappush(h, (t + d[r], k))
    return max(t for t, _ in h), sum(d) / nwarp
res = {"index": [], "lpt_prev": [], "lpt_oracle": []}
for wi in range(0, nw, 8):
    d = d2[wi]
    for name, order in [("index", range(128)), ("lpt_prev", np.argsort(-d1[wi], kind="stable")),
                        ("lpt_oracle", np.argsort(-d, kind="stable"))]:
        m, ideal = makespan(d, order)
        res[name].append(m / ideal)
print({k: round(float(np.mean(v)), 4) for k, v in res.items()}, "(makespan / ideal, simulated)")
