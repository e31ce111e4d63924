"""delta_local dynamics injected into the REAL reference (fixture generation only).

The reference has no delta_local model (engine.py:32).  This shim patches it
in from outside /root/reference, with the definition DESIGN.md §2 gives:
action (dx, dy, dyaw[, head]) in the ego frame, clipped to delta_bounds;
x += dx cos h - dy sin h, y += dx sin h + dy cos h, h = wrap(h + dyaw),
v = clip(hypot(dx, dy) / dt, +-v_max); a 4th column is the head rotation.
  * SimConfig validation: DYNAMICS_MODELS (engine.py:32, 60-61);
  * dynamics branch: World.step calls dyn.step_invertible_arr for every
    non-classic model (engine.py:393-403); the proxy below receives column 0
    of the live action rows, whose .base is the whole [live] matrix;
  * head column: World.step reads column 2 as head rotation (engine.py:408-411),
    so actions are reordered to (dx, dy, head, dyaw) with head = 0 if absent.
"""
import math
import types

import numpy as np
from drivesim import engine as E
from drivesim.geometry import wrap_angle_arr

BOUNDS = ((-6.0, 6.0), (-6.0, 6.0), (-math.pi, math.pi))   # config.DEFAULT_DELTA_BOUNDS


def _delta_local(px, py, h, v, a0, a1, dt, v_max=E.dyn.DEFAULT_V_MAX):
    act = a0.base                                  # (dx, dy, head, dyaw) live rows
    dx, dy, dyaw = (np.clip(act[:, c], *BOUNDS[k]) for k, c in enumerate((0, 1, 3)))
    ch, sh = np.frompyfunc(math.cos, 1, 1)(h).astype(float), np.frompyfunc(math.sin, 1, 1)(h).astype(float)
    return (px + (dx * ch - dy * sh), py + (dx * sh + dy * ch), wrap_angle_arr(h + dyaw),
            np.clip(np.hypot(dx, dy) / dt, -v_max, v_max))


def install():
    E.DYNAMICS_MODELS = ("classic", "invertible", "delta_local")
    dyn, inv, orig, active = types.SimpleNamespace(**vars(E.dyn)), E.dyn.step_invertible_arr, E.World.step, [False]
    dyn.step_invertible_arr = lambda *a, **k: (_delta_local if active[0] else inv)(*a, **k)
    E.dyn = dyn

    def step(self, actions, obs_out=None):
        active[0] = self.cfg.dynamics == "delta_local"
        if active[0] and actions is not None:
            a = np.asarray(actions, float)
            head = a[:, 3:4] if a.shape[1] > 3 else np.zeros((len(a), 1))
            actions = np.concatenate([a[:, :2], head, a[:, 2:3]], 1)
        return orig(self, actions, obs_out)
    E.World.step = step
