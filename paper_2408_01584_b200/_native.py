"""ctypes binding of libdrivesim_b200.so (include/drivesim_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the shared object is missing, every entry point
raises ``ImportError`` -- the step never silently runs on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DS_LIB_PATH (dev only): an alternative build of the same library, for A/B timing
LIB_PATH = os.environ.get("DS_LIB_PATH") or os.path.join(_HERE, "libdrivesim_b200.so")
ABI_VERSION = 4
OBS_F32, OBS_BF16 = 0, 1   # ds_set_obs_format element types

DS_OK = 0
DS_E_INVALID = -1
DS_E_ACTION_COUNT = -2
DS_E_CUDA = -3
DS_E_CAPACITY = -4
DS_E_OVERFLOW = -5

DYN = {"classic": 0, "invertible": 1, "delta_local": 2}
COLL = {"ignore": 0, "remove_agent": 1, "end_episode": 2}
OBS = {"radial": 0, "lidar": 1, "view_cone": 2}

# mutable flag bits (DS_F_*)
F_PRESENT = 0x001
F_REMOVED = 0x002
F_PENDING = 0x004
F_GOAL_REACHED = 0x008
F_COLLIDED = 0x010
F_OFFROAD = 0x020
F_GOAL_EVER = 0x040
F_COLL_EVER = 0x080
F_OFF_EVER = 0x100
F_DONE = 0x200

_p = C.c_void_p


class DsConfig(C.Structure):
    _fields_ = [("dynamics", C.c_int32), ("collision_behavior", C.c_int32),
                ("obs_mode", C.c_int32), ("n_rays", C.c_int32),
                ("max_agents_obs", C.c_int32), ("max_road_points_obs", C.c_int32),
                ("obs_width", C.c_int32), ("reserved0", C.c_int32),
                ("radius", C.c_double), ("fov", C.c_double), ("max_range", C.c_double),
                ("goal_tolerance", C.c_double), ("accel_lo", C.c_double),
                ("accel_hi", C.c_double), ("steer_lo", C.c_double), ("steer_hi", C.c_double),
                ("v_max", C.c_double), ("delta_lo", C.c_double * 3),
                ("delta_hi", C.c_double * 3), ("grid_cell", C.c_double)]


TABLE_PTRS = [
    "a_off", "c_off", "r_off", "num_steps", "dt",
    "kind", "length", "width", "half_l", "half_w", "circumradius", "goal_x", "goal_y",
    "sflags", "ctrl_row", "row_agent",
    "rep_x", "rep_y", "rep_h", "rep_v", "rep_valid", "rep_present",
    "grid_x0", "grid_y0", "grid_nx", "grid_ny", "grid_cell_off",
    "p_off", "pt_cell_start", "gpt_x", "gpt_y", "gpt_h", "gpt_kind", "gpt_id",
    "eseg_cell_start", "eseg_ax", "eseg_ay", "eseg_bx", "eseg_by",
    "aseg_cell_start", "aseg_ax", "aseg_ay", "aseg_bx", "aseg_by", "aseg_id", "aseg_edge",
    "s_off", "gpt_xy", "grid_eps", "gpt_rec", "eseg_rel", "agent_rec", "eseg_rec", "aseg_rec",
]


class DsTables(C.Structure):
    _fields_ = ([("n_worlds", C.c_int32), ("n_agents", C.c_int32), ("n_rows", C.c_int32),
                 ("max_agents", C.c_int32), ("max_points", C.c_int32), ("reserved0", C.c_int32)]
                + [(n, _p) for n in TABLE_PTRS])


STATE_PTRS = ["x", "y", "heading", "speed", "head_angle", "flags", "t", "episode_over",
              "ring", "ring_head"]


class DsState(C.Structure):
    _fields_ = [(n, _p) for n in STATE_PTRS] + [("ring_cap", C.c_int32),
                                                ("reserved0", C.c_int32), ("obs_hint", _p),
                                                ("status", _p)]


STATUS_BAD_ACTION_INDEX = 1


class DsStepArgs(C.Structure):
    _fields_ = [("actions", _p), ("action_idx", _p), ("act_dim", C.c_int32),
                ("replay", C.c_int32), ("grid_accel", _p), ("grid_steer", _p),
                ("n_accel", C.c_int32), ("n_steer", C.c_int32), ("obs", _p),
                ("rewards", _p), ("dones", _p), ("info", _p), ("obs_scale", _p),
                ("auto_reset", C.c_int32), ("serial", C.c_int32), ("sel_idx", _p),
                ("reserved0", C.c_int32), ("events", _p * 3)]


EXPORTS = ["ds_abi_version", "ds_lidar_supported", "ds_struct_sizes", "ds_last_error", "ds_create", "ds_destroy", "ds_reset", "ds_step",
           "ds_observe", "ds_set_obs_format", "ds_sample_categorical", "ds_decimate_scratch_bytes", "ds_decimate_polylines", "ds_episode_drain", "ds_status", "ds_gumbel_noise", "ds_goal_seek", "ds_host_hypot_libm", "ds_host_hypot_cpython",
           "ds_host_hypot_port", "ds_host_wrap_port", "ds_host_road_headings"]

_lib = None


def lib():
    """Load (once) and return the CDLL; raises ImportError when not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                          "(there is no CPU fallback for the batched step)")
    L = C.CDLL(LIB_PATH)
    L.ds_abi_version.restype = C.c_int
    L.ds_struct_sizes.argtypes = [_p]
    L.ds_struct_sizes.restype = None
    L.ds_last_error.restype = C.c_char_p
    L.ds_create.argtypes = [C.POINTER(DsTables), C.POINTER(DsConfig), C.POINTER(DsState),
                            C.c_int, C.POINTER(_p)]
    L.ds_destroy.argtypes = [_p]
    L.ds_reset.argtypes = [_p, _p, _p, _p, _p, _p, _p, _p]
    L.ds_step.argtypes = [_p, C.POINTER(DsStepArgs), _p]
    L.ds_observe.argtypes = [_p, _p, _p, _p, _p, _p]
    L.ds_episode_drain.argtypes = [_p, _p, C.c_int32, C.POINTER(C.c_int32), _p]
    L.ds_set_obs_format.argtypes = [_p, C.c_int, C.c_int]
    L.ds_decimate_scratch_bytes.argtypes = [C.c_int64]
    L.ds_gumbel_noise.argtypes = [_p, C.c_int64, _p, _p]
    L.ds_goal_seek.argtypes = [_p, _p, _p]
    L.ds_status.argtypes = [_p, _p, C.c_int, _p]
    L.ds_decimate_polylines.argtypes = [_p, _p, _p, C.c_int64, _p, C.c_double, _p, _p,
                                        C.c_int64, _p]
    L.ds_sample_categorical.argtypes = [_p, C.c_int, C.c_int64, C.c_int32, C.c_int64,
                                        C.c_uint64, C.c_uint64, _p, _p]
    for n in ("ds_host_hypot_libm", "ds_host_hypot_cpython", "ds_host_hypot_port"):
        getattr(L, n).argtypes = [_p, _p, C.c_int64, _p]
    L.ds_host_road_headings.argtypes = [_p, _p, _p, C.c_int64, _p]
    L.ds_host_wrap_port.argtypes = [_p, C.c_int64, _p]
    for n in EXPORTS:
        if n not in ("ds_abi_version", "ds_last_error", "ds_struct_sizes", "ds_lidar_supported",
                     "ds_decimate_scratch_bytes"):
            getattr(L, n).restype = C.c_int
    L.ds_decimate_scratch_bytes.restype = C.c_int64
    if L.ds_abi_version() != ABI_VERSION:
        raise ImportError("libdrivesim_b200.so ABI version mismatch; rebuild")
    sizes = (C.c_int64 * 4)()
    L.ds_struct_sizes(sizes)
    mine = (C.sizeof(DsConfig), C.sizeof(DsTables), C.sizeof(DsState), C.sizeof(DsStepArgs))
    if tuple(sizes) != mine:
        raise ImportError(f"C-ABI struct layout mismatch: lib {tuple(sizes)} vs ctypes {mine}")
    _lib = L
    return L


def lidar_supported() -> bool:
    """True once the library implements the LiDAR / view-cone kernel."""
    return bool(lib().ds_lidar_supported())


class NativeError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc == DS_OK:
        return
    msg = lib().ds_last_error().decode(errors="replace")
    if rc in (DS_E_INVALID, DS_E_CAPACITY):
        raise ValueError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p)


def host_hypot_libm(x, y) -> np.ndarray:
    x, y = _f64(x), _f64(y)
    out = np.empty_like(x)
    check(lib().ds_host_hypot_libm(_ptr(x), _ptr(y), x.size, _ptr(out)), "hypot_libm")
    return out


def host_hypot_cpython(x, y) -> np.ndarray:
    x, y = _f64(x), _f64(y)
    out = np.empty_like(x)
    check(lib().ds_host_hypot_cpython(_ptr(x), _ptr(y), x.size, _ptr(out)), "hypot_cpython")
    return out


def host_hypot_port(x, y) -> np.ndarray:
    x, y = _f64(x), _f64(y)
    out = np.empty_like(x)
    check(lib().ds_host_hypot_port(_ptr(x), _ptr(y), x.size, _ptr(out)), "hypot_port")
    return out


def host_wrap_port(x) -> np.ndarray:
    x = _f64(x)
    out = np.empty_like(x)
    check(lib().ds_host_wrap_port(_ptr(x), x.size, _ptr(out)), "wrap_port")
    return out


def host_road_headings(x, y, poly_pt_off) -> np.ndarray:
    x, y = _f64(x), _f64(y)
    off = np.ascontiguousarray(poly_pt_off, dtype=np.int64)
    out = np.zeros_like(x)
    check(lib().ds_host_road_headings(_ptr(x), _ptr(y), _ptr(off), max(len(off) - 1, 0),
                                      _ptr(out)), "road_headings")
    return out
