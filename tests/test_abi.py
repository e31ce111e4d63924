"""The C-ABI library loads without a GPU and exports every symbol declared in
include/drivesim_b200.h, with struct layouts matching the ctypes mirror."""

import ctypes
import os
import re

import pytest

from paper_2408_01584_b200 import _native as N

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "drivesim_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ds_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("ds_create", "ds_reset", "ds_step", "ds_observe", "ds_episode_drain",
                     "ds_destroy", "ds_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_struct_layouts_match():
    N.lib()   # raises ImportError on any size mismatch
    sizes = (ctypes.c_int64 * 4)()
    N.lib().ds_struct_sizes(sizes)
    assert tuple(sizes) == (ctypes.sizeof(N.DsConfig), ctypes.sizeof(N.DsTables),
                            ctypes.sizeof(N.DsState), ctypes.sizeof(N.DsStepArgs))
    assert N.lib().ds_abi_version() == N.ABI_VERSION


def test_create_rejects_bad_config_without_touching_cuda():
    tab, cfg, st = N.DsTables(), N.DsConfig(), N.DsState()
    cfg.dynamics = 7
    h = ctypes.c_void_p()
    rc = N.lib().ds_create(ctypes.byref(tab), ctypes.byref(cfg), ctypes.byref(st), 0,
                           ctypes.byref(h))
    assert rc == N.DS_E_INVALID
    assert b"dynamics" in N.lib().ds_last_error()
    with pytest.raises(ValueError):
        N.check(rc, "ds_create")


def test_product_path_has_no_cpu_fallback(monkeypatch):
    """Without the built library the engine raises instead of running on CPU."""
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", "/nonexistent/libdrivesim_b200.so")
    with pytest.raises(ImportError):
        N.lib()
