"""Binary world files (paper_2408_01584_b200/worldfile.py):
raw scenes and packed World tables round-trip bit for bit, reference
prepared-scenario JSON (scenario.py:416-454) converts losslessly, and a
converted golden scene still reproduces the reference's own trajectory."""

import numpy as np
import pytest

from golden_util import load, sha
from paper_2408_01584_b200 import worldfile as wf
from paper_2408_01584_b200.config import SimConfig
from paper_2408_01584_b200.packing import PackedWorlds, RawWorlds, pack
from paper_2408_01584_b200.scenario import serialize_prepared
from paper_2408_01584_b200.synthetic import WaymoSpec, generate, to_scenarios


def _fields(cls):
    import dataclasses
    return [f.name for f in dataclasses.fields(cls) if f.name not in ("names", "extra")]


def _same(a, b, cls):
    assert list(a.names) == list(b.names)
    for n in _fields(cls):
        x, y = getattr(a, n), getattr(b, n)
        assert x.dtype == y.dtype and x.shape == y.shape and np.array_equal(x, y), n


@pytest.mark.parametrize("mmap", [True, False])
def test_raw_round_trip(tmp_path, mmap):
    raw = generate(WaymoSpec(n_worlds=3, n_agents=20, n_points=500, seed=3, quantize=False))
    p = str(tmp_path / "scenes.dsw")
    wf.save_raw(p, raw)
    _same(wf.load_raw(p, mmap=mmap), raw, RawWorlds)


def test_ragged_and_empty_worlds_round_trip(tmp_path):
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from ragged import ragged_batch
    raw = ragged_batch(seed=1, num_steps=12)
    p = str(tmp_path / "ragged.dsw")
    wf.save_raw(p, raw)
    _same(wf.load_raw(p), raw, RawWorlds)


def test_packed_round_trip_and_config_check(tmp_path):
    raw = generate(WaymoSpec(n_worlds=2, n_agents=16, n_points=300, seed=4))
    cfg = SimConfig(init_mode="all_valid", max_controlled_per_world=10)
    pw = pack(raw, cfg)
    p = str(tmp_path / "tables.dsw")
    wf.save_packed(p, pw, cfg)
    _same(wf.load_packed(p, cfg), pw, PackedWorlds)
    with pytest.raises(ValueError):      # packed for a different controlled-set rule
        wf.load_packed(p, SimConfig(init_mode="all_nontrivial"))
    with pytest.raises(ValueError):      # not raw tables
        wf.load_raw(p)


def test_reference_json_converts_losslessly(tmp_path):
    """prepared-scenario JSON (the reference's on-disk form) -> world file ->
    the same flat scene, then the reference's golden trajectory again."""
    z, raw, cfg = load("templates_classic_remove_radial")
    docs = [serialize_prepared(p) for p in to_scenarios(raw)]
    p = str(tmp_path / "templates.dsw")
    got = wf.convert_prepared_json(docs, p)
    _same(got, raw, RawWorlds)
    back = wf.load_raw(p)
    _same(back, raw, RawWorlds)
    from oracle.oracle import OracleBatch
    ora = OracleBatch(back, cfg)
    assert sha(ora.observations) == z["obs_sha256"][0]
    for t in range(1, 11):
        obs, *_ = ora.step(z["actions"][t - 1].astype(np.float64))
        assert sha(obs) == z["obs_sha256"][t]


def test_corrupt_files_are_rejected(tmp_path):
    raw = generate(WaymoSpec(n_worlds=1, n_agents=4, n_points=50, seed=5))
    p = tmp_path / "w.dsw"
    wf.save_raw(str(p), raw)
    data = p.read_bytes()
    (tmp_path / "magic.dsw").write_bytes(b"NOTWORLD" + data[8:])
    (tmp_path / "version.dsw").write_bytes(data[:8] + (99).to_bytes(4, "little") + data[12:])
    (tmp_path / "short.dsw").write_bytes(data[:len(data) - 200])
    for name in ("magic", "version", "short"):
        with pytest.raises(ValueError):
            wf.load_raw(str(tmp_path / f"{name}.dsw"))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["raw", "packed"])
def test_batch_from_file_matches_from_raw(tmp_path, kind):
    import torch
    from paper_2408_01584_b200.engine import SimBatch, random_actions
    raw = generate(WaymoSpec(n_worlds=3, n_agents=24, n_points=600, seed=6, quantize=False))
    cfg = SimConfig(init_mode="all_valid", collision_behavior="remove_agent")
    p = str(tmp_path / "w.dsw")
    if kind == "raw":
        wf.save_raw(p, raw)
    else:
        wf.save_packed(p, pack(raw, cfg), cfg)
    a, b = SimBatch.from_raw(raw, cfg, device="cuda:0"), SimBatch.from_file(p, cfg, device="cuda:0")
    for t in range(20):
        act = random_actions(a.n_controlled, cfg, 1, t, "cuda:0")
        a.step(act)
        b.step(act)
    torch.cuda.synchronize()
    assert torch.equal(a.observations, b.observations) and torch.equal(a._x, b._x)
    a.close()
    b.close()
