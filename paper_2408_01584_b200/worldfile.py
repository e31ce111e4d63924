"""Packed binary world files: prepared scenarios on disk in the
flat SoA form the batch consumes, loadable without building a single
per-object Python value.

The reference stores one prepared scenario per JSON document
(scenario.py:188-305 writes it, load_prepared scenario.py:418-454 reads it
back into ObjectLog / LoggedStep / Vec2 objects, and World.__init__ then
walks those objects again, engine.py:173-314).  A world file holds a whole
batch as typed arrays instead:

    offset 0   magic  b"DSWORLD\\0"                     8 bytes
    offset 8   u32    format version (FORMAT_VERSION)
    offset 12  u32    header length H (bytes)
    offset 16  header UTF-8 JSON, H bytes:
                 {"kind": "raw" | "packed", "n_worlds": W, "names": [...],
                  "meta": {...},                        (packed: the SimConfig
                                                         fields the tables depend on)
                  "arrays": [{"name", "dtype", "shape", "offset", "nbytes"}, ...]}
    D = 16 + H rounded up to 64: the data section -- every array's bytes,
               little-endian, C order, at D + offset (offsets 64-byte aligned)

``load_raw`` / ``load_packed`` map the file (np.memmap, read-only) and hand
the arrays to ``RawWorlds`` / ``PackedWorlds`` as they are: loading 4096
C3-sized worlds is a few milliseconds of header parsing plus page-ins.
``convert_prepared_json`` turns reference prepared-scenario JSON documents
into a world file.  A version or layout mismatch raises ``ValueError``.
"""

from __future__ import annotations

import dataclasses
import json
import os
import struct

import numpy as np

from .packing import PackedWorlds, RawWorlds, pack, raw_from_prepared

MAGIC = b"DSWORLD\0"
FORMAT_VERSION = 1
_ALIGN = 64
_PREFIX = struct.Struct("<8sII")


def _array_fields(cls) -> list:
    return [f.name for f in dataclasses.fields(cls) if f.name not in ("names", "extra")]


def _data_start(header_len: int) -> int:
    return -(-(_PREFIX.size + header_len) // _ALIGN) * _ALIGN


def _write(path: str, kind: str, names: list, arrays: dict, meta: dict) -> None:
    entries, off, blobs = [], 0, []
    for name, a in arrays.items():
        a = np.ascontiguousarray(a)
        if a.dtype.kind not in "biuf":
            raise ValueError(f"{name}: unsupported dtype {a.dtype}")
        a = a.astype(a.dtype.newbyteorder("<"), copy=False)
        entries.append({"name": name, "dtype": a.dtype.str, "shape": list(a.shape),
                        "offset": off, "nbytes": int(a.nbytes)})   # offset: from the data start
        blobs.append(a)
        off += -(-int(a.nbytes) // _ALIGN) * _ALIGN
    hb = json.dumps({"kind": kind, "n_worlds": len(names), "names": list(names), "meta": meta,
                     "arrays": entries}).encode()
    data0 = _data_start(len(hb))
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(_PREFIX.pack(MAGIC, FORMAT_VERSION, len(hb)))
        f.write(hb)
        for e, a in zip(entries, blobs):
            f.seek(data0 + e["offset"])
            f.write(a.tobytes())
        f.truncate(data0 + off)
    os.replace(tmp, path)


def _read(path: str, kind: str, mmap: bool):
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        prefix = f.read(_PREFIX.size)
        if len(prefix) < _PREFIX.size:
            raise ValueError(f"{path}: not a world file (too short)")
        magic, version, hlen = _PREFIX.unpack(prefix)
        if magic != MAGIC:
            raise ValueError(f"{path}: not a world file (bad magic)")
        if version != FORMAT_VERSION:
            raise ValueError(f"{path}: world file version {version}, this reader is "
                             f"{FORMAT_VERSION}")
        hb = f.read(hlen)
        if len(hb) < hlen:
            raise ValueError(f"{path}: truncated header")
        header = json.loads(hb.decode())
    if header.get("kind") != kind:
        raise ValueError(f"{path}: holds {header.get('kind')!r} tables, expected {kind!r}")
    data0 = _data_start(hlen)
    out = {}
    for e in header["arrays"]:
        start = data0 + e["offset"]
        if e["offset"] % _ALIGN or start + e["nbytes"] > size:
            raise ValueError(f"{path}: array {e['name']} outside the file (truncated?)")
        shape, dt = tuple(e["shape"]), np.dtype(e["dtype"])
        if mmap and e["nbytes"]:
            out[e["name"]] = np.asarray(np.memmap(path, dtype=dt, mode="r", offset=start,
                                                  shape=shape))
        else:
            with open(path, "rb") as f:
                f.seek(start)
                buf = f.read(e["nbytes"])
            out[e["name"]] = np.frombuffer(buf, dtype=dt).reshape(shape).copy()
    return header, out


def save_raw(path: str, raw: RawWorlds) -> None:
    """Write a RawWorlds batch (prepared scenarios, flat) to ``path``."""
    _write(path, "raw", raw.names, {n: getattr(raw, n) for n in _array_fields(RawWorlds)}, {})


def load_raw(path: str, mmap: bool = True) -> RawWorlds:
    """Read a world file written by save_raw (memory-mapped by default)."""
    header, arrs = _read(path, "raw", mmap)
    missing = set(_array_fields(RawWorlds)) - set(arrs)
    if missing:
        raise ValueError(f"{path}: missing arrays {sorted(missing)}")
    raw = RawWorlds(names=list(header["names"]), **{n: arrs[n] for n in _array_fields(RawWorlds)})
    if raw.n_worlds != header["n_worlds"] or len(raw.a_off) != raw.n_worlds + 1:
        raise ValueError(f"{path}: inconsistent world count")
    return raw


def _pack_meta(cfg) -> dict:
    return {"init_mode": cfg.init_mode, "max_controlled_per_world": cfg.max_controlled_per_world}


def save_packed(path: str, pw: PackedWorlds, cfg) -> None:
    """Write the World.__init__ tables of a batch (packing.pack output) so a
    later run skips the packing; the SimConfig fields they depend on (the
    controlled-set rule) are recorded and checked on load."""
    _write(path, "packed", pw.names, {n: getattr(pw, n) for n in _array_fields(PackedWorlds)},
           _pack_meta(cfg))


def load_packed(path: str, cfg, mmap: bool = True) -> PackedWorlds:
    header, arrs = _read(path, "packed", mmap)
    if header["meta"] != _pack_meta(cfg):
        raise ValueError(f"{path}: packed for {header['meta']}, the config asks for "
                         f"{_pack_meta(cfg)}")
    return PackedWorlds(names=list(header["names"]),
                        **{n: arrs[n] for n in _array_fields(PackedWorlds)})


def convert_prepared_json(docs, path: str, decimation_threshold: float = 0.05,
                          controllable_threshold: float = 2.0) -> RawWorlds:
    """Reference prepared-scenario JSON documents (text, or paths to files) ->
    one world file; plain scenario documents are preprocessed on the way
    (load_prepared, scenario.py:434-454).  Returns the RawWorlds written."""
    from .scenario import load_prepared
    preps = []
    for d in docs:
        text = d
        if not d.lstrip().startswith("{"):
            with open(d) as f:
                text = f.read()
        preps.append(load_prepared(text, decimation_threshold, controllable_threshold))
    raw = raw_from_prepared(preps)
    save_raw(path, raw)
    return raw


def pack_file(raw_path: str, packed_path: str, cfg) -> PackedWorlds:
    """World file -> packed-table file (pack once, load many times)."""
    pw = pack(load_raw(raw_path), cfg)
    save_packed(packed_path, pw, cfg)
    return pw
