"""UNND containers (src/formats.py): v1 datasets, v2 packaged models, v3 checkpoints.

The dataset flavour is on the hot path: its sha256 is the content hash that
keys every epoch's shuffle (src/store.py:74-76).  The model flavour is what
``package`` writes from separated parameters (src/separate.py:39-72,
src/formats.py:157-181); the checkpoint flavour is what a paused job's
``Checkpoint.encode`` writes (src/train.py:57-99, src/formats.py:188-207).
All must be byte-identical to the reference's:
little-endian, a canonical JSON header (sorted keys, no whitespace) for
models, then float32 sections ``name(u8 len) rank(u8) dims(u32...) data``.
"""
from __future__ import annotations

import struct

import numpy as np

from .errors import FormatError

import json

MAGIC = b"UNND"
VERSION_DATASET = 1
VERSION_MODEL = 2
VERSION_CHECKPOINT = 3
DATASET_SECTIONS = ("train_x", "train_y", "test_x", "test_y")


def _section(name: str, arr) -> bytes:
    raw = name.encode("utf-8")
    if len(raw) > 255:
        raise FormatError(f"section name too long: {name!r}")
    arr = np.ascontiguousarray(arr, dtype="<f4")
    if arr.ndim > 255:
        raise FormatError(f"section {name!r}: rank {arr.ndim} too large")
    head = struct.pack("<B", len(raw)) + raw + struct.pack("<B", arr.ndim)
    head += b"".join(struct.pack("<I", d) for d in arr.shape)
    return head + arr.tobytes()


def encode_dataset(splits: dict) -> bytes:
    missing = [s for s in DATASET_SECTIONS if s not in splits]
    if missing:
        raise FormatError(f"dataset missing sections {missing}")
    extra = [s for s in splits if s not in DATASET_SECTIONS]
    if extra:
        raise FormatError(f"dataset has unexpected sections {sorted(extra)}")
    body = b"".join(_section(name, splits[name]) for name in DATASET_SECTIONS)
    return MAGIC + struct.pack("<HH", VERSION_DATASET, len(DATASET_SECTIONS)) + body


def decode_dataset(blob: bytes) -> dict:
    view = memoryview(blob)
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(view):
            raise FormatError("truncated container")
        chunk = view[pos:pos + n]
        pos += n
        return chunk

    if bytes(take(4)) != MAGIC:
        raise FormatError("bad magic: not a container file")
    (version,) = struct.unpack("<H", take(2))
    if version != VERSION_DATASET:
        raise FormatError(f"expected format version {VERSION_DATASET}, got {version}")
    (count,) = struct.unpack("<H", take(2))
    out = {}
    for _ in range(count):
        (nlen,) = struct.unpack("<B", take(1))
        name = bytes(take(nlen)).decode("utf-8")
        (rank,) = struct.unpack("<B", take(1))
        shape = tuple(struct.unpack("<I", take(4))[0] for _ in range(rank))
        n = int(np.prod(shape)) if shape else 1
        arr = np.frombuffer(bytes(take(4 * n)), dtype="<f4").reshape(shape).astype(np.float32)
        if name in out:
            raise FormatError(f"duplicate section {name!r}")
        out[name] = arr
    if pos != len(view):
        raise FormatError("trailing bytes after final section")
    missing = [s for s in DATASET_SECTIONS if s not in out]
    if missing:
        raise FormatError(f"dataset missing sections {missing}")
    extra = [s for s in out if s not in DATASET_SECTIONS]
    if extra:
        raise FormatError(f"dataset has unexpected sections {sorted(extra)}")
    for split in ("train", "test"):
        xs, ys = out[f"{split}_x"].shape, out[f"{split}_y"].shape
        if not xs or not ys or xs[0] != ys[0]:
            raise FormatError(f"{split} split rows disagree: x {xs}, y {ys}")
    return out


# --------------------------------------------------------------------------- models (v2)


def canonical_json(obj) -> bytes:
    """Sorted keys, no whitespace: identical content, identical bytes (src/formats.py:36-37)."""
    return json.dumps(obj, sort_keys=True, separators=(",", ":")).encode("utf-8")


def encode_model(header: dict, params: dict, order: list) -> bytes:
    """magic, u16 version 2, u32 header length, canonical JSON header, u16 section count, the
    parameter sections in ``order`` (src/formats.py:157-170)."""
    if sorted(order) != sorted(params):
        raise FormatError("parameter order does not cover the parameter set")
    head = canonical_json(header)
    parts = [MAGIC, struct.pack("<H", VERSION_MODEL), struct.pack("<I", len(head)), head,
             struct.pack("<H", len(order))]
    parts += [_section(pid, params[pid]) for pid in order]
    return b"".join(parts)


def _reader(blob: bytes, version: int):
    """(take, done) over a container body after its magic and version."""
    view = memoryview(blob)
    pos = [0]

    def take(n):
        if pos[0] + n > len(view):
            raise FormatError("truncated container")
        chunk = bytes(view[pos[0]:pos[0] + n])
        pos[0] += n
        return chunk

    if take(4) != MAGIC:
        raise FormatError("bad magic: not a container file")
    (got,) = struct.unpack("<H", take(2))
    if got != version:
        raise FormatError(f"expected format version {version}, got {got}")
    return take, lambda: pos[0] == len(view)


def _header_and_sections(blob: bytes, version: int) -> tuple:
    """u32-prefixed JSON header, u16 section count, the sections; no duplicates, no trailing
    bytes (src/formats.py:98-107)."""
    take, done = _reader(blob, version)
    (hlen,) = struct.unpack("<I", take(4))
    header = json.loads(take(hlen).decode("utf-8"))
    (count,) = struct.unpack("<H", take(2))
    sections = {}
    for _ in range(count):
        name = take(take(1)[0]).decode("utf-8")
        rank = take(1)[0]
        shape = tuple(struct.unpack("<I", take(4))[0] for _ in range(rank))
        n = int(np.prod(shape)) if shape else 1
        if name in sections:
            raise FormatError(f"duplicate section {name!r}")
        sections[name] = np.frombuffer(take(4 * n), dtype="<f4").reshape(shape).astype(np.float32)
    if not done():
        raise FormatError("trailing bytes after final section")
    return header, sections


def decode_model(blob: bytes) -> tuple:
    """Inverse of encode_model; checks the header's declared parameter count (src/formats.py:173-181)."""
    header, sections = _header_and_sections(blob, VERSION_MODEL)
    declared = header.get("param_count")
    actual = sum(int(a.size) for a in sections.values())
    if declared is not None and declared != actual:
        raise FormatError(f"header says {declared} parameters, file holds {actual}")
    return header, sections


# --------------------------------------------------------------------------- checkpoints (v3)


def encode_checkpoint(header: dict, sections: dict, order: list) -> bytes:
    """The v2 layout under version 3: header, then the named sections in ``order``
    (src/formats.py:188-201)."""
    if sorted(order) != sorted(sections):
        raise FormatError("section order does not cover the section set")
    head = canonical_json(header)
    parts = [MAGIC, struct.pack("<H", VERSION_CHECKPOINT), struct.pack("<I", len(head)), head,
             struct.pack("<H", len(order))]
    parts += [_section(name, sections[name]) for name in order]
    return b"".join(parts)


def decode_checkpoint(blob: bytes) -> tuple:
    return _header_and_sections(blob, VERSION_CHECKPOINT)
