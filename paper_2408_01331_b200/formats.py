"""UNND v1 dataset container (src/formats.py:27-120).

Only the dataset flavour is needed on the hot path: its sha256 is the
content hash that keys every epoch's shuffle (src/store.py:74-76), so the
encoding must be byte-identical to the reference's.
"""
from __future__ import annotations

import struct

import numpy as np

from .errors import FormatError

MAGIC = b"UNND"
VERSION_DATASET = 1
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
