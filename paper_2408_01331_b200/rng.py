"""Keyed Philox streams (src/rng.py:18-28).

A stream is named by its key parts only: sha256 over the 0x1f-joined UTF-8
labels, first 16 bytes as the Philox key.  Initial weights and every
epoch's batch order are drawn on the host from these streams, so they are
bit-identical to the reference by construction before being uploaded.
"""
from __future__ import annotations

import hashlib

import numpy as np


def stream(*key_parts) -> np.random.Generator:
    material = b"\x1f".join(str(part).encode("utf-8") for part in key_parts)
    key = np.frombuffer(hashlib.sha256(material).digest()[:16], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def permutation(n: int, *key_parts) -> np.ndarray:
    return stream(*key_parts).permutation(n)
