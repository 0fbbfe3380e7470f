"""The reference's modeled per-model device footprint, for reporting next to measured HBM bytes.

BASELINE.json's metric includes "HBM bytes/model"; BASELINE.md asks for it next to what the
reference's cost model (src/memory.py:98-145, ``estimate_model``) predicts for the same model.
This restates the two graph-dependent terms of that model — weights + gradients
(2 * params * 4 B) and batch-scaled node outputs (batch * per-sample activation bytes) — and the
calibration constants it adds per model load (900 MB ephemeral x 1.1 fragmentation, 300 MB
device context, src/memory.py:42-44).  Host-side arithmetic only; it is not on the hot path.
"""
from __future__ import annotations

import numpy as np

from . import engine

BYTES_PER_VALUE = 4
MB = 1024 * 1024
EPHEMERAL_PER_LOAD = 900 * MB
FRAGMENTATION = 1.1
DEVICE_CONTEXT = 300 * MB


def activation_bytes(graph) -> int:
    """Per-sample bytes over every node output (src/memory.py:98-106)."""
    total = 0
    for nid, shape in engine.infer_shapes(graph).items():
        if nid == "input":
            continue
        total += int(np.prod(shape)) * BYTES_PER_VALUE if shape else BYTES_PER_VALUE
    return total


def reference_model_bytes(jobs: list) -> dict:
    """Mean over `jobs` of the reference's modeled footprint terms (bytes per model)."""
    wg = [2 * engine.param_count(j.graph) * BYTES_PER_VALUE for j in jobs]
    io = [j.hypers.batch_size * activation_bytes(j.graph) for j in jobs]
    const = int(EPHEMERAL_PER_LOAD * FRAGMENTATION) + DEVICE_CONTEXT
    return {"weights_grads": int(np.mean(wg)), "io_tensors": int(np.mean(io)),
            "graph_terms": int(np.mean(wg) + np.mean(io)),
            "with_load_constants": int(np.mean(wg) + np.mean(io) + const),
            "source": "reference cost model src/memory.py:98-145 (dataset term excluded)"}
