"""Optimizer state and the step-decay schedule (src/optim.py:16-49).

The update arithmetic itself runs on the GPU (hnn_multi_tensor_sgd /
hnn_multi_tensor_adam); this module keeps the host-visible state record and
the constants, evaluated exactly as the reference does: ``F32(lr)``, and
Adam's bias corrections computed in float64 then rounded to float32.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8
DECAY_FACTOR = 0.1


def lr_at_epoch(base_lr: float, milestones, epoch: int) -> float:
    """Rate during zero-based ``epoch``: one x0.1 drop per passed one-based milestone."""
    return base_lr * (DECAY_FACTOR ** sum(1 for m in milestones if epoch + 1 >= m))


def adam_corrections(step: int) -> tuple:
    """(F32(1-b1^t), F32(1-b2^t)) for 1-based step t (src/optim.py:75-76)."""
    return float(np.float32(1.0 - ADAM_BETA1 ** step)), float(np.float32(1.0 - ADAM_BETA2 ** step))


@dataclass
class OptimizerState:
    """Per-job optimizer record.  On the device path the moment buffers live
    in the hybrid's packed arenas; these dicts are filled only by snapshots."""

    kind: str
    momentum: float = 0.0
    step: int = 0
    velocity: dict = field(default_factory=dict)
    m1: dict = field(default_factory=dict)
    m2: dict = field(default_factory=dict)

    @classmethod
    def fresh(cls, kind: str, momentum: float = 0.0) -> "OptimizerState":
        if kind not in ("sgd", "adam"):
            raise ValueError(f"unknown optimizer {kind!r}")
        return cls(kind=kind, momentum=momentum)
