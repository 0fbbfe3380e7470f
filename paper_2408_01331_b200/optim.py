"""Optimizer state, the step-decay schedule and ``apply_update`` (src/optim.py:16-87).

The update arithmetic runs on the GPU (hnn_multi_tensor_sgd /
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


def apply_update(state: OptimizerState, params: dict, grads: dict, lr: float) -> None:
    """One optimizer step over every parameter, in place (src/optim.py:52-87) — one launch of the
    multi-tensor kernel on the device.

    numpy ``params`` are updated in place and the state's moment dicts hold numpy arrays, as in
    the reference; CUDA-tensor params are updated in place on the device (moments then stay
    CUDA tensors).  The kernel evaluates the reference's float32 expression order, so the
    result is bit-identical to the numpy update for the same gradients."""
    import numpy as np_

    from . import _native as N
    from .runtime import STATUS_DTYPE, STEP_DTYPE, OPT_CHUNK, _align4, _dev_table, _ptr
    from . import devops

    torch = devops._torch()
    dev = devops._dev()
    state.step += 1
    pids = sorted(params)
    missing = [pid for pid in pids if pid not in grads]
    if missing:
        raise KeyError(missing[0])
    on_device = isinstance(params[pids[0]], torch.Tensor) if pids else False
    sizes = [int(np_.prod(params[pid].shape)) for pid in pids]
    offs = np_.concatenate([[0], np_.cumsum([_align4(n) for n in sizes])]).astype(np_.int64)
    total = int(max(offs[-1], 4))
    kind = N.OPT_ADAM if state.kind == "adam" else (N.OPT_SGD_MOMENTUM if state.momentum else N.OPT_SGD)
    moments = {N.OPT_ADAM: (state.m1, state.m2), N.OPT_SGD_MOMENTUM: (state.velocity, None), N.OPT_SGD: (None, None)}[kind]

    def pack(src):
        arena = torch.zeros(total, dtype=torch.float32, device=dev)
        if src is None:
            return None
        for pid, o, n in zip(pids, offs, sizes):
            a = src.get(pid) if isinstance(src, dict) else None
            if a is not None:
                arena[o:o + n].copy_(devops._to_dev(a)[0].reshape(-1))
        return arena

    p_ar, g_ar = pack(params), pack(grads)
    m_ar = pack(moments[0]) if moments[0] is not None else None
    v_ar = pack(moments[1]) if moments[1] is not None else None
    row = np_.zeros(1, dtype=STEP_DTYPE)
    row["active"], row["opt_step"], row["lr"] = 1, state.step, np_.float32(lr)
    row["bias1"], row["bias2"] = adam_corrections(state.step)
    st = np_.zeros(1, dtype=STATUS_DTYPE)
    st["alive"] = 1
    cur = torch.from_numpy(row.view(np_.uint8).copy()).to(dev)
    status = torch.from_numpy(st.view(np_.uint8).copy()).to(dev)
    chunks = -(-total // OPT_CHUNK)
    seg = N.OptSegment(_ptr(p_ar), _ptr(g_ar), _ptr(m_ar), _ptr(v_ar), total, 0, kind, float(np_.float32(state.momentum)),
                       0, chunks, 0)
    table = _dev_table(N.OptSegment, [seg], dev)
    entry = "hnn_multi_tensor_adam" if kind == N.OPT_ADAM else "hnn_multi_tensor_sgd"
    N.call(entry, _ptr(table), 1, chunks, _ptr(cur), _ptr(status), devops._stream())
    torch.cuda.current_stream().synchronize()

    def unpack(arena, dst, in_place):
        for pid, o, n in zip(pids, offs, sizes):
            shape = tuple(params[pid].shape)
            if in_place:
                if on_device:
                    params[pid].copy_(arena[o:o + n].view(shape))
                else:
                    params[pid][...] = arena[o:o + n].view(shape).cpu().numpy()
            else:
                v = arena[o:o + n].view(shape).clone()
                dst[pid] = v if on_device else v.cpu().numpy()

    unpack(p_ar, None, True)
    if m_ar is not None:
        unpack(m_ar, moments[0], False)
    if v_ar is not None:
        unpack(v_ar, moments[1], False)
