"""Operator plugin registry — the reference's ``OP_KINDS`` surface (src/ops.py:285-368).

Each :class:`OpKind` keeps the reference's fields: attribute spec, per-sample
shape rule, parameter shapes, ``forward(x, params, attrs[, targets]) ->
(y, aux)`` and ``backward(dy, aux, params, attrs) -> (dx | None, grads)``.
Shape rules run on the host.  ``forward``/``backward`` run on the GPU
through the C-ABI kernels (see :mod:`.devops`): they accept numpy arrays
(copied to ``cuda:0`` and back, like the reference's ndarray contract) or
CUDA torch tensors (kept on the device).  There is no CPU implementation:
without the CUDA library these raise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np


def _pos_int(v):
    return isinstance(v, int) and not isinstance(v, bool) and v > 0


def _nonneg_int(v):
    return isinstance(v, int) and not isinstance(v, bool) and v >= 0


def conv_extent(size: int, kernel: int, stride: int, padding: int) -> int:
    """Output length of a strided window sweep (src/ops.py:28-29)."""
    return (size + 2 * padding - kernel) // stride + 1


# ---------------------------------------------------------------- shape rules


def _dense_out(shape, attrs):
    if len(shape) != 1:
        raise ValueError(f"dense expects a flat input, got {shape}")
    return (attrs["units"],)


def _conv_out(shape, attrs):
    if len(shape) != 3:
        raise ValueError(f"conv2d expects (channels, h, w), got {shape}")
    _, h, w = shape
    k, s, p = attrs["kernel"], attrs.get("stride", 1), attrs.get("padding", 0)
    oh, ow = conv_extent(h, k, s, p), conv_extent(w, k, s, p)
    if oh < 1 or ow < 1:
        raise ValueError(f"kernel {k} too large for input {shape}")
    return (attrs["filters"], oh, ow)


def _pool_out(shape, attrs):
    if len(shape) != 3:
        raise ValueError(f"maxpool2d expects (channels, h, w), got {shape}")
    c, h, w = shape
    k = attrs["kernel"]
    s = attrs.get("stride", k)
    oh, ow = conv_extent(h, k, s, 0), conv_extent(w, k, s, 0)
    if oh < 1 or ow < 1:
        raise ValueError(f"pool kernel {k} too large for input {shape}")
    return (c, oh, ow)


def _flatten_out(shape, attrs):
    return (int(np.prod(shape)),) if shape else (1,)


def _sce_out(shape, attrs):
    if len(shape) != 1:
        raise ValueError(f"softmax-cross-entropy expects logits, got {shape}")
    return ()


def _embed_out(shape, attrs):
    if len(shape) != 1:
        raise ValueError(f"embedding-lookup expects token indices, got {shape}")
    return (shape[0], attrs["dim"])


def _no_params(shape, attrs):
    return {}


# ------------------------------------------------------------ device bridges


def _device_forward(name):
    def run(x, params, attrs, targets=None):
        from . import devops

        return devops.forward(name, x, params, attrs, targets)

    run.__name__ = f"{name}_forward"
    return run


def _device_backward(name):
    def run(dy, aux, params, attrs):
        from . import devops

        return devops.backward(name, dy, aux, params, attrs)

    run.__name__ = f"{name}_backward"
    return run


@dataclass(frozen=True)
class OpKind:
    name: str
    attr_spec: dict
    infer_shape: Callable
    param_shapes: Callable
    forward: Callable
    backward: Callable
    loss_head: bool = False
    takes_targets: bool = False


def _kind(name, attr_spec, infer, params, **flags):
    return OpKind(name, attr_spec, infer, params, _device_forward(name), _device_backward(name), **flags)


OP_KINDS: dict = {
    k.name: k
    for k in (
        _kind(
            "dense",
            {"units": (True, _pos_int)},
            _dense_out,
            lambda s, a: {"weight": (a["units"], s[0]), "bias": (a["units"],)},
        ),
        _kind("relu", {}, lambda s, a: tuple(s), _no_params),
        _kind(
            "conv2d",
            {
                "filters": (True, _pos_int),
                "kernel": (True, _pos_int),
                "stride": (False, _pos_int),
                "padding": (False, _nonneg_int),
            },
            _conv_out,
            lambda s, a: {"weight": (a["filters"], s[0], a["kernel"], a["kernel"]), "bias": (a["filters"],)},
        ),
        _kind("maxpool2d", {"kernel": (True, _pos_int), "stride": (False, _pos_int)}, _pool_out, _no_params),
        _kind("flatten", {}, _flatten_out, _no_params),
        _kind("softmax-cross-entropy", {}, _sce_out, _no_params, loss_head=True, takes_targets=True),
        _kind(
            "embedding-lookup",
            {"vocab": (True, _pos_int), "dim": (True, _pos_int)},
            _embed_out,
            lambda s, a: {"table": (a["vocab"], a["dim"])},
        ),
    )
}


def kaiming_bound(fan_in: int) -> float:
    """Uniform bound for relu-gain layers (src/ops.py:371-373)."""
    return math.sqrt(6.0 / fan_in)


def init_node_params(node_id: str, op: str, shapes: dict, seed: int, rng_stream) -> dict:
    """Seeded initial values for one node (src/ops.py:376-398): keyed by (seed, pid), zero biases."""
    out = {}
    for pname, shape in shapes.items():
        pid = f"{node_id}.{pname}"
        if pname == "bias":
            out[pid] = np.zeros(shape, dtype=np.float32)
            continue
        if op == "dense":
            bound = kaiming_bound(shape[1])
        elif op == "conv2d":
            bound = kaiming_bound(shape[1] * shape[2] * shape[3])
        elif op == "embedding-lookup":
            bound = 1.0 / math.sqrt(shape[1])
        else:
            bound = 1.0
        out[pid] = rng_stream("init", seed, pid).uniform(-bound, bound, size=shape).astype(np.float32)
    return out


def check_class_indices(targets, classes: int) -> np.ndarray:
    """Float-coded labels -> int64, rejecting fractional or out-of-range values (src/ops.py:203-211)."""
    flat = np.asarray(targets).reshape(-1)
    as_int = flat.astype(np.int64)
    if not np.all(as_int == flat):
        raise ValueError("targets must hold integral class indices")
    if as_int.size and (as_int.min() < 0 or as_int.max() >= classes):
        raise ValueError(f"target class out of range [0, {classes})")
    return as_int


def softmax_cross_entropy(logits, targets):
    """Mean SCE loss and dlogits on the GPU (src/ops.py:243-251)."""
    from . import devops

    return devops.softmax_cross_entropy(logits, targets)
