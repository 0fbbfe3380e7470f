"""numpy restatement of hybridnn's training arithmetic (test oracle, see __init__).

Graphs are duck-typed: anything with ``input_shape``, ``output`` and
``nodes`` (each with ``node_id``, ``op``, ``inputs``, ``attrs``) works, so
both the reference's ModelGraph and the product's mirror type are accepted.
All arrays are float32 as in the reference (src/tensor.py:9-14).
"""
from __future__ import annotations

import hashlib
import math

import numpy as np

__all__ = [
    "keyed_generator", "keyed_permutation", "graph_chain", "out_shape", "param_layout",
    "init_model", "epoch_batches", "op_forward", "op_backward", "sce_loss_and_grad",
    "model_forward", "model_backward", "OracleOptimizer", "lr_for_epoch", "train_step",
    "standalone_training", "evaluate_split", "blob_splits", "image_splits",
    "dataset_digest", "encode_dataset",
]

F = np.float32
_ADAM_B1, _ADAM_B2, _ADAM_EPS = 0.9, 0.999, 1e-8


# --------------------------------------------------------------------------
# keyed random streams — src/rng.py:18-28


def keyed_generator(*parts) -> np.random.Generator:
    """Philox keyed by the first 16 bytes of sha256 over 0x1f-joined labels (src/rng.py:18-23)."""
    digest = hashlib.sha256(b"\x1f".join(str(p).encode("utf-8") for p in parts)).digest()
    return np.random.Generator(np.random.Philox(key=np.frombuffer(digest[:16], dtype=np.uint64)))


def keyed_permutation(n: int, *parts) -> np.ndarray:
    """src/rng.py:26-28."""
    return keyed_generator(*parts).permutation(n)


# --------------------------------------------------------------------------
# dataset container hash — src/formats.py:27-39,71-82 and src/store.py:55-56


def encode_dataset(splits: dict) -> bytes:
    """UNND v1 bytes: magic, u16 version=1, u16 count=4, then 4 named f32 sections."""
    import struct

    chunks = [b"UNND", struct.pack("<HH", 1, 4)]
    for name in ("train_x", "train_y", "test_x", "test_y"):
        arr = np.ascontiguousarray(splits[name], dtype="<f4")
        raw = name.encode("utf-8")
        chunks.append(struct.pack("<B", len(raw)) + raw + struct.pack("<B", arr.ndim))
        chunks.append(b"".join(struct.pack("<I", d) for d in arr.shape))
        chunks.append(arr.tobytes())
    return b"".join(chunks)


def dataset_digest(splits: dict) -> str:
    return hashlib.sha256(encode_dataset(splits)).hexdigest()


def blob_splits(tag, stream_name, classes, features, train_n, test_n, sigma=0.5):
    """Gaussian blobs around U(-2,2) centres (pkg/tests/conftest.py:59-70, keyed by ``tag``)."""
    centres = keyed_generator(tag, stream_name, "centers").uniform(-2.0, 2.0, size=(classes, features))
    out = {}
    for split, n in (("train", train_n), ("test", test_n)):
        g = keyed_generator(tag, stream_name, split)
        y = g.integers(0, classes, size=n)
        out[f"{split}_x"] = (centres[y] + g.normal(0.0, sigma, size=(n, features))).astype(F)
        out[f"{split}_y"] = y.astype(F)
    return out


def image_splits(tag, stream_name, classes, shape, train_n, test_n, sigma=0.35):
    """Noisy per-class patterns (src/demo.py:113-124 / pkg/tests/conftest.py:73-84)."""
    pats = keyed_generator(tag, stream_name, "patterns").uniform(0.0, 1.0, size=(classes,) + tuple(shape))
    out = {}
    for split, n in (("train", train_n), ("test", test_n)):
        g = keyed_generator(tag, stream_name, split)
        y = g.integers(0, classes, size=n)
        out[f"{split}_x"] = (pats[y] + g.normal(0.0, sigma, size=(n,) + tuple(shape))).astype(F)
        out[f"{split}_y"] = y.astype(F)
    return out


# --------------------------------------------------------------------------
# graph helpers — src/engine.py:22-52, src/ops.py:28-190


def graph_chain(graph) -> list:
    """Nodes in execution order.  Every valid graph is a chain (one input per
    node, src/model.py:114-117, everything reaches the output :129-137)."""
    by_id = {n.node_id: n for n in graph.nodes}
    chain, cur = [], graph.output
    while cur != "input":
        node = by_id[cur]
        chain.append(node)
        cur = node.inputs[0]
    return chain[::-1]


def _conv_len(size, k, s, p):
    return (size + 2 * p - k) // s + 1


def out_shape(op, in_shape, attrs):
    """Per-sample output shapes (src/ops.py:36-39,74-82,137-146,181-182,214-217,258-261)."""
    if op == "dense":
        return (attrs["units"],)
    if op == "relu":
        return tuple(in_shape)
    if op == "conv2d":
        c, h, w = in_shape
        k, s, p = attrs["kernel"], attrs.get("stride", 1), attrs.get("padding", 0)
        return (attrs["filters"], _conv_len(h, k, s, p), _conv_len(w, k, s, p))
    if op == "maxpool2d":
        c, h, w = in_shape
        k = attrs["kernel"]
        s = attrs.get("stride", k)
        return (c, _conv_len(h, k, s, 0), _conv_len(w, k, s, 0))
    if op == "flatten":
        return (int(np.prod(in_shape)),) if in_shape else (1,)
    if op == "softmax-cross-entropy":
        return ()
    if op == "embedding-lookup":
        return (in_shape[0], attrs["dim"])
    raise ValueError(op)


def _node_param_shapes(op, in_shape, attrs):
    """src/ops.py:42-43,85-88,264-265."""
    if op == "dense":
        return {"weight": (attrs["units"], in_shape[0]), "bias": (attrs["units"],)}
    if op == "conv2d":
        k = attrs["kernel"]
        return {"weight": (attrs["filters"], in_shape[0], k, k), "bias": (attrs["filters"],)}
    if op == "embedding-lookup":
        return {"table": (attrs["vocab"], attrs["dim"])}
    return {}


def param_layout(graph) -> dict:
    """{pid: shape} in graph declaration order (src/engine.py:42-52)."""
    shapes = {"input": tuple(graph.input_shape)}
    for node in graph_chain(graph):
        shapes[node.node_id] = out_shape(node.op, shapes[node.inputs[0]], node.attrs)
    specs = {}
    for node in graph.nodes:
        for name, shp in _node_param_shapes(node.op, shapes[node.inputs[0]], node.attrs).items():
            specs[f"{node.node_id}.{name}"] = tuple(shp)
    return specs


def init_model(graph, seed: int) -> dict:
    """Kaiming-uniform weights from keyed streams, zero biases (src/engine.py:59-69, src/ops.py:371-398)."""
    ops = {n.node_id: n.op for n in graph.nodes}
    params = {}
    for pid, shp in param_layout(graph).items():
        node_id, name = pid.rsplit(".", 1)
        if name == "bias":
            params[pid] = np.zeros(shp, dtype=F)
            continue
        op = ops[node_id]
        if op == "dense":
            bound = math.sqrt(6.0 / shp[1])
        elif op == "conv2d":
            bound = math.sqrt(6.0 / (shp[1] * shp[2] * shp[3]))
        elif op == "embedding-lookup":
            bound = 1.0 / math.sqrt(shp[1])
        else:
            bound = 1.0
        params[pid] = keyed_generator("init", seed, pid).uniform(-bound, bound, size=shp).astype(F)
    return params


def epoch_batches(train_x, train_y, digest, batch_size, seed, epoch):
    """[(x, y, idx)] for one epoch (src/store.py:68-81): keyed permutation, remainder kept."""
    n = train_x.shape[0]
    perm = keyed_permutation(n, "shuffle", digest, seed, epoch)
    return [
        (train_x[perm[s:s + batch_size]], train_y[perm[s:s + batch_size]], perm[s:s + batch_size])
        for s in range(0, n, batch_size)
    ]


# --------------------------------------------------------------------------
# op arithmetic — src/ops.py


def _im2col(x, k, s, oh, ow):
    """cols[n, c, i, j, oh, ow] = x[n, c, i + s*oh, j + s*ow] (src/ops.py:91-97)."""
    n, c = x.shape[:2]
    cols = np.empty((n, c, k, k, oh, ow), dtype=F)
    for i in range(k):
        for j in range(k):
            cols[:, :, i, j] = x[:, :, i:i + s * oh:s, j:j + s * ow:s]
    return cols


def op_forward(op, x, p, attrs):
    """Returns (y, saved) mirroring each kind's forward (src/ops.py:46-48,62-63,100-113,149-161,185-186,268-271)."""
    if op == "dense":
        return x @ p["weight"].T + p["bias"], {"x": x}
    if op == "relu":
        return np.maximum(x, F(0.0)), {"mask": x > 0}
    if op == "conv2d":
        k, s, pad = attrs["kernel"], attrs.get("stride", 1), attrs.get("padding", 0)
        w = p["weight"]
        if pad:
            x = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
        n, c, h, wd = x.shape
        oh, ow = _conv_len(h, k, s, 0), _conv_len(wd, k, s, 0)
        cols = _im2col(x, k, s, oh, ow)
        y = np.matmul(cols.reshape(n, c * k * k, oh * ow).transpose(0, 2, 1), w.reshape(w.shape[0], -1).T)
        y += p["bias"]
        y = np.ascontiguousarray(y.transpose(0, 2, 1).reshape(n, w.shape[0], oh, ow))
        return y, {"cols": cols, "in_shape": x.shape, "padding": pad}
    if op == "maxpool2d":
        k = attrs["kernel"]
        s = attrs.get("stride", k)
        n, c, h, w = x.shape
        oh, ow = _conv_len(h, k, s, 0), _conv_len(w, k, s, 0)
        win = np.empty((n, c, oh, ow, k, k), dtype=F)
        for i in range(k):
            for j in range(k):
                win[:, :, :, :, i, j] = x[:, :, i:i + s * oh:s, j:j + s * ow:s]
        flat = win.reshape(n, c, oh, ow, k * k)
        idx = flat.argmax(axis=-1)
        y = np.ascontiguousarray(np.take_along_axis(flat, idx[..., None], axis=-1)[..., 0])
        return y, {"idx": idx, "in_shape": x.shape}
    if op == "flatten":
        return np.ascontiguousarray(x.reshape(x.shape[0], -1)), {"in_shape": x.shape}
    if op == "embedding-lookup":
        table = p["table"]
        flat = x.reshape(-1)
        as_int = flat.astype(np.int64)
        if not np.all(as_int == flat):
            raise ValueError("targets must hold integral class indices")
        if as_int.size and (as_int.min() < 0 or as_int.max() >= table.shape[0]):
            raise ValueError("index out of range")
        idx = as_int.reshape(x.shape)
        return np.ascontiguousarray(table[idx]), {"idx": idx}
    raise ValueError(op)


def op_backward(op, dy, saved, p, attrs):
    """Returns (dx, {name: grad}) (src/ops.py:51-55,66-67,116-130,164-174,189-190,274-278)."""
    if op == "dense":
        return dy @ p["weight"], {"weight": dy.T @ saved["x"], "bias": dy.sum(axis=0)}
    if op == "relu":
        return dy * saved["mask"], {}
    if op == "conv2d":
        k, s = attrs["kernel"], attrs.get("stride", 1)
        cols, padded, pad = saved["cols"], saved["in_shape"], saved["padding"]
        db = dy.sum(axis=(0, 2, 3))
        dw = np.einsum("nfhw,ncijhw->fcij", dy, cols, dtype=F, casting="same_kind")
        dcols = np.einsum("nfhw,fcij->ncijhw", dy, p["weight"], dtype=F, casting="same_kind")
        oh, ow = dy.shape[2], dy.shape[3]
        dxp = np.zeros(padded, dtype=F)
        for i in range(k):
            for j in range(k):
                dxp[:, :, i:i + s * oh:s, j:j + s * ow:s] += dcols[:, :, i, j]
        if pad:
            dxp = dxp[:, :, pad:-pad, pad:-pad]
        return np.ascontiguousarray(dxp), {"weight": dw, "bias": db}
    if op == "maxpool2d":
        k = attrs["kernel"]
        s = attrs.get("stride", k)
        idx = saved["idx"]
        dx = np.zeros(saved["in_shape"], dtype=F)
        ni, ci, oi, wi = np.indices(idx.shape)
        np.add.at(dx, (ni, ci, oi * s + idx // k, wi * s + idx % k), dy)
        return dx, {}
    if op == "flatten":
        return dy.reshape(saved["in_shape"]), {}
    if op == "embedding-lookup":
        table = p["table"]
        dt = np.zeros_like(table)
        np.add.at(dt, saved["idx"].reshape(-1), dy.reshape(-1, table.shape[1]))
        return None, {"table": dt}
    raise ValueError(op)


def _class_indices(targets, classes):
    """src/ops.py:203-211."""
    flat = np.asarray(targets).reshape(-1)
    as_int = flat.astype(np.int64)
    if not np.all(as_int == flat):
        raise ValueError("targets must hold integral class indices")
    if as_int.size and (as_int.min() < 0 or as_int.max() >= classes):
        raise ValueError(f"target class out of range [0, {classes})")
    return as_int


def sce_loss_and_grad(logits, targets):
    """Mean softmax cross-entropy and d/dlogits (src/ops.py:220-251)."""
    t = _class_indices(targets, logits.shape[1])
    shifted = logits - logits.max(axis=1, keepdims=True)
    lse = np.log(np.exp(shifted).sum(axis=1))
    logp = shifted[np.arange(logits.shape[0]), t] - lse
    loss = F(-np.mean(logp, dtype=F))
    grad = np.exp(shifted - lse[:, None])
    grad[np.arange(logits.shape[0]), t] -= F(1.0)
    grad *= F(1.0) / F(logits.shape[0])
    return np.asarray(loss, dtype=F), grad


def model_forward(graph, params, x, targets=None):
    """Returns (logits, tape) — the chain evaluated like src/engine.py:82-113.

    A loss-head output node is not evaluated here: callers apply
    :func:`sce_loss_and_grad` to its input, which is what
    src/train.py:232-240 does with the same arithmetic.
    """
    tape = []
    h = np.ascontiguousarray(np.asarray(x, dtype=F))
    for node in graph_chain(graph):
        if node.op == "softmax-cross-entropy":
            break
        p = {k.rsplit(".", 1)[1]: v for k, v in params.items() if k.rsplit(".", 1)[0] == node.node_id}
        y, saved = op_forward(node.op, h, p, node.attrs)
        tape.append((node, p, saved))
        h = y
    return h, tape


def model_backward(tape, dlogits):
    """Reverse replay (src/engine.py:120-151); grads keyed by pid."""
    grads = {}
    d = dlogits
    for node, p, saved in reversed(tape):
        dx, dp = op_backward(node.op, d, saved, p, node.attrs)
        for name, g in dp.items():
            grads[f"{node.node_id}.{name}"] = g
        d = dx
    return grads


# --------------------------------------------------------------------------
# optimizer — src/optim.py:16-87


def lr_for_epoch(base, milestones, epoch):
    """src/optim.py:22-30."""
    return base * (0.1 ** sum(1 for m in milestones if epoch + 1 >= m))


class OracleOptimizer:
    """In-place SGD/momentum/Adam with the reference's f32 evaluation order."""

    def __init__(self, kind, momentum=0.0):
        self.kind, self.momentum, self.step = kind, momentum, 0
        self.slots = {}

    def apply(self, params, grads, lr):
        self.step += 1
        lr32 = F(lr)
        if self.kind == "sgd":
            for pid in sorted(params):
                g = grads[pid]
                if self.momentum:
                    prev = self.slots.get(pid)
                    g = g.copy() if prev is None else F(self.momentum) * prev + g
                    self.slots[pid] = g
                params[pid] -= lr32 * g
            return
        b1, b2, eps = F(_ADAM_B1), F(_ADAM_B2), F(_ADAM_EPS)
        c1 = F(1.0 - _ADAM_B1 ** self.step)
        c2 = F(1.0 - _ADAM_B2 ** self.step)
        for pid in sorted(params):
            g = grads[pid]
            m, v = self.slots.get(pid, (None, None))
            m = (F(1.0) - b1) * g if m is None else b1 * m + (F(1.0) - b1) * g
            v = (F(1.0) - b2) * g * g if v is None else b2 * v + (F(1.0) - b2) * g * g
            self.slots[pid] = (m, v)
            params[pid] -= lr32 * (m / c1) / (np.sqrt(v / c2) + eps)


# --------------------------------------------------------------------------
# training loop — src/train.py:223-279,453-476


def train_step(graph, params, x, y, opt, lr):
    """One batch (src/train.py:223-256). Returns (loss, correct); no update if loss non-finite."""
    with np.errstate(over="ignore", invalid="ignore"):
        logits, tape = model_forward(graph, params, x)
        loss, dlogits = sce_loss_and_grad(logits, y)
    if not np.isfinite(float(loss)):
        return float(loss), 0
    grads = model_backward(tape, dlogits)
    opt.apply(params, grads, lr)
    t = _class_indices(y, logits.shape[1])
    return float(loss), int((logits.argmax(axis=1) == t).sum())


def standalone_training(graph, splits, digest, epochs, batch_size, lr, optimizer, seed,
                        milestones=(), momentum=0.0, observer=None, max_steps=None):
    """train_standalone (src/train.py:453-476) plus per-epoch curve rows like
    Trainer._run_slice (:394-427).  ``observer(step, params, loss)`` sees every step."""
    params = init_model(graph, seed)
    opt = OracleOptimizer(optimizer, momentum)
    curve, step = [], 0
    for epoch in range(epochs):
        rate = lr_for_epoch(lr, milestones, epoch)
        loss_sum, correct, seen = 0.0, 0, 0
        for bx, by, _ in epoch_batches(splits["train_x"], splits["train_y"], digest, batch_size, seed, epoch):
            loss, c = train_step(graph, params, bx, by, opt, rate)
            if not np.isfinite(loss):
                return params, opt, curve, ("abort", epoch, step)
            loss_sum += loss * bx.shape[0]
            correct += c
            seen += bx.shape[0]
            if observer is not None:
                observer(step, params, loss)
            step += 1
            if max_steps is not None and step >= max_steps:
                return params, opt, curve, None
        curve.append((epoch, loss_sum / seen, correct / seen))
    return params, opt, curve, None


def evaluate_split(graph, params, x, y, batch_size):
    """src/train.py:259-279."""
    total = x.shape[0]
    if total == 0:
        return 0.0, 0.0
    loss_sum, correct = 0.0, 0
    for s in range(0, total, batch_size):
        bx, by = x[s:s + batch_size], y[s:s + batch_size]
        with np.errstate(over="ignore", invalid="ignore"):
            logits, _ = model_forward(graph, params, bx)
            loss, _ = sce_loss_and_grad(logits, by)
        loss_sum += float(loss) * bx.shape[0]
        correct += int((logits.argmax(axis=1) == _class_indices(by, logits.shape[1])).sum())
    return loss_sum / total, correct / total
