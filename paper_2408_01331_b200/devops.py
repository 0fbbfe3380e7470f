"""Single-model device execution of the op registry (the plugin API path).

``OP_KINDS[name].forward/backward`` land here: each call runs the same
grouped kernels as the hybrid trainer with a one-problem table.  Inputs may
be numpy arrays (copied to ``cuda:0``; results come back as numpy, matching
the reference's ndarray contract) or CUDA tensors (results stay on the
device).  The ``aux`` dict keeps device tensors between forward and backward.
"""
from __future__ import annotations

import numpy as np

from . import _native as N
from .errors import HybridnnError
from .ops import check_class_indices, conv_extent
from .runtime import STEP_DTYPE, STATUS_DTYPE, UnsupportedGraphError, _dev_table, _ptr


def _torch():
    import torch

    return torch


def _dev():
    torch = _torch()
    if not torch.cuda.is_available():
        raise HybridnnError("no CUDA device: device ops have no CPU fallback")
    N.load()
    return torch.device("cuda")


def _to_dev(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(_dev(), dtype=torch.float32).contiguous(), True
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32))).to(_dev()), False


def _back(t, keep):
    return t if keep else t.cpu().numpy()


def _cur(rows: int):
    torch = _torch()
    r = np.zeros(1, dtype=STEP_DTYPE)
    r["active"], r["rows"] = 1, rows
    return torch.from_numpy(r.view(np.uint8).copy()).to(_dev())


def _stream():
    return _torch().cuda.current_stream().cuda_stream


def _embed(op, x, table, y, dy, dtable):
    """One-problem hnn_embedding launch: x [B, L] token ids (validated), table [V, D]."""
    torch = _torch()
    B, L = x.shape
    V, D = table.shape
    blocks = -(-(B * L) // 8) if op == N.HNN_FWD else -(-V // 8)
    prob = N.EmbedProblem(x=_ptr(x), table=_ptr(table), y=_ptr(y), dy=_ptr(dy), dtable=_ptr(dtable), cap=B, len=L,
                          ldx=L, dim=D, vocab=V, model=0, block_base=0, blocks=blocks)
    t = torch.frombuffer(bytearray(N.table_bytes(N.EmbedProblem, [prob])), dtype=torch.uint8).to(_dev())
    N.call("hnn_embedding", op, _ptr(t), 1, blocks, _ptr(_cur(B)), 0, _stream())


def _gemm(op, rows, d):
    prec = N.PREC_SIMT
    tm, tn = N.tile_shape(op, prec)
    tiles_n = -(-d["n"] // tn)
    prob = N.GemmProblem(tile_base=0, tiles_n=tiles_n, model=0, **d)
    t = _dev_table(N.GemmProblem, [prob], _dev())
    cur = _cur(rows)
    N.call("hnn_grouped_gemm", op, prec, _ptr(t), 1, -(-d["m"] // tm) * tiles_n, _ptr(cur), 0, _stream())
    _torch().cuda.current_stream().synchronize()


def _conv(op, x, w, b, y, dy, dx, attrs, rows, dw=None, db=None):
    torch = _torch()
    n, c, h, wd = x.shape
    f, _, k, _ = w.shape
    s, p = attrs.get("stride", 1), attrs.get("padding", 0)
    oh, ow = conv_extent(h, k, s, p), conv_extent(wd, k, s, p)
    direct = N.conv_direct_ok(c, h, wd, f, k, oh, ow)
    split_len = 2048
    splits = -(-n // N.CONV_DIRECT_BCHUNK) if direct else -(-n * oh * ow // split_len)
    partial = torch.zeros(splits * f * (c * k * k + 1), dtype=torch.float32, device=x.device)
    common = dict(x=_ptr(x), weight=_ptr(w), bias=_ptr(b), y=_ptr(y), dy=_ptr(dy), dx=_ptr(dx), mask=0,
                  partial=_ptr(partial), dw=_ptr(dw), db=_ptr(db), cap=n, c=c, h=h, w=wd, f=f, k=k, stride=s,
                  pad=p, oh=oh, ow=ow, model=0, relu=0, splits=splits, split_len=split_len)
    cols = c * k * k + 1
    if direct:
        tiles_n = 1
        tiles = splits if op == N.HNN_WGRAD else n
    else:
        tm, tn = N.conv_tile_shape(op)
        if op == N.HNN_FWD:
            tiles_n, tiles = -(-f // tn), -(-(n * oh * ow) // tm) * -(-f // tn)
        elif op == N.HNN_DGRAD:
            tiles_n, tiles = -(-c // tn), -(-(n * h * wd) // tm) * -(-c // tn)
        else:
            tiles_n = -(-cols // tn)
            tiles = splits * -(-f // tm) * tiles_n
    t = _dev_table(N.ConvProblem, [N.ConvProblem(tile_base=0, tiles_n=tiles_n, **common)], x.device)
    cur = _cur(rows)
    if direct:
        N.call("hnn_grouped_conv_direct", op, _ptr(t), 1, tiles, N.conv_direct_smem(op, c, h, wd, f, k, oh, ow),
               _ptr(cur), 0, _stream())
    else:
        N.call("hnn_grouped_conv", op, _ptr(t), 1, tiles, _ptr(cur), 0, _stream())
    if op == N.HNN_WGRAD:
        nblk = -(-(f * cols) // 256)
        N.call("hnn_conv_wgrad_reduce", _ptr(t), 1, nblk, _ptr(cur), 0, _stream())
    torch.cuda.current_stream().synchronize()


def _pool(op, x, y, idx, dy, dx, attrs):
    n, c, h, w = x.shape
    k = attrs["kernel"]
    s = attrs.get("stride", k)
    oh, ow = conv_extent(h, k, s, 0), conv_extent(w, k, s, 0)
    mode, blocks = N.pool_mode_blocks(op, n, c, h, w, k, s, oh, ow, (_ptr(x), _ptr(dx)) if op != N.HNN_FWD else (_ptr(x),))
    prob = N.PoolProblem(_ptr(x), _ptr(y), _ptr(idx), _ptr(dy), _ptr(dx), 0, n, c, h, w, k, s, oh, ow, 0, 0,
                         blocks, mode)
    t = _dev_table(N.PoolProblem, [prob], x.device)
    N.call("hnn_grouped_maxpool", op, _ptr(t), 1, blocks, _ptr(_cur(n)), 0, _stream())
    _torch().cuda.current_stream().synchronize()


def _relu(op, x, y, dy, dx):
    n = x.shape[0]
    row = int(np.prod(x.shape[1:])) if x.dim() > 1 else 1
    blocks = -(-(n * row) // 256)
    prob = N.ReluProblem(_ptr(x), _ptr(y), _ptr(dy), _ptr(dx), n, row, 0, 0, blocks, 0)
    t = _dev_table(N.ReluProblem, [prob], x.device)
    N.call("hnn_grouped_relu", op, _ptr(t), 1, blocks, _ptr(_cur(n)), 0, _stream())
    _torch().cuda.current_stream().synchronize()


def sce_device(logits, labels_i32, with_grad=True):
    """(loss f32 tensor[1], dlogits or None, correct int) for one logits block on the device."""
    torch = _torch()
    B, Cc = logits.shape
    dl = torch.empty_like(logits) if with_grad else None
    status = torch.from_numpy(np.zeros(1, dtype=STATUS_DTYPE).view(np.uint8).copy()).to(logits.device)
    loss = torch.zeros(1, dtype=torch.float32, device=logits.device)
    corr = torch.zeros(1, dtype=torch.int32, device=logits.device)
    prob = N.SceProblem(_ptr(logits), _ptr(labels_i32), _ptr(dl), Cc, Cc, B, 0)
    t = _dev_table(N.SceProblem, [prob], logits.device)
    N.call("hnn_sce_fused", _ptr(t), 1, B, Cc, _ptr(_cur(B)), _ptr(status), 0, _ptr(loss), _ptr(corr), _stream())
    torch.cuda.current_stream().synchronize()
    return loss, dl, int(corr.item())


def softmax_cross_entropy(logits, targets):
    torch = _torch()
    x, keep = _to_dev(logits)
    t = torch.from_numpy(check_class_indices(_host(targets), x.shape[1]).astype(np.int32)).to(x.device)
    loss, dl, _ = sce_device(x, t)
    return np.float32(loss.item()), _back(dl, keep)


def _host(a):
    torch = _torch()
    return a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


def forward(name, x, params, attrs, targets=None):
    torch = _torch()
    xd, keep = _to_dev(x)
    P = {k: _to_dev(v)[0] for k, v in params.items()}
    if name == "dense":
        B, K = xd.shape
        U = P["weight"].shape[0]
        y = torch.empty(B, U, dtype=torch.float32, device=xd.device)
        _gemm(N.HNN_FWD, B, dict(a=_ptr(xd), b=_ptr(P["weight"]), c=_ptr(y), bias=_ptr(P["bias"]), mask=0, dbias=0,
                                 m=B, n=U, k=K, lda=K, ldb=K, ldc=U, relu=0))
        return _back(y, keep), {"x": xd, "keep": keep}
    if name == "relu":
        y = torch.empty_like(xd)
        _relu(N.HNN_FWD, xd, y, None, None)
        return _back(y, keep), {"x": xd, "keep": keep}
    if name == "conv2d":
        n, c, h, w = xd.shape
        k, s, p = attrs["kernel"], attrs.get("stride", 1), attrs.get("padding", 0)
        f = P["weight"].shape[0]
        y = torch.empty(n, f, conv_extent(h, k, s, p), conv_extent(w, k, s, p), dtype=torch.float32,
                        device=xd.device)
        _conv(N.HNN_FWD, xd, P["weight"], P["bias"], y, None, None, attrs, n)
        return _back(y, keep), {"x": xd, "keep": keep}
    if name == "maxpool2d":
        n, c, h, w = xd.shape
        k = attrs["kernel"]
        s = attrs.get("stride", k)
        if k * k > 256:
            raise UnsupportedGraphError("pool windows above 16x16 are not supported")
        oh, ow = conv_extent(h, k, s, 0), conv_extent(w, k, s, 0)
        y = torch.empty(n, c, oh, ow, dtype=torch.float32, device=xd.device)
        idx = torch.empty(n * c * oh * ow, dtype=torch.uint8, device=xd.device)
        _pool(N.HNN_FWD, xd, y, idx, None, None, attrs)
        return _back(y, keep), {"x": xd, "idx": idx, "keep": keep}
    if name == "flatten":
        y = xd.reshape(xd.shape[0], -1)
        return _back(y, keep), {"in_shape": tuple(xd.shape), "keep": keep}
    if name == "softmax-cross-entropy":
        if targets is None:
            raise ValueError("softmax-cross-entropy needs batch targets")
        t = check_class_indices(_host(targets), xd.shape[1])
        if t.shape[0] != xd.shape[0]:
            raise ValueError("targets batch dimension does not match logits")
        loss, dl, _ = sce_device(xd, torch.from_numpy(t.astype(np.int32)).to(xd.device))
        return np.asarray(loss.item(), dtype=np.float32), {"dlogits": dl, "keep": keep}
    if name == "embedding-lookup":
        table = P["table"]
        check_class_indices(_host(x), table.shape[0])  # same errors as the reference (ops.py:268-270)
        xx = xd.reshape(xd.shape[0], -1).contiguous()
        y = torch.empty(xx.shape[0], xx.shape[1], table.shape[1], dtype=torch.float32, device=xd.device)
        _embed(N.HNN_FWD, xx, table, y, None, None)
        return _back(y.reshape(*xd.shape, table.shape[1]), keep), {"x": xx, "keep": keep}
    raise UnsupportedGraphError(f"op {name!r} has no device kernel")


def backward(name, dy, aux, params, attrs):
    torch = _torch()
    keep = aux.get("keep", False)
    P = {k: _to_dev(v)[0] for k, v in params.items()}
    if name == "softmax-cross-entropy":
        scale = float(np.float32(_host(dy)))
        dl = aux["dlogits"] if scale == 1.0 else aux["dlogits"] * scale
        return _back(dl, keep), {}
    dyd = _to_dev(dy)[0]
    if name == "dense":
        x = aux["x"]
        B, K = x.shape
        U = P["weight"].shape[0]
        dx = torch.empty(B, K, dtype=torch.float32, device=x.device)
        dw = torch.empty(U, K, dtype=torch.float32, device=x.device)
        db = torch.empty(U, dtype=torch.float32, device=x.device)
        _gemm(N.HNN_DGRAD, B, dict(a=_ptr(dyd), b=_ptr(P["weight"]), c=_ptr(dx), bias=0, mask=0, dbias=0, m=B, n=K,
                                   k=U, lda=U, ldb=K, ldc=K, relu=0))
        _gemm(N.HNN_WGRAD, B, dict(a=_ptr(dyd), b=_ptr(x), c=_ptr(dw), bias=0, mask=0, dbias=_ptr(db), m=U, n=K, k=B,
                                   lda=U, ldb=K, ldc=K, relu=0))
        return _back(dx, keep), {"weight": _back(dw, keep), "bias": _back(db, keep)}
    if name == "relu":
        x = aux["x"]
        dx = torch.empty_like(x)
        _relu(N.HNN_DGRAD, x, None, dyd, dx)
        return _back(dx, keep), {}
    if name == "conv2d":
        x = aux["x"]
        dx = torch.empty_like(x)
        dw = torch.empty_like(P["weight"])
        db = torch.empty_like(P["bias"])
        _conv(N.HNN_DGRAD, x, P["weight"], P["bias"], None, dyd, dx, attrs, x.shape[0])
        _conv(N.HNN_WGRAD, x, P["weight"], P["bias"], None, dyd, None, attrs, x.shape[0], dw, db)
        return _back(dx, keep), {"weight": _back(dw, keep), "bias": _back(db, keep)}
    if name == "maxpool2d":
        x = aux["x"]
        dx = torch.empty_like(x)
        _pool(N.HNN_DGRAD, x, None, aux["idx"], dyd, dx, attrs)
        return _back(dx, keep), {}
    if name == "flatten":
        return _back(dyd.reshape(aux["in_shape"]), keep), {}
    if name == "embedding-lookup":
        table = P["table"]
        dt = torch.empty_like(table)
        _embed(N.HNN_WGRAD, aux["x"], table, None, dyd.contiguous(), dt)
        return None, {"table": _back(dt, keep)}  # indices carry no gradient
    raise UnsupportedGraphError(f"op {name!r} has no device kernel")


def graph_forward(graph, params: dict, batch, targets=None):
    """Chain forward of one model on the device; returns logits (or the loss for a loss head)."""
    from .engine import chain
    from .ops import OP_KINDS

    torch = _torch()
    h = _to_dev(batch)[0]
    for node in chain(graph):
        kind = OP_KINDS[node.op]
        p = {k.rsplit(".", 1)[1]: v for k, v in params.items() if k.rsplit(".", 1)[0] == node.node_id}
        h, _ = forward(node.op, h, p, node.attrs, targets if kind.takes_targets else None)
    return h.cpu().numpy() if isinstance(h, torch.Tensor) else h
