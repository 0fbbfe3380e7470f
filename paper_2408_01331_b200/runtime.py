"""Device runtime for a merged hybrid: packing, launch plans, lockstep steps.

A :class:`DeviceHybrid` owns, for the models of one rank:

* packed HBM arenas — params / grads / moment-1 / moment-2, one contiguous
  16-byte-aligned segment per model, tensors inside in the reference's
  param_specs order (src/engine.py:42-52);
* per-model activation buffers ([batch, features], NCHW for images) and two
  ping-pong gradient buffers;
* compiled launch plans: every model's op chain is lowered to *stages*
  (dense / conv with relu fused into the producer, max-pool, stand-alone
  relu; flatten is a view) and stage ``w`` of every model runs in the same
  grouped launch per kind ("wave");
* the per-step schedule (``hnn_step_row`` per model) in device memory, read
  by every kernel through the ``cur`` row block that ``hnn_step_begin``
  refreshes, so a whole step is a fixed launch sequence that can be replayed
  as a CUDA graph.

Everything here calls the C-ABI (``_native``); nothing computes on the CPU.
"""
from __future__ import annotations

import os

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import HybridnnError, ShapeMismatchError
from .ops import OP_KINDS, conv_extent

STEP_DTYPE = np.dtype([("active", "<i4"), ("rows", "<i4"), ("perm_base", "<i4"), ("epoch", "<i4"),
                       ("batch", "<i4"), ("opt_step", "<i4"), ("lr", "<f4"), ("bias1", "<f4"),
                       ("bias2", "<f4"), ("reserved", "<i4", (3,))])
STATUS_DTYPE = np.dtype([("alive", "<i4"), ("abort_epoch", "<i4"), ("abort_batch", "<i4"),
                         ("last_correct", "<i4"), ("last_loss", "<f4"), ("reserved", "<i4"),
                         ("loss_sum", "<f8"), ("correct_sum", "<i8"), ("seen", "<i8")])
assert STEP_DTYPE.itemsize == 48 and STATUS_DTYPE.itemsize == 48

OPT_CHUNK = 4096
CONV_SPLIT_LEN = 2048
TC_MIN_DIM = 64  # smallest M/N/K worth a tcgen05 tile; smaller problems stay on CUDA cores


class UnsupportedGraphError(HybridnnError):
    """The graph uses something the device path does not implement."""


def _torch():
    import torch

    return torch


RSC_STAGE_MAX = 512 * 9  # k*k*channels one (r, s, c) weight-permute CTA stages (csrc/conv_tc.cu RSC_MAX)


def _implicit_tiles(oh: int, ow: int, rows: int = 128) -> bool:
    """A GEMM tile of `rows` output pixels is whole rows of one image, or whole images (4D TMA box)."""
    return ow <= rows and rows % ow == 0 and ((oh * ow) % rows == 0 or rows % (oh * ow) == 0)


def _parity_offsets(c: int, f: int) -> list:
    """Element offsets of the four parity-class weight blocks [c, kh*kw*f] inside wpar (9*c*f)."""
    offs, o = [], 0
    for q in range(4):
        offs.append(o)
        o += c * f * (1 + (q >> 1)) * (1 + (q & 1))
    return offs


def _align4(n: int) -> int:
    return (n + 3) // 4 * 4


# --------------------------------------------------------------------------- stages


@dataclass
class Stage:
    kind: str                  # dense | conv | pool | relu
    node_id: str
    attrs: dict
    in_shape: tuple
    out_shape: tuple
    relu: bool = False         # relu fused into this producer's epilogue
    mask_input: bool = False   # grad wrt input is multiplied by (input > 0) (producer had a fused relu)
    needs_dx: bool = False     # some parameter lives upstream
    params: tuple = ()         # pids (weight, bias) in the model namespace
    # filled when buffers are bound
    ld_in: int = 0
    ld_out: int = 0
    x = None
    y = None
    dy = None
    dx = None
    idx = None
    partial = None
    splits: int = 0
    # tensor-core conv lowering (im2col + CTA-pair GEMM)
    tc: bool = False
    ksplit: int = 1
    ksplit_len: int = 0
    cols = None
    dyt = None
    bpart = None
    kkp: int = 0
    wpad = None
    dg_fwd: bool = False
    wflip = None
    bf16: bool = False
    pix_ld: int = 0
    colst = None
    dyk = None
    wt = None
    fld: int = 0
    im_fwd: bool = False       # implicit-GEMM forward over xh (NHWC bf16 copy of x)
    im_dg: bool = False        # implicit-GEMM input gradient over dyt (NHWC dy)
    xh = None
    im_wg: bool = False        # implicit-GEMM weight gradient (B = xh, MN-major)
    par_dg: bool = False       # stride-2 input gradient as four parity-class implicit convs
    wpar = None
    xh_next = None             # the next conv's xh, written by this conv's forward epilogue
    xh_from_prev: bool = False # xh is written by the previous conv's forward epilogue


def lower_graph(graph) -> tuple:
    """Chain of nodes -> (stages, logits_features, loss_head).  Raises for unsupported graphs."""
    from .engine import chain, infer_shapes

    nodes = chain(graph)
    shapes = infer_shapes(graph)
    loss_head = OP_KINDS[nodes[-1].op].loss_head
    body = nodes[:-1] if loss_head else nodes
    stages: list = []
    i = 0
    while i < len(body):
        n = body[i]
        ins = shapes[n.inputs[0]]
        outs = shapes[n.node_id]
        if n.op in ("dense", "conv2d"):
            st = Stage("dense" if n.op == "dense" else "conv", n.node_id, dict(n.attrs), ins, outs,
                       params=(f"{n.node_id}.weight", f"{n.node_id}.bias"))
            # fuse a following relu when its consumer's backward can apply the mask
            if i + 1 < len(body) and body[i + 1].op == "relu":
                j = i + 2
                while j < len(body) and body[j].op == "flatten":
                    j += 1
                if j < len(body) and body[j].op in ("dense", "conv2d", "maxpool2d"):
                    st.relu = True
                    i += 1
            stages.append(st)
        elif n.op == "maxpool2d":
            if n.attrs["kernel"] ** 2 > 256:
                raise UnsupportedGraphError(f"node {n.node_id!r}: pool windows above 16x16 are not supported")
            stages.append(Stage("pool", n.node_id, dict(n.attrs), ins, outs))
        elif n.op == "relu":
            stages.append(Stage("relu", n.node_id, {}, ins, outs))
        elif n.op == "flatten":
            if stages:
                stages[-1].out_shape = outs  # a view: same memory, flat per-sample shape
        elif n.op == "embedding-lookup":
            if stages:
                raise UnsupportedGraphError(f"node {n.node_id!r}: embedding-lookup must read the model input")
            stages.append(Stage("embed", n.node_id, dict(n.attrs), ins, outs, params=(f"{n.node_id}.table",)))
        else:
            raise UnsupportedGraphError(f"node {n.node_id!r}: op {n.op!r} cannot appear here")
        i += 1
    if not stages:
        raise UnsupportedGraphError("graph has no parameterised or elementwise stage")
    final = shapes[body[-1].node_id]
    if len(final) != 1:
        raise ShapeMismatchError(body[-1].node_id, f"softmax-cross-entropy needs flat logits, got {final}")
    seen_param = False
    for k, st in enumerate(stages):
        st.needs_dx = seen_param
        if st.kind in ("dense", "conv", "embed"):
            seen_param = True
        if k > 0 and stages[k - 1].relu:
            st.mask_input = True
    return stages, final[0], loss_head


# --------------------------------------------------------------------------- models / datasets


@dataclass
class ModelSlot:
    """One model on this rank: graph, hyper-parameters and arena placement."""

    index: int
    job_id: str
    graph: object
    batch_size: int
    optimizer: str
    momentum: float
    specs: dict                  # pid -> shape (param_specs order)
    stages: list = field(default_factory=list)
    classes: int = 0
    offsets: dict = field(default_factory=dict)  # pid -> float offset in the arena
    seg_off: int = 0
    seg_len: int = 0
    sample_shape: tuple = ()
    batch_x = None
    batch_y = None
    grads_buf: list = field(default_factory=list)

    @property
    def opt_kind(self) -> int:
        if self.optimizer == "adam":
            return N.OPT_ADAM
        return N.OPT_SGD_MOMENTUM if self.momentum else N.OPT_SGD


class DeviceDataset:
    """A dataset resident in HBM once: samples as f32, labels as int32 class ids."""

    def __init__(self, ds, device):
        torch = _torch()
        from .ops import check_class_indices

        self.content_hash = ds.content_hash
        self.sample_shape = tuple(ds.train_x.shape[1:])
        self.n_train, self.n_test = int(ds.train_x.shape[0]), int(ds.test_x.shape[0])
        ytr = check_class_indices(ds.train_y, 1 << 30).astype(np.int32)
        yte = check_class_indices(ds.test_y, 1 << 30).astype(np.int32) if self.n_test else np.zeros(0, np.int32)
        self.train_x = torch.from_numpy(np.ascontiguousarray(ds.train_x, dtype=np.float32)).to(device)
        self.test_x = torch.from_numpy(np.ascontiguousarray(ds.test_x, dtype=np.float32)).to(device)
        self.train_y = torch.from_numpy(ytr).to(device)
        self.test_y = torch.from_numpy(yte).to(device)
        self.max_label = int(max(ytr.max(initial=0), yte.max(initial=0)))
        self._finish(device)

    @classmethod
    def from_tensors(cls, content_hash, train_x, train_y, test_x, test_y, max_label, device):
        """Wrap tensors already on the device (e.g. received through an NCCL broadcast)."""
        self = cls.__new__(cls)
        self.content_hash = content_hash
        self.sample_shape = tuple(train_x.shape[1:])
        self.n_train, self.n_test = int(train_x.shape[0]), int(test_x.shape[0])
        self.train_x, self.train_y, self.test_x, self.test_y = train_x, train_y, test_x, test_y
        self.max_label = int(max_label)
        self._finish(device)
        return self

    def _finish(self, device):
        torch = _torch()
        self.identity = torch.arange(max(self.n_test, 1), dtype=torch.int32, device=device)
        self.nbytes = int(sum(t.numel() * t.element_size() for t in (self.train_x, self.train_y, self.test_x,
                                                                          self.test_y)))


# --------------------------------------------------------------------------- launches


# kernel families for the roofline (bench.py) and the ncu traffic map (tools/ncu_traffic.py)
GEMM_FAMILY = {N.PREC_SIMT: "gemm/simt", N.PREC_SIMT_SKINNY: "gemm/skinny", N.PREC_3XTF32: "gemm/tc-3xtf32",
               N.PREC_3XTF32_PAIR: "gemm/tc2-3xtf32", N.PREC_BF16_PAIR: "gemm/tc2-bf16"}
ENTRY_FAMILY = {"hnn_multi_tensor_adam": "optimizer", "hnn_multi_tensor_sgd": "optimizer", "hnn_sce_fused": "sce",
                "hnn_gather_rows": "gather", "hnn_splitk_epilogue": "splitk_epilogue",
                "hnn_grouped_conv": "conv/simt", "hnn_grouped_conv_direct": "conv/direct",
                "hnn_grouped_conv_direct_ex": "conv/direct", "hnn_skinny_backward": "gemm/skinny",
                "hnn_logits_tail": "logits_tail",
                "hnn_conv_wgrad_reduce": "conv/wgrad_reduce", "hnn_embedding": "embed",
                "hnn_grouped_maxpool": "pool", "hnn_grouped_relu": "relu", "hnn_conv_tc_aux": "conv/tc_aux"}


class Launch:
    """One C-ABI call with its device-resident problem table."""

    def __init__(self, entry: str, args: tuple, table=None, label: str = "", flops: int = 0, nbytes: int = 0):
        self.entry, self.args, self.table, self.label = entry, args, table, label
        # algorithmic work of one launch (all problems, full batches): the roofline numerators
        self.flops, self.nbytes = flops, nbytes
        if entry == "hnn_grouped_gemm":
            self.family = GEMM_FAMILY[args[1]]
        else:
            self.family = ENTRY_FAMILY.get(entry, entry)

    def run(self, stream) -> None:
        N.call(self.entry, *self.args, stream)


def _dev_table(cls, rows, device, extra: bytes = b""):
    torch = _torch()
    raw = N.table_bytes(cls, rows) + extra
    t = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)
    return t


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def C_addr(cobj) -> int:
    import ctypes

    return ctypes.addressof(cobj)


def C_addr_bytes(buf: bytearray) -> int:
    import ctypes

    return ctypes.addressof((ctypes.c_char * len(buf)).from_buffer(buf))


_TF32_CHECKED: set = set()


def tf32_truncation_selftest(device) -> float:
    """Assert the hardware fact the 3xTF32 GEMMs rely on (gemm_tc2.cu:11-13): a kind::tf32 MMA fed
    raw fp32 operands uses their TRUNCATED tf32 value, so hi = x (no conversion) and the converters'
    lo = x - trunc_tf32(x) add back to x exactly.  One 64 x 64 x 64 pair-GEMM forward on operands
    x = 1 + 2^-11 + 2^-12 (truncation gives hi = 1, round-to-nearest would give 1 + 2^-10): the
    3xTF32 result is 64 x^2 to 5.4e-7 (the dropped lo*lo term) when the hardware truncates and off by
    2^-9 when it rounds.  Runs once per device and process (DeviceHybrid construction); raises
    DeviceError if the assumption fails.  Returns the measured relative error."""
    torch = _torch()
    key = str(device)
    if key in _TF32_CHECKED:
        return 0.0
    _TF32_CHECKED.add(key)  # (the probe hybrid below must not recurse into the check)
    from . import zoo
    from .unify import merge

    x = 1.0 + 2.0 ** -11 + 2.0 ** -12
    job = zoo.TrainingJob("tf32-selftest", zoo.mlp(64, (64,), 16), "-", zoo.HyperParams(1, 64, 1.0), 0, 0)
    dev = merge([job]).materialize(device)
    s = dev.slots[0]
    st = s.stages[0]
    dev.upload_params(0, {pid: np.full(shp, x if pid.endswith("weight") else 0.0, np.float32)
                          for pid, shp in s.specs.items()})
    fake = DeviceDataset.from_tensors("-", torch.zeros(64, 64, device=dev.device), torch.zeros(64, dtype=torch.int32,
                                      device=dev.device), torch.zeros(1, 64, device=dev.device),
                                      torch.zeros(1, dtype=torch.int32, device=dev.device), 0, dev.device)
    dev.bind_datasets([fake], 64)
    dev.build_plans()
    probe = [l for l in dev.forward_plan if l.label.startswith("fwd0/dense/")]  # (+ a split-K epilogue)
    if not any(l.label == "fwd0/dense/tc2" for l in probe):  # tensor cores routed off: nothing to check
        return 0.0
    rows = np.zeros((1, 1), dtype=STEP_DTYPE)
    rows["active"], rows["rows"] = 1, 64
    dev.load_schedule(rows)
    s.batch_x.fill_(x)
    dev.run_plan(probe)
    got = st.y[:, :64].double().cpu().numpy()
    err = float(np.max(np.abs(got - 64.0 * x * x)) / (64.0 * x * x))
    if not np.isfinite(err) or err > 1e-5:
        from .errors import DeviceError

        raise DeviceError("tf32_truncation_selftest", -1,
                          f"3xTF32 GEMM error {err:.2e} on operands with sub-tf32 bits: the tensor core does not "
                          "truncate raw fp32 operands to tf32 as gemm_tc2.cu assumes (expected <= 1e-5)")
    return err


class DeviceHybrid:
    """Packed device state + launch plans for the models of one rank."""

    def __init__(self, slots: list, device=None, use_tensor_cores: bool = True, fuse_optimizer: bool = True,
                 keep_grads: bool = False, conv_precision: str = "f32"):
        torch = _torch()
        # fuse_optimizer: dense layers apply SGD/Adam in their weight-gradient epilogue (the
        # gradient never round-trips HBM); keep_grads: still store dW/db (tests, diagnostics)
        self.fuse_optimizer, self.keep_grads = fuse_optimizer, keep_grads
        N.load()
        if not torch.cuda.is_available():
            raise HybridnnError("no CUDA device: the hybrid trainer has no CPU fallback")
        self.device = torch.device(device or "cuda")
        self.slots = slots
        self.n = len(slots)
        self.use_tc = use_tensor_cores
        if conv_precision not in ("f32", "bf16"):
            raise ValueError(f"conv_precision must be 'f32' or 'bf16', not {conv_precision!r}")
        # tensor-core convolutions: "f32" = 3xTF32 (fp32 parity), "bf16" = kind::f16 with bf16
        # operands, fp32 accumulation and fp32 master weights (BASELINE C4)
        self.conv_bf16 = conv_precision == "bf16"
        # CTA-pair tcgen05 GEMM (HNN_TC_PAIR=0: single-CTA kernel)
        # conv layers with at least this many filters use the tensor-core conv path
        self.tc_conv_min_f = int(os.environ.get("HNN_TC_CONV_MIN_F", "64"))
        self.use_pairs = os.environ.get("HNN_TC_PAIR", "1") != "0"
        # bf16 tensor-core convs read NHWC activations through 4D TMA maps where the shape allows
        self.implicit_conv = os.environ.get("HNN_IMPLICIT_CONV", "1") != "0"
        if os.environ.get("HNN_FUSE_OPT", "1") == "0":  # SGD / momentum in the multi-tensor pass
            self.fuse_optimizer = False
        off = 0
        for s in slots:
            s.stages, s.classes, _ = lower_graph(s.graph)
            s.sample_shape = tuple(s.graph.input_shape)
            s.seg_off = off
            for pid, shp in s.specs.items():
                s.offsets[pid] = off
                off += _align4(int(np.prod(shp)))
            s.seg_len = off - s.seg_off
        self.arena_len = max(off, 4)
        f32 = dict(dtype=torch.float32, device=self.device)
        self.params = torch.zeros(self.arena_len, **f32)
        self.grads = torch.zeros(self.arena_len, **f32)
        need_m = any(s.opt_kind != N.OPT_SGD for s in slots)
        need_v = any(s.opt_kind == N.OPT_ADAM for s in slots)
        self.m1 = torch.zeros(self.arena_len, **f32) if need_m else None
        self.m2 = torch.zeros(self.arena_len, **f32) if need_v else None
        self.cur = torch.zeros(self.n * 48, dtype=torch.uint8, device=self.device)
        self.counter = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.status = torch.zeros(self.n * 48, dtype=torch.uint8, device=self.device)
        self.eval_status = torch.zeros(self.n * 48, dtype=torch.uint8, device=self.device)
        self.loss_out = torch.zeros(self.n, **f32)
        self.correct_out = torch.zeros(self.n, dtype=torch.int32, device=self.device)
        self.sched = None
        self.reset_status()
        self._bind_buffers()
        self.train_plan: list = []
        self.eval_plan: list = []
        self.forward_plan: list = []
        self.graph = None
        self.datasets = {}
        if self.use_tc and self.use_pairs:
            tf32_truncation_selftest(self.device)

    # ------------------------------------------------------------------ buffers
    def _bind_buffers(self):
        torch = _torch()
        dev = self.device
        # every model's input batch lives in one arena so a host-fed step is a single H2D copy
        lds, xo, yo = [], [], []
        xoff = yoff = 0
        for s in self.slots:
            sample = int(np.prod(s.sample_shape))
            ld0 = _align4(sample) if s.stages[0].kind == "dense" else sample
            lds.append(ld0)
            xo.append(xoff)
            yo.append(yoff)
            xoff += _align4(s.batch_size * ld0)
            yoff += _align4(s.batch_size)
        self.batch_arena = torch.zeros(max(xoff, 4), dtype=torch.float32, device=dev)
        self.label_arena = torch.zeros(max(yoff, 4), dtype=torch.int32, device=dev)
        self.batch_layout = list(zip(xo, yo, lds))
        for s, ld0, a, b in zip(self.slots, lds, xo, yo):
            cap = s.batch_size
            s.batch_x = self.batch_arena[a:a + cap * ld0].view(cap, ld0)
            s.batch_y = self.label_arena[b:b + cap]
            prev_out, prev_ld = s.batch_x, ld0
            widest = ld0
            dcols_need = dgb_need = 0
            for st in s.stages:
                st.x, st.ld_in = prev_out, prev_ld
                feats = int(np.prod(st.out_shape))
                if st.kind == "dense":
                    st.ld_out = _align4(feats)
                elif st.kind == "embed":
                    st.ld_out = feats  # [len, dim] rows back to back
                elif st.kind == "relu":
                    st.ld_out = st.ld_in
                else:
                    st.ld_out = feats
                st.y = torch.zeros(cap, st.ld_out, dtype=torch.float32, device=dev)
                if st.kind == "pool":
                    st.idx = torch.zeros(cap * feats, dtype=torch.uint8, device=dev)
                if st.kind == "conv":
                    c, h, w = st.in_shape
                    f, oh, ow = self._conv_out(st)
                    k = st.attrs["kernel"]
                    # small layers (LeNet-class) use the direct shared-memory kernels; layers with
                    # C*k*k and F >= 64 go to the tensor cores (im2col + CTA-pair 3xTF32 GEMM)
                    st.direct = N.conv_direct_ok(c, h, w, f, k, oh, ow)
                    kk = c * k * k
                    stride = st.attrs.get("stride", 1)
                    st.tc = (self.use_tc and self.use_pairs and kk >= 16 and f >= self.tc_conv_min_f
                             and (k <= 3 or (k <= 5 and stride == 1)) and stride <= 2
                             and (not st.direct or self.tc_conv_min_f < 64))
                    if st.tc:
                        pix = cap * oh * ow
                        st.bf16 = self.conv_bf16
                        # cols / weight rows padded to 16 bytes for TMA (8 bf16 / 4 fp32 elements)
                        st.kkp = -(-kk // 8) * 8 if st.bf16 else _align4(kk)
                        wdt = torch.bfloat16 if st.bf16 else torch.float32
                        st.wpad = (torch.zeros(f * st.kkp, dtype=wdt, device=dev)
                                   if (st.kkp != kk or st.bf16) else None)
                        kk = st.kkp
                        kq = 64 if st.bf16 else 32  # K block of the GEMM
                        tiles_mn = -(-f // 256) * -(-kk // 256)
                        split = max(1, min(-(-148 // tiles_mn), -(-pix // 1024)))
                        st.ksplit_len = -(-(-(-pix // split)) // kq) * kq
                        st.ksplit = -(-pix // st.ksplit_len)
                        st.pix_ld = -(-pix // 8) * 8
                        # implicit-GEMM forward (bf16, stride 1, 64-channel K blocks, output tiles of
                        # whole rows / images): the GEMM reads an NHWC copy of x through a 4D TMA map,
                        # no cols matrix (im2col still writes the weight-gradient copy colst)
                        st.im_fwd = (self.implicit_conv and st.bf16 and stride == 1 and c % 64 == 0
                                     and k * k * c <= RSC_STAGE_MAX and _implicit_tiles(oh, ow))
                        st.xh = torch.zeros(cap * h * w * c, dtype=wdt, device=dev) if st.im_fwd else None
                        # implicit weight gradient too (B = the same NHWC copy, MN-major, 64-pixel K
                        # blocks): needs the zero-filled copy im2col writes for "same" layers
                        st.im_wg = (st.im_fwd and stride == 1 and (oh, ow) == (h, w) and _implicit_tiles(oh, ow, 64)
                                    and st.ksplit_len % 64 == 0)
                        st.cols = None if st.im_fwd else torch.zeros(pix * kk, dtype=wdt, device=dev)
                        st.bpart = torch.zeros(cap * -(-(oh * ow) // 32) * f, dtype=torch.float32, device=dev)
                        st.partial = torch.zeros(st.ksplit * (-(-f // 32) * 32) * kk, dtype=torch.float32,
                                                 device=dev)
                        if st.bf16:  # pixel-contiguous (K-major) weight-gradient operands
                            st.colst = None if st.im_wg else torch.zeros(kk * st.pix_ld, dtype=wdt, device=dev)
                            st.dyk = torch.zeros(f * st.pix_ld, dtype=wdt, device=dev)
                        # input gradient: stride 1 -> a forward conv of dy (im2col of dy, flipped
                        # weights; scratch [cap*H*W, F*k*k]); stride 2 -> dcols GEMM + col2im
                        st.dg_fwd = st.attrs.get("stride", 1) == 1 and (f * k * k) % 8 == 0
                        st.fld = -(-f // 8) * 8 if st.bf16 else _align4(f)  # dyt rows: 16 bytes
                        # implicit-GEMM input gradient: a forward conv of the NHWC dy (dyt) with the
                        # flipped weights, no im2col of dy
                        st.im_dg = (self.implicit_conv and st.bf16 and st.needs_dx and st.dg_fwd and f % 64 == 0
                                    and k * k * f <= RSC_STAGE_MAX and _implicit_tiles(h, w))
                        # stride-2 3x3 input gradient as four stride-1 implicit convs of the NHWC dy
                        # (one per output parity class), no dcols / col2im
                        st.par_dg = (self.implicit_conv and st.bf16 and st.needs_dx and not st.dg_fwd and k == 3
                                     and stride == 2 and st.attrs.get("padding", 0) == 1 and (h, w) == (2 * oh, 2 * ow)
                                     and f % 64 == 0 and _implicit_tiles(oh, ow))
                        st.wpar = torch.zeros(9 * c * f, dtype=wdt, device=dev) if st.par_dg else None
                        if not st.bf16 or (st.needs_dx and not st.dg_fwd) or st.im_dg:
                            st.dyt = torch.zeros(pix * st.fld, dtype=wdt, device=dev)
                        if st.needs_dx and st.dg_fwd:
                            st.wflip = torch.zeros(c * f * k * k, dtype=wdt, device=dev)
                            if st.bf16 and not st.im_dg:
                                dgb_need = max(dgb_need, cap * h * w * f * k * k)
                            else:
                                dcols_need = max(dcols_need, cap * h * w * f * k * k)
                        elif st.needs_dx and not st.par_dg:
                            dcols_need = max(dcols_need, pix * kk)
                            if st.bf16:
                                st.wt = torch.zeros(kk * f, dtype=wdt, device=dev)
                    else:
                        st.splits = (-(-cap // N.CONV_DIRECT_BCHUNK) if st.direct
                                     else -(-cap * oh * ow // CONV_SPLIT_LEN))
                        st.partial = torch.zeros(st.splits * f * (c * k * k + 1), dtype=torch.float32, device=dev)
                widest = max(widest, st.ld_out, st.ld_in)
                prev_out, prev_ld = st.y, st.ld_out
            s.grads_buf = [torch.zeros(cap * widest, dtype=torch.float32, device=dev) for _ in range(2)]
            # one DGRAD column scratch per model: a tensor-core conv's dcols lives only between its
            # DGRAD GEMM and col2im, inside one backward wave
            s.dcols = torch.zeros(max(dcols_need, 4), dtype=torch.float32, device=dev) if dcols_need else None
            s.dgcols = torch.zeros(dgb_need, dtype=torch.bfloat16, device=dev) if dgb_need else None
            for k, st in enumerate(s.stages):
                st.dy = s.grads_buf[k % 2][: cap * st.ld_out].view(cap, st.ld_out)
                st.dx = s.grads_buf[(k + 1) % 2][: cap * st.ld_in].view(cap, st.ld_in)

    @staticmethod
    def _conv_out(st):
        c, h, w = st.in_shape
        k, s_, p = st.attrs["kernel"], st.attrs.get("stride", 1), st.attrs.get("padding", 0)
        return st.attrs["filters"], conv_extent(h, k, s_, p), conv_extent(w, k, s_, p)

    def reset_status(self, which=None):
        st = np.zeros(self.n, dtype=STATUS_DTYPE)
        st["alive"] = 1
        st["abort_epoch"] = -1
        st["abort_batch"] = -1
        torch = _torch()
        target = self.status if which is None else which
        target.copy_(torch.from_numpy(st.view(np.uint8)).to(self.device))

    def read_status(self, which=None) -> np.ndarray:
        src = self.status if which is None else which
        return src.cpu().numpy().view(STATUS_DTYPE).copy()

    def reset_accumulators(self, models: list):
        """Zero loss_sum / correct_sum / seen of the given models (alive flags untouched)."""
        if not models:
            return
        st = self.read_status()
        for m in models:
            st["loss_sum"][m] = 0.0
            st["correct_sum"][m] = 0
            st["seen"][m] = 0
        self.status.copy_(_torch().from_numpy(st.view(np.uint8)).to(self.device))

    # ------------------------------------------------------------------ params
    def upload_params(self, m: int, params: dict):
        s = self.slots[m]
        host = np.zeros(s.seg_len, dtype=np.float32)
        for pid, shp in s.specs.items():
            a = np.ascontiguousarray(params[pid], dtype=np.float32)
            if a.shape != tuple(shp):
                raise ShapeMismatchError(pid, f"shape {a.shape} != {tuple(shp)}")
            o = s.offsets[pid] - s.seg_off
            host[o:o + a.size] = a.reshape(-1)
        self.params[s.seg_off:s.seg_off + s.seg_len].copy_(_torch().from_numpy(host))

    def _download(self, arena, m: int) -> dict:
        s = self.slots[m]
        host = arena[s.seg_off:s.seg_off + s.seg_len].cpu().numpy()
        out = {}
        for pid, shp in s.specs.items():
            o = s.offsets[pid] - s.seg_off
            out[pid] = host[o:o + int(np.prod(shp))].reshape(shp).copy()
        return out

    def download_params(self, m: int) -> dict:
        return self._download(self.params, m)

    def download_grads(self, m: int) -> dict:
        return self._download(self.grads, m)

    def download_moments(self, m: int) -> tuple:
        s = self.slots[m]
        m1 = self._download(self.m1, m) if s.opt_kind != N.OPT_SGD else {}
        m2 = self._download(self.m2, m) if s.opt_kind == N.OPT_ADAM else {}
        return m1, m2

    def upload_moments(self, m: int, m1: dict, m2: dict):
        s = self.slots[m]
        for arena, src in ((self.m1, m1), (self.m2, m2)):
            if arena is None or not src:
                continue
            host = np.zeros(s.seg_len, dtype=np.float32)
            for pid, a in src.items():
                o = s.offsets[pid] - s.seg_off
                host[o:o + a.size] = np.asarray(a, dtype=np.float32).reshape(-1)
            arena[s.seg_off:s.seg_off + s.seg_len].copy_(_torch().from_numpy(host))

    def pview(self, arena, m: int, pid: str):
        s = self.slots[m]
        o = s.offsets[pid]
        return arena[o:o + int(np.prod(s.specs[pid]))]

    # ------------------------------------------------------------------ datasets
    def bind_datasets(self, by_model: list, perm_capacity: int):
        """by_model[m] = DeviceDataset of model m.  Builds the gather tables."""
        torch = _torch()
        self.model_data = by_model
        self.perm = torch.zeros(self.n, max(perm_capacity, 1), dtype=torch.int32, device=self.device)
        for s, d in zip(self.slots, by_model):
            if tuple(d.sample_shape) != tuple(s.sample_shape):
                raise ShapeMismatchError("input", f"job {s.job_id!r}: dataset samples {d.sample_shape} "
                                                  f"!= graph input {s.sample_shape}")
            if d.max_label >= s.classes:
                raise ValueError(f"target class out of range [0, {s.classes})")
            if s.stages[0].kind == "embed":
                # token ids checked once here (the reference checks each batch in _embed_fwd,
                # src/ops.py:268-270, via check_class_indices): integral and inside the vocabulary
                vocab = s.stages[0].attrs["vocab"]
                for x in (d.train_x, d.test_x):
                    if x.numel() and bool((x != torch.trunc(x)).any()):
                        raise ValueError("targets must hold integral class indices")
                    if x.numel() and bool(((x < 0) | (x >= vocab)).any()):
                        raise ValueError(f"target class out of range [0, {vocab})")
        self._gather_train = self._gather_launch(train=True)
        self._gather_eval = self._gather_launch(train=False)

    def _gather_launch(self, train: bool):
        rows = []
        for s, d in zip(self.slots, self.model_data):
            rows.append(N.GatherProblem(
                _ptr(d.train_x if train else d.test_x), _ptr(d.train_y if train else d.test_y),
                _ptr(self.perm[s.index]) if train else _ptr(d.identity),
                _ptr(s.batch_x), _ptr(s.batch_y), int(np.prod(s.sample_shape)), s.batch_x.shape[1],
                s.batch_size, s.index))
        t = _dev_table(N.GatherProblem, rows, self.device)
        cap = max(s.batch_size for s in self.slots)
        nbytes = sum(r.cap * (8 * r.sample + 8) for r in rows)
        return Launch("hnn_gather_rows", (_ptr(t), len(rows), cap, _ptr(self.cur)), t, "gather", nbytes=nbytes)

    # ------------------------------------------------------------------ plans
    def _stage_waves(self):
        depth = max(len(s.stages) for s in self.slots)
        return [[(s, s.stages[w]) for s in self.slots if w < len(s.stages)] for w in range(depth)]

    def _route_tc(self, op, d) -> bool:
        """Dense problems big and aligned enough for the tcgen05 tiles go to the 3xTF32 kernels.
        The CTA-pair kernel takes short batches too (64 rows: a quarter of its 256-row tile still
        beats the FFMA path 3x on C5's first layer); the single-CTA kernel needs 128 rows."""
        # (the 10-class logits forward on the pair kernel at tile width 64 measured slower than the
        # streaming skinny kernel: C3 39 -> 67 us, profiles/r02/narrow_fwd_ab_v7.txt)
        if d["m"] < (32 if self.use_pairs else 128) or d["n"] < 64 or d["k"] < 64:
            return False
        if op == N.HNN_WGRAD and d["m"] > 4096:
            return False
        if any(d[k] % 4 for k in ("lda", "ldb", "ldc")):
            return False
        return all(d[k] % 16 == 0 for k in ("a", "b", "c"))

    @staticmethod
    def _route_skinny(op, d) -> bool:
        """One GEMM dimension <= 16 (the logits layer): the streaming kernels of gemm_skinny.cu.
        DGRAD / WGRAD use float4 column quads, so they also need 16-byte rows."""
        if op == N.HNN_FWD:
            return d["n"] <= 16
        small = d["k"] if op == N.HNN_DGRAD else d["m"]
        if small > 16 or d["n"] % 4:
            return False
        if any(d[k] % 4 for k in ("ldb", "ldc")) or (op == N.HNN_DGRAD and d["mask"] and d["ldc"] % 4):
            return False
        ptrs = ("b", "c", "mask") if op == N.HNN_DGRAD else ("b", "c", "opt_w", "opt_wm", "opt_wv")
        return all(d.get(k, 0) % 16 == 0 for k in ptrs)

    def _pair_schedule(self, probs, rows, total_tiles, tm, narrow=False) -> bytes:
        """Longest-processing-time assignment of a CTA-pair launch's tiles to its pairs (the
        table trailer read by gemm_tc2.cu): int32 npairs, offsets[npairs + 1], tile ids.
        Cost of a tile = its 32-wide K blocks + a fixed epilogue share.  Which pair computes a
        tile never changes the tile's arithmetic (bit-exact isolation).  narrow: the kernel gives a
        ragged n's last column tile the narrowest width covering the rest (fp32 input / weight
        gradients, gemm_tc2.cu tile_info), so its cost uses that width."""
        torch = _torch()
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        npairs = max(1, min(total_tiles, sms // 2))
        costs = []
        for pr, (s, d) in zip(probs, rows):
            split = d.get("ksplit", 1) if d.get("ksplit_len") else 1
            kb = -(-(d["ksplit_len"] if split > 1 else d["k"]) // 32)
            tiles = pr.tiles_n * -(-d["m"] // tm) * split
            for i in range(tiles):
                tn = pr.tile_n  # MMA and operand time scale with the tile's columns
                if narrow:
                    rem = d["n"] - ((i // split) % pr.tiles_n) * pr.tile_n
                    if rem < tn:
                        tn = 64 if rem <= 64 else (128 if rem <= 128 else tn)
                costs.append((kb * (0.5 + 0.5 * tn / 256) + 3, pr.tile_base + i))
        costs.sort(key=lambda c: (-c[0], c[1]))
        import heapq

        heap = [(0, p) for p in range(npairs)]
        lists = [[] for _ in range(npairs)]
        for cost, tile in costs:
            load, p = heapq.heappop(heap)
            lists[p].append(tile)
            heapq.heappush(heap, (load + cost, p))
        offs = np.zeros(npairs + 1, dtype=np.int32)
        offs[1:] = np.cumsum([len(l) for l in lists])
        ids = np.array([t for l in lists for t in l], dtype=np.int32)
        return np.concatenate([np.array([npairs], np.int32), offs, ids]).tobytes()

    def _gemm_launch(self, op, items, label):
        """items: list of (slot, stage).  Splits into SIMT / 3xTF32 launches."""
        groups = {N.PREC_SIMT: [], N.PREC_SIMT_SKINNY: [], N.PREC_3XTF32: [], N.PREC_3XTF32_PAIR: []}
        for s, st in items:
            d = self._gemm_problem(op, s, st)
            groups[self._gemm_prec(op, d)].append((s, d))
        out = []
        for prec, rows in groups.items():
            if rows:
                out += self._emit_gemm(op, prec, rows, label)
        return out

    def _gemm_prec(self, op, d) -> int:
        if self.use_tc and self._route_tc(op, d):
            # CTA-pair 256x256 tiles (one launch per wave, LPT-scheduled); HNN_TC_PAIR=0
            # selects the single-CTA 128x128 kernel
            return N.PREC_3XTF32_PAIR if self.use_pairs else N.PREC_3XTF32
        if self._route_skinny(op, d):
            return N.PREC_SIMT_SKINNY
        return N.PREC_SIMT

    def _skinny_backward(self, items):
        """Dense layers of a backward wave whose input gradient and weight gradient both take the
        skinny kernels (the <= 10-class logits layer), without a fused optimizer: one fused launch
        (hnn_skinny_backward) reads their input once for both.  Returns (launches, fused items)."""
        if os.environ.get("HNN_SKINNY_FUSED", "1") == "0":
            return [], []
        pairs = []
        for s, st in items:
            if st.kind != "dense" or not st.needs_dx:
                continue
            dg, wg = self._gemm_problem(N.HNN_DGRAD, s, st), self._gemm_problem(N.HNN_WGRAD, s, st)
            if (self._gemm_prec(N.HNN_DGRAD, dg) == N.PREC_SIMT_SKINNY and self._gemm_prec(N.HNN_WGRAD, wg)
                    == N.PREC_SIMT_SKINNY and not wg.get("opt_w") and wg["m"] <= 10 and dg["k"] == wg["m"]):
                pairs.append((s, st, dg, wg))
        if not pairs:
            return [], []
        tn = 4 * 32  # columns per CTA (gemm_skinny.cu WG_QUADS float4 quads)
        wp, dp, base = [], [], 0
        for s, st, dg, wg in sorted(pairs, key=lambda t: -t[3]["n"]):
            tiles = -(-wg["n"] // tn)
            wp.append(N.GemmProblem(tile_base=base, tiles_n=tiles, model=s.index, **wg))
            dp.append(N.GemmProblem(tile_base=base, tiles_n=tiles, model=s.index, **dg))
            base += tiles
        t = _dev_table(N.GemmProblem, wp + dp, self.device)
        import ctypes

        size = ctypes.sizeof(N.GemmProblem)
        nbytes = sum(4 * (2 * d["m"] * d["n"] + w["k"] * w["m"] * 2 + w["m"] * w["n"]) for _, _, d, w in pairs)
        flops = sum(4 * w["m"] * w["n"] * w["k"] for _, _, _, w in pairs)
        label = "dense/skinny_bwd"
        launch = Launch("hnn_skinny_backward", (_ptr(t), _ptr(t) + size * len(wp), len(wp), base, _ptr(self.cur),
                                                _ptr(self.status)), t, label, flops=flops, nbytes=nbytes)
        return [launch], [(s, st) for s, st, _, _ in pairs]

    def _gemm_problem(self, op, s, st) -> dict:
        """The grouped-GEMM problem dict of dense stage st of slot s for op."""
        if True:
            cap = s.batch_size
            K, U = int(np.prod(st.in_shape)), st.out_shape[0]
            w = self.pview(self.params, s.index, st.params[0])
            b = self.pview(self.params, s.index, st.params[1])
            if op == N.HNN_FWD:
                d = dict(a=_ptr(st.x), b=_ptr(w), c=_ptr(st.y), bias=_ptr(b), mask=0, dbias=0, m=cap, n=U, k=K,
                         lda=st.ld_in, ldb=K, ldc=st.ld_out, relu=int(st.relu))
            elif op == N.HNN_DGRAD:
                d = dict(a=_ptr(st.dy), b=_ptr(w), c=_ptr(st.dx), bias=0, mask=_ptr(st.x) if st.mask_input else 0,
                         dbias=0, m=cap, n=K, k=U, lda=st.ld_out, ldb=K, ldc=st.ld_in, relu=0)
            else:
                gw = self.pview(self.grads, s.index, st.params[0])
                gb = self.pview(self.grads, s.index, st.params[1])
                fuse = self._fused(s)
                keep = self.keep_grads or not fuse
                d = dict(a=_ptr(st.dy), b=_ptr(st.x), c=_ptr(gw) if keep else 0, bias=0, mask=0,
                         dbias=_ptr(gb) if keep else 0, m=U, n=K, k=cap, lda=st.ld_out, ldb=st.ld_in, ldc=K, relu=0)
                if fuse:
                    kind = s.opt_kind
                    arena = lambda a, pid: _ptr(self.pview(a, s.index, pid)) if a is not None else 0
                    d.update(opt_w=arena(self.params, st.params[0]), opt_b=arena(self.params, st.params[1]),
                             opt_wm=arena(self.m1, st.params[0]) if kind != N.OPT_SGD else 0,
                             opt_bm=arena(self.m1, st.params[1]) if kind != N.OPT_SGD else 0,
                             opt_wv=arena(self.m2, st.params[0]) if kind == N.OPT_ADAM else 0,
                             opt_bv=arena(self.m2, st.params[1]) if kind == N.OPT_ADAM else 0,
                             opt_kind=kind, opt_momentum=float(np.float32(s.momentum)))
            return d

    def _pair_tile_cap(self, op, rows, tm) -> int:
        """Widest pair-tile width (256 / 128 / 64) for one launch: narrower tiles put more CTA pairs
        to work when a launch has fewer tiles than pairs (C5's 32 batch-64 forward GEMMs: 32
        tiles at 256 columns, 64 at 128).  Cost model per tile: K blocks * (0.5 + 0.5 * width / 256)
        + 3 (the A operand streams whatever the width; the _pair_schedule model); makespan =
        max(total / pairs, largest tile).  The width never changes a tile's per-element arithmetic."""
        pairs = self._sm_count() // 2
        best, best_cost = 256, None
        for cap in (256, 128, 64):
            total, largest = 0.0, 0.0
            for _, d in rows:
                w = min(cap, 64 if d["n"] <= 64 else (128 if d["n"] <= 128 else 256))
                # a tile's time scales with its K blocks (the long-K tiles of a sparse launch set its
                # makespan: C3 on 8 GPUs, 4 models per launch, K up to 2048)
                split = d.get("ksplit", 1) if op == N.HNN_WGRAD else 1
                kb = -(-(d["ksplit_len"] if split > 1 else d["k"]) // 32)
                cost = kb * (0.5 + 0.5 * w / 256) + 3
                n_tiles = -(-d["m"] // tm) * -(-d["n"] // w) * split
                total += n_tiles * cost
                largest = max(largest, cost)
            c = max(total / pairs, largest)
            if best_cost is None or c < best_cost * 0.95:
                best, best_cost = cap, c
        return best

    def _sm_count(self) -> int:
        torch = _torch()
        if getattr(self, "_sms", None) is None:
            dev = torch.device(self.device) if self.device is not None else None
            self._sms = (torch.cuda.get_device_properties(dev).multi_processor_count
                         if dev is not None and dev.type == "cuda" else 148)
        return self._sms

    def _emit_gemm(self, op, prec, rows, label):
        """One grouped-GEMM launch over rows = [(slot, problem dict)] (dense layers or lowered convs)."""
        out = []
        if True:
            tm, tn = N.tile_shape(op, prec)
            # heaviest problems first: their tiles start in the first wave (LPT over SMs)
            rows = sorted(rows, key=lambda r: -(r[1]["m"] * r[1]["n"] * r[1]["k"]))
            probs, base = [], 0
            cap = self._pair_tile_cap(op, rows, tm) if prec in (N.PREC_3XTF32_PAIR, N.PREC_BF16_PAIR) else tn
            finals = []
            if prec == N.PREC_3XTF32_PAIR and op == N.HNN_FWD:
                rows, finals = self._split_k_forward(rows, tm, cap)
            for s, d in rows:
                tn_p = tn
                if prec in (N.PREC_3XTF32_PAIR, N.PREC_BF16_PAIR):  # narrowest pair tile covering n
                    tn_p = min(cap, 64 if d["n"] <= 64 else (128 if d["n"] <= 128 else 256))
                    if d.get("im_c") and op == N.HNN_WGRAD:
                        tn_p = 128  # implicit weight gradient: one tap's 64 channels per CTA
                    d = dict(d, tile_n=tn_p)
                tiles_m, tiles_n = -(-d["m"] // tm), -(-d["n"] // tn_p)
                probs.append(N.GemmProblem(tile_base=base, tiles_n=tiles_n, model=s.index, **d))
                base += tiles_m * tiles_n * (d.get("ksplit", 1) if op in (N.HNN_WGRAD, N.HNN_FWD) else 1)
            keep = None
            if prec in (N.PREC_3XTF32, N.PREC_3XTF32_PAIR, N.PREC_BF16_PAIR):
                torch = _torch()
                maps = bytearray(128 * 4 * len(probs))
                host = (N.GemmProblem * len(probs))(*probs)
                enc = "hnn_gemm_bf16_encode" if prec == N.PREC_BF16_PAIR else "hnn_gemm_tc_encode"
                N.call(enc, op, C_addr(host), len(probs), C_addr_bytes(maps))
                keep = torch.frombuffer(maps, dtype=torch.uint8).to(self.device)
                for i, pr in enumerate(probs):
                    pr.tmap_a = _ptr(keep) + 512 * i
                    pr.tmap_b = _ptr(keep) + 512 * i + 128
                    pr.tmap_c = _ptr(keep) + 512 * i + 256
                    pr.tmap_xh = _ptr(keep) + 512 * i + 384
            extra = b""
            if prec in (N.PREC_3XTF32_PAIR, N.PREC_BF16_PAIR):
                extra = self._pair_schedule(probs, rows, base, tm,
                                            narrow=prec == N.PREC_3XTF32_PAIR and op != N.HNN_FWD)
            t = _dev_table(N.GemmProblem, probs, self.device, extra)
            flops = sum(2 * d["m"] * d["n"] * d["k"] for _, d in rows)
            # bytes: A + B read once, C written once (fp32); a fused optimizer adds its p/m/v traffic
            nbytes = sum(4 * (d["m"] * d["k"] + d["k"] * d["n"] + (d["m"] * d["n"] if d.get("c") else 0))
                         for _, d in rows)
            per_param = {N.OPT_SGD: 8, N.OPT_SGD_MOMENTUM: 16, N.OPT_ADAM: 24}
            nbytes += sum(per_param[d["opt_kind"]] * d["m"] * (d["n"] + 1) for _, d in rows if d.get("opt_w"))
            launch = Launch("hnn_grouped_gemm", (op, prec, _ptr(t), len(probs), base, _ptr(self.cur),
                                                 _ptr(self.status)), t,
                            f"{label}/{ {N.PREC_SIMT: 'simt', N.PREC_SIMT_SKINNY: 'simt16', N.PREC_3XTF32: 'tc', N.PREC_3XTF32_PAIR: 'tc2', N.PREC_BF16_PAIR: 'bf16'}[prec] }",
                            flops=flops, nbytes=nbytes)
            launch.maps = keep
            out.append(launch)
            if finals:  # the split-K forward's partial sums -> bias / relu output
                eprobs, ebase = [], 0
                for d in finals:
                    nb = max(1, min(-(-(d["m"] * d["n"]) // 256), 2 * self._sm_count()))
                    eprobs.append(N.GemmProblem(a=d["partial"], c=d["c"], bias=d["bias"], relu=d["relu"], m=d["m"],
                                                n=d["n"], k=d["k"], lda=d["n"], ldc=d["ldc"], ksplit=d["ksplit"],
                                                model=d["model"], tile_base=ebase, tiles_n=nb))
                    ebase += nb
                et = _dev_table(N.GemmProblem, eprobs, self.device)
                el = Launch("hnn_splitk_epilogue", (_ptr(et), len(eprobs), ebase, _ptr(self.cur), _ptr(self.status)),
                            et, f"{label}/splitk")
                el.keep = [d["keep"] for d in finals]
                out.append(el)
        return out

    def _split_k_forward(self, rows, tm, cap):
        """A CTA-pair forward launch with fewer tiles than a third of the pairs and long-K dense
        problems (C1's two 64 x 784 x 256 first layers: 2 tiles for 74 pairs) splits every such
        problem's K into 128-term ranges — exactly the tensor-core accumulation chunks of the
        unsplit kernel — whose raw sums a second launch adds in order before the bias / relu
        (hnn_splitk_epilogue).  That is the unsplit kernel's own promotion order, so the result is
        bit-identical to not splitting (model isolation does not depend on the launch's
        composition); the launch just spreads over K/128 times more CTA pairs.
        Returns the rewritten rows and the epilogue descriptions."""
        torch = _torch()
        pairs = self._sm_count() // 2
        tiles = 0
        for _, d in rows:
            w = min(cap, 64 if d["n"] <= 64 else (128 if d["n"] <= 128 else 256))
            tiles += -(-d["m"] // tm) * -(-d["n"] // w)
        if os.environ.get("HNN_SPLITK_FWD", "1") == "0" or tiles * 3 > pairs:
            return rows, []
        out, finals = [], []
        for s, d in rows:
            dense = d.get("c_mode", 0) == 0 and d.get("row_mult", 1) == 1 and not d.get("im_c")
            if not (dense and d["k"] >= 2 * N.chunk_terms(N.PREC_3XTF32_PAIR)):  # (at least two chunks)
                out.append((s, d))
                continue
            length = N.chunk_terms(N.PREC_3XTF32_PAIR)  # one promotion chunk (gemm_tc2.cu)
            split = -(-d["k"] // length)
            mp = -(-d["m"] // 32) * 32
            part = torch.empty(split * mp * d["n"], dtype=torch.float32, device=self.device)
            finals.append(dict(partial=_ptr(part), c=d["c"], bias=d["bias"], relu=d["relu"], m=d["m"], n=d["n"],
                               k=d["k"], ldc=d["ldc"], ksplit=split, model=s.index, keep=part))
            out.append((s, dict(d, c=_ptr(part), ldc=d["n"], bias=0, relu=0, ksplit=split, ksplit_len=length)))
        return out, finals

    def _conv_launch(self, op, items, label):
        out = []
        tc = [(s, st) for s, st in items if getattr(st, "tc", False)]
        if tc:
            out += self._conv_tc_launches(op, tc, label)
        for direct in (False, True):
            group = [(s, st) for s, st in items if getattr(st, "direct", False) == direct
                     and not getattr(st, "tc", False)]
            if group:
                out += self._conv_group(op, group, label + ("/direct" if direct else ""), direct)
        return out

    def _same_conv(self, st) -> bool:
        c, h, w = st.in_shape
        _, oh, ow = self._conv_out(st)
        return st.attrs.get("stride", 1) == 1 and (oh, ow) == (h, w)

    def _convtc_aux(self, aux, items, label, blocks_of, nbytes=None):
        probs, base = [], 0
        for s, st in items:
            c, h, w = st.in_shape
            f, oh, ow = self._conv_out(st)
            k = st.attrs["kernel"]
            W = self.pview(self.grads, s.index, st.params[0])
            B = self.pview(self.grads, s.index, st.params[1])
            nb = blocks_of(s, st)
            dyt = st.dyt
            if aux == N.CONVTC_IM2COL:  # (im2col's dyt = the NHWC copy of x, "same" implicit layers)
                dyt = st.xh if (st.im_fwd and self._same_conv(st) and not st.xh_from_prev) else None
            probs.append(N.ConvTcProblem(
                x=_ptr(st.x), cols=_ptr(st.cols), dy=_ptr(st.dy), dyt=_ptr(dyt),
                dcols=_ptr(s.dcols) if s.dcols is not None else 0, dx=_ptr(st.dx),
                mask=_ptr(st.x) if st.mask_input else 0, partial=_ptr(st.partial), dw=_ptr(W), db=_ptr(B),
                bpart=_ptr(st.bpart), weight=_ptr(self.pview(self.params, s.index, st.params[0])),
                wpad=_ptr(st.wt if aux == N.CONVTC_WT_WEIGHTS else st.wpad), colst=_ptr(st.colst), rsc=int(st.im_wg),
                dyk=_ptr(st.dyk), bf16=int(st.bf16), pix_ld=st.pix_ld, cap=s.batch_size, c=c, h=h, w=w, f=f, k=k,
                stride=st.attrs.get("stride", 1), pad=st.attrs.get("padding", 0), oh=oh, ow=ow, kk=c * k * k,
                kkp=st.kkp,
                ksplit=st.ksplit, ksplit_len=st.ksplit_len, model=s.index, block_base=base, blocks=nb))
            base += nb
        if nbytes is None:  # algorithmic bytes (read + write) for the roofline
            nbytes = 0
            for pr in probs:
                esz = 2 if pr.bf16 else 4
                pix_out, pix_in = pr.cap * pr.oh * pr.ow, pr.cap * pr.h * pr.w
                if aux == N.CONVTC_IM2COL:
                    if pr.bf16 and not pr.cols and not pr.colst:  # only the NHWC copy
                        nbytes += (4 + 2) * pr.c * pix_in
                    else:
                        nbytes += (4 * pr.c * pix_in + esz * pix_out * pr.kkp * ((1 if pr.cols else 0) + (1 if pr.colst else 0))
                                   + (2 * pr.c * pix_in if pr.dyt else 0))
                elif aux == N.CONVTC_TRANSPOSE_DY:
                    nbytes += 4 * pr.f * pix_out + esz * pr.f * pix_out * ((1 if pr.dyt else 0) + (1 if pr.dyk else 0))
                elif aux == N.CONVTC_COL2IM:
                    nbytes += 4 * pix_out * pr.kkp + 4 * pr.c * pix_in * (3 if pr.mask else 2)
                elif aux == N.CONVTC_WGRAD_REDUCE:
                    nbytes += 4 * pr.f * pr.kkp * (pr.ksplit + 1) + 4 * pr.f * (pr.cap + 1)
                else:
                    nbytes += (4 + esz) * pr.f * pr.kkp
        t = _dev_table(N.ConvTcProblem, probs, self.device)
        max_k = max(st.attrs["kernel"] for _, st in items)
        return Launch("hnn_conv_tc_aux", (aux, _ptr(t), len(probs), base, max_k, _ptr(self.cur), _ptr(self.status)),
                      t, label, nbytes=nbytes)

    def _conv_dgrad_as_fwd(self, items, label, grid):
        """Stride-1 conv input gradient = conv(dy, flipped weights, pad k-1-p): flip the weights,
        im2col dy into the model's scratch, one forward-type CTA-pair GEMM writing NCHW dx with the
        relu mask of x (no dcols round trip through col2im)."""
        out, cols = [], []
        imp = [(s, st) for s, st in items if st.im_dg]
        if imp:  # NHWC dy (+ the weight-gradient copies and bias partials of the same transpose)
            out.append(self._convtc_aux(N.CONVTC_TRANSPOSE_DY, imp, f"{label}/tc/transpose",
                                        lambda s, st: N.transpose_blocks(s.batch_size,
                                                                         self._conv_out(st)[1] * self._conv_out(st)[2],
                                                                         self._conv_out(st)[0])))
        for s, st in items:
            if st.im_dg:
                continue
            c, h, w = st.in_shape
            f, oh, ow = self._conv_out(st)
            k = st.attrs["kernel"]
            p = st.attrs.get("padding", 0)
            kf = f * k * k
            # im2col over dy: channels F, spatial OH x OW -> H x W, padding k-1-p
            dst = s.dgcols if st.bf16 else s.dcols
            cols.append((s, N.ConvTcProblem(x=_ptr(st.dy), cols=_ptr(dst), cap=s.batch_size, c=f, h=oh, w=ow,
                                            f=c, k=k, stride=1, pad=k - 1 - p, oh=h, ow=w, kk=kf, kkp=kf,
                                            model=s.index, bf16=int(st.bf16))))
        max_k = max(st.attrs["kernel"] for _, st in items)
        # (the flipped weights come from the step's prep launch: conv_weight_prep)
        if cols:
            out.append(self._aux_table(N.CONVTC_IM2COL, cols, f"{label}/tc/im2col_dy",
                                       lambda pr: -(-(pr.cap * pr.oh * pr.ow) // 32) * -(-pr.c // 32), max_k))
        by_prec, fins = {}, []
        for s, st in items:
            c, h, w = st.in_shape
            f, oh, ow = self._conv_out(st)
            k = st.attrs["kernel"]
            kf = f * k * k
            src = s.dgcols if st.bf16 else s.dcols
            d = dict(a=_ptr(src), b=_ptr(st.wflip), c=_ptr(st.dx), bias=0,
                     mask=_ptr(st.x) if st.mask_input else 0, dbias=0, m=s.batch_size * h * w, n=c,
                     k=kf, lda=kf, ldb=kf, ldc=c, relu=0, row_mult=h * w, c_mode=1)
            if st.im_dg:  # conv of the NHWC dy, pad k-1-p, onto the h x w input grid
                d.update(a=_ptr(st.dyt), lda=st.fld, im_c=f, im_k=k, im_pad=k - 1 - st.attrs.get("padding", 0),
                         im_h=oh, im_w=ow, im_oh=h, im_ow=w, im_n=s.batch_size)
            d, fin = self._fwd_split(s, st, d)
            if fin is not None:
                fins.append(fin)
            by_prec.setdefault(N.PREC_BF16_PAIR if st.bf16 else N.PREC_3XTF32_PAIR, []).append((s, d))
        for prec, rows in by_prec.items():
            out += self._emit_gemm(N.HNN_FWD, prec, rows, f"{label}/tc/dgfwd")
        if fins:
            out.append(self._splitk_finish(fins, f"{label}/tc/dgfwd/splitk"))
        return out

    def _aux_table(self, aux, probs_by_slot, label, blocks_of, max_k):
        probs, base = [], 0
        for s, pr in probs_by_slot:
            nb = blocks_of(pr)
            pr.block_base, pr.blocks = base, nb
            probs.append(pr)
            base += nb
        t = _dev_table(N.ConvTcProblem, probs, self.device)
        return Launch("hnn_conv_tc_aux", (aux, _ptr(t), len(probs), base, max_k, _ptr(self.cur), _ptr(self.status)),
                      t, label)

    def _fwd_split(self, s, st, d):
        """K split of a bf16 forward-type conv GEMM whose output tiles fill few CTA pairs (ResNet /
        VGG layers at 8x8 and below: 4-32 tiles of 256 x n for 74 pairs, K up to 4608).  A fixed
        function of the problem's own shape and the device's SM count (never of the launch's other
        problems), so model isolation stays bit-exact: S = min(pairs // tiles, K blocks // 8) ranges
        of whole 64-element K blocks, raw partial sums stacked [S, m rounded to 32, n] and finished
        in order by HNN_CONVTC_SPLITK_FWD (+ bias, relu, NCHW, NHWC copy, relu mask).  Returns
        (problem dict, finish description or None)."""
        if not st.bf16 or os.environ.get("HNN_CONV_SPLITK", "0") == "0":  # measured slower on every C4 layer (off)
            return d, None
        M, F, K = d["m"], d["n"], d["k"]
        tn = 64 if F <= 64 else (128 if F <= 128 else 256)
        tiles = -(-M // 256) * -(-F // tn)
        nkb = -(-K // 64)
        S = min(self._sm_count() // 2 // tiles, nkb // 8)
        if S < 2:
            return d, None
        L = -(-nkb // S) * 64
        S = -(-K // L)
        mp = -(-M // 32) * 32
        part = _torch().empty(S * mp * F, dtype=_torch().float32, device=self.device)
        fin = dict(partial=part, ksplit=S, pix_ld=mp, f=F, cap=s.batch_size, hw=d["row_mult"], dx=d["c"],
                   mask=d.get("mask", 0), db=d.get("bias", 0), relu=d.get("relu", 0), dyt=d.get("xh_out", 0),
                   model=s.index)
        d2 = dict(d, c=_ptr(part), ldc=F, c_mode=0, bias=0, relu=0, mask=0, xh_out=0, ksplit=S, ksplit_len=L)
        return d2, fin

    def _splitk_finish(self, fins, label):
        """One HNN_CONVTC_SPLITK_FWD launch for the split problems of a forward-type GEMM launch."""
        probs, base = [], 0
        for f in fins:
            M = f["cap"] * f["hw"]
            nb = -(-M // 32) * -(-f["f"] // 32)
            # (the finish kernel only needs the plane size: oh = hw, ow = 1)
            probs.append(N.ConvTcProblem(partial=_ptr(f["partial"]), dx=f["dx"], mask=f["mask"], db=f["db"],
                                         dyt=f["dyt"], cap=f["cap"], f=f["f"], oh=f["hw"], ow=1, ksplit=f["ksplit"],
                                         pix_ld=f["pix_ld"], rsc=int(f["relu"]), bf16=1, model=f["model"],
                                         block_base=base, blocks=nb))
            base += nb
        t = _dev_table(N.ConvTcProblem, probs, self.device)
        nbytes = sum(4 * f["cap"] * f["hw"] * f["f"] * (f["ksplit"] + 1 + (1 if f["mask"] else 0))
                     + (2 * f["cap"] * f["hw"] * f["f"] if f["dyt"] else 0) for f in fins)
        launch = Launch("hnn_conv_tc_aux", (N.CONVTC_SPLITK_FWD, _ptr(t), len(probs), base, 3, _ptr(self.cur),
                                            _ptr(self.status)), t, label, nbytes=nbytes)
        launch.keep = [f["partial"] for f in fins]
        return launch

    def _conv_tc_launches(self, op, items, label):
        """Tensor-core conv layers of one wave: im2col / transpose / col2im / split reduce around
        CTA-pair GEMMs (csrc/conv_tc.cu, csrc/gemm_tc2.cu): 3xTF32 on fp32 operands, or kind::f16 on
        bf16 operand copies (every operand K-major: pixel-contiguous copies for the weight gradient)."""
        def geo(st):  # GEMM K = C*k*k padded to kkp
            c, h, w = st.in_shape
            f, oh, ow = self._conv_out(st)
            return c, h, w, f, oh, ow, st.kkp

        def weight(s, st):  # GEMM B operand rows [f, kkp]: the weights, or their padded / bf16 copy
            return _ptr(st.wpad) if st.wpad is not None else _ptr(self.pview(self.params, s.index, st.params[0]))

        def grid(total):
            return max(1, min(-(-total // 256), 4 * 148))

        def prec(st):
            return N.PREC_BF16_PAIR if st.bf16 else N.PREC_3XTF32_PAIR

        def gemms(op_, rows_by_prec, lab):
            res = []
            for pr, rows in rows_by_prec.items():
                res += self._emit_gemm(op_, pr, rows, lab)
            return res

        out = []
        if op == N.HNN_FWD:
            # (the padded weight copies come from the step's prep launch: conv_weight_prep)
            # NHWC bf16 copies of the inputs for the implicit-GEMM layers: written by the im2col
            # launch for "same" layers (output pixel = input pixel), a transpose otherwise
            imp = [(s, st) for s, st in items if st.im_fwd and not self._same_conv(st) and not st.xh_from_prev]
            if imp:
                probs = []
                for s, st in imp:
                    c, h, w = st.in_shape
                    probs.append((s, N.ConvTcProblem(dy=_ptr(st.x), dyt=_ptr(st.xh), cap=s.batch_size, f=c, oh=h,
                                                     ow=w, model=s.index, bf16=1)))
                out.append(self._aux_table(N.CONVTC_TRANSPOSE_DY, probs, f"{label}/tc/nhwc",
                                           lambda pr: N.transpose_blocks(pr.cap, pr.oh * pr.ow, pr.f), 3))
            # (no im2col at all for a layer whose NHWC input came from the previous epilogue and
            # whose weight gradient is implicit too)
            cols_items = [(s, st) for s, st in items if not (st.xh_from_prev and st.im_wg)]
            if cols_items:
                out.append(self._convtc_aux(
                    N.CONVTC_IM2COL, cols_items, f"{label}/tc/im2col",
                    lambda s, st: (-(-(s.batch_size * geo(st)[4] * geo(st)[5]) // 256)
                                   if st.bf16 and geo(st)[0] * st.attrs["kernel"] ** 2 <= 32  # (first layers)
                                   else -(-(s.batch_size * geo(st)[4] * geo(st)[5]) // 32) * -(-geo(st)[0] // 32))))
            rows, fins = {}, []
            for s, st in items:
                c, h, w, f, oh, ow, kk = geo(st)
                B = self.pview(self.params, s.index, st.params[1])
                d = dict(a=_ptr(st.cols), b=weight(s, st), c=_ptr(st.y), bias=_ptr(B), mask=0, dbias=0,
                         m=s.batch_size * oh * ow, n=f, k=kk, lda=kk, ldb=kk, ldc=f, relu=int(st.relu),
                         row_mult=oh * ow, c_mode=1)
                if st.im_fwd:
                    d.update(a=_ptr(st.xh), lda=c, im_c=c, im_k=st.attrs["kernel"], im_pad=st.attrs.get("padding", 0),
                             im_h=h, im_w=w, im_oh=oh, im_ow=ow, im_n=s.batch_size)
                if st.xh_next is not None:
                    d.update(xh_out=_ptr(st.xh_next))
                d, fin = self._fwd_split(s, st, d)
                if fin is not None:
                    fins.append(fin)
                rows.setdefault(prec(st), []).append((s, d))
            out += gemms(N.HNN_FWD, rows, f"{label}/tc")
            if fins:
                out.append(self._splitk_finish(fins, f"{label}/tc/splitk"))
            return out
        tiles_t = lambda s, st: N.transpose_blocks(s.batch_size, geo(st)[4] * geo(st)[5], geo(st)[3])
        if op == N.HNN_DGRAD:
            # (only stages whose input gradient is needed reach here)
            fw = [(s, st) for s, st in items if st.dg_fwd]
            if fw:
                out += self._conv_dgrad_as_fwd(fw, label, grid)
            items = [(s, st) for s, st in items if not st.dg_fwd]
            if not items:
                return out
            out.append(self._convtc_aux(N.CONVTC_TRANSPOSE_DY, items, f"{label}/tc/transpose", tiles_t))
            par = [(s, st) for s, st in items if st.par_dg]
            if par:
                prow = []
                for s, st in par:
                    c, h, w, f, oh, ow, kk = geo(st)
                    for q, off in enumerate(_parity_offsets(c, f)):
                        kh, kw = 1 + (q >> 1), 1 + (q & 1)
                        prow.append((s, dict(a=_ptr(st.dyt), b=_ptr(st.wpar) + 2 * off, c=_ptr(st.dx), bias=0,
                                             mask=_ptr(st.x) if st.mask_input else 0, dbias=0,
                                             m=s.batch_size * oh * ow, n=c, k=kh * kw * f, lda=st.fld,
                                             ldb=kh * kw * f, ldc=c, relu=0, row_mult=oh * ow, c_mode=2 + q,
                                             im_c=f, im_k=kh, im_kw=kw, im_pad=0, im_h=oh, im_w=ow, im_oh=oh,
                                             im_ow=ow, im_n=s.batch_size)))
                out += self._emit_gemm(N.HNN_FWD, N.PREC_BF16_PAIR, prow, f"{label}/tc/dgpar")
            items = [(s, st) for s, st in items if not st.par_dg]
            if not items:
                return out
            rows = {}
            for s, st in items:
                c, h, w, f, oh, ow, kk = geo(st)
                if st.bf16:  # B = w^T [kkp, f] (K-major)
                    d = dict(a=_ptr(st.dyt), b=_ptr(st.wt), ldb=f)
                else:
                    d = dict(a=_ptr(st.dyt), b=weight(s, st), ldb=kk)
                rows.setdefault(prec(st), []).append(
                    (s, dict(d, c=_ptr(s.dcols), bias=0, mask=0, dbias=0, m=s.batch_size * oh * ow, n=kk, k=f,
                             lda=st.fld, ldc=kk, relu=0, row_mult=oh * ow)))
            out += gemms(N.HNN_DGRAD, rows, f"{label}/tc")
            out.append(self._convtc_aux(N.CONVTC_COL2IM, items, f"{label}/tc/col2im",
                                        lambda s, st: (s.batch_size * geo(st)[1] * -(-geo(st)[2] // 32)
                                                       * -(-geo(st)[0] // 16))))
            return out
        # WGRAD (the transpose already ran in this wave's DGRAD phase when the stage needs dx)
        fresh = [(s, st) for s, st in items if not (st.needs_dx and not st.dg_fwd) and not st.im_dg]
        if fresh:
            out.append(self._convtc_aux(N.CONVTC_TRANSPOSE_DY, fresh, f"{label}/tc/transpose", tiles_t))
        rows = {}
        for s, st in items:
            c, h, w, f, oh, ow, kk = geo(st)
            if st.im_wg:  # A = dy [f, pixels]; B read from the NHWC x, columns (r, s, c)
                d = dict(a=_ptr(st.dyk), b=_ptr(st.xh), lda=st.pix_ld, ldb=c, tile_n=128, im_c=c,
                         im_k=st.attrs["kernel"], im_pad=st.attrs.get("padding", 0), im_h=h, im_w=w, im_oh=oh,
                         im_ow=ow, im_n=s.batch_size)
            elif st.bf16:  # A = dy [f, pixels], B = cols^T [kkp, pixels]: both pixel-contiguous
                d = dict(a=_ptr(st.dyk), b=_ptr(st.colst), lda=st.pix_ld, ldb=st.pix_ld)
            else:
                d = dict(a=_ptr(st.dyt), b=_ptr(st.cols), lda=st.fld, ldb=kk)
            rows.setdefault(prec(st), []).append(
                (s, dict(d, c=_ptr(st.partial), bias=0, mask=0, dbias=0, m=f, n=kk, k=s.batch_size * oh * ow,
                         ldc=kk, relu=0, row_mult=oh * ow, ksplit=st.ksplit, ksplit_len=st.ksplit_len)))
        out += gemms(N.HNN_WGRAD, rows, f"{label}/tc")
        # (the split partials are summed for every layer at once before the optimizer: conv_reduce_all)
        return out

    @staticmethod
    def _aux_grid(total):
        return max(1, min(-(-total // 256), 4 * 148))

    def _tc_conv_stages(self):
        return [(s, st) for w in self._stage_waves() for s, st in w if st.kind == "conv" and getattr(st, "tc", False)]

    def conv_weight_prep(self, train: bool) -> list:
        """One launch per weight transform for every tensor-core conv layer of the step (the
        weights only change in the optimizer, after the backward): the padded GEMM copies for
        the forward, and for training the flipped (stride-1 input gradient as a forward conv) and
        transposed (stride-2 dcols GEMM) copies.  Per-layer launches of these cost ~13 us each."""
        stages = self._tc_conv_stages()
        out = []
        blocks = lambda s, st: self._aux_grid(self._conv_out(st)[0] * st.kkp)
        padded = [(s, st) for s, st in stages if st.wpad is not None and not st.im_fwd]
        if padded:
            out.append(self._convtc_aux(N.CONVTC_PAD_WEIGHTS, padded, "prep/conv/tc/padw", blocks))
        rsc = [(s, st) for s, st in stages if st.im_fwd]
        if rsc:  # (r, s, c)-ordered K for the implicit-GEMM forward: one CTA per filter (grid-stride)
            out.append(self._convtc_aux(N.CONVTC_PAD_WEIGHTS_RSC, rsc, "prep/conv/tc/padw_rsc",
                                        lambda s, st: min(self._conv_out(st)[0], 148)))
        if not train:
            return out
        flips, flips_rsc = [], []
        for s, st in stages:
            if st.needs_dx and st.dg_fwd:
                c = st.in_shape[0]
                f = self._conv_out(st)[0]
                k = st.attrs["kernel"]
                W = self.pview(self.params, s.index, st.params[0])
                (flips_rsc if st.im_dg else flips).append(
                    (s, N.ConvTcProblem(weight=_ptr(W), wpad=_ptr(st.wflip), c=c, f=f, k=k, model=s.index,
                                        bf16=int(st.bf16))))
        if flips_rsc:  # one CTA per input channel (grid-stride)
            out.append(self._aux_table(N.CONVTC_FLIP_WEIGHTS_RSC, flips_rsc, "prep/conv/tc/flipw_rsc",
                                       lambda pr: min(pr.c, 148),
                                       max(pr.k for _, pr in flips_rsc)))
        if flips:
            max_k = max(pr.k for _, pr in flips)
            out.append(self._aux_table(N.CONVTC_FLIP_WEIGHTS, flips, "prep/conv/tc/flipw",
                                       lambda pr: self._aux_grid(pr.c * pr.f * pr.k * pr.k), max_k))
        par = []
        for s, st in stages:
            if st.par_dg:
                c, f = st.in_shape[0], self._conv_out(st)[0]
                W = self.pview(self.params, s.index, st.params[0])
                for q, off in enumerate(_parity_offsets(c, f)):
                    par.append((s, N.ConvTcProblem(weight=_ptr(W), wpad=_ptr(st.wpar) + 2 * off, c=c, f=f, k=3,
                                                   ksplit=q, model=s.index, bf16=1)))
        if par:
            out.append(self._aux_table(N.CONVTC_PARITY_WEIGHTS, par, "prep/conv/tc/parity_w",
                                       lambda pr: self._aux_grid(pr.c * pr.f * (1 + (pr.ksplit >> 1)) * (1 + (pr.ksplit & 1))),
                                       3))
        wt = [(s, st) for s, st in stages if st.needs_dx and not st.dg_fwd and st.bf16 and not st.par_dg]
        if wt:
            out.append(self._convtc_aux(N.CONVTC_WT_WEIGHTS, wt, "prep/conv/tc/wt", blocks))
        return out

    def conv_reduce_all(self) -> list:
        """The weight / bias gradients of every tensor-core conv layer from their split partials,
        one launch after the last weight-gradient GEMM (each layer has its own partial buffers)."""
        out = []
        if self._pending_reduce:  # SIMT / direct conv layers: hnn_conv_wgrad_reduce
            red, base = [], 0
            for pr in self._pending_reduce:
                n = -(-(pr.f * (pr.c * pr.k * pr.k + 1)) // 256)
                pr.tile_base = base
                red.append(pr)
                base += n
            rt = _dev_table(N.ConvProblem, red, self.device)
            out.append(Launch("hnn_conv_wgrad_reduce", (_ptr(rt), len(red), base, _ptr(self.cur), _ptr(self.status)),
                              rt, "bwd/conv/reduce"))
        stages = self._tc_conv_stages()
        if stages:
            out.append(self._convtc_aux(N.CONVTC_WGRAD_REDUCE, stages, "bwd/conv/tc/reduce",
                                        lambda s, st: self._aux_grid(self._conv_out(st)[0] * st.kkp
                                                                     + self._conv_out(st)[0])))
        return out

    def _conv_group(self, op, items, label, direct):
        tm, tn = N.conv_tile_shape(op)
        probs, base, red, rbase = [], 0, [], 0
        flops = smem = threads = 0
        for s, st in items:
            c, h, w = st.in_shape
            f, oh, ow = self._conv_out(st)
            k = st.attrs["kernel"]
            W = self.pview(self.params, s.index, st.params[0])
            B = self.pview(self.params, s.index, st.params[1])
            common = dict(x=_ptr(st.x), weight=_ptr(W), bias=_ptr(B), y=_ptr(st.y), dy=_ptr(st.dy),
                          dx=_ptr(st.dx), mask=_ptr(st.x) if (op == N.HNN_DGRAD and st.mask_input) else 0,
                          partial=_ptr(st.partial), dw=_ptr(self.pview(self.grads, s.index, st.params[0])),
                          db=_ptr(self.pview(self.grads, s.index, st.params[1])), cap=s.batch_size, c=c, h=h, w=w,
                          f=f, k=k, stride=st.attrs.get("stride", 1), pad=st.attrs.get("padding", 0), oh=oh, ow=ow,
                          model=s.index, relu=int(st.relu), splits=st.splits, split_len=CONV_SPLIT_LEN)
            cols = c * k * k + 1
            fold = getattr(st, "pool_fold", None)
            if direct and fold is not None and op != N.HNN_FWD:  # (the pool's backward in the dy staging)
                common.update(pool_dy=_ptr(fold.dy), pool_idx=_ptr(fold.idx),
                              pool_mask=_ptr(fold.x) if fold.mask_input else 0)
            pfwd = getattr(st, "pool_fwd", None)
            if direct and pfwd is not None and op == N.HNN_FWD:  # (the pool's forward in the x staging)
                common.update(pool_x=_ptr(pfwd.x), pool_idx=_ptr(pfwd.idx))
            if direct:
                tiles_n = 1
                tiles = st.splits if op == N.HNN_WGRAD else s.batch_size
                smem = max(smem, N.conv_direct_smem(op, c, h, w, f, k, oh, ow))
                threads = max(threads, N.conv_direct_threads(op, c, h, w, f, k, oh, ow))
            elif op == N.HNN_FWD:
                tiles_n = -(-f // tn)
                tiles = -(-(s.batch_size * oh * ow) // tm) * tiles_n
            elif op == N.HNN_DGRAD:
                tiles_n = -(-c // tn)
                tiles = -(-(s.batch_size * h * w) // tm) * tiles_n
            else:
                tiles_n = -(-cols // tn)
                tiles = st.splits * -(-f // tm) * tiles_n
            if op == N.HNN_WGRAD:
                red.append(N.ConvProblem(tile_base=rbase, tiles_n=tiles_n, **common))
                rbase += -(-(f * cols) // 256)
            probs.append(N.ConvProblem(tile_base=base, tiles_n=tiles_n, **common))
            base += tiles
            flops += 2 * s.batch_size * oh * ow * f * c * k * k
        t = _dev_table(N.ConvProblem, probs, self.device)
        if direct:
            pooled = op == N.HNN_FWD and any(getattr(st, "pool_fwd", None) is not None for _, st in items)
            args = (N.CONV_DIRECT_FWD_POOLED if pooled else op, _ptr(t), len(probs), base, smem, threads,
                    _ptr(self.cur), _ptr(self.status))
            out = [Launch("hnn_grouped_conv_direct_ex", args, t, label, flops=flops)]
        else:
            out = [Launch("hnn_grouped_conv", (op, _ptr(t), len(probs), base, _ptr(self.cur), _ptr(self.status)), t,
                          label, flops=flops)]
        if op == N.HNN_WGRAD:  # split partials summed with every other layer's (conv_reduce_all)
            self._pending_reduce += red
        return out

    def _embed_launch(self, op, items, label):
        probs, base = [], 0
        for s, st in items:
            length, dim, vocab = st.in_shape[0], st.attrs["dim"], st.attrs["vocab"]
            nb = -(-(s.batch_size * length) // 8) if op == N.HNN_FWD else -(-vocab // 8)
            probs.append(N.EmbedProblem(x=_ptr(st.x), table=_ptr(self.pview(self.params, s.index, st.params[0])),
                                        y=_ptr(st.y), dy=_ptr(st.dy),
                                        dtable=_ptr(self.pview(self.grads, s.index, st.params[0])),
                                        cap=s.batch_size, len=length, ldx=st.ld_in, dim=dim, vocab=vocab,
                                        model=s.index, block_base=base, blocks=nb))
            base += nb
        t = _dev_table(N.EmbedProblem, probs, self.device)
        nbytes = sum(4 * p.cap * p.len * (2 * p.dim + 1) if op == N.HNN_FWD
                     else 4 * (p.vocab * p.dim + p.cap * p.len * (p.dim + 1)) for p in probs)
        return [Launch("hnn_embedding", (op, _ptr(t), len(probs), base, _ptr(self.cur), _ptr(self.status)), t,
                       label, nbytes=nbytes)]

    def _pool_launch(self, op, items, label):
        probs, base = [], 0
        for s, st in items:
            c, h, w = st.in_shape
            k = st.attrs["kernel"]
            stride = st.attrs.get("stride", k)
            oh, ow = conv_extent(h, k, stride, 0), conv_extent(w, k, stride, 0)
            if s.batch_size * c * h * w >= 2 ** 31:  # (the pool kernels index in 32 bits)
                raise UnsupportedGraphError(f"{st.node_id}: pooled tensor above 2^31 elements")
            mode, blocks = N.pool_mode_blocks(op, s.batch_size, c, h, w, k, stride, oh, ow,
                                              (_ptr(st.x), _ptr(st.dx)) if op != N.HNN_FWD else (_ptr(st.x),))
            probs.append(N.PoolProblem(_ptr(st.x), _ptr(st.y), _ptr(st.idx), _ptr(st.dy), _ptr(st.dx),
                                       _ptr(st.x) if st.mask_input else 0, s.batch_size, c, h, w, k, stride, oh,
                                       ow, s.index, base, blocks, mode,
                                       _ptr(st.xh_next) if op == N.HNN_FWD else 0))
            base += blocks
        nbytes = sum(4 * p.cap * p.c * (p.h * p.w + p.oh * p.ow) + p.cap * p.c * p.oh * p.ow for p in probs)
        t = _dev_table(N.PoolProblem, probs, self.device)
        return [Launch("hnn_grouped_maxpool", (op, _ptr(t), len(probs), base, _ptr(self.cur), _ptr(self.status)),
                       t, label, nbytes=nbytes)]

    def _relu_launch(self, op, items, label):
        probs, base = [], 0
        for s, st in items:
            if s.batch_size * st.ld_in >= 2 ** 31:  # (the relu kernel indexes in 32 bits)
                raise UnsupportedGraphError(f"{st.node_id}: relu tensor above 2^31 elements")
            blocks = -(-(s.batch_size * st.ld_in) // 256)
            probs.append(N.ReluProblem(_ptr(st.x), _ptr(st.y), _ptr(st.dy), _ptr(st.dx), s.batch_size, st.ld_in,
                                       s.index, base, blocks, 0))
            base += blocks
        t = _dev_table(N.ReluProblem, probs, self.device)
        nbytes = sum((8 if op == N.HNN_FWD else 12) * p.cap * p.row for p in probs)
        return [Launch("hnn_grouped_relu", (op, _ptr(t), len(probs), base, _ptr(self.cur), _ptr(self.status)), t,
                       label, nbytes=nbytes)]

    def _wave_launches(self, op, items, label):
        by_kind: dict = {}
        for s, st in items:
            by_kind.setdefault(st.kind, []).append((s, st))
        out = []
        for kind, group in by_kind.items():
            if kind == "dense":
                out += self._gemm_launch(op, group, f"{label}/dense")
            elif kind == "conv":
                out += self._conv_launch(op, group, f"{label}/conv")
            elif kind == "pool":
                if op == N.HNN_FWD:  # (pools folded into the next direct conv's input staging: no launch)
                    group = [(s, st) for s, st in group if not getattr(st, "fwd_folded", False)]
                if group:
                    out += self._pool_launch(N.HNN_FWD if op == N.HNN_FWD else N.HNN_DGRAD, group, f"{label}/pool")
            elif kind == "embed":
                if op == N.HNN_FWD:  # (an embedding never needs an input gradient: it reads the input)
                    out += self._embed_launch(N.HNN_FWD, group, f"{label}/embed")
            else:
                out += self._relu_launch(N.HNN_FWD if op == N.HNN_FWD else N.HNN_DGRAD, group, f"{label}/relu")
        return out

    def _sce_launch(self, train: bool, skip=()):
        probs = []
        for s in self.slots:
            last = s.stages[-1]
            if id(last) in skip:
                continue
            probs.append(N.SceProblem(_ptr(last.y), _ptr(s.batch_y), _ptr(last.dy) if train else 0, last.ld_out,
                                      s.classes, s.batch_size, s.index))
        t = _dev_table(N.SceProblem, probs, self.device)
        cap = max(s.batch_size for s in self.slots)
        ncls = max(s.classes for s in self.slots)
        status = self.status if train else self.eval_status
        nbytes = sum(p.cap * (4 * p.classes * (2 if train else 1) + 4) for p in probs)
        return Launch("hnn_sce_fused", (_ptr(t), len(probs), cap, ncls, _ptr(self.cur), _ptr(status), int(train),
                                        _ptr(self.loss_out), _ptr(self.correct_out)), t,
                      "sce" if train else "sce/eval", nbytes=nbytes)

    def _fused(self, s) -> bool:
        """Dense weight gradients of model s feed the optimizer inside their epilogue.

        Only for SGD / momentum (a multiply-subtract per element): Adam's three IEEE
        divisions and square root per element would leave the tensor-core pipeline waiting
        on eight epilogue warps (measured 2.5x slower), so Adam keeps the full-occupancy
        multi-tensor kernel."""
        return self.fuse_optimizer and s.opt_kind != N.OPT_ADAM

    def _unfused_ranges(self, s) -> list:
        """(offset, count) arena ranges of model s updated by the multi-tensor kernel."""
        if not self._fused(s):
            return [(s.seg_off, s.seg_len)]
        fused = {pid for st in s.stages if st.kind == "dense" for pid in st.params}
        out = []
        for pid, shp in s.specs.items():
            if pid in fused:
                continue
            off, cnt = s.offsets[pid], _align4(int(np.prod(shp)))
            if out and out[-1][0] + out[-1][1] == off:
                out[-1] = (out[-1][0], out[-1][1] + cnt)
            else:
                out.append((off, cnt))
        return out

    def _optimizer_order(self):
        """(slot, offset, count) ranges in the order the multi-tensor kernel walks them: grouped by
        stage, first stage first.  Backward runs the stages in reverse, so the first stage's
        gradients were written last and are still in L2 when the optimizer starts."""
        items = []
        for s in self.slots:
            ranges = self._unfused_ranges(s)
            if len(ranges) == 1 and ranges[0] == (s.seg_off, s.seg_len):  # split by stage
                ranges = []
                for st in s.stages:
                    if not st.params:
                        continue
                    offs = [s.offsets[pid] for pid in st.params]
                    end = max(s.offsets[pid] + _align4(int(np.prod(s.specs[pid]))) for pid in st.params)
                    ranges.append((min(offs), end - min(offs)))
            for r in ranges:
                stage = next((k for k, st in enumerate(s.stages) for pid in st.params
                              if s.offsets[pid] <= r[0] < s.offsets[pid] + _align4(int(np.prod(s.specs[pid])))), 0)
                items.append((stage, s.index, s, r[0], r[1]))
        items.sort(key=lambda t: (t[0], t[1]))
        covered = sum(t[4] for t in items)
        assert covered == sum(c for s in self.slots for _, c in self._unfused_ranges(s)), "optimizer ranges"
        return [(t[2], t[3], t[4]) for t in items]

    def _optimizer_launch(self):
        segs, base = [], 0
        for s, off, cnt in self._optimizer_order():
            kind = s.opt_kind
            if True:
                chunks = -(-cnt // OPT_CHUNK)
                segs.append(N.OptSegment(
                    _ptr(self.params) + 4 * off, _ptr(self.grads) + 4 * off,
                    (_ptr(self.m1) + 4 * off) if kind != N.OPT_SGD else 0,
                    (_ptr(self.m2) + 4 * off) if kind == N.OPT_ADAM else 0,
                    cnt, s.index, kind, float(np.float32(s.momentum)), base, chunks, 0))
                base += chunks
        if not segs:
            return []
        t = _dev_table(N.OptSegment, segs, self.device)
        entry = "hnn_multi_tensor_adam" if any(s.kind == N.OPT_ADAM for s in segs) else "hnn_multi_tensor_sgd"
        per = {N.OPT_SGD: 12, N.OPT_SGD_MOMENTUM: 20, N.OPT_ADAM: 28}
        nbytes = sum(per[s.kind] * s.count for s in segs)
        return [Launch(entry, (_ptr(t), len(segs), base, _ptr(self.cur), _ptr(self.status)), t, "optimizer",
                       nbytes=nbytes)]

    def _link_nhwc_producers(self):
        """A bf16 conv whose output feeds an implicit-GEMM "same" conv directly writes that conv's
        NHWC input from its forward epilogue (second TMA store per block), so the consumer needs
        no NHWC copy launch."""
        for s in self.slots:
            for a, b in zip(s.stages, s.stages[1:]):
                a.xh_next, b.xh_from_prev = None, False
            for a, b in zip(s.stages, s.stages[1:]):
                if (a.kind == "pool" and b.kind == "conv" and getattr(b, "tc", False) and b.im_fwd
                        and self._same_conv(b) and b.x is a.y):  # the pool writes the NHWC copy
                    a.xh_next, b.xh_from_prev = b.xh, True
                    continue
                if not (a.kind == b.kind == "conv" and getattr(a, "tc", False) and getattr(b, "tc", False)):
                    continue
                f, oh, ow = self._conv_out(a)
                if (a.bf16 and b.im_fwd and self._same_conv(b) and b.x is a.y and (oh * ow) % 32 == 0
                        and f % 8 == 0):
                    a.xh_next, b.xh_from_prev = b.xh, True

    def _link_pool_folds(self):
        """A direct (LeNet-class) conv whose output feeds a 2 x 2 / stride-2 max-pool on even planes
        stages its dy through the pool's backward (hnn_conv_problem.pool_*: argmax select + relu mask,
        maxpool2_bwd's arithmetic, so bit-identical) and the pool's backward launch is dropped (C2's
        first pool gradient alone was a 45 us launch).  The conv then reads the pool's dy, which
        lives in the ping-pong buffer its own dx would overwrite, so a conv that needs dx gets a
        dx buffer of its own (and the stage below reads its dy from there).  Forward: a direct conv
        whose input is such a pool's output computes the pool while staging its input (writing the
        pool's y and argmax) and the pool's forward launch is dropped.  HNN_POOL_FOLD=0: off; =bwd:
        backward folds only."""
        torch = _torch()
        mode = os.environ.get("HNN_POOL_FOLD", "1")
        even22 = lambda b: (b.attrs["kernel"] == 2 and b.attrs.get("stride", 2) == 2
                            and b.in_shape[1] % 2 == 0 and b.in_shape[2] % 2 == 0)
        for s in self.slots:
            for st in s.stages:
                st.pool_fold, st.folded, st.pool_fwd, st.fwd_folded = None, False, None, False
            if mode == "0":
                continue
            for a, b in zip(s.stages, s.stages[1:]):
                if (mode != "bwd" and a.kind == "pool" and b.kind == "conv" and getattr(b, "direct", False)
                        and b.x is a.y and even22(a) and getattr(a, "xh_next", None) is None):
                    b.pool_fwd, a.fwd_folded = a, True
            for k, (a, b) in enumerate(zip(s.stages, s.stages[1:])):
                if not (a.kind == "conv" and getattr(a, "direct", False) and b.kind == "pool" and b.x is a.y):
                    continue
                if not even22(b):
                    continue
                a.pool_fold, b.folded = b, True
                if a.needs_dx and getattr(a, "fold_dx", None) is None:
                    cap = s.batch_size
                    a.fold_dx = torch.zeros(cap * a.ld_in, dtype=torch.float32, device=self.device)
                    a.dx = a.fold_dx.view(cap, a.ld_in)
                    s.stages[k - 1].dy = a.dx

    def _tail_eligible(self, s) -> bool:
        """Models whose logits layer takes the fused tail (hnn_logits_tail): a final plain dense layer
        with <= 16 classes, 16-byte rows and a small input (cap * K <= 16K floats: C1 / C5's 64 x 256,
        LeNet's 128 x 84; measured slower than the grouped skinny launches for C3's 256 x 128 and the
        CNNs' 128 x 512, profiles/r02/logits_tail_ab_v10.txt).  A function of the model's own shape
        only, so isolation and sharding never change a model's path.  Opt-in (HNN_LOGITS_TAIL=1):
        eager per-launch times favour it (C5 0.150 -> 0.133 ms), but in the graph-replayed step the
        four programmatically-dependent launches it replaces overlap their tails and it measured level
        or slower (C5 0.111 -> 0.110, C1 0.0615 -> 0.0636, C2 0.482 -> 0.496 ms)."""
        if os.environ.get("HNN_LOGITS_TAIL", "0") != "1":  # (off by default: see below)
            return False
        st = s.stages[-1]
        if st.kind != "dense" or st.relu or len(st.params) != 2:
            return False
        K, U = int(np.prod(st.in_shape)), st.out_shape[0]
        return (U <= 16 and U == s.classes and K % 4 == 0 and st.ld_in % 4 == 0 and K <= 2048
                and s.batch_size * K <= 16 * 1024
                and N.tail_smem(s.batch_size, K, U) <= 200 * 1024)

    def _logits_tail(self):
        """(launch or None, ids of the tail stages): the fused logits tail of every eligible model."""
        probs, done, smem = [], set(), 0
        for s in self.slots:
            if not self._tail_eligible(s):
                continue
            st = s.stages[-1]
            K, U = int(np.prod(st.in_shape)), st.out_shape[0]
            fuse = self._fused(s)
            keep = self.keep_grads or not fuse
            arena = lambda a, pid: _ptr(self.pview(a, s.index, pid)) if a is not None else 0
            probs.append(N.TailProblem(
                x=_ptr(st.x), w=arena(self.params, st.params[0]), b=arena(self.params, st.params[1]),
                logits=_ptr(st.y), labels=_ptr(s.batch_y), dx=_ptr(st.dx) if st.needs_dx else 0,
                mask=_ptr(st.x) if st.mask_input else 0,
                dw=arena(self.grads, st.params[0]) if keep else 0, db=arena(self.grads, st.params[1]) if keep else 0,
                opt_w=arena(self.params, st.params[0]) if fuse else 0, opt_b=arena(self.params, st.params[1]) if fuse else 0,
                opt_wm=arena(self.m1, st.params[0]) if fuse and s.opt_kind != N.OPT_SGD else 0,
                opt_bm=arena(self.m1, st.params[1]) if fuse and s.opt_kind != N.OPT_SGD else 0,
                ldx=st.ld_in, ld_logits=st.ld_out, ld_dx=st.ld_in, cap=s.batch_size, k=K, classes=U, model=s.index,
                opt_kind=s.opt_kind, opt_momentum=float(np.float32(s.momentum))))
            smem = max(smem, N.tail_smem(s.batch_size, K, U))
            done.add(id(st))
        if not probs:
            return None, done
        t = _dev_table(N.TailProblem, probs, self.device)
        flops = sum(6 * p.cap * p.k * p.classes for p in probs)
        launch = Launch("hnn_logits_tail", (_ptr(t), len(probs), smem, _ptr(self.cur), _ptr(self.status),
                                            _ptr(self.loss_out), _ptr(self.correct_out)), t, "tail/logits+sce+bwd",
                        flops=flops)
        return launch, done

    def build_plans(self):
        waves = self._stage_waves()
        self._pending_reduce = []
        self._link_nhwc_producers()
        self._link_pool_folds()
        fwd = []
        for w, items in enumerate(waves):
            fwd += self._wave_launches(N.HNN_FWD, items, f"fwd{w}")
        # training: eligible models' logits layers leave their waves for the fused tail launch
        tail, tail_ids = self._logits_tail()
        fwd_train = fwd
        if tail is not None:
            fwd_train = []
            for w, items in enumerate(waves):
                rest = [(s, st) for s, st in items if id(st) not in tail_ids]
                if rest:
                    fwd_train += self._wave_launches(N.HNN_FWD, rest, f"fwd{w}")
        sce_train = [] if tail is not None and all(id(s.stages[-1]) in tail_ids for s in self.slots) else \
            [self._sce_launch(True, skip=tail_ids)]
        bwd = []
        for w in range(len(waves) - 1, -1, -1):
            items = [(s, st) for s, st in waves[w] if id(st) not in tail_ids]
            # input gradients first: with optimizer fusion the weight-gradient launch updates W in
            # place, and this wave's DGRAD must still read the pre-update W (src/engine.py:120-151
            # computes every gradient before apply_update)
            fused_l, fused = self._skinny_backward(items)
            for l in fused_l:
                l.label = f"bwd{w}/dense/skinny_bwd"
            done = {id(st) for _, st in fused}
            dg = [(s, st) for s, st in items if st.needs_dx and id(st) not in done and not st.folded]
            if dg:
                bwd += self._wave_launches(N.HNN_DGRAD, dg, f"bwd{w}")
            bwd += fused_l
            for kind in ("dense", "conv", "embed"):
                grp = [(s, st) for s, st in items if st.kind == kind and id(st) not in done]
                if grp:
                    if kind == "dense":
                        bwd += self._gemm_launch(N.HNN_WGRAD, grp, f"bwd{w}/dense/wgrad")
                    elif kind == "conv":
                        bwd += self._conv_launch(N.HNN_WGRAD, grp, f"bwd{w}/conv/wgrad")
                    else:
                        bwd += self._embed_launch(N.HNN_WGRAD, grp, f"bwd{w}/embed/wgrad")
        self.forward_plan = self.conv_weight_prep(False) + fwd
        self.train_plan = ([self._gather_train] + self.conv_weight_prep(True) + fwd_train + ([tail] if tail else [])
                           + sce_train + bwd + self.conv_reduce_all() + self._optimizer_launch())
        self.eval_plan = [self._gather_eval] + self.conv_weight_prep(False) + fwd + [self._sce_launch(False)]
        self.graph = None

    # ------------------------------------------------------------------ running
    def load_schedule(self, rows: np.ndarray):
        """rows: [T, n] STEP_DTYPE.  Uploads and rewinds the step counter."""
        torch = _torch()
        flat = np.ascontiguousarray(rows).view(np.uint8).reshape(-1)
        need = flat.size
        if self.sched is None or self.sched.numel() < need:
            self.sched = torch.zeros(max(need, 48 * self.n * 64), dtype=torch.uint8, device=self.device)
            self.graph = None  # the graph captured the old schedule pointer
        self.sched[:need].copy_(torch.from_numpy(flat))
        self.counter.zero_()

    def _stream(self):
        torch = _torch()
        return torch.cuda.current_stream(self.device).cuda_stream

    def run_plan(self, plan: list, stream=None):
        stream = self._stream() if stream is None else stream
        N.call("hnn_step_begin", _ptr(self.sched), _ptr(self.counter), _ptr(self.cur), self.n, stream)
        for launch in plan:
            launch.run(stream)

    def train_steps(self, count: int, use_graph: bool = False, host_fed: bool = False):
        """Run `count` scheduled training steps (stream-ordered, asynchronous).

        host_fed: the batch arenas were filled by the caller (H2D), so the gather is skipped.
        """
        plan = self.train_plan[1:] if host_fed else self.train_plan
        if not use_graph:
            for _ in range(count):
                self.run_plan(plan)
            return
        torch = _torch()
        graphs = self.__dict__.setdefault("_graphs", {})
        if self.graph is None:
            graphs.clear()
            self.graph = True
        g = graphs.get(host_fed)
        if g is None:
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            g = torch.cuda.CUDAGraph()
            # thread-local capture: host loader threads may sync events while a step is captured
            with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
                self.run_plan(plan, side.cuda_stream)
            torch.cuda.current_stream(self.device).wait_stream(side)
            graphs[host_fed] = g
        for _ in range(count):
            g.replay()

    def launch_count(self, train: bool = True) -> int:
        return 1 + len(self.train_plan if train else self.eval_plan)

    def perm_upload(self, m: int, perm: np.ndarray):
        self.perm[m, : perm.size].copy_(_torch().from_numpy(perm.astype(np.int32)))
