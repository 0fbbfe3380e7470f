"""ctypes binding of the C-ABI library (include/hnn_b200.h).

The library is the product: if it is missing, cannot be loaded, or no CUDA
device is present, every device entry point raises — there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import DeviceError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libhnn_b200.so"

HNN_FWD, HNN_DGRAD, HNN_WGRAD = 0, 1, 2
PREC_SIMT, PREC_3XTF32, PREC_SIMT_SKINNY, PREC_3XTF32_PAIR, PREC_BF16_PAIR = 0, 1, 2, 3, 4
CONVTC_IM2COL, CONVTC_TRANSPOSE_DY, CONVTC_COL2IM, CONVTC_WGRAD_REDUCE, CONVTC_PAD_WEIGHTS = 0, 1, 2, 3, 4
CONVTC_TRANSPOSE_HW_TILES = 4  # (hnn_b200.h)


def transpose_blocks(cap: int, hw: int, f: int) -> int:
    """Blocks of one HNN_CONVTC_TRANSPOSE_DY problem: 32 channels x CONVTC_TRANSPOSE_HW_TILES
    consecutive (sample, 32-pixel run) units per block."""
    return -(-(cap * -(-hw // 32)) // CONVTC_TRANSPOSE_HW_TILES) * -(-f // 32)
CONVTC_FLIP_WEIGHTS, CONVTC_WT_WEIGHTS, CONVTC_PAD_WEIGHTS_RSC, CONVTC_FLIP_WEIGHTS_RSC = 5, 6, 7, 8
CONVTC_PARITY_WEIGHTS, CONVTC_SPLITK_FWD = 9, 10
OPT_SGD, OPT_SGD_MOMENTUM, OPT_ADAM = 0, 1, 2
CONV_DIRECT_BCHUNK = 1

P = C.c_uint64  # device pointers travel as integers
I = C.c_int32


class StepRow(C.Structure):
    _fields_ = [("active", I), ("rows", I), ("perm_base", I), ("epoch", I), ("batch", I), ("opt_step", I),
                ("lr", C.c_float), ("bias1", C.c_float), ("bias2", C.c_float), ("reserved", I * 3)]


class ModelStatus(C.Structure):
    _fields_ = [("alive", I), ("abort_epoch", I), ("abort_batch", I), ("last_correct", I),
                ("last_loss", C.c_float), ("reserved", I), ("loss_sum", C.c_double),
                ("correct_sum", C.c_int64), ("seen", C.c_int64)]


class GatherProblem(C.Structure):
    _fields_ = [("src_x", P), ("src_y", P), ("perm", P), ("dst_x", P), ("dst_y", P),
                ("sample", I), ("ld_dst", I), ("cap", I), ("model", I)]


class GemmProblem(C.Structure):
    _fields_ = [("a", P), ("b", P), ("c", P), ("bias", P), ("mask", P), ("dbias", P),
                ("m", I), ("n", I), ("k", I), ("lda", I), ("ldb", I), ("ldc", I),
                ("model", I), ("relu", I), ("tile_base", I), ("tiles_n", I), ("tmap_a", P), ("tmap_b", P),
                ("tmap_c", P), ("opt_w", P), ("opt_wm", P), ("opt_wv", P), ("opt_b", P), ("opt_bm", P),
                ("opt_bv", P), ("opt_kind", I), ("opt_momentum", C.c_float),
                ("row_mult", I), ("c_mode", I), ("ksplit", I), ("ksplit_len", I), ("tile_n", I), ("im_kw", I),
                ("im_c", I), ("im_k", I), ("im_pad", I), ("im_h", I), ("im_w", I), ("im_oh", I), ("im_ow", I),
                ("im_n", I), ("xh_out", P), ("tmap_xh", P)]

    def __init__(self, **kw):
        kw.setdefault("row_mult", 1)
        kw.setdefault("ksplit", 1)
        super().__init__(**kw)


class ConvProblem(C.Structure):
    _fields_ = [("x", P), ("weight", P), ("bias", P), ("y", P), ("dy", P), ("dx", P), ("mask", P),
                ("partial", P), ("dw", P), ("db", P),
                ("cap", I), ("c", I), ("h", I), ("w", I), ("f", I), ("k", I), ("stride", I), ("pad", I),
                ("oh", I), ("ow", I), ("model", I), ("relu", I), ("tile_base", I), ("tiles_n", I),
                ("splits", I), ("split_len", I), ("pool_dy", P), ("pool_idx", P), ("pool_mask", P),
                ("pool_x", P)]


class ConvTcProblem(C.Structure):
    _fields_ = [("x", P), ("cols", P), ("dy", P), ("dyt", P), ("dcols", P), ("dx", P), ("mask", P),
                ("partial", P), ("dw", P), ("db", P), ("bpart", P), ("weight", P), ("wpad", P),
                ("cap", I), ("c", I), ("h", I), ("w", I), ("f", I), ("k", I), ("stride", I), ("pad", I),
                ("oh", I), ("ow", I), ("kk", I), ("kkp", I), ("ksplit", I), ("ksplit_len", I),
                ("model", I), ("block_base", I), ("blocks", I), ("colst", P), ("dyk", P), ("bf16", I),
                ("pix_ld", I), ("rsc", I), ("reserved", I)]


class EmbedProblem(C.Structure):
    _fields_ = [("x", P), ("table", P), ("y", P), ("dy", P), ("dtable", P), ("cap", I), ("len", I), ("ldx", I),
                ("dim", I), ("vocab", I), ("model", I), ("block_base", I), ("blocks", I)]


class PoolProblem(C.Structure):
    _fields_ = [("x", P), ("y", P), ("idx", P), ("dy", P), ("dx", P), ("mask", P),
                ("cap", I), ("c", I), ("h", I), ("w", I), ("k", I), ("stride", I), ("oh", I), ("ow", I),
                ("model", I), ("block_base", I), ("blocks", I), ("mode", I), ("xh", P)]


POOL_ELEMENTWISE, POOL_WINDOWS_2X2 = 0, 1  # (hnn_b200.h)
CONV_DIRECT_FWD_POOLED = 16  # (hnn_b200.h: hnn_grouped_conv_direct_ex op, forward with folded max-pools)
# HNN_POOL_WINDOWS_PER_BLOCK: the library's build constant (the override is for variant builds only)
POOL_WINDOWS_PER_BLOCK = int(os.environ.get("HNN_POOL_WINDOWS_PER_BLOCK", "1024"))


def pool_mode_blocks(op: int, cap: int, c: int, h: int, w: int, k: int, stride: int, oh: int, ow: int,
                     ptrs=()):
    """(mode, blocks) of one hnn_pool_problem: 2 x 2 / stride 2 windows on even planes run in window
    mode (HNN_POOL_WINDOWS_PER_BLOCK windows per block, both directions); other pools one element per
    thread, 256 per block.  ptrs: the plane-sized tensors the window form moves as float2 (8-byte
    aligned or elementwise).  HNN_POOL_WINDOWS=0 forces the elementwise form (A/B, tests)."""
    import os

    if (k == 2 and stride == 2 and h % 2 == 0 and w % 2 == 0 and all(p % 8 == 0 for p in ptrs)
            and os.environ.get("HNN_POOL_WINDOWS", "1") != "0"):
        return POOL_WINDOWS_2X2, -(-(cap * c * oh * ow) // POOL_WINDOWS_PER_BLOCK)
    return POOL_ELEMENTWISE, -(-(cap * c * (oh * ow if op == HNN_FWD else h * w)) // 256)


class ReluProblem(C.Structure):
    _fields_ = [("x", P), ("y", P), ("dy", P), ("dx", P), ("cap", I), ("row", I), ("model", I),
                ("block_base", I), ("blocks", I), ("reserved", I)]


class SceProblem(C.Structure):
    _fields_ = [("logits", P), ("labels", P), ("dlogits", P), ("ld", I), ("classes", I), ("cap", I), ("model", I)]


class HostGatherItem(C.Structure):
    _fields_ = [("dst_x", P), ("dst_y", P), ("src_x", P), ("src_y", P), ("idx", P), ("ld_dst", C.c_int64),
                ("ld_src", C.c_int64), ("cols", C.c_int64), ("n", C.c_int64), ("cap", C.c_int64)]


class HostFedIO(C.Structure):
    _fields_ = [("host_x", P), ("stage_x", P), ("arena_x", P), ("x_bytes", C.c_int64), ("host_y", P), ("stage_y", P),
                ("arena_y", P), ("y_bytes", C.c_int64), ("out_dev", P * 2), ("out_host", P * 2),
                ("out_bytes", C.c_int64 * 2)]


class TailProblem(C.Structure):
    _fields_ = [("x", P), ("w", P), ("b", P), ("logits", P), ("labels", P), ("dx", P), ("mask", P), ("dw", P),
                ("db", P), ("opt_w", P), ("opt_wm", P), ("opt_b", P), ("opt_bm", P), ("ldx", I), ("ld_logits", I),
                ("ld_dx", I), ("cap", I), ("k", I), ("classes", I), ("model", I), ("opt_kind", I),
                ("opt_momentum", C.c_float), ("reserved", I)]


class OptSegment(C.Structure):
    _fields_ = [("param", P), ("grad", P), ("m", P), ("v", P), ("count", C.c_int64), ("model", I), ("kind", I),
                ("momentum", C.c_float), ("chunk_base", I), ("chunks", I), ("reserved", I)]


STRUCTS = {
    "hnn_step_row": StepRow, "hnn_model_status": ModelStatus, "hnn_gather_problem": GatherProblem,
    "hnn_gemm_problem": GemmProblem, "hnn_conv_problem": ConvProblem, "hnn_pool_problem": PoolProblem,
    "hnn_relu_problem": ReluProblem, "hnn_convtc_problem": ConvTcProblem, "hnn_embed_problem": EmbedProblem, "hnn_sce_problem": SceProblem, "hnn_opt_segment": OptSegment,
    "hnn_host_gather_item": HostGatherItem, "hnn_hostfed_io": HostFedIO,
    "hnn_tail_problem": TailProblem,
}

# every symbol include/hnn_b200.h declares, with its ctypes signature
VP = C.c_void_p
SIGNATURES = {
    "hnn_step_begin": [P, P, P, C.c_int, VP],
    "hnn_gather_rows": [P, C.c_int, C.c_int, P, VP],
    "hnn_host_gather_rows": [VP, C.c_int64, VP, VP, C.c_int64, VP, VP, C.c_int64, C.c_int64],
    "hnn_host_gather_batch": [VP, C.c_int, C.c_int],
    "hnn_hostfed_create": [C.POINTER(VP)],
    "hnn_hostfed_destroy": [VP],
    "hnn_hostfed_step": [VP, C.c_int, VP, VP, VP, VP, C.POINTER(VP)],
    "hnn_event_synchronize": [VP],
    "hnn_gemm_tile_shape": [C.c_int, C.c_int, C.POINTER(I), C.POINTER(I)],
    "hnn_gemm_chunk_terms": [C.c_int, C.POINTER(I)],
    "hnn_grouped_gemm": [C.c_int, C.c_int, P, C.c_int, C.c_int, P, P, VP],
    "hnn_skinny_backward": [P, P, C.c_int, C.c_int, P, P, VP],
    "hnn_splitk_epilogue": [P, C.c_int, C.c_int, P, P, VP],
    "hnn_gemm_tc_encode": [C.c_int, C.c_void_p, C.c_int, C.c_void_p],
    "hnn_gemm_bf16_encode": [C.c_int, C.c_void_p, C.c_int, C.c_void_p],
    "hnn_conv_tile_shape": [C.c_int, C.POINTER(I), C.POINTER(I)],
    "hnn_grouped_conv": [C.c_int, P, C.c_int, C.c_int, P, P, VP],
    "hnn_conv_wgrad_reduce": [P, C.c_int, C.c_int, P, P, VP],
    "hnn_grouped_conv_direct": [C.c_int, P, C.c_int, C.c_int, C.c_int, P, P, VP],
    "hnn_conv_direct_smem": [C.c_int] * 8,
    "hnn_conv_direct_threads": [C.c_int] * 8,
    "hnn_grouped_conv_direct_ex": [C.c_int, P, C.c_int, C.c_int, C.c_int, C.c_int, P, P, VP],
    "hnn_grouped_maxpool": [C.c_int, P, C.c_int, C.c_int, P, P, VP],
    "hnn_grouped_relu": [C.c_int, P, C.c_int, C.c_int, P, P, VP],
    "hnn_tail_smem": [C.c_int, C.c_int, C.c_int],
    "hnn_logits_tail": [P, C.c_int, C.c_int, P, P, P, P, VP],
    "hnn_sce_fused": [P, C.c_int, C.c_int, C.c_int, P, P, C.c_int, P, P, VP],
    "hnn_multi_tensor_sgd": [P, C.c_int, C.c_int, P, P, VP],
    "hnn_multi_tensor_adam": [P, C.c_int, C.c_int, P, P, VP],
    "hnn_selftest_div_sqrt": [VP, VP, VP, VP, C.c_int64, VP],
    "hnn_conv_tc_aux": [C.c_int, P, C.c_int, C.c_int, C.c_int, P, P, VP],
    "hnn_embedding": [C.c_int, P, C.c_int, C.c_int, P, P, VP],
    "hnn_struct_size": [C.c_char_p],
    "hnn_last_error": [],
    "hnn_version": [],
}

_lib = None


def load(path: Path = LIB_PATH):
    """Load (once) and type the library; raises if it is not built.  HNN_LIB_VARIANT=NAME loads
    _lib/variants/NAME/libhnn_b200.so instead (A/B builds of tools/build_variant.sh)."""
    global _lib
    if _lib is not None:
        return _lib
    variant = os.environ.get("HNN_LIB_VARIANT")
    if variant and path == LIB_PATH:
        path = LIB_PATH.parent / "variants" / variant / LIB_PATH.name
    if not path.exists():
        raise DeviceError("load", -1, f"{path} is missing — run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(str(path))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_char_p if name in ("hnn_last_error", "hnn_version") else C.c_int
    for name, cls in STRUCTS.items():
        got = lib.hnn_struct_size(name.encode())
        if got != C.sizeof(cls):
            raise DeviceError("load", -1, f"ABI mismatch for {name}: library {got} bytes, binding {C.sizeof(cls)}")
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    lib = load()
    status = getattr(lib, name)(*args)
    if status != 0:
        raise DeviceError(name, status, lib.hnn_last_error().decode(errors="replace"))


def tile_shape(op: int, prec: int) -> tuple:
    tm, tn = I(), I()
    call("hnn_gemm_tile_shape", op, prec, C.byref(tm), C.byref(tn))
    return tm.value, tn.value


def chunk_terms(prec: int) -> int:
    t = I()
    call("hnn_gemm_chunk_terms", prec, C.byref(t))
    return t.value


def conv_tile_shape(op: int) -> tuple:
    tm, tn = I(), I()
    call("hnn_conv_tile_shape", op, C.byref(tm), C.byref(tn))
    return tm.value, tn.value


def conv_direct_smem(op, c, h, w, f, k, oh, ow) -> int:
    return int(load().hnn_conv_direct_smem(op, c, h, w, f, k, oh, ow))


def tail_smem(cap, k, classes) -> int:
    return int(load().hnn_tail_smem(cap, k, classes))


def conv_direct_threads(op, c, h, w, f, k, oh, ow) -> int:
    return int(load().hnn_conv_direct_threads(op, c, h, w, f, k, oh, ow))


def conv_direct_ok(c, h, w, f, k, oh, ow) -> bool:
    """Whether a conv layer fits the direct (shared-memory, per-sample) kernels."""
    if f * (c * k * k + 1) > 16 * 256:
        return False
    return all(conv_direct_smem(op, c, h, w, f, k, oh, ow) <= 200 * 1024 for op in (HNN_FWD, HNN_DGRAD, HNN_WGRAD))


def table_bytes(cls, rows: list) -> bytes:
    arr = (cls * len(rows))(*rows)
    return bytes(arr)
