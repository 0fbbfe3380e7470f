"""Probe the grouped GEMM kernels op by op against float64 numpy (debug / evidence tool)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes

import numpy as np
import torch

from paper_2408_01331_b200 import _native as N
from paper_2408_01331_b200.runtime import STEP_DTYPE, _dev_table, _ptr


TIME = False


def run(op, prec, M, Nn, K, rows=None, seed=0, dbg=0):
    g = np.random.default_rng(seed)
    dev = torch.device("cuda")
    cap = M if op != N.HNN_WGRAD else K
    rows = rows or cap
    if op == N.HNN_FWD:
        A = g.standard_normal((M, K)).astype(np.float32); B = g.standard_normal((Nn, K)).astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64).T
        bias = g.standard_normal(Nn).astype(np.float32); ref = ref + bias
        ref[rows:] = 0
        d = dict(m=M, n=Nn, k=K, lda=K, ldb=K, ldc=Nn)
    elif op == N.HNN_DGRAD:
        A = g.standard_normal((M, K)).astype(np.float32); B = g.standard_normal((K, Nn)).astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64); ref[rows:] = 0
        bias = np.zeros(1, np.float32)
        d = dict(m=M, n=Nn, k=K, lda=K, ldb=Nn, ldc=Nn)
    else:
        A = g.standard_normal((K, M)).astype(np.float32); B = g.standard_normal((K, Nn)).astype(np.float32)
        A[rows:] = 0; B[rows:] = 0
        ref = A.astype(np.float64).T @ B.astype(np.float64)
        bias = np.zeros(1, np.float32)
        d = dict(m=M, n=Nn, k=K, lda=M, ldb=Nn, ldc=Nn)
    a = torch.from_numpy(A).to(dev); b = torch.from_numpy(B).to(dev)
    c = torch.full((d["m"], d["n"]), 7.0, device=dev)
    bi = torch.from_numpy(bias).to(dev)
    db = torch.zeros(d["m"], device=dev)
    tm, tn = N.tile_shape(op, prec)
    tiles_n = -(-d["n"] // tn)
    prob = N.GemmProblem(a=_ptr(a), b=_ptr(b), c=_ptr(c), bias=_ptr(bi) if op == 0 else 0, mask=0,
                         dbias=_ptr(db) if op == 2 else 0, model=0, relu=dbg << 8, tile_base=0, tiles_n=tiles_n, **d)
    keep = None
    if prec == N.PREC_3XTF32:
        maps = bytearray(512)
        host = (N.GemmProblem * 1)(prob)
        N.call("hnn_gemm_tc_encode", op, ctypes.addressof(host), 1,
               ctypes.addressof((ctypes.c_char * 512).from_buffer(maps)))
        keep = torch.frombuffer(maps, dtype=torch.uint8).to(dev)
        prob.tmap_a, prob.tmap_b, prob.tmap_c = _ptr(keep), _ptr(keep) + 128, _ptr(keep) + 256
    t = _dev_table(N.GemmProblem, [prob], dev)
    r = np.zeros(1, STEP_DTYPE); r["active"] = 1; r["rows"] = rows
    cur = torch.from_numpy(r.view(np.uint8).copy()).to(dev)
    N.call("hnn_grouped_gemm", op, prec, _ptr(t), 1, -(-d["m"] // tm) * tiles_n, _ptr(cur), 0,
           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    if TIME:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            N.call("hnn_grouped_gemm", op, prec, _ptr(t), 1, -(-d["m"] // tm) * tiles_n, _ptr(cur), 0,
                   torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"  time op={op} prec={prec} {M}x{Nn}x{K}: {ms*1e3:.1f} us  {2*M*Nn*K/ms/1e9:.1f} TF/s")
    got = c.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref) / (np.abs(ref).max() + 1e-30)
    return float(err.max()), got, ref


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "bisect":
    TIME = True
    for shape in ((256, 2048, 2048), (2048, 2048, 256)):
        for dbg in (0,):
            print("dbg", dbg, "(1: no lo MMAs, 2: no conversion, 4: no stores, 8: no promotion)")
            run(0, 1, *shape, dbg=dbg)
    sys.exit(0)

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "trunc":
    for op in (0, 1, 2):
        for dbg in (0, 1):
            e, got, ref = run(op, 1, 256, 384, 784, dbg=dbg)
            print(f"op={op} raw-hi={dbg} maxrel={e:.3e}")
    sys.exit(0)

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "time":
    TIME = True
    for shape in ((256, 2048, 2048), (2048, 2048, 256), (256, 1024, 784), (4096, 4096, 256)):
        for op in (0, 1, 2):
            run(op, 1, *shape)
    sys.exit(0)

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "variants":
    for op in (1, 2):
        for dbg in range(4):
            e, got, ref = run(op, 1, 128, 128, 32, dbg=dbg)
            print(f"op={op} dbg={dbg} maxrel={e:.3e} got={got[0,:3].round(3).tolist()} ref={ref[0,:3].round(3).tolist()} got10={got[10,5]:.3f} ref10={ref[10,5]:.3f}")
    sys.exit(0)

if __name__ == "__main__":
    for op in (0, 1, 2):
        for (M, Nn, K) in ((128, 128, 32), (128, 128, 64), (256, 256, 784), (256, 384, 256), (384, 784, 256)):
            for prec in (0, 1):
                e, got, ref = run(op, prec, M, Nn, K)
                bad = np.argwhere(np.abs(got - ref) / (np.abs(ref).max()) > 1e-4)
                print(f"op={op} prec={prec} M={M} N={Nn} K={K} maxrel={e:.3e} nbad={len(bad)} first={bad[:3].tolist()}")
