"""Tile widths / K splits / tile counts of every pair-GEMM launch of a (sharded) workload's step (debug tool).
usage: python tools/tile_dump.py WORKLOAD [R/N]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2408_01331_b200 import _native as N

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
shard = tuple(int(v) for v in sys.argv[2].split("/")) if len(sys.argv) > 2 else None
torch.cuda.set_device(0)
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank(wl, 0, 1, torch.device("cuda", 0), shard)
for l in dev.train_plan:
    if l.entry != "hnn_grouped_gemm" or l.args[1] not in (N.PREC_3XTF32_PAIR, N.PREC_BF16_PAIR):
        continue
    n = l.args[3]
    raw = l.table.cpu().numpy().tobytes()[: n * C.sizeof(N.GemmProblem)]
    probs = (N.GemmProblem * n).from_buffer_copy(raw)
    print(l.label, "tiles", l.args[4], [(p.m, p.n, p.k, p.tile_n, p.ksplit, p.tiles_n) for p in probs])
