"""Wait-cycle breakdown of the CTA-pair GEMM (build with -DHNN_TC2_TRACE; debug tool).
usage: python tools/tc2_trace.py path/to/trace/libhnn_b200.so"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_2408_01331_b200 import _native as N

lib = N.load(Path(sys.argv[1]))
import torch

import bench

torch.cuda.set_device(0)
wl = sys.argv[2] if len(sys.argv) > 2 else "c3"
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank(wl, 0, 1, torch.device("cuda", 0))
meta = ds
rows = bench.schedule(jobs, meta, 200)
bench.upload_perms(dev, jobs, meta)
dev.load_schedule(rows)
dev.train_steps(3, use_graph=False)
torch.cuda.synchronize()
buf = np.zeros(296 * 16, dtype=np.uint64)
fn = lib.hnn_debug_tc2_trace
fn.argtypes = [C.c_void_p, C.c_int]
st = torch.cuda.current_stream().cuda_stream
for launch in dev.train_plan:
    if not launch.label.endswith(("/tc2", "/bf16")):
        continue
    fn(buf.ctypes.data, 1)
    reps = 5
    for _ in range(reps):
        launch.run(st)
    torch.cuda.synchronize()
    fn(buf.ctypes.data, 1)
    t = buf.reshape(296, 16)[:148].astype(np.float64) / reps
    lead = t[0::2]
    tot = t[:, 15].mean()
    print(f"{launch.label:26s} CTA life {tot:9.0f} clk | MMA wait lo {lead[:, 0].mean():8.0f} acc {lead[:, 1].mean():8.0f}"
          f" | conv wait raw {t[:, 2].mean() / 2:8.0f} | TMA wait empty {t[:, 3].mean():8.0f}"
          f" | acc warps wait full {t[:, 4].mean() / 8:8.0f}")
    print(f"{'':26s} MMA issue {lead[:, 5].mean():8.0f} | acc promote {t[:, 6].mean() / 8:8.0f} epilogue {t[:, 7].mean() / 8:8.0f}"
          f" | end barrier (per warp) {t[:, 8].mean() / 12:8.0f} | life min/max {t[:, 15].min():.0f}/{t[:, 15].max():.0f}")
    print(f"{'':26s} acc tile_info {t[:, 9].mean() / 8:8.0f} | bias+tmem ld (bf16) {t[:, 10].mean() / 8:8.0f}")
