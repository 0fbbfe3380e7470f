"""Per-launch times of one C3 step for a given library build (debug tool).
usage: python tools/plan_times.py [path/to/libhnn_b200.so] [workload] [R/N: rank R's shard of an N-GPU run]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_01331_b200 import _native as N

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    N.load(Path(sys.argv[1]))
import torch

import bench

wl = sys.argv[2] if len(sys.argv) > 2 else "c3"
torch.cuda.set_device(0)
shard = tuple(int(v) for v in sys.argv[3].split("/")) if len(sys.argv) > 3 else None
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank(wl, 0, 1, torch.device("cuda", 0), shard)
meta = ds
rows = bench.schedule(jobs, meta, 200)
bench.upload_perms(dev, jobs, meta)
dev.load_schedule(rows)
dev.train_steps(3, use_graph=False)
torch.cuda.synchronize()
per = bench.kernel_profile(dev, 5)
for l, t in zip(dev.train_plan, per):
    fl = f"{l.flops / t / 1e9:8.1f} TF/s" if l.flops else f"{l.nbytes / t / 1e6:8.1f} GB/s"
    print(f"{l.label:32s} {t:.3f} ms {fl}")
print(f"sum {per.sum():.3f} ms")
