"""Optimizer duration in-step vs alone, after each preceding launch (debug tool)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2408_01331_b200 import _native as N

torch.cuda.set_device(0)
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank("c3", 0, 1, torch.device("cuda", 0))
meta = ds
rows = bench.schedule(jobs, meta, 400)
bench.upload_perms(dev, jobs, meta)
dev.load_schedule(rows)
dev.train_steps(5, use_graph=True)
dev.train_steps(50, use_graph=True)
torch.cuda.synchronize()
dev.load_schedule(rows)
per = bench.kernel_profile(dev, 5)
for l, t in zip(dev.train_plan, per):
    print(f"{l.label:32s} {t:.3f}")
st = torch.cuda.current_stream().cuda_stream
opt = dev.train_plan[-1]


def timed(pre, n=5):
    tot = 0
    for _ in range(n):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        opt.run(st)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / n


print("opt alone", timed(lambda: None))
for i, l in enumerate(dev.train_plan[:-1]):
    print(f"after {l.label:28s} {timed(lambda: l.run(st)):.3f}")
print("after full eager prefix", timed(lambda: [x.run(st) for x in dev.train_plan[:-1]]))
cur = dev.cur.cpu().numpy()
print(cur[:4])

# value classes of the optimizer inputs in this (slow) state
def classes(name, t):
    x = t.float()
    a = x.abs()
    tiny = torch.finfo(torch.float32).tiny
    print(f"{name}: n={x.numel()} zero={int((x == 0).sum())} denorm={int(((a > 0) & (a < tiny)).sum())} "
          f"nonfinite={int((~torch.isfinite(x)).sum())} absmin_nz={float(a[a > 0].min()) if (a > 0).any() else 0:.3e} absmax={float(a.max()):.3e}")


for nm in ("params", "grads", "m1", "m2"):
    classes(nm, getattr(dev, nm))
row = dev.cur.cpu().numpy()[0]
print("row", row)
