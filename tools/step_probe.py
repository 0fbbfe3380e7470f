"""Per-launch timing of one C3 step, three ways (debug / evidence tool):
   (1) eager step with events between launches, (2) each launch repeated alone x10, (3) graph replay."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2408_01331_b200 import _native as N

torch.cuda.set_device(0)
dev_t = torch.device("cuda", 0)
workload = sys.argv[1] if len(sys.argv) > 1 else "c3"
jobs, hy, dev, ddev, meta, ds, comm = bench.build_rank(workload, 0, 1, dev_t)
rows = bench.schedule(jobs, meta, 200)
bench.upload_perms(dev, jobs, meta)
dev.load_schedule(rows)
dev.train_steps(3, use_graph=False)
torch.cuda.synchronize()
per = bench.kernel_profile(dev, 5)
s = torch.cuda.current_stream()
alone = []
for launch in dev.train_plan:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        launch.run(s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    alone.append(e0.elapsed_time(e1) / 10)
dev.load_schedule(rows)
dev.train_steps(3, use_graph=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
dev.train_steps(20, use_graph=True)
e1.record()
torch.cuda.synchronize()
print(f"graph step {e0.elapsed_time(e1)/20:.3f} ms; eager sum {per.sum():.3f} ms; alone sum {sum(alone):.3f} ms")
for l, a, b in zip(dev.train_plan, per, alone):
    work = f"{l.flops/1e9:.2f} GF -> {l.flops/a/1e9:.1f} TF/s" if l.flops else f"{l.nbytes/1e6:.1f} MB -> {l.nbytes/a/1e6:.0f} GB/s"
    print(f"{l.label:28s} in-step {a:.3f} ms  alone {b:.3f} ms  {work}")
