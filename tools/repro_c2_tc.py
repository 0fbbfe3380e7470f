"""Run one LeNet step launch by launch with a sync after each (debug tool)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench

torch.cuda.set_device(0)
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank("c2", 0, 1, torch.device("cuda", 0))
meta = ds
rows = bench.schedule(jobs, meta, 20)
bench.upload_perms(dev, jobs, meta)
dev.load_schedule(rows)
from paper_2408_01331_b200 import _native as N

st = torch.cuda.current_stream().cuda_stream
N.call("hnn_step_begin", int(dev.sched.data_ptr()), int(dev.counter.data_ptr()), int(dev.cur.data_ptr()), dev.n, st)
for l in dev.train_plan:
    print(l.label, flush=True)
    l.run(st)
    torch.cuda.synchronize()
print("ok")
