"""Time the multi-tensor optimizer of a library variant in the early and the converged C3 state.
usage: python tools/opt_variants.py path/to/libhnn_b200.so  (debug tool)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2408_01331_b200 import _native as N

N.load(Path(sys.argv[1]))
import torch

import bench

torch.cuda.set_device(0)
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank("c3", 0, 1, torch.device("cuda", 0))
meta = ds
rows = bench.schedule(jobs, meta, 400)
bench.upload_perms(dev, jobs, meta)
st = torch.cuda.current_stream().cuda_stream
opt = dev.train_plan[-1]


def timed(n=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        opt.run(st)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


dev.load_schedule(rows)
dev.train_steps(3, use_graph=True)
early = timed()
dev.load_schedule(rows)
dev.train_steps(60, use_graph=True)
late = timed()
gbs = opt.nbytes / 1e9
print(f"{sys.argv[1]}: early {early:.3f} ms ({gbs / early * 1e3:.0f} GB/s)  converged {late:.3f} ms ({gbs / late * 1e3:.0f} GB/s)")
