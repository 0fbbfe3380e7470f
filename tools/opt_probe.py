"""Why is the optimizer 2x slower next to other kernels? (debug tool)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2408_01331_b200 import _native as N

torch.cuda.set_device(0)
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank("c3", 0, 1, torch.device("cuda", 0))
meta = ds
rows = bench.schedule(jobs, meta, 400)
bench.upload_perms(dev, jobs, meta)
dev.load_schedule(rows)
dev.train_steps(3, use_graph=False)
torch.cuda.synchronize()
st = torch.cuda.current_stream().cuda_stream
opt, gather = dev.train_plan[-1], dev.train_plan[0]
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")


def one(label, pre, n=10):
    tot = 0.0
    for _ in range(n):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        opt.run(st)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    print(f"{label:40s} optimizer {tot / n:.3f} ms")


one("after optimizer", lambda: opt.run(st))
one("after gather", lambda: gather.run(st))
one("after 512MB memset (L2 flush)", lambda: flush.zero_())
one("after step_begin (counter advances)", lambda: N.call("hnn_step_begin", int(dev.sched.data_ptr()),
                                                         int(dev.counter.data_ptr()), int(dev.cur.data_ptr()),
                                                         dev.n, st))
one("after fwd0", lambda: dev.train_plan[1].run(st))
one("nothing before", lambda: None)
