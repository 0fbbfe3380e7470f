"""Host data-loader throughput on this box: hnn_host_gather_batch for one C3 step at several thread
counts, and the pinned H2D copy of the same bytes (debug tool)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2408_01331_b200.train import HostBatchLoader

print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
torch.cuda.set_device(0)
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank("c3", 0, 1, torch.device("cuda", 0))
rows = bench.schedule(jobs, ds, 40)
for th in (1, 2, 4, 8, 12, 16):
    ld = HostBatchLoader(hy, {j.job_id: ds for j in jobs}, rows, threads=th)
    asm = ld.asm
    x, y = ld.bufs[0]
    perms = {m: asm.perm(dev.slots[m], 0) for m in range(dev.n)}
    its = [asm.items(x, y, rows[t], perms) for t in range(8)]
    asm.gather(its[0], th)
    t0 = time.perf_counter()
    for it in its:
        asm.gather(it, th)
    dt = (time.perf_counter() - t0) / len(its)
    nbytes = dev.batch_arena.numel() * 4
    print(f"threads {th:2d}: gather {dt * 1e3:.3f} ms/step  {nbytes / dt / 1e9:.1f} GB/s")
    ld.close()
sx = torch.empty_like(dev.batch_arena)
x = torch.zeros(dev.batch_arena.numel(), dtype=torch.float32).pin_memory()
sx.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    sx.copy_(x, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 20
print(f"H2D pinned {x.numel() * 4 / 1e6:.1f} MB: {dt * 1e3:.3f} ms  {x.numel() * 4 / dt / 1e9:.1f} GB/s")
