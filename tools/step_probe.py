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
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank(workload, 0, 1, dev_t)
meta = ds
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
g_ms = e0.elapsed_time(e1) / 20
dev.load_schedule(rows)
dev.train_steps(3, use_graph=False)
torch.cuda.synchronize()
e0.record()
dev.train_steps(20, use_graph=False)
e1.record()
torch.cuda.synchronize()
def timed(fn, n=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


st = torch.cuda.current_stream().cuda_stream
dev.load_schedule(rows)
sb = timed(lambda: N.call("hnn_step_begin", int(dev.sched.data_ptr()), int(dev.counter.data_ptr()),
                          int(dev.cur.data_ptr()), dev.n, st))
dev.load_schedule(rows)
dev.run_plan([])
plan_only = timed(lambda: [l.run(st) for l in dev.train_plan])
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    for l in dev.train_plan:
        l.run(st)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"step_begin alone {sb*1e3:.1f} us; plan without step_begin {plan_only:.3f} ms; host issue {1e3*(t1-t0)/20:.3f} ms/step, drain {1e3*(t2-t1):.3f} ms")
# per-step events, host far ahead: steps issued back to back, events only around each whole step
evs = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
dev.load_schedule(rows)
torch.cuda.synchronize()
for i in range(20):
    evs[i].record()
    dev.run_plan(dev.train_plan)
evs[20].record()
torch.cuda.synchronize()
print("per-step ms:", [round(evs[i].elapsed_time(evs[i+1]), 3) for i in range(20)][-3:])
for mode in ("timing-events", "plain-events", "sync-events"):
    marks = [torch.cuda.Event(enable_timing=(mode == "timing-events")) for _ in range(len(dev.train_plan))]
    def one():
        for l, m in zip(dev.train_plan, marks):
            l.run(st)
            m.record()
    dev.load_schedule(rows)
    print(mode, "step", round(timed(one), 3), "ms")
# which kernel pair slows down? time each consecutive pair back to back
pairs = []
opt = dev.train_plan[-1]
for a_, b_ in [(x, opt) for x in dev.train_plan[:-1]] + [(opt, dev.train_plan[0]), (opt, dev.train_plan[1])]:
    pairs.append((a_.label, b_.label, round(timed(lambda: (a_.run(st), b_.run(st)), 10), 3)))
print(pairs)
print(f"graph step {g_ms:.3f} ms; eager whole step {e0.elapsed_time(e1)/20:.3f} ms; eager per-launch sum {per.sum():.3f} ms; alone sum {sum(alone):.3f} ms")
for l, a, b in zip(dev.train_plan, per, alone):
    work = f"{l.flops/1e9:.2f} GF -> {l.flops/a/1e9:.1f} TF/s" if l.flops else f"{l.nbytes/1e6:.1f} MB -> {l.nbytes/a/1e6:.0f} GB/s"
    print(f"{l.label:28s} in-step {a:.3f} ms  alone {b:.3f} ms  {work}")
