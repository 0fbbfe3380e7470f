"""Can the HBM-bound optimizer run beside the smem-bound pair GEMM?  Times C3's last weight-gradient
GEMM on P CTA pairs, the multi-tensor Adam on G CTAs, and both on two streams at once.
usage: python tools/overlap_probe.py  (debug tool)"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench

torch.cuda.set_device(0)
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank("c3", 0, 1, torch.device("cuda", 0))
rows = bench.schedule(jobs, ds, 400)
bench.upload_perms(dev, jobs, ds)
dev.load_schedule(rows)
dev.train_steps(40, use_graph=True)
torch.cuda.synchronize()
plan = {l.label: l for l in dev.train_plan}
wg0, wg1, dg1, opt = plan["bwd0/dense/wgrad/tc2"], plan["bwd1/dense/wgrad/tc2"], plan["bwd1/dense/tc2"], dev.train_plan[-1]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, n=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def env(k, v):
    if v is None:
        os.environ.pop(k, None)
    else:
        os.environ[k] = str(v)


def both(gemms, pairs, grid):
    def fn():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        s2.wait_event(ev)
        env("HNN_TC2_PAIRS", pairs)
        for g in gemms:
            g.run(s1.cuda_stream)
        env("HNN_OPT_GRID", grid)
        opt.run(s2.cuda_stream)
        e1, e2 = torch.cuda.Event(), torch.cuda.Event()
        e1.record(s1)
        e2.record(s2)
        torch.cuda.current_stream().wait_event(e1)
        torch.cuda.current_stream().wait_event(e2)
    return fn


st = torch.cuda.current_stream().cuda_stream
print(f"optimizer {opt.nbytes / 1e9:.3f} GB")
for g in (None, 96, 64, 48, 36, 24, 16):
    env("HNN_OPT_GRID", g)
    t = timed(lambda: opt.run(st))
    print(f"adam grid {g or 148:>4}: {t:.3f} ms  {opt.nbytes / t / 1e6:.0f} GB/s  ({opt.nbytes / t / 1e6 / (g or 148):.1f} GB/s per CTA)")
env("HNN_OPT_GRID", None)
for p in (None, 64, 56, 48):
    env("HNN_TC2_PAIRS", p)
    print(f"pairs {p or 74:>3}: wg0 {timed(lambda: wg0.run(st)):.3f}  dg1 {timed(lambda: dg1.run(st)):.3f}  "
          f"wg1 {timed(lambda: wg1.run(st)):.3f} ms")
env("HNN_TC2_PAIRS", None)
serial = timed(lambda: (dg1.run(st), wg0.run(st), opt.run(st)))
print(f"serial dg1 + wg0 + adam: {serial:.3f} ms")
for p in (64, 56, 48):
    for order in ("gemm_first",):
        t = timed(both([dg1, wg0], p, 148 - 2 * p))
        print(f"concurrent pairs {p} + adam grid {148 - 2 * p}: {t:.3f} ms")
env("HNN_TC2_PAIRS", None)
env("HNN_OPT_GRID", None)
