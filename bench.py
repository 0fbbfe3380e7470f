"""Benchmark: aggregate train samples/s of N merged models on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c2|c4|c5|c1] [--impl reference]

``--gpus N`` with N > 1 outside torchrun re-launches itself under
``torch.distributed.run`` (one process per GPU, NCCL); under torchrun the ranks come from
RANK / LOCAL_RANK / WORLD_SIZE.

Default workload: C3 (BASELINE.json configs[2]) — 32 heterogeneous MLPs 784-h-h-10,
h_i = 128*(1 + i mod 16), Adam lr 1e-3, batch 256, synthetic MNIST-shaped blob data
(60,000 x 784), the 32 models IN TOTAL sharded by model identity over the N GPUs with
``parallel.shard_jobs`` (LPT by FLOP/step: strong scaling).  C5 is 32 models per GPU (256 over
8), C4 4 per GPU (32 over 8), C2 8 LeNet-5 per GPU, C1 2 MLPs per GPU: weak scaling.  No gradient
collective exists (sub-models share nothing); NCCL broadcasts the dataset once and carries the
max-over-ranks timing.

One "step" = one lockstep optimizer step of every model of the rank on its next batch.
  value    device-resident throughput: inputs already in HBM, CUDA events around exactly K
           graph-replayed steps, max over ranks; the K-step region is repeated R times
           (R = enough repeats for >= 1 s of timed steps) and the median repeat is reported.
  e2e      the public host-fed API (train.HostFedStepper over train.HostBatchLoader): host
           threads gather every step's batches from the host datasets (the reference's
           store.batches work) into pinned buffers, each step copies them H2D and reads the
           per-model losses back; CUDA events around K steps, max over ranks.
  roofline the kernel FAMILY with the largest summed share of an eager step, each launch timed
           with CUDA events on its stream; traffic = ncu dram bytes of that family per step from
           the committed capture profiles/*/traffic_<workload>.json (null when absent).
  cpu_baseline the reference algorithm (the numpy oracle port) on the host cores, bounded sample:
           median of 5 repeats x 20 steps per model (one process per core).
--impl reference runs only that CPU arm (rank 0) and prints its own line with the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

METRIC = "Aggregate train samples/s over N merged models"
UNIT = "samples/s"
WORKLOADS = {
    "c3": "C3: 32 heterogeneous MLPs 784-h-h-10 (h=128*(1+i%16)) in total, sharded by model identity over the "
          "GPUs, Adam lr 1e-3, batch 256, synthetic MNIST-shaped blob 60000x784",
    "c2": "C2: 8 LeNet-5 per GPU, SGD lr 0.01, batch 128, synthetic CIFAR-shaped 50000x3x32x32",
    "c5": "C5: 32 MLP 784-256-10 per GPU (256 over 8), SGD lr 10^(-3+2i/255), batch 64, MNIST-shaped blob",
    "c1": "C1: 2 MLP 784-256-10 per GPU, SGD lr 0.01/0.05, batch 64, MNIST-shaped blob",
    "c4": "C4: 4 CNNs per GPU (32 over 8): ResNet-18-plain, VGG-11-noBN, 2 LeNet-5; SGD lr 1e-3, batch 128, "
          "bf16 tensor-core convs, synthetic CIFAR-shaped 50000x3x32x32",
}
MODELS_PER_GPU = {"c2": 8, "c5": 32, "c1": 2, "c4": 4}
C3_TOTAL = 32
# the fp32 GEMMs run as 3xTF32: 3 tcgen05 kind::tf32 MMAs per useful product; measured tf32
# issue rate 1070 TF/s (profiles/r01/mma_rate_micro.txt, cta_group::2 256x256x8) -> 357 useful
TF32_RATE = 1070.2
TRIPLE_TF32_PEAK = round(TF32_RATE / 3, 1)


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_dataset(workload):
    from paper_2408_01331_b200 import zoo

    if workload in ("c2", "c4"):
        return zoo.image_dataset()
    return zoo.blob_dataset()


def workload_jobs(workload, ds, world):
    """Every job of the workload at world size N (global model ids)."""
    from paper_2408_01331_b200 import zoo

    if workload == "c3":
        return zoo.config_jobs("c3", ds, count=C3_TOTAL)
    return zoo.config_jobs(workload, ds, count=MODELS_PER_GPU[workload] * world)


def bench_config(workload, jobs, world):
    """The config dict both arms print (identical keys and values)."""
    return {"workload": WORKLOADS[workload], "models": len(jobs),
            "global_batch": int(sum(j.hypers.batch_size for j in jobs)),
            "parallelism": f"model-identity sharding over {world} GPU(s) (parallel.shard_jobs, LPT by FLOP/step)",
            "l2": "per-step working set (params + grads + optimizer state + activations) exceeds the 126 MB L2; "
                  "no flush"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- CPU arm


_CPU_DATA = {}


def _cpu_worker(args):
    """Reference algorithm (oracle port) for one model: `steps` batches from its epoch-0 order.

    The dataset is inherited through fork (module global), never pickled."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits

    import oracle

    graph, seed, lr, opt, batch, steps = args
    xs, ys, digest = _CPU_DATA["x"], _CPU_DATA["y"], _CPU_DATA["digest"]
    with threadpool_limits(1):
        params = oracle.init_model(graph, seed)
        o = oracle.OracleOptimizer(opt)
        perm = oracle.keyed_permutation(xs.shape[0], "shuffle", digest, seed, 0)
        t0 = time.perf_counter()
        done = 0
        for b in range(steps):
            idx = perm[b * batch:(b + 1) * batch]
            oracle.train_step(graph, params, xs[idx], ys[idx], o, lr)
            done += idx.size
        return done, time.perf_counter() - t0


def cpu_baseline(jobs, ds, steps_per_model, repeats=5):
    """Aggregate samples/s of the reference algorithm over all host cores: one process per core
    (the SURVEY 8(d) "embarrassingly parallel" plan (ii)), each model training `steps_per_model`
    batches of its epoch-0 order with the store.batches gather inside the timed loop.

    Per repeat: samples / (sum of per-model step times / processes), i.e. the per-model work
    packed onto the cores.  Reported: the median of `repeats` repeats."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    procs = min(cores, len(jobs))
    _CPU_DATA.update(x=ds.train_x, y=ds.train_y, digest=ds.content_hash)
    work = [(j.graph, j.hypers.seed, j.hypers.learning_rate, j.hypers.optimizer, j.hypers.batch_size,
             steps_per_model) for j in jobs]
    ctx = mp.get_context("fork")
    values, walls = [], []
    with ctx.Pool(procs) as pool:
        for _ in range(repeats):
            t0 = time.perf_counter()
            res = pool.map(_cpu_worker, work, chunksize=1)
            walls.append(time.perf_counter() - t0)
            samples = sum(r[0] for r in res)
            busy = sum(r[1] for r in res)
            values.append(samples / (busy / procs))
    med = float(np.median(values))
    return {"value": round(med, 2), "unit": UNIT, "cores": procs, "kind": "port",
            "cpu": f"{cpu_model()} ({cores} cores visible)",
            "repeats": [round(v, 1) for v in values],
            "sample": f"median of {repeats} repeats; each: {steps_per_model} steps x {len(jobs)} models of the "
                      f"workload through the oracle's numpy restatement of hybridnn run_batch + store.batches "
                      f"gather, {procs} processes, 1 BLAS thread each; {samples} samples per repeat, "
                      f"{busy:.1f} core-seconds, {float(np.median(walls)):.1f}s wall"}


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    def __init__(self, index=0):
        self.index, self.proc, self.path = index, None, Path(f"/tmp/hnn_clocks_{os.getpid()}.csv")

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = [r.split(", ") for r in self.path.read_text().strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        # samples under load: the sampler runs for the whole timed region (>= 1 s of steps)
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------- GPU arm


def build_rank(workload, rank, world, device, shard_of=None):
    """This rank's jobs (model-identity shard of the workload), hybrid, device dataset, plans."""
    from paper_2408_01331_b200 import merge
    from paper_2408_01331_b200.parallel import RankGroup, shard_jobs

    comm = RankGroup(rank, world, device) if world > 1 else None
    # every rank keeps a host copy for the host-fed (e2e) arm; HBM copies come from rank 0's broadcast
    ds = make_dataset(workload)
    if comm is not None:
        ddev, _ = comm.share_dataset(ds if rank == 0 else None, device)
    else:
        from paper_2408_01331_b200.runtime import DeviceDataset

        ddev = DeviceDataset(ds, device)
    all_jobs = workload_jobs(workload, ds, world if shard_of is None else shard_of[1])
    jobs = shard_jobs(all_jobs, world)[rank] if shard_of is None else shard_jobs(all_jobs, shard_of[1])[shard_of[0]]
    hy = merge(jobs)
    # C4 is specified on bf16 tensor cores (BASELINE.json configs[3]); the other configs are fp32
    dev = hy.materialize(device, conv_precision="bf16" if workload == "c4" else "f32")
    dev.bind_datasets([ddev] * dev.n, ddev.n_train)
    dev.build_plans()
    return all_jobs, jobs, hy, dev, ddev, ds, comm


def schedule(jobs, meta, steps):
    """Rows for `steps` lockstep steps from epoch 0 (wrapping the epoch-0 order past its end)."""
    from paper_2408_01331_b200.runtime import STEP_DTYPE
    from paper_2408_01331_b200.train import _bias
    from paper_2408_01331_b200.optim import lr_at_epoch

    rows = np.zeros((steps, len(jobs)), dtype=STEP_DTYPE)
    n = meta.sample_count
    for m, j in enumerate(jobs):
        B = j.hypers.batch_size
        spe = -(-n // B)
        lr = float(np.float32(lr_at_epoch(j.hypers.learning_rate, (), 0)))
        for t in range(steps):
            b = t % spe
            b1, b2 = _bias(t + 1)
            rows[t, m] = (1, min(B, n - b * B), b * B, 0, b, t + 1, lr, b1, b2, (0, 0, 0))
    return rows


def upload_perms(dev, jobs, meta):
    from paper_2408_01331_b200 import rng

    for m, j in enumerate(jobs):
        dev.perm_upload(m, rng.permutation(meta.sample_count, "shuffle", meta.content_hash, j.hypers.seed, 0))


def kernel_profile(dev, steps):
    """Average duration of every launch of an eager step (CUDA events on the launch stream)."""
    import torch

    from paper_2408_01331_b200 import _native as N

    stream = torch.cuda.current_stream()
    plan = dev.train_plan
    totals = np.zeros(len(plan))
    for _ in range(steps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(plan) + 1)]
        N.call("hnn_step_begin", int(dev.sched.data_ptr()), int(dev.counter.data_ptr()), int(dev.cur.data_ptr()),
               dev.n, stream.cuda_stream)
        evs[0].record(stream)
        for i, launch in enumerate(plan):
            launch.run(stream.cuda_stream)
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        totals += [evs[i].elapsed_time(evs[i + 1]) for i in range(len(plan))]
    return totals / steps  # ms


def traffic_record(workload):
    """ncu DRAM bytes per step by kernel family from the newest committed capture, or None."""
    found = sorted(REPO.glob(f"profiles/r*/traffic_{workload}.json"))
    if not found:
        return None, None
    return json.loads(found[-1].read_text()), str(found[-1].relative_to(REPO))


def roofline(dev, per_launch_ms, workload):
    """The kernel family with the largest summed share of the step, against its roofline.

    achieved = the family's algorithmic bytes (or useful FLOPs) per step / its summed launch time;
    tensor-core families use their instruction's measured peak (3xTF32: tf32 rate / 3; bf16:
    MEASURED_PEAKS burst, the kernels are timed alone), HBM families the measured copy bandwidth."""
    hbm, tf_burst, tf_sus, kind = peaks()
    fams = {}
    for launch, ms in zip(dev.train_plan, per_launch_ms):
        f = fams.setdefault(launch.family, {"ms": 0.0, "flops": 0, "nbytes": 0, "launches": 0, "tensor": False})
        f["ms"] += ms
        f["flops"] += launch.flops
        f["nbytes"] += launch.nbytes
        f["launches"] += 1
        f["tensor"] = f["tensor"] or launch.family.startswith("gemm/tc2") or launch.family.startswith("gemm/tc")
    total = float(per_launch_ms.sum())

    def frac_of(fname, fam):  # each family against its own roofline (reported next to the dominant one)
        sec_ = fam["ms"] / 1e3
        if fam["tensor"] and fam["flops"]:
            pk = tf_burst if fname.endswith("bf16") else TRIPLE_TF32_PEAK
            return {"bound": "tensor", "achieved": round(fam["flops"] / sec_ / 1e12, 2), "peak": pk, "unit": "TFLOP/s",
                    "frac": round(fam["flops"] / sec_ / 1e12 / pk, 4), "share_of_step": round(fam["ms"] / total, 4)}
        if fam["nbytes"]:
            return {"bound": "hbm", "achieved": round(fam["nbytes"] / sec_ / 1e9, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(fam["nbytes"] / sec_ / 1e9 / hbm, 4), "share_of_step": round(fam["ms"] / total, 4)}
        return None

    name, f = max(fams.items(), key=lambda kv: kv[1]["ms"])
    sec = f["ms"] / 1e3
    rec, src = traffic_record(workload)
    traffic = None
    if rec is not None and name in rec.get("families", {}):
        traffic = rec["families"][name]["dram_bytes_per_step"]
    shares = {k: round(v["ms"] / total, 4) for k, v in sorted(fams.items(), key=lambda kv: -kv[1]["ms"])}
    others = {k: frac_of(k, v) for k, v in sorted(fams.items(), key=lambda kv: -kv[1]["ms"])[:4] if k != name}
    out = {"kernel": name, "launches_per_step": f["launches"], "share_of_step": round(f["ms"] / total, 4),
           "ms_per_step": round(f["ms"], 4), "family_shares": shares,
           "other_families": {k: v for k, v in others.items() if v is not None},
           "traffic_unit": "DRAM bytes per step of this family (ncu --set full, one eager step)",
           "traffic_source": src}
    if f["tensor"] and f["flops"]:
        bf16 = name.endswith("bf16")
        peak = tf_burst if bf16 else TRIPLE_TF32_PEAK
        achieved = f["flops"] / sec / 1e12
        out.update({"bound": "tensor", "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic,
                    "algorithmic": f"{f['flops']} useful FLOP per step (2*m*n*k per problem)",
                    "peak_source": (f"{kind} bf16 burst (MEASURED_PEAKS.json)" if bf16 else
                                    f"3xTF32 useful-FLOP ceiling = measured tf32 tcgen05 rate {TF32_RATE} TF/s / 3 "
                                    "(profiles/r01/mma_rate_micro.txt)")})
    elif f["flops"] and not f["nbytes"]:
        # CUDA-core FP32 kernels (the direct convolutions of LeNet-class layers): the FFMA roofline,
        # nominal (148 SMs x 128 FMA lanes x 2 FLOP x the 1965 MHz max clock; no measured figure)
        peak = round(148 * 128 * 2 * 1.965e9 / 1e12, 1)
        achieved = f["flops"] / sec / 1e12
        out.update({"bound": "fp32-fma", "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic,
                    "algorithmic": f"{f['flops']} useful FLOP per step (2*B*OH*OW*F*C*k*k per conv)",
                    "peak_source": "nominal FFMA peak, 148 SMs x 128 lanes x 2 x 1.965 GHz"})
    else:
        achieved = f["nbytes"] / sec / 1e9
        out.update({"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(achieved / hbm, 4), "traffic": traffic,
                    "algorithmic": f"{f['nbytes']} bytes per step (SURVEY 8(d) per-unit bytes x units)",
                    "peak_source": f"{kind} HBM copy (MEASURED_PEAKS.json)"})
    return out


def _reduce(x, world, device, op):
    """All-reduce one scalar over the ranks (NCCL on the device; gloo on a host tensor)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = device if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def _max_over_ranks(x, world, device):
    import torch.distributed as dist

    return _reduce(x, world, device, dist.ReduceOp.MAX)


def _sum_over_ranks(x, world, device):
    import torch.distributed as dist

    return _reduce(x, world, device, dist.ReduceOp.SUM)


def gpu_arm(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # HNN_BENCH_ONE_GPU=1: every rank on cuda:0 with gloo (exercises the multi-rank bench on a
    # one-GPU box; NCCL refuses two ranks on one device).  Never set for a measurement.
    one_gpu = os.environ.get("HNN_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
    shard_of = tuple(int(v) for v in args.shard.split("/")) if args.shard else None
    all_jobs, jobs, hy, dev, ddev, ds, comm = build_rank(args.workload, rank, world, device, shard_of)
    meta = ds
    upload_perms(dev, jobs, meta)
    sync = lambda: (torch.cuda.synchronize(), dist.barrier() if world > 1 else None)

    # ---- warm-up (graph capture) and a calibration of the step time
    dev.load_schedule(schedule(jobs, meta, args.warmup))
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev.train_steps(1, use_graph=True)
    c0.record()
    dev.train_steps(args.warmup - 1, use_graph=True)
    c1.record()
    torch.cuda.synchronize()
    est = _max_over_ranks(c0.elapsed_time(c1) / max(args.warmup - 1, 1), world, device)
    repeats = int(min(max(1, np.ceil(args.min_seconds * 1e3 / (args.steps * est))), 1000))

    # ---- device-resident timed run: `repeats` x exactly K graph-replayed steps
    rows = schedule(jobs, meta, 1 + repeats * args.steps + 8)
    samples_rank = [int(rows["rows"][1 + r * args.steps: 1 + (r + 1) * args.steps].sum()) for r in range(repeats)]
    dev.load_schedule(rows)
    dev.train_steps(1, use_graph=True)  # (re)capture on the new schedule buffer, untimed
    times = []
    with ClockSampler(local) as clocks:
        for r in range(repeats):
            sync()
            start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record()
            dev.train_steps(args.steps, use_graph=True)
            stop.record()
            torch.cuda.synchronize()
            times.append(_max_over_ranks(start.elapsed_time(stop), world, device))
    samples_all = [_sum_over_ranks(s, world, device) for s in samples_rank]
    med = int(np.argsort(times)[len(times) // 2])
    ms = times[med]
    value = samples_all[med] / (ms / 1e3)

    # ---- per-kernel timing for the roofline (eager, same schedule)
    dev.load_schedule(rows)
    per_launch = kernel_profile(dev, min(5, args.steps))
    roof = roofline(dev, per_launch, args.workload)

    # ---- e2e through the host-fed public API, host batch assembly included
    from paper_2408_01331_b200.train import HostBatchLoader, HostFedStepper

    e_rows = schedule(jobs, meta, args.warmup + args.steps + 8)
    loader = HostBatchLoader(hy, {j.job_id: ds for j in jobs}, e_rows, threads=args.loader_threads)
    stepper = HostFedStepper(hy, {j.job_id: ds for j in jobs})
    dev.load_schedule(e_rows)
    for i in range(args.warmup):
        stepper.step(loader.next())
    stepper.finish()
    sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        stepper.step(loader.next())
    stepper.finish()
    e1.record()
    torch.cuda.synchronize()
    loader.close()
    ems = _max_over_ranks(e0.elapsed_time(e1), world, device)
    e_samples = _sum_over_ranks(int(e_rows["rows"][args.warmup:args.warmup + args.steps].sum()), world, device)
    e2e = {"value": round(e_samples / (ems / 1e3), 1), "unit": UNIT,
           "h2d_bytes_per_step": stepper.h2d_bytes_per_step, "d2h_bytes_per_step": stepper.d2h_bytes_per_step,
           "ms_per_step": round(ems / args.steps, 4),
           "api": "paper_2408_01331_b200.train.HostFedStepper.step(HostBatchLoader.next()): host threads gather "
                  f"each step's batches from the host dataset ({args.loader_threads} threads, store.batches order) "
                  "into pinned memory -> one H2D copy per arena -> the step's kernels -> losses D2H"}

    peak_alloc = torch.cuda.max_memory_allocated(device)
    n_models = len(jobs)
    from paper_2408_01331_b200 import memory

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong" if args.workload == "c3" else "weak", "vs_baseline": None,
        "dtype": "bf16 conv operands, f32 accumulate / dense / optimizer" if args.workload == "c4" else "f32",
        "data": "synthetic (keyed-Philox blob/image generators of the reference), random-init weights from the "
                "reference's keyed init",
        "config": bench_config(args.workload, all_jobs, world),
        "repeats": repeats, "timed_s": round(sum(times) / 1e3, 3),
        **({"diagnostic_shard": args.shard, "shard_models": len(jobs)} if args.shard else {}),
        "repeat_ms": [round(t, 3) for t in times],
        "hbm_bytes_per_model": int((peak_alloc - ddev.nbytes) / n_models + ddev.nbytes / n_models),
        "reference_modeled_bytes_per_model": memory.reference_model_bytes(jobs),
        "gpu_launches": dev.launch_count() * args.steps,
        "e2e": e2e, "roofline": roof, "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(all_jobs, ds, args.cpu_steps, args.cpu_repeats)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    ds = make_dataset(args.workload)
    all_jobs = workload_jobs(args.workload, ds, world)
    # warmup: one short pass so page-ins / pool start-up are not timed
    if args.warmup:
        cpu_baseline(all_jobs[:2], ds, 1, repeats=1)
    base = cpu_baseline(all_jobs, ds, args.cpu_steps, args.cpu_repeats)
    line = {"metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong" if args.workload == "c3" else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": bench_config(args.workload, all_jobs, world),
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run, one rank per GPU."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=20)
    ap.add_argument("--cpu-repeats", type=int, default=5)
    ap.add_argument("--min-seconds", type=float, default=1.0)
    ap.add_argument("--loader-threads", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    # diagnostic: time only shard R of an N-GPU run on this one GPU (per-GPU work at N GPUs)
    ap.add_argument("--shard", default=None, metavar="R/N")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        sys.exit(_relaunch(args))
    if world and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
