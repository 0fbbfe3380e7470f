"""Lockstep training of a merged hybrid on the GPU — the hot path's host side.

Mirrors hybridnn.train (src/train.py:42-476): ``Trainer(hybrid, plan, jobs,
datasets, ...)`` with the same hooks and report types, ``evaluate``,
``train_standalone`` and checkpoints.  The difference is the schedule: the
reference runs one (job, epoch) slice at a time; here every live job steps
in lockstep, one grouped launch sequence per step for all of them
(SURVEY.md finding 3 — a job's trajectory does not depend on the order).

Per job the arithmetic is the reference's: the same keyed initial values and
epoch permutations, ``lr_at_epoch``, the optimizer step counter t, a
non-finite loss aborting only that job before its update
(src/train.py:239-243, 408-418), sample-weighted epoch curves accumulated in
float64 (:419-426) and the test split evaluated in order at completion
(:259-279, 429-446).  Schedule-dependent outputs (``completion_index``,
``executed``) follow the lockstep order instead of the plan's slice order.
"""
from __future__ import annotations

import os

import time
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from . import formats
from .errors import StateError, UnknownJobError
from .model import TrainingJob
from .optim import ADAM_BETA1, ADAM_BETA2, OptimizerState, lr_at_epoch
from .runtime import STEP_DTYPE, DeviceDataset
from .unify import HybridModel, merge, qualify, unqualify

F32 = np.float32


@lru_cache(maxsize=None)
def _bias(t: int) -> tuple:
    """Adam corrections for 1-based step t, evaluated like src/optim.py:75-76."""
    return float(F32(1.0 - ADAM_BETA1 ** t)), float(F32(1.0 - ADAM_BETA2 ** t))


# --------------------------------------------------------------------------- checkpoints


@dataclass
class Checkpoint:
    """One job's resumable state at an epoch boundary (src/train.py:42-99)."""

    job_id: str
    completed_epochs: int
    data_cursor: int
    optimizer_kind: str
    optimizer_step: int
    momentum: float
    params: dict
    slot_m: dict = field(default_factory=dict)
    slot_v: dict = field(default_factory=dict)
    slot_momentum: dict = field(default_factory=dict)

    _TAGS = (("p", "params"), ("m", "slot_m"), ("v", "slot_v"), ("mom", "slot_momentum"))

    def encode(self) -> bytes:
        """UNND v3 bytes, identical to the reference's for the same state (src/train.py:57-80):
        canonical JSON header {job_id, completed_epochs, data_cursor, optimizer{kind, step,
        momentum}}, then sections "p/", "m/", "v/", "mom/" + param id in sorted name order."""
        header = {"job_id": self.job_id, "completed_epochs": self.completed_epochs, "data_cursor": self.data_cursor,
                  "optimizer": {"kind": self.optimizer_kind, "step": self.optimizer_step, "momentum": self.momentum}}
        sections = {f"{tag}/{pid}": arr for tag, attr in self._TAGS for pid, arr in getattr(self, attr).items()}
        return formats.encode_checkpoint(header, sections, sorted(sections))

    @classmethod
    def decode(cls, blob: bytes) -> "Checkpoint":
        """Inverse of :meth:`encode` (src/train.py:82-99); unknown section tags are a StateError."""
        header, sections = formats.decode_checkpoint(blob)
        opt = header["optimizer"]
        out = cls(header["job_id"], int(header["completed_epochs"]), int(header["data_cursor"]), opt["kind"],
                  int(opt["step"]), float(opt.get("momentum", 0.0)), {})
        by_tag = {tag: getattr(out, attr) for tag, attr in cls._TAGS}
        for name, arr in sections.items():
            tag, _, pid = name.partition("/")
            if tag not in by_tag or not pid:
                raise StateError(f"unrecognized checkpoint section {name!r}")
            by_tag[tag][pid] = arr
        return out


def make_checkpoint(hybrid: HybridModel, job_id: str) -> Checkpoint:
    sub = hybrid.sub(job_id)
    params = {unqualify(job_id, k): v.copy() for k, v in hybrid.sub_params(job_id).items()}
    m1 = m2 = {}
    if hybrid.on_device(job_id):
        m1, m2 = hybrid.device.download_moments(sub.slot)
    else:
        opt = sub.optimizer
        m1 = {unqualify(job_id, k): v.copy() for k, v in (opt.m1 or opt.velocity).items()}
        m2 = {unqualify(job_id, k): v.copy() for k, v in opt.m2.items()}
    opt = sub.optimizer
    adam = opt.kind == "adam"
    return Checkpoint(job_id, sub.completed_epochs, sub.completed_epochs, opt.kind, opt.step, opt.momentum, params,
                      slot_m=m1 if adam else {}, slot_v=m2 if adam else {},
                      slot_momentum=m1 if (not adam and opt.momentum) else {})


def restore_checkpoint(hybrid: HybridModel, ckpt: Checkpoint) -> None:
    """Load a checkpoint into the matching sub-model (src/train.py:102-149)."""
    sub = hybrid.sub(ckpt.job_id)
    expect = {unqualify(ckpt.job_id, pid) for pid in sub.param_ids()}
    if sorted(expect) != sorted(ckpt.params):
        raise StateError(f"checkpoint for {ckpt.job_id!r} does not match the submitted model: parameter sets differ")
    current = {unqualify(ckpt.job_id, k): v for k, v in hybrid.sub_params(ckpt.job_id).items()}
    for pid, arr in ckpt.params.items():
        if current[pid].shape != arr.shape:
            raise StateError(f"checkpoint shape {arr.shape} != model shape {current[pid].shape} for parameter {pid!r}")
    if sub.optimizer.kind != ckpt.optimizer_kind:
        raise StateError(f"checkpoint optimizer {ckpt.optimizer_kind!r} != job optimizer {sub.optimizer.kind!r}")
    hybrid.set_sub_params(ckpt.job_id, ckpt.params)
    opt = sub.optimizer
    opt.step, opt.momentum = ckpt.optimizer_step, ckpt.momentum
    q = lambda d: {qualify(ckpt.job_id, k): np.array(v, copy=True) for k, v in d.items()}
    if hybrid.on_device(ckpt.job_id):
        # the device copy is the truth: no host moments left behind to be re-uploaded later
        hybrid.device.upload_moments(sub.slot, ckpt.slot_m or ckpt.slot_momentum, ckpt.slot_v)
        opt.m1, opt.m2, opt.velocity = {}, {}, {}
    else:
        opt.m1, opt.m2, opt.velocity = q(ckpt.slot_m), q(ckpt.slot_v), q(ckpt.slot_momentum)
    sub.completed_epochs = ckpt.completed_epochs


# --------------------------------------------------------------------------- reports


@dataclass
class JobResult:
    job_id: str
    status: str = "training"
    slices_executed: int = 0
    completion_index: int | None = None
    epochs_completed: int = 0
    curve: list = field(default_factory=list)
    final_train_loss: float | None = None
    final_train_accuracy: float | None = None
    final_test_loss: float | None = None
    final_test_accuracy: float | None = None
    abort_reason: str | None = None
    wall_time: float = 0.0

    def to_dict(self, with_wall: bool = False) -> dict:
        out = {
            "job_id": self.job_id, "status": self.status, "slices_executed": self.slices_executed,
            "completion_index": self.completion_index, "epochs_completed": self.epochs_completed,
            "curve": [[e, l, a] for e, l, a in self.curve], "final_train_loss": self.final_train_loss,
            "final_train_accuracy": self.final_train_accuracy, "final_test_loss": self.final_test_loss,
            "final_test_accuracy": self.final_test_accuracy, "abort_reason": self.abort_reason,
        }
        if with_wall:
            out["wall_time"] = self.wall_time
        return out


@dataclass
class TrainReport:
    policy: str
    jobs: dict
    executed: list = field(default_factory=list)
    simulated_unified_time: float = 0.0
    simulated_baseline_time: float = 0.0
    memory_trace_ref: str | None = None
    wall_time: float = 0.0
    steps: int = 0             # lockstep device steps executed
    samples: int = 0           # training rows consumed across all jobs

    def to_dict(self, with_wall: bool = False) -> dict:
        out = {
            "policy": self.policy, "jobs": {j: r.to_dict(with_wall) for j, r in sorted(self.jobs.items())},
            "executed": [[j, e] for j, e in self.executed], "simulated_unified_time": self.simulated_unified_time,
            "simulated_baseline_time": self.simulated_baseline_time, "memory_trace_ref": self.memory_trace_ref,
        }
        if with_wall:
            out["wall_time"] = self.wall_time
        return out


# --------------------------------------------------------------------------- the trainer


class _Track:
    """Lockstep bookkeeping of one job."""

    def __init__(self, job, slot, dataset, epochs):
        self.job, self.slot, self.dataset, self.epochs = job, slot, dataset, list(epochs)
        hp = job.hypers
        self.batch = hp.batch_size
        self.n = dataset.sample_count
        self.spe = -(-self.n // self.batch)
        self.total = self.spe * len(self.epochs)
        self.opt_base = 0
        self.done = False

    def epoch_index(self, t):
        return t // self.spe


class Trainer:
    """Runs a plan over a hybrid, all live jobs in lockstep on the GPU.

    Hooks are the reference's (src/train.py:294-325).  Extra keyword options:
    ``use_graph`` (replay each step as a CUDA graph), ``use_tensor_cores``,
    ``device``, ``comm`` (a :class:`paper_2408_01331_b200.parallel.RankGroup`
    for multi-GPU dataset broadcast / metric gather), ``conv_precision``
    ("f32": 3xTF32 tensor-core convolutions, fp32 parity; "bf16": bf16 operands with fp32
    accumulation and fp32 master weights, the BASELINE C4 setting).
    """

    def __init__(self, hybrid: HybridModel, plan, jobs: list, datasets: dict, completion_sink=None,
                 pause_sink=None, pause_poll=None, step_observer=None, slice_observer=None, *,
                 use_graph: bool = True, use_tensor_cores: bool = True, device=None, comm=None,
                 loss_observer=None, fuse_optimizer: bool = True, keep_grads: bool = False,
                 conv_precision: str = "f32"):
        self.hybrid = hybrid
        self.conv_precision = conv_precision
        self.plan = plan
        jobs = [TrainingJob.coerce(j) for j in jobs]
        self.jobs = {j.job_id: j for j in jobs}
        self.datasets = datasets
        self.completion_sink, self.pause_sink, self.pause_poll = completion_sink, pause_sink, pause_poll
        self.step_observer, self.slice_observer = step_observer, slice_observer
        # loss_observer(job_id, step, loss, correct): per-step device losses (forces one-step windows)
        self.loss_observer = loss_observer
        self.use_graph, self.use_tc, self.device_name, self.comm = use_graph, use_tensor_cores, device, comm
        self.fuse_optimizer, self.keep_grads = fuse_optimizer, keep_grads
        self._pause_requests: set = set()
        self.results = {j.job_id: JobResult(job_id=j.job_id, epochs_completed=j.completed_epochs) for j in jobs}
        self.checkpoints: dict = {}
        self._executed: list = []
        self._exec_keys: list = []          # (lockstep step, job order) of each executed slice
        self._completion_keys: dict = {}
        self._local: set = set(self.jobs)
        self._device_data: dict = {}
        self.device = None
        for job_id in self.jobs:
            if job_id not in hybrid.sub_models:
                raise UnknownJobError(job_id)
            if job_id not in datasets:
                raise StateError(f"job {job_id!r}: dataset not resolved")

    def request_pause(self, job_id: str) -> None:
        if job_id not in self.jobs:
            raise UnknownJobError(job_id)
        status = self.results[job_id].status
        if status in ("complete", "aborted"):
            raise StateError(f"job {job_id!r} is already {status}")
        self._pause_requests.add(job_id)

    # ------------------------------------------------------------------ setup
    def _epochs_from_plan(self) -> dict:
        out = {jid: [] for jid in self.jobs}
        for s in self.plan.slices:
            if s.job_id in out:
                out[s.job_id].append(s.epoch)
        return out

    def _local_ids(self) -> list:
        """Jobs this process trains: all of them, or its model-identity shard (parallel.shard_jobs)."""
        if self.comm is None or self.comm.world == 1:
            return list(self.jobs)
        from .parallel import shard_jobs

        return [j.job_id for j in shard_jobs(list(self.jobs.values()), self.comm.world)[self.comm.rank]]

    def _device(self, local):
        """Materialise with this Trainer's options.  Single-process: every sub-model of the hybrid
        (jobs of other Trainers ride along untouched); sharded: only this rank's jobs."""
        return self.hybrid.materialize(self.device_name, use_tensor_cores=self.use_tc,
                                       fuse_optimizer=self.fuse_optimizer, keep_grads=self.keep_grads,
                                       conv_precision=self.conv_precision,
                                       local=None if self.comm is None else local)

    def _upload_datasets(self, dev) -> list:
        by_model = [None] * dev.n
        cache = self._device_data
        wanted = [self.datasets[s.job_id] for s in dev.slots if s.job_id in self.jobs]
        if self.comm is not None:
            missing = [d for d in wanted if d.content_hash not in cache]
            cache.update(self.comm.share_datasets(missing, dev.device))
        for ds in wanted:
            if ds.content_hash not in cache:
                cache[ds.content_hash] = DeviceDataset(ds, dev.device)
        for s in dev.slots:
            if s.job_id in self.jobs:
                by_model[s.index] = cache[self.datasets[s.job_id].content_hash]
        # models of the hybrid not trained by this Trainer borrow any dataset of the right shape
        for i, d in enumerate(by_model):
            if d is None:
                slot = dev.slots[i]
                match = [v for v in cache.values() if tuple(v.sample_shape) == tuple(slot.sample_shape)]
                if not match:
                    raise StateError(f"job {slot.job_id!r}: dataset not resolved")
                by_model[i] = match[0]
        return by_model

    def _prepare_device(self, local):
        dev = self._device(local)
        by_model = self._upload_datasets(dev)
        dev.bind_datasets(by_model, max(d.n_train for d in by_model))
        dev.build_plans()
        dev.reset_status()
        self.device = dev
        return dev

    # ------------------------------------------------------------------ run
    def run(self) -> TrainReport:
        started = time.perf_counter()
        epochs = self._epochs_from_plan()
        local = self._local_ids()
        self._local = set(local)
        # a resumed job may arrive with nothing left to do (src/train.py:339-341); its test
        # evaluation runs on the device, so the device is set up first, with this Trainer's options
        finished = [jid for jid in local if self.jobs[jid].completed_epochs >= self.jobs[jid].hypers.epochs]
        live = [jid for jid in local if jid not in finished and epochs[jid]]
        steps_run, samples = 0, 0
        if live or finished:
            dev = self._prepare_device(local)
        for jid in finished:
            self._complete(jid, key=(-1, self._order(jid)))
        # pause requests pending before the first slice apply immediately (src/train.py:343)
        self._apply_pauses()
        live = [jid for jid in live if self.results[jid].status == "training"]
        if live:
            tracks = {}
            for jid in live:
                sub = self.hybrid.sub(jid)
                tr = _Track(self.jobs[jid], sub.slot, self.datasets[jid], epochs[jid])
                tr.opt_base = sub.optimizer.step
                tracks[jid] = tr
            steps_run, samples = self._lockstep(dev, tracks)
        self._apply_pauses(force_all=True)
        if self.comm is not None and self.comm.world > 1:
            steps_run, samples = self._gather(local, steps_run, samples)
        report = TrainReport(self.plan.policy, self.results, executed=list(self._executed),
                             wall_time=time.perf_counter() - started, steps=steps_run, samples=samples)
        return report

    def _order(self, jid) -> int:
        return list(self.jobs).index(jid)

    def _gather(self, local, steps_run, samples) -> tuple:
        """Sharded run: all-gather every rank's job results, slice log and checkpoints, then
        broadcast each job's final state from its owner, so every rank returns the report (and
        holds the parameters) a single-process run over all jobs would have produced."""
        comm = self.comm
        mine = {
            "results": {jid: self.results[jid] for jid in local},
            "log": [(k, e) for k, e in zip(self._exec_keys, self._executed)],
            "completions": {jid: self._completion_keys[jid] for jid in local if jid in self._completion_keys},
            "checkpoints": {jid: c for jid, c in self.checkpoints.items() if jid in self._local},
            "state": {jid: (self.hybrid.sub(jid).optimizer.step, self.hybrid.sub(jid).completed_epochs)
                      for jid in local},
            "steps": steps_run, "samples": samples,
        }
        every = comm.all_gather_object(mine)
        owners, state, log = {}, {}, []
        for r, part in enumerate(every):
            for jid, res in part["results"].items():
                owners[jid] = r
                if r != comm.rank:
                    self.results[jid] = res
            state.update(part["state"])
            log += part["log"]
            self.checkpoints.update(part["checkpoints"])
        log.sort(key=lambda t: t[0])
        self._exec_keys = [k for k, _ in log]
        self._executed = [e for _, e in log]
        # completion_index = slices executed up to and including the job's last slice (lockstep order)
        for part in every:
            for jid, key in part["completions"].items():
                self.results[jid].completion_index = sum(1 for k in self._exec_keys if k <= key)
        comm.exchange_models(self.hybrid, owners, state)
        return max(p["steps"] for p in every), sum(p["samples"] for p in every)

    def _boundaries(self, tracks) -> list:
        pts = {0}
        for tr in tracks.values():
            pts.update(range(tr.spe, tr.total + 1, tr.spe))
        if self.step_observer is not None or self.loss_observer is not None:
            pts.update(range(0, max(tr.total for tr in tracks.values()) + 1))
        return sorted(pts)

    def _window_rows(self, tracks, t0, t1) -> np.ndarray:
        width = self.device.n if self.device is not None else len(self.hybrid.sub_models)
        rows = np.zeros((t1 - t0, width), dtype=STEP_DTYPE)
        for tr in tracks.values():
            if tr.done:
                continue
            lo, hi = t0, min(t1, tr.total)
            if hi <= lo:
                continue
            hp = tr.job.hypers
            for t in range(lo, hi):
                i, b = divmod(t, tr.spe)
                e = tr.epochs[i]
                step = tr.opt_base + t + 1
                b1, b2 = _bias(step)
                rows[t - t0, tr.slot] = (1, min(tr.batch, tr.n - b * tr.batch), b * tr.batch, e, b, step,
                                         float(F32(lr_at_epoch(hp.learning_rate, hp.lr_milestones, e))), b1, b2,
                                         (0, 0, 0))
        return rows

    def _lockstep(self, dev, tracks) -> tuple:
        from concurrent.futures import ThreadPoolExecutor

        from . import rng

        bounds = self._boundaries(tracks)
        horizon = max(tr.total for tr in tracks.values())
        # epoch permutations (src/store.py:74-76) are computed by host threads one epoch ahead,
        # while the device trains the current one; a boundary only uploads the ready result
        pool = ThreadPoolExecutor(max_workers=4)
        perm_of = lambda tr, e: rng.permutation(tr.n, "shuffle", tr.dataset.content_hash, tr.job.hypers.seed, e)
        ahead = {(tr.slot, tr.epochs[0]): pool.submit(perm_of, tr, tr.epochs[0]) for tr in tracks.values()}
        try:
            return self._lockstep_windows(dev, tracks, bounds, horizon, pool, perm_of, ahead)
        finally:
            pool.shutdown(wait=False, cancel_futures=True)

    def _lockstep_windows(self, dev, tracks, bounds, horizon, pool, perm_of, ahead) -> tuple:
        steps_run, samples = 0, 0
        for t0, t1 in zip(bounds[:-1], bounds[1:]):
            if t0 >= horizon or all(tr.done for tr in tracks.values()):
                break
            starting = []
            for tr in tracks.values():
                if not tr.done and t0 < tr.total and t0 % tr.spe == 0:
                    i = t0 // tr.spe
                    e = tr.epochs[i]
                    fut = ahead.pop((tr.slot, e), None)
                    perm = fut.result() if fut is not None else perm_of(tr, e)
                    dev.perm_upload(tr.slot, perm)
                    starting.append(tr.slot)
                    if i + 1 < len(tr.epochs):
                        nxt = tr.epochs[i + 1]
                        ahead[(tr.slot, nxt)] = pool.submit(perm_of, tr, nxt)
            dev.reset_accumulators(starting)
            rows = self._window_rows(tracks, t0, t1)
            samples += int(rows["rows"][rows["active"] == 1].sum())
            dev.load_schedule(rows)
            wall0 = time.perf_counter()
            dev.train_steps(t1 - t0, use_graph=self.use_graph)
            steps_run += t1 - t0
            if self.loss_observer is not None:
                losses = dev.loss_out.cpu().numpy()
                hits = dev.correct_out.cpu().numpy()
                for tr in tracks.values():
                    if not tr.done and t0 < tr.total:
                        self.loss_observer(tr.job.job_id, t0, float(losses[tr.slot]), int(hits[tr.slot]))
            if self.step_observer is not None:
                alive = dev.read_status()["alive"]
                for tr in tracks.values():
                    if not tr.done and t0 < tr.total and alive[tr.slot]:
                        self.step_observer(tr.job.job_id, self.hybrid.sub_params(tr.job.job_id))
            st = dev.read_status()  # synchronises the stream
            elapsed = time.perf_counter() - wall0
            self._poll_pauses()  # once per window: every hit is kept until its job's boundary
            for tr in tracks.values():
                if tr.done or t0 >= tr.total:
                    continue
                res = self.results[tr.job.job_id]
                res.wall_time += elapsed
                row = st[tr.slot]
                if not row["alive"]:
                    res.status = "aborted"
                    res.abort_reason = (f"non-finite loss in job {tr.job.job_id} at epoch {int(row['abort_epoch'])}"
                                        f", batch {int(row['abort_batch'])}")
                    tr.done = True
                    continue
                if t1 % tr.spe == 0 and t1 <= tr.total:
                    i = t1 // tr.spe - 1
                    e = tr.epochs[i]
                    seen = int(row["seen"])
                    loss, acc = float(row["loss_sum"]) / seen, int(row["correct_sum"]) / seen
                    res.curve.append((e, loss, acc))
                    res.final_train_loss, res.final_train_accuracy = loss, acc
                    res.slices_executed += 1
                    res.epochs_completed = e + 1
                    sub = self.hybrid.sub(tr.job.job_id)
                    sub.completed_epochs = e + 1
                    sub.optimizer.step = tr.opt_base + t1
                    key = (t1, self._order(tr.job.job_id))
                    self._executed.append((tr.job.job_id, e))
                    self._exec_keys.append(key)
                    if self.slice_observer is not None:
                        self.slice_observer(tr.job.job_id, e)
                    if e == tr.job.hypers.epochs - 1:
                        tr.done = True
                        self._complete(tr.job.job_id, key)
                    elif tr.job.job_id in self._pause_requests:
                        tr.done = True
                        self._pause(tr.job.job_id)
        return steps_run, samples

    # ------------------------------------------------------------------ completion / pause
    def _poll_pauses(self):
        """Call pause_poll once and keep every hit for a job of this Trainer that is still training
        (the reference's poll consumes its markers, src/workspace.py:293-301, so a hit must not be
        dropped just because its job is mid-epoch right now)."""
        if self.pause_poll is None:
            return
        for jid in self.pause_poll():
            if jid in self.jobs and self.results[jid].status == "training":
                self._pause_requests.add(jid)

    def _pause(self, job_id):
        self._pause_requests.discard(job_id)
        ckpt = make_checkpoint(self.hybrid, job_id)
        self.checkpoints[job_id] = ckpt
        self.results[job_id].status = "paused"
        if self.pause_sink is not None:
            self.pause_sink(job_id, ckpt)

    def _apply_pauses(self, force_all=False):
        """Checkpoint and stop every job with a pending pause request (reference _apply_pauses)."""
        self._poll_pauses()
        wanted = {j for j in self._pause_requests if j in self._local}
        self._pause_requests -= wanted
        for jid in sorted(wanted):
            if self.results[jid].status == "training":
                self._pause(jid)

    def _complete(self, job_id: str, key: tuple) -> None:
        result = self.results[job_id]
        ds = self.datasets[job_id]
        loss, acc = evaluate_hybrid(self.hybrid, [job_id], {job_id: ds})[job_id]
        result.status = "complete"
        result.completion_index = len(self._executed)
        self._completion_keys[job_id] = key
        result.final_test_loss, result.final_test_accuracy = loss, acc
        if self.completion_sink is not None:
            self.completion_sink(job_id, self.hybrid.snapshot(), result)


# --------------------------------------------------------------------------- host-fed steps


class HostFedStepper:
    """Step a materialised hybrid from HOST batches (the reference's run_batch contract, all jobs at once).

    Each :meth:`step` copies one lockstep step's batches — every job's ``x`` and integer
    labels, laid out like the device batch arena — from pinned host memory into HBM with
    one H2D copy per arena, runs the step's kernels (no device gather), and copies the
    per-job loss and correct count back to pinned host memory.  The schedule rows
    (rows / lr / optimizer step) come from :meth:`DeviceHybrid.load_schedule` as usual.

    The H2D copies run on their own stream into one of two HBM staging buffers, so step t's
    upload overlaps step t-1's kernels (the way a data loader prefetches); the step itself
    waits for its upload, moves the staged batch into the arena with one device copy, and
    frees the staging buffer for step t+2.
    """

    def __init__(self, hybrid: HybridModel, datasets: dict, use_graph: bool = True):
        import torch

        self.hybrid, self.dev, self.use_graph = hybrid, hybrid.device, use_graph
        if self.dev is None or not self.dev.train_plan:
            raise StateError("materialise the hybrid and build its plans before host-fed stepping")
        self.datasets = datasets
        self.loss_host = torch.zeros(self.dev.n, dtype=torch.float32).pin_memory()
        self.hits_host = torch.zeros(self.dev.n, dtype=torch.int32).pin_memory()
        self.h2d_bytes_per_step = int(self.dev.batch_arena.numel() * 4 + self.dev.label_arena.numel() * 4)
        self.d2h_bytes_per_step = int(self.dev.n * 8)
        self.copy_stream = torch.cuda.Stream(device=self.dev.device)
        self.staging = [(torch.empty_like(self.dev.batch_arena), torch.empty_like(self.dev.label_arena))
                        for _ in range(2)]
        self.staging_free = [None, None]
        self.steps_issued = 0
        self.dev.train_steps(0, use_graph=use_graph, host_fed=True)  # capture the step graph up front
        # graph-replayed steps go through one native call per step (hnn_hostfed_step: the staged
        # copies, the graph launch and the output D2H), the per-step Python of the stream-context
        # path below being the bound of the small configs' end-to-end step (C5: 0.3 ms)
        self._ctx = None
        if use_graph and os.environ.get("HNN_HOSTFED_NATIVE", "1") == "1":
            import ctypes

            from . import _native as N

            ctx = ctypes.c_void_p()
            N.call("hnn_hostfed_create", ctypes.byref(ctx))
            self._ctx = ctx
            self._io = N.HostFedIO()
            self._io.x_bytes = self.dev.batch_arena.numel() * 4
            self._io.y_bytes = self.dev.label_arena.numel() * 4
            self._io.arena_x = self.dev.batch_arena.data_ptr()
            self._io.arena_y = self.dev.label_arena.data_ptr()
            self._io.out_dev[0], self._io.out_host[0] = self.dev.loss_out.data_ptr(), self.loss_host.data_ptr()
            self._io.out_dev[1], self._io.out_host[1] = self.dev.correct_out.data_ptr(), self.hits_host.data_ptr()
            self._io.out_bytes[0], self._io.out_bytes[1] = self.dev.n * 4, self.dev.n * 4

    def __del__(self):
        if getattr(self, "_ctx", None) is not None:
            from . import _native as N

            try:
                torch_sync = __import__("torch").cuda.synchronize
                torch_sync(self.dev.device)
                N.call("hnn_hostfed_destroy", self._ctx)
            except Exception:
                pass
            self._ctx = None

    def _graph_exec(self) -> int:
        g = self.dev.__dict__.get("_graphs", {}).get(True)
        if g is None:  # (re-planned device: capture again)
            self.dev.train_steps(0, use_graph=True, host_fed=True)
            g = self.dev._graphs[True]
        h = g.raw_cuda_graph_exec()
        if not isinstance(h, int):  # a capsule on some builds
            import ctypes

            ctypes.pythonapi.PyCapsule_GetPointer.restype = ctypes.c_void_p
            ctypes.pythonapi.PyCapsule_GetPointer.argtypes = [ctypes.py_object, ctypes.c_char_p]
            h = ctypes.pythonapi.PyCapsule_GetPointer(h, None)
        return h

    def stage_epoch_batches(self, rows, count: int = 2, host_datasets: dict | None = None) -> list:
        """Pinned host copies of the first `count` steps' batches (store.batches order, src/store.py:68-81),
        each model from its own dataset and its row's epoch permutation."""
        fill = _BatchAssembler(self.hybrid, host_datasets or self.datasets)
        staged = []
        for t in range(count):
            x, y = fill.buffers()
            for slot in self.dev.slots:
                fill.fill(x, y, rows[t], slot.index)
            staged.append((x, y))
        return staged

    def step(self, host_batch) -> None:
        """Enqueue one step from a host batch: a ``(x, y)`` pair of pinned arena-layout tensors or a
        :class:`HostBatchLoader` batch (its buffer is handed back once the H2D copy has run)."""
        import torch

        x, y = host_batch[0], host_batch[1]
        k = self.steps_issued % 2
        sx, sy = self.staging[k]
        if self._ctx is not None:
            import ctypes

            from . import _native as N

            io = self._io
            io.host_x, io.host_y = x.data_ptr(), y.data_ptr()
            io.stage_x, io.stage_y = sx.data_ptr(), sy.data_ptr()
            ev = ctypes.c_void_p()
            N.call("hnn_hostfed_step", self._ctx, k, ctypes.byref(io), self._graph_exec(),
                   torch.cuda.current_stream(self.dev.device).cuda_stream, self.copy_stream.cuda_stream,
                   ctypes.byref(ev))
            self.steps_issued += 1
            if isinstance(host_batch, LoadedBatch):
                host_batch.release(_NativeEvent(ev.value))
            return
        compute = torch.cuda.current_stream(self.dev.device)
        with torch.cuda.stream(self.copy_stream):
            if self.staging_free[k] is not None:  # step t-2 has moved its batch out
                self.copy_stream.wait_event(self.staging_free[k])
            sx.copy_(x, non_blocking=True)
            sy.copy_(y, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(self.copy_stream)
        if isinstance(host_batch, LoadedBatch):
            host_batch.release(ready)
        compute.wait_event(ready)
        self.dev.batch_arena.copy_(sx, non_blocking=True)
        self.dev.label_arena.copy_(sy, non_blocking=True)
        free = torch.cuda.Event()
        free.record(compute)
        self.staging_free[k] = free
        self.steps_issued += 1
        self.dev.train_steps(1, use_graph=self.use_graph, host_fed=True)
        self.loss_host.copy_(self.dev.loss_out, non_blocking=True)
        self.hits_host.copy_(self.dev.correct_out, non_blocking=True)

    def finish(self) -> dict:
        import torch

        torch.cuda.current_stream().synchronize()
        return {s.job_id: (float(self.loss_host[s.index]), int(self.hits_host[s.index])) for s in self.dev.slots}


def C_sizeof(cls) -> int:
    import ctypes

    return ctypes.sizeof(cls)


class _BatchAssembler:
    """Host-side batch gather into the device batch-arena layout (the reference's store.batches:
    ``train_x[perm[s:s+B]]``, src/store.py:68-81).  One step of every model is ONE native call
    (``hnn_host_gather_batch``: the rows of all models split over host threads, GIL released);
    the per-step Python work is a vectorised update of the item table."""

    def __init__(self, hybrid: HybridModel, datasets: dict):
        from . import _native as N

        self.hybrid, self.dev, self.datasets = hybrid, hybrid.device, datasets
        self._perms: dict = {}
        self._src: dict = {}
        n = self.dev.n
        dt = np.dtype([(name, np.uint64 if ctype is N.P else np.int64) for name, ctype in N.HostGatherItem._fields_])
        assert dt.itemsize == C_sizeof(N.HostGatherItem)
        self.item_dtype = dt
        self.static = np.zeros(n, dtype=dt)  # destination offsets (filled per buffer), sources, widths
        self.caps = np.zeros(n, dtype=np.int64)
        for slot in self.dev.slots:
            m = slot.index
            xo, yo, ld = self.dev.batch_layout[m]
            d = self.datasets[slot.job_id]
            sample = int(np.prod(slot.sample_shape))
            src, ys = self._sources(slot.job_id, d, sample)
            self.static[m]["dst_x"] = 4 * xo
            self.static[m]["dst_y"] = 4 * yo
            self.static[m]["src_x"] = src.ctypes.data
            self.static[m]["src_y"] = ys.ctypes.data
            self.static[m]["ld_dst"] = ld
            self.static[m]["ld_src"] = sample
            self.static[m]["cols"] = sample
            self.caps[m] = slot.batch_size

    def buffers(self) -> tuple:
        import torch

        return (torch.zeros(self.dev.batch_arena.numel(), dtype=torch.float32).pin_memory(),
                torch.zeros(self.dev.label_arena.numel(), dtype=torch.int32).pin_memory())

    def perm(self, slot, epoch: int) -> np.ndarray:
        from . import rng

        key = (slot.index, epoch)
        p = self._perms.get(key)
        if p is None:
            d = self.datasets[slot.job_id]
            p = np.ascontiguousarray(rng.permutation(d.sample_count, "shuffle", d.content_hash,
                                                     self.hybrid.sub(slot.job_id).hypers.seed, epoch), dtype=np.int64)
            self._perms = {k: v for k, v in self._perms.items() if k[0] != slot.index}  # one epoch per slot
            self._perms[key] = p
        return p

    def items(self, x, y, row, perms: dict) -> np.ndarray:
        """The step's item table for buffers (x, y): model m gathers its `rows` indices of `perms[m]`
        from perm_base on (inactive models: no item rows).  Vectorised (per-step Python is the bound
        of the small configs' end-to-end step)."""
        it = self.static.copy()
        it["dst_x"] += np.uint64(x.data_ptr())
        it["dst_y"] += np.uint64(y.data_ptr())
        active = row["active"].astype(bool)
        it["n"] = np.where(active, row["rows"], 0)
        it["cap"] = np.where(active, self.caps, 0)
        base = np.zeros(len(it), dtype=np.uint64)
        for m, p in perms.items():
            base[m] = p.ctypes.data
        it["idx"] = np.where(active, base + 8 * row["perm_base"].astype(np.uint64), 0)
        return it

    def step_items(self, x, y, row) -> np.ndarray:
        """items() for a schedule row, with the per-model permutation pointers cached across steps
        (recomputed only for models whose epoch changed): no per-model Python on ordinary steps."""
        n = self.dev.n
        if not hasattr(self, "_ptr"):
            self._ptr = np.zeros(n, dtype=np.uint64)
            self._ep = np.full(n, -1, dtype=np.int64)
            self._keep = [None] * n
        active = row["active"].astype(bool)
        epochs = row["epoch"].astype(np.int64)
        for m in np.nonzero(active & (epochs != self._ep))[0]:
            p = self.perm(self.dev.slots[int(m)], int(epochs[m]))
            self._keep[m], self._ptr[m], self._ep[m] = p, p.ctypes.data, epochs[m]
        it = self.static.copy()
        it["dst_x"] += np.uint64(x.data_ptr())
        it["dst_y"] += np.uint64(y.data_ptr())
        it["n"] = np.where(active, row["rows"], 0)
        it["cap"] = np.where(active, self.caps, 0)
        it["idx"] = np.where(active, self._ptr + 8 * row["perm_base"].astype(np.uint64), 0)
        return it, list(self._keep)  # (the permutation arrays the raw pointers refer to)

    def gather(self, items: np.ndarray, threads: int) -> None:
        from . import _native as N

        N.call("hnn_host_gather_batch", items.ctypes.data, len(items), int(threads))

    def fill(self, x, y, row, m: int, perm=None) -> None:
        """Gather model m's rows of step `row` into the pinned arenas x / y."""
        slot = self.dev.slots[m]
        if not row[m]["active"]:
            return
        perm = self.perm(slot, int(row[m]["epoch"])) if perm is None else perm
        it = self.items(x, y, row, {m: perm})[m:m + 1]
        self.gather(it, 1)

    def _sources(self, job_id, d, sample):
        got = self._src.get(job_id)
        if got is None:
            got = (np.ascontiguousarray(d.train_x.reshape(d.train_x.shape[0], sample), dtype=np.float32),
                   np.ascontiguousarray(d.train_y, dtype=np.float32))
            self._src[job_id] = got
        return got


class _NativeEvent:
    """A CUDA event owned by the native host-fed context (hnn_hostfed_step's copied event)."""

    def __init__(self, handle: int):
        self.handle = handle

    def synchronize(self) -> None:
        from . import _native as N

        N.call("hnn_event_synchronize", self.handle)


class LoadedBatch(tuple):
    """One step's pinned (x, y) arena buffers from a :class:`HostBatchLoader`."""

    def release(self, copied_event) -> None:
        self.loader._recycle(self.slot_index, copied_event)


class HostBatchLoader:
    """Host data loader for :class:`HostFedStepper`: worker threads gather every upcoming step's
    batches — each model's rows of its epoch permutation from its host dataset, the reference's
    ``store.batches`` work (src/store.py:68-81) — into a ring of pinned arena-layout buffers,
    ``depth`` steps ahead of the device.  A buffer is refilled only after the H2D copy that
    read it has completed (the CUDA event the stepper hands back)."""

    def __init__(self, hybrid: HybridModel, datasets: dict, rows: np.ndarray, threads: int = 8, depth: int = 3):
        from concurrent.futures import ThreadPoolExecutor

        self.asm = _BatchAssembler(hybrid, datasets)
        self.rows = rows
        self.depth = depth
        self.threads = max(1, min(64, int(threads)))
        self.bufs = [self.asm.buffers() for _ in range(depth)]
        # one worker: each step is one native call that fans out over `threads` host threads
        self.pool = ThreadPoolExecutor(1)
        self.pending: list = [None] * depth
        self.t_next = 0
        self.t_issue = 0
        # permutations are computed on the caller's thread before any worker needs them
        for t in range(min(depth, rows.shape[0])):
            self._issue(t % depth, None)

    def _issue(self, k: int, after) -> None:
        t = self.t_issue
        self.t_issue += 1
        if t >= self.rows.shape[0]:
            self.pending[k] = None
            return
        row = self.rows[t]
        x, y = self.bufs[k]
        items, keep = self.asm.step_items(x, y, row)

        def job():
            if after is not None:
                after.synchronize()
            self.asm.gather(items, self.threads)
            del keep[:]  # (kept alive until the gather has read them)

        self.pending[k] = [self.pool.submit(job)]

    def next(self) -> LoadedBatch:
        """The next step's batch (blocks until its gather is complete)."""
        k = self.t_next % self.depth
        futs = self.pending[k]
        if futs is None:
            raise StateError("HostBatchLoader: schedule exhausted")
        for f in futs:
            f.result()
        self.t_next += 1
        out = LoadedBatch(self.bufs[k])
        out.loader, out.slot_index = self, k
        return out

    def _recycle(self, k: int, copied_event) -> None:
        self._issue(k, copied_event)

    def close(self) -> None:
        self.pool.shutdown(wait=True)


# --------------------------------------------------------------------------- one model, one batch


def run_batch(graph, params, order, batch, optimizer, lr, observer=None) -> tuple:
    """Forward, loss, backward, update for one batch of one model; returns (loss, correct)
    (src/train.py:223-256) — the reference's step, each stage on the device kernels.

    A non-finite loss returns ``(loss, 0)`` before any gradient or update (the caller's abort
    signal).  ``correct`` counts argmax hits of the pre-update logits.  The Trainer does not go
    through here: it runs every model's step as one grouped launch sequence (:mod:`.runtime`)."""
    from . import devops, engine
    from .errors import MissingGradientError
    from .ops import OP_KINDS, check_class_indices
    from .optim import apply_update

    torch = devops._torch()
    output_node = graph.node(graph.output)
    if OP_KINDS[output_node.op].loss_head:
        loss, tape = engine.forward(graph, params, batch.x, targets=batch.y, order=order)
        logits = tape.outputs[output_node.inputs[0]]
        upstream = np.float32(1.0)
    else:
        logits, tape = engine.forward(graph, params, batch.x, order=order)
        logits_dev = devops._to_dev(logits)[0]
        t = torch.from_numpy(check_class_indices(devops._host(batch.y), logits_dev.shape[1]).astype(np.int32))
        loss_t, upstream, _ = devops.sce_device(logits_dev, t.to(logits_dev.device))
        loss = np.float32(loss_t.item())
        if tape.host:
            upstream = upstream.cpu().numpy()
    loss_value = float(loss)
    if not np.isfinite(loss_value):
        return loss_value, 0
    grads = engine.backward(graph, params, tape, upstream)
    missing = [pid for pid in params if pid not in grads]
    if missing:
        raise MissingGradientError(missing[0])
    extra = [pid for pid in grads if pid not in params]
    if extra:
        raise MissingGradientError(extra[0], extra=True)
    apply_update(optimizer, params, grads, lr)
    if observer is not None:
        observer(params)
    logits_host = devops._host(logits)
    targets = check_class_indices(devops._host(batch.y), logits_host.shape[1])
    return loss_value, int((logits_host.argmax(axis=1) == targets).sum())


# --------------------------------------------------------------------------- evaluation


def evaluate_hybrid(hybrid: HybridModel, job_ids: list, datasets: dict, **options) -> dict:
    """Test-split loss/accuracy of several sub-models in one lockstep forward pass (src/train.py:259-279).

    Uses the hybrid's device as bound by its Trainer.  A hybrid that was never set up for the
    device is materialised here (``options``: the Trainer's materialisation options) with each
    sub-model bound to its own dataset from ``datasets``; sub-models without one borrow a dataset
    of their input shape, and evaluating a job without a dataset is an error."""
    dev = hybrid.device
    if dev is None or not dev.eval_plan:
        dev = hybrid.materialize(**options)
        cache = {}
        for ds in datasets.values():
            cache.setdefault(ds.content_hash, ds)
        by_model = []
        uploaded = {}
        for slot in dev.slots:
            ds = datasets.get(slot.job_id)
            if ds is None:
                ds = next((d for d in cache.values() if tuple(d.sample_shape) == tuple(slot.sample_shape)), None)
            if ds is None:
                raise StateError(f"job {slot.job_id!r}: dataset not resolved")
            if ds.content_hash not in uploaded:
                uploaded[ds.content_hash] = DeviceDataset(ds, dev.device)
            by_model.append(uploaded[ds.content_hash])
        dev.bind_datasets(by_model, max(d.n_train for d in by_model))
        dev.build_plans()
    out = {}
    todo = []
    for jid in job_ids:
        n_test = datasets[jid].test_x.shape[0]
        if n_test == 0:
            out[jid] = (0.0, 0.0)
        else:
            todo.append(jid)
    if not todo:
        return out
    for jid in todo:
        if not hybrid.on_device(jid):
            raise StateError(f"job {jid!r} is held by another rank; evaluate it where it trained")
    slots = {jid: hybrid.sub(jid).slot for jid in todo}
    for jid in todo:
        if dev.model_data[slots[jid]].content_hash != datasets[jid].content_hash:
            raise StateError(f"job {jid!r}: evaluation dataset differs from the bound one")
    steps = {jid: -(-datasets[jid].test_x.shape[0] // dev.slots[slots[jid]].batch_size) for jid in todo}
    T = max(steps.values())
    rows = np.zeros((T, dev.n), dtype=STEP_DTYPE)
    for jid in todo:
        m, B, n = slots[jid], dev.slots[slots[jid]].batch_size, datasets[jid].test_x.shape[0]
        for t in range(steps[jid]):
            rows[t, m]["active"] = 1
            rows[t, m]["rows"] = min(B, n - t * B)
            rows[t, m]["perm_base"] = t * B
    dev.reset_status(dev.eval_status)
    dev.load_schedule(rows)
    for _ in range(T):
        dev.run_plan(dev.eval_plan)
    st = dev.read_status(dev.eval_status)
    for jid in todo:
        row = st[slots[jid]]
        total = int(row["seen"])
        out[jid] = (float(row["loss_sum"]) / total, int(row["correct_sum"]) / total)
    return out


def evaluate(graph, params, order, x, y, batch_size: int) -> tuple:
    """Reference-signature evaluate (src/train.py:259-279) for one model, on the GPU."""
    from . import store
    from .model import HyperParams

    job = TrainingJob("eval", graph, "eval", HyperParams(1, batch_size, 1.0), 0, 0)
    h = merge([job])
    h.set_sub_params("eval", {k.split("/", 1)[-1]: v for k, v in params.items()})
    ds = store.Dataset("eval", x[:1].astype(np.float32), np.zeros(1, np.float32),
                       np.ascontiguousarray(x, dtype=np.float32), np.asarray(y, dtype=np.float32))
    return evaluate_hybrid(h, ["eval"], {"eval": ds})["eval"]


# --------------------------------------------------------------------------- standalone


def train_standalone(job, dataset, step_observer=None, **options) -> tuple:
    """Train one model alone (src/train.py:453-476) — the same device path with one slot."""
    job = TrainingJob.coerce(job)
    hybrid = merge([job])
    from .schedule import make_plan

    observer = None
    if step_observer is not None:
        observer = lambda jid, p: step_observer(jid, {unqualify(jid, k): v for k, v in p.items()})
    trainer = Trainer(hybrid, make_plan("fcfs", [job]), [job], {job.job_id: dataset}, step_observer=observer,
                      **options)
    report = trainer.run()
    res = report.jobs[job.job_id]
    if res.status == "aborted":
        raise StateError(f"non-finite loss in standalone run of {job.job_id} at epoch "
                         f"{res.abort_reason.split('epoch ')[1].split(',')[0]}")
    params = {unqualify(job.job_id, k): v for k, v in hybrid.sub_params(job.job_id).items()}
    sub = hybrid.sub(job.job_id)
    opt = OptimizerState(sub.optimizer.kind, sub.optimizer.momentum, sub.optimizer.step)
    return params, opt
