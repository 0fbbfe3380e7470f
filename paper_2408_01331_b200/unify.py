"""merge(): build the hybrid model — the entry side of the drop-in boundary.

Same contract as hybridnn.unify (src/unify.py:100-198): every job is
validated and failures are gathered into one MergeError; parameters are
initialised on the host from keyed streams (bit-identical to the reference,
independent of merge order); ids are namespaced ``"<job>/<node>"``.

What changes is where the parameters live.  The first time the hybrid is
used on the device, :class:`HybridModel` packs every sub-model into grouped
HBM arenas (see :mod:`.runtime`) and from then on the device copy is the
truth: ``params`` / ``sub_params`` return host copies (the reference returns
views, src/unify.py:121-123 — aliasing cannot cross the PCIe boundary), and
``snapshot()`` is a host-side deep copy exactly like the reference's.
"""
from __future__ import annotations

import copy
from dataclasses import dataclass, field

import numpy as np

from . import engine
from .errors import GraphValidationError, HybridnnError, MergeError, StateError, UnknownJobError
from .model import INPUT_ID, ModelGraph, OpNode, TrainingJob, validate_graph
from .optim import OptimizerState

GLOBAL_INPUT = "hybrid/input"
GLOBAL_OUTPUT = "hybrid/output"
CRITERION = "softmax-cross-entropy"


def qualify(job_id: str, node_id: str) -> str:
    return f"{job_id}/{node_id}"


def unqualify(job_id: str, qualified: str) -> str:
    head = f"{job_id}/"
    if not qualified.startswith(head):
        raise HybridnnError(f"node {qualified!r} is not namespaced under job {job_id!r}")
    return qualified[len(head):]


def namespace_graph(job_id: str, graph: ModelGraph) -> ModelGraph:
    """Copy with node ids prefixed; the reserved input reference stays as-is."""
    return ModelGraph(
        graph.name,
        tuple(graph.input_shape),
        [OpNode(qualify(job_id, n.node_id), n.op,
                [r if r == INPUT_ID else qualify(job_id, r) for r in n.inputs], dict(n.attrs))
         for n in graph.nodes],
        qualify(job_id, graph.output),
    )


@dataclass(frozen=True)
class RoutingNode:
    node_id: str
    routes: dict


@dataclass
class SubModel:
    job_id: str
    graph: ModelGraph       # namespaced
    original: ModelGraph    # as submitted
    optimizer: OptimizerState
    criterion: str = CRITERION
    completed_epochs: int = 0
    order: list = field(default_factory=list)
    slot: int = -1          # index in the device arenas
    hypers: object = None

    def param_ids(self) -> list:
        return [qualify(self.job_id, pid) for pid in engine.param_specs(self.original)]


class _ParamView(dict):
    """``hybrid.params`` of a device-backed hybrid: a host copy taken on access."""


class HybridModel:
    """All sub-models plus the parameter store (host until first device use, then HBM)."""

    def __init__(self, sub_models: dict, params: dict, global_input: RoutingNode, global_output: RoutingNode):
        self.sub_models = sub_models
        self._host_params = params
        self.global_input = global_input
        self.global_output = global_output
        self.device = None  # runtime.DeviceHybrid once materialised

    # ---------------------------------------------------------------- reference surface
    def sub(self, job_id: str) -> SubModel:
        try:
            return self.sub_models[job_id]
        except KeyError:
            raise UnknownJobError(job_id) from None

    def job_ids(self) -> list:
        return list(self.sub_models)

    def node_count(self) -> int:
        return sum(len(s.graph.nodes) for s in self.sub_models.values()) + 2

    def on_device(self, job_id: str) -> bool:
        """True when the job's state lives in this process's HBM arenas (its slot is local)."""
        return self.device is not None and self.sub(job_id).slot >= 0

    @property
    def params(self) -> dict:
        if self.device is None:
            return self._host_params
        out = _ParamView()
        for jid in self.sub_models:
            out.update(self.sub_params(jid))
        return out

    def sub_params(self, job_id: str) -> dict:
        sub = self.sub(job_id)
        if not self.on_device(job_id):
            if self.device is None:
                return {pid: self._host_params[pid] for pid in sub.param_ids()}
            return {pid: np.array(self._host_params[pid], copy=True) for pid in sub.param_ids()}
        host = self.device.download_params(sub.slot)
        return {qualify(job_id, pid): arr for pid, arr in host.items()}

    def snapshot(self) -> "HybridModel":
        snap = HybridModel(copy.deepcopy(self.sub_models),
                           {pid: np.array(a, copy=True) for pid, a in self.params.items()},
                           self.global_input, self.global_output)
        for jid, sub in snap.sub_models.items():
            sub.slot = -1
            if not self.on_device(jid):
                continue  # host-held state was deep-copied with the sub-model
            m1, m2 = self.device.download_moments(self.sub_models[jid].slot)
            kind = sub.optimizer.kind
            if kind == "adam":
                sub.optimizer.m1 = {qualify(jid, k): v for k, v in m1.items()}
                sub.optimizer.m2 = {qualify(jid, k): v for k, v in m2.items()}
            elif m1:
                sub.optimizer.velocity = {qualify(jid, k): v for k, v in m1.items()}
        return snap

    # ---------------------------------------------------------------- device side
    def set_sub_params(self, job_id: str, params: dict) -> None:
        """Write a sub-model's parameters (namespaced or bare ids) into the store."""
        sub = self.sub(job_id)
        bare = {(unqualify(job_id, k) if k.startswith(job_id + "/") else k): np.asarray(v, dtype=np.float32)
                for k, v in params.items()}
        if not self.on_device(job_id):
            for pid, arr in bare.items():
                self._host_params[qualify(job_id, pid)][...] = arr
        else:
            self.device.upload_params(sub.slot, bare)

    def materialize(self, device=None, use_tensor_cores: bool = True, fuse_optimizer: bool = True,
                    keep_grads: bool = False, conv_precision: str = "f32", local=None):
        """Pack sub-models into device arenas (idempotent).

        ``local``: the job ids this process holds in HBM (model-identity sharding over ranks,
        :mod:`.parallel`); the others keep their state on the host.  Default: every job.
        Host-held optimizer moments (a restored checkpoint, a released device) are uploaded
        here, once, with the parameters."""
        want = [jid for jid in self.sub_models if local is None or jid in set(local)]
        if self.device is not None:
            if [s.job_id for s in self.device.slots] == want:
                return self.device
            self.release_device()
        from .runtime import DeviceHybrid, ModelSlot

        slots = []
        for sub in self.sub_models.values():
            sub.slot = -1
        for i, jid in enumerate(want):
            sub = self.sub_models[jid]
            sub.slot = i
            hp = sub.hypers
            slots.append(ModelSlot(i, jid, sub.original, hp.batch_size if hp else 1, sub.optimizer.kind,
                                   sub.optimizer.momentum, engine.param_specs(sub.original)))
        dev = DeviceHybrid(slots, device=device, use_tensor_cores=use_tensor_cores, fuse_optimizer=fuse_optimizer,
                           keep_grads=keep_grads, conv_precision=conv_precision)
        for jid in want:
            sub = self.sub_models[jid]
            dev.upload_params(sub.slot, {unqualify(jid, pid): self._host_params[pid] for pid in sub.param_ids()})
            opt = sub.optimizer
            if opt.m1 or opt.m2 or opt.velocity:
                strip = lambda d: {unqualify(jid, k): v for k, v in d.items()}
                dev.upload_moments(sub.slot, strip(opt.m1 or opt.velocity), strip(opt.m2))
                # the device copy is the truth from here on: drop the host moments so a later
                # run can never re-upload stale ones (they are re-read by snapshot / checkpoints)
                opt.m1, opt.m2, opt.velocity = {}, {}, {}
        self.device = dev
        return dev

    def release_device(self) -> None:
        """Copy every device-held sub-model's parameters and moments back to the host and drop
        the device arenas (before re-packing a different local set)."""
        dev = self.device
        if dev is None:
            return
        for jid, sub in self.sub_models.items():
            if sub.slot < 0:
                continue
            for pid, arr in dev.download_params(sub.slot).items():
                self._host_params[qualify(jid, pid)] = arr
            m1, m2 = dev.download_moments(sub.slot)
            q = lambda d: {qualify(jid, k): v for k, v in d.items()}
            if sub.optimizer.kind == "adam":
                sub.optimizer.m1, sub.optimizer.m2 = q(m1), q(m2)
            elif m1:
                sub.optimizer.velocity = q(m1)
            sub.slot = -1
        self.device = None

    def store_remote(self, job_id: str, params: dict, m1: dict, m2: dict, step: int, completed_epochs: int) -> None:
        """Host state of a sub-model trained on another rank (bare ids), after a gather."""
        sub = self.sub(job_id)
        if self.on_device(job_id):
            raise StateError(f"job {job_id!r} is held on this rank's device")
        for pid, arr in params.items():
            self._host_params[qualify(job_id, pid)] = np.array(arr, dtype=np.float32, copy=True)
        q = lambda d: {qualify(job_id, k): np.array(v, dtype=np.float32, copy=True) for k, v in d.items()}
        opt = sub.optimizer
        if opt.kind == "adam":
            opt.m1, opt.m2 = q(m1), q(m2)
        elif m1:
            opt.velocity = q(m1)
        opt.step = step
        sub.completed_epochs = completed_epochs


def merge(jobs: list) -> HybridModel:
    """Validate every job, then embed each sub-graph with keyed initial values (src/unify.py:135-184)."""
    if not jobs:
        raise StateError("cannot merge an empty job list")
    jobs = [TrainingJob.coerce(j) for j in jobs]
    failures: dict = {}
    seen: set = set()
    for job in jobs:
        problems = []
        if job.job_id in seen:
            problems.append("duplicate job id")
        seen.add(job.job_id)
        try:
            validate_graph(job.graph)
        except GraphValidationError as exc:
            problems.extend(exc.diagnostics)
        if problems:
            failures[job.job_id] = problems
    if failures:
        raise MergeError(failures)
    subs: dict = {}
    params: dict = {}
    for job in jobs:
        for pid, arr in engine.init_params(job.graph, job.hypers.seed).items():
            params[qualify(job.job_id, pid)] = arr
        subs[job.job_id] = SubModel(
            job.job_id, namespace_graph(job.job_id, job.graph), job.graph,
            OptimizerState.fresh(job.hypers.optimizer), completed_epochs=job.completed_epochs,
            order=[qualify(job.job_id, nid) for nid in validate_graph(job.graph)], hypers=job.hypers)
    entry = RoutingNode(GLOBAL_INPUT, {j.job_id: qualify(j.job_id, INPUT_ID) for j in jobs})
    exit_ = RoutingNode(GLOBAL_OUTPUT, {j.job_id: subs[j.job_id].graph.output for j in jobs})
    return HybridModel(subs, params, entry, exit_)


def route(hybrid: HybridModel, job_id: str, batch, targets=None) -> np.ndarray:
    """Forward a batch through exactly one sub-model on the device (src/unify.py:187-198).

    Returns the graph output: logits, or the scalar loss for a loss-head graph
    (``targets`` required then).
    """
    from . import devops

    sub = hybrid.sub(job_id)
    params = {unqualify(job_id, k): v for k, v in hybrid.sub_params(job_id).items()}
    return devops.graph_forward(sub.original, params, batch, targets)
