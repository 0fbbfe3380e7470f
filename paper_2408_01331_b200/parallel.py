"""Multi-GPU plumbing: model-identity sharding, dataset broadcast, metric gather.

Sub-models share nothing (src/unify.py:1-9), so the natural partition is by
model: each rank trains its own shard with no gradient collective.  NCCL
(over NVLink/NVSwitch) carries exactly two things:

* the shared dataset, broadcast once from rank 0's HBM into every rank's HBM
  (:meth:`RankGroup.share_dataset`);
* per-model metrics ``[loss_sum, correct, seen, alive]`` gathered at the end
  (:meth:`RankGroup.gather_metrics`).

With the ``gloo`` backend the same code runs on CPU tensors (tests).
"""
from __future__ import annotations

import json

import numpy as np


def flops_per_sample(graph) -> int:
    """fwd + wgrad for every layer + dgrad for every layer but the first (= 6*MACs - 2*MACs_first)."""
    from .engine import chain, infer_shapes

    shapes = infer_shapes(graph)
    macs = []
    for n in chain(graph):
        if n.op == "dense":
            macs.append(int(np.prod(shapes[n.inputs[0]])) * n.attrs["units"])
        elif n.op == "conv2d":
            c = shapes[n.inputs[0]][0]
            f, oh, ow = shapes[n.node_id]
            macs.append(c * n.attrs["kernel"] ** 2 * f * oh * ow)
    return 6 * sum(macs) - 2 * (macs[0] if macs else 0)


def shard_jobs(jobs: list, world: int) -> list:
    """Deterministic longest-processing-time assignment by FLOP/step; returns one job list per rank.

    Ties break on job order so every rank computes the same partition independently.
    """
    load = [0] * world
    out = [[] for _ in range(world)]
    cost = [(flops_per_sample(j.graph) * j.hypers.batch_size, i) for i, j in enumerate(jobs)]
    for c, i in sorted(cost, key=lambda t: (-t[0], t[1])):
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(jobs[i])
        load[r] += c
    return [sorted(part, key=lambda j: jobs.index(j)) for part in out]


class DatasetMeta:
    """Host-side facts about a dataset a non-root rank received by broadcast."""

    def __init__(self, content_hash, n_train, n_test, sample_shape):
        self.content_hash = content_hash
        self.sample_count = n_train
        self.n_test = n_test
        self.sample_shape = tuple(sample_shape)


class RankGroup:
    """This process's rank in a torch.distributed group (one process per GPU)."""

    def __init__(self, rank: int, world: int, device, group=None):
        self.rank, self.world, self.device, self.group = rank, world, device, group

    def _dist(self):
        import torch.distributed as dist

        return dist

    def share_dataset(self, ds, device=None):
        """Rank 0 uploads `ds` once and broadcasts it device-to-device; returns (DeviceDataset, meta)."""
        import torch

        from .runtime import DeviceDataset

        dist = self._dist()
        device = device or self.device
        if self.rank == 0:
            dd = DeviceDataset(ds, device)
            head = json.dumps({"hash": dd.content_hash, "x": list(dd.train_x.shape), "tx": list(dd.test_x.shape),
                               "max": dd.max_label}).encode()
            blob = torch.zeros(1024, dtype=torch.uint8, device=device)
            blob[: len(head)] = torch.frombuffer(bytearray(head), dtype=torch.uint8).to(device)
        else:
            blob = torch.zeros(1024, dtype=torch.uint8, device=device)
        dist.broadcast(blob, 0, group=self.group)
        head = json.loads(bytes(blob.cpu().numpy()).rstrip(b"\x00").decode())
        if self.rank != 0:
            f32, i32 = dict(dtype=torch.float32, device=device), dict(dtype=torch.int32, device=device)
            tx = torch.empty(head["x"], **f32)
            ty = torch.empty(head["x"][0], **i32)
            vx = torch.empty(head["tx"], **f32)
            vy = torch.empty(head["tx"][0], **i32)
        else:
            tx, ty, vx, vy = dd.train_x, dd.train_y, dd.test_x, dd.test_y
        for t in (tx, ty, vx, vy):
            dist.broadcast(t, 0, group=self.group)
        if self.rank != 0:
            dd = DeviceDataset.from_tensors(head["hash"], tx, ty, vx, vy, head["max"], device)
        meta = ds if ds is not None else DatasetMeta(head["hash"], head["x"][0], head["tx"][0], head["x"][1:])
        return dd, meta

    def gather_metrics(self, job_ids: list, stats: np.ndarray) -> dict:
        """All-gather per-model rows [loss_sum, correct, seen, alive] (float64) keyed by job id."""
        import torch

        dist = self._dist()
        local = torch.tensor(np.asarray(stats, dtype=np.float64).reshape(-1, 4), device=self.device)
        n = torch.tensor([local.shape[0]], device=self.device)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(sizes, n, group=self.group)
        width = int(max(s.item() for s in sizes))
        pad = torch.zeros(width, 4, dtype=torch.float64, device=self.device)
        pad[: local.shape[0]] = local
        bufs = [torch.zeros_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad, group=self.group)
        names = [None] * self.world
        dist.all_gather_object(names, list(job_ids), group=self.group)
        out = {}
        for r in range(self.world):
            rows = bufs[r].cpu().numpy()[: int(sizes[r].item())]
            out.update({jid: rows[i] for i, jid in enumerate(names[r])})
        return out
