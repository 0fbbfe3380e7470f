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
    """This process's rank in a torch.distributed group (one process per GPU).

    With the ``nccl`` backend the collectives run device-to-device over NVLink; with ``gloo``
    (CPU tests, or several ranks sharing one GPU in the GPU tests) device tensors are staged
    through host memory.  Every method is a collective: all ranks call it in the same order.
    """

    def __init__(self, rank: int, world: int, device, group=None):
        self.rank, self.world, self.device, self.group = rank, world, device, group

    def _dist(self):
        import torch.distributed as dist

        return dist

    def _staged(self, t) -> bool:
        return t.is_cuda and self._dist().get_backend(self.group) == "gloo"

    def broadcast(self, t, src: int) -> None:
        dist = self._dist()
        if self._staged(t):
            host = t.cpu()
            dist.broadcast(host, src, group=self.group)
            t.copy_(host)
        else:
            dist.broadcast(t, src, group=self.group)

    def all_gather(self, bufs: list, t) -> None:
        dist = self._dist()
        if self._staged(t):
            host = [b.cpu() for b in bufs]
            dist.all_gather(host, t.cpu(), group=self.group)
            for b, h in zip(bufs, host):
                b.copy_(h)
        else:
            dist.all_gather(bufs, t, group=self.group)

    def all_gather_object(self, obj) -> list:
        out = [None] * self.world
        self._dist().all_gather_object(out, obj, group=self.group)
        return out

    def share_dataset(self, ds, device=None):
        """Rank 0 uploads `ds` once and broadcasts it device-to-device; returns (DeviceDataset, meta).

        The hot-path form (bench.py): every rank trains on rank 0's dataset.  The Trainer uses
        :meth:`share_datasets`, which first agrees on the set of datasets."""
        from .runtime import DeviceDataset

        device = device or self.device
        dd = head = None
        if self.rank == 0:
            dd = DeviceDataset(ds, device)
            head = {"hash": dd.content_hash, "x": list(dd.train_x.shape), "tx": list(dd.test_x.shape),
                    "max": dd.max_label}
        head = self.all_gather_object(head)[0]
        dd = self._broadcast_dataset(head, dd, 0, device)
        meta = ds if ds is not None else DatasetMeta(head["hash"], head["x"][0], head["tx"][0], head["x"][1:])
        return dd, meta

    def _broadcast_dataset(self, head, dd, src, device):
        import torch

        from .runtime import DeviceDataset

        if self.rank != src:
            f32, i32 = dict(dtype=torch.float32, device=device), dict(dtype=torch.int32, device=device)
            tx = torch.empty(head["x"], **f32)
            ty = torch.empty(head["x"][0], **i32)
            vx = torch.empty(head["tx"], **f32)
            vy = torch.empty(head["tx"][0], **i32)
        else:
            tx, ty, vx, vy = dd.train_x, dd.train_y, dd.test_x, dd.test_y
        for t in (tx, ty, vx, vy):
            self.broadcast(t, src)
        if self.rank != src:
            dd = DeviceDataset.from_tensors(head["hash"], tx, ty, vx, vy, head["max"], device)
        return dd

    def share_datasets(self, datasets: list, device=None) -> dict:
        """Agree on every rank's datasets, then broadcast each one once; returns {hash: DeviceDataset}
        holding the datasets THIS rank asked for.

        ``datasets``: the store.Dataset objects (or metadata with ``content_hash`` only) this rank
        needs.  All ranks exchange (hash, shape, holds-data) first; each distinct hash, in sorted
        order, is uploaded by the lowest rank holding its arrays and broadcast to all ranks.  A
        receiving rank that also holds the dataset checks the broadcast header against its own
        copy (the content hash covers the bytes), so a rank can never train on another rank's
        data under its own hash."""
        from .errors import StateError
        from .runtime import DeviceDataset

        device = device or self.device
        mine = {}
        for d in datasets:
            if d is None:
                continue
            has = getattr(d, "train_x", None) is not None
            info = {"data": has}
            if has:
                info.update(x=list(d.train_x.shape), tx=list(d.test_x.shape))
            prev = mine.get(d.content_hash)
            if prev is None or (has and not prev[1]["data"]):
                mine[d.content_hash] = (d, info)
        every = self.all_gather_object({h: info for h, (_, info) in mine.items()})
        out = {}
        for h in sorted({h for inf in every for h in inf}):
            owners = [r for r, inf in enumerate(every) if h in inf and inf[h]["data"]]
            if not owners:
                raise StateError(f"dataset {h[:12]}...: no rank holds its arrays")
            src = owners[0]
            dd = None
            if self.rank == src:
                dd = DeviceDataset(mine[h][0], device)
                head = {"hash": h, "x": list(dd.train_x.shape), "tx": list(dd.test_x.shape), "max": dd.max_label}
            else:
                head = None
            head = self.all_gather_object(head)[src]
            if head["hash"] != h:
                raise StateError(f"dataset broadcast out of order: expected {h[:12]}, got {head['hash'][:12]}")
            if h in mine and mine[h][1]["data"] and self.rank != src:
                local = mine[h][1]
                if local["x"] != head["x"] or local["tx"] != head["tx"]:
                    raise StateError(f"dataset {h[:12]}...: rank {self.rank} holds shapes {local['x']}/{local['tx']}"
                                     f", rank {src} broadcast {head['x']}/{head['tx']}")
            dd = self._broadcast_dataset(head, dd, src, device)
            if h in mine:
                out[h] = dd
            else:
                del dd
        return out

    def gather_metrics(self, job_ids: list, stats: np.ndarray) -> dict:
        """All-gather per-model rows [loss_sum, correct, seen, alive] (float64) keyed by job id."""
        import torch

        local = torch.tensor(np.asarray(stats, dtype=np.float64).reshape(-1, 4), device=self.device)
        n = torch.tensor([local.shape[0]], device=self.device)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        self.all_gather(sizes, n)
        width = int(max(s.item() for s in sizes))
        pad = torch.zeros(width, 4, dtype=torch.float64, device=self.device)
        pad[: local.shape[0]] = local
        bufs = [torch.zeros_like(pad) for _ in range(self.world)]
        self.all_gather(bufs, pad)
        names = self.all_gather_object(list(job_ids))
        out = {}
        for r in range(self.world):
            rows = bufs[r].cpu().numpy()[: int(sizes[r].item())]
            out.update({jid: rows[i] for i, jid in enumerate(names[r])})
        return out

    def exchange_models(self, hybrid, owners: dict, meta: dict) -> None:
        """Broadcast each job's final parameters and optimizer moments from its owning rank, so
        every rank's hybrid holds every job afterwards (host-side for the jobs of other ranks).

        owners: {job_id: rank}; meta: {job_id: (optimizer step, completed epochs)}.  One
        device-to-device broadcast per arena segment (params, then m1 / m2 when present)."""
        import torch

        from . import engine

        for jid in sorted(owners, key=list(hybrid.sub_models).index):
            src = owners[jid]
            sub = hybrid.sub(jid)
            specs = engine.param_specs(sub.original)
            sizes = [int(np.prod(s)) for s in specs.values()]
            total = sum(-(-n // 4) * 4 for n in sizes)
            kind = sub.optimizer.kind
            narenas = 1 + (2 if kind == "adam" else (1 if sub.optimizer.momentum else 0))
            if self.rank == src:
                dev = hybrid.device
                slot = dev.slots[sub.slot]
                arenas = [dev.params, dev.m1, dev.m2][:narenas]
                flat = torch.stack([a[slot.seg_off:slot.seg_off + slot.seg_len] for a in arenas])
            else:
                flat = torch.empty(narenas, total, dtype=torch.float32, device=self.device)
            self.broadcast(flat, src)
            if self.rank == src:
                continue
            host = flat.cpu().numpy()
            unpack = []
            for row in host:
                d, o = {}, 0
                for (pid, shp), n in zip(specs.items(), sizes):
                    d[pid] = row[o:o + n].reshape(shp).copy()
                    o += -(-n // 4) * 4
                unpack.append(d)
            params, m1, m2 = unpack[0], (unpack[1] if narenas > 1 else {}), (unpack[2] if narenas > 2 else {})
            step, epochs = meta[jid]
            hybrid.store_remote(jid, params, m1, m2, step, epochs)
