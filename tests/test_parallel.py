"""Multi-rank host logic on CPU (gloo, world size 2): sharding, dataset broadcast, metric gather."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2408_01331_b200 import store, zoo
from paper_2408_01331_b200.parallel import RankGroup, flops_per_sample, shard_jobs


def test_flops_per_sample_matches_baseline_table():
    # BASELINE.md "Configs": 818,176 (MLP 784-256-10), 3,204,720 (LeNet-5)
    assert flops_per_sample(zoo.mlp()) == 818176
    assert flops_per_sample(zoo.lenet5()) == 3204720
    assert flops_per_sample(zoo.vgg11_nobn()) == 913078272
    assert flops_per_sample(zoo.resnet18_plain()) == 3291248640


def test_shard_jobs_is_deterministic_balanced_and_complete():
    ds = store.from_splits(oracle.blob_splits("t", "p", 2, 784, 8, 2))
    jobs = zoo.config_jobs("c3", ds)
    for world in (1, 2, 4, 8):
        parts = shard_jobs(jobs, world)
        assert parts == shard_jobs(list(jobs), world)
        assert sorted(j.job_id for p in parts for j in p) == sorted(j.job_id for j in jobs)
        loads = [sum(flops_per_sample(j.graph) * j.hypers.batch_size for j in p) for p in parts]
        assert max(loads) <= 1.15 * (sum(loads) / world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, splits, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = RankGroup(rank, world, torch.device("cpu"))
    ds = store.from_splits(splits) if rank == 0 else None
    dd, meta = comm.share_dataset(ds, torch.device("cpu"))
    stats = np.array([[1.5 + rank, 10 * rank, 64, 1]], dtype=np.float64)
    gathered = comm.gather_metrics([f"m{rank}"], stats)
    out[rank] = (dd.content_hash, dd.train_x.numpy().copy(), dd.train_y.numpy().copy(), meta.sample_count,
                 {k: v.tolist() for k, v in gathered.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_dataset_broadcast_and_metric_gather_with_gloo():
    import torch.multiprocessing as mp

    splits = oracle.blob_splits("t", "bcast", 3, 6, 20, 5)
    ref = store.from_splits(splits)
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, _free_port(), splits, out), nprocs=2, join=True)
        res = dict(out)
    for rank in (0, 1):
        h, x, y, n, gathered = res[rank]
        assert h == ref.content_hash and n == 20
        assert np.array_equal(x, ref.train_x)
        assert np.array_equal(y, ref.train_y.astype(np.int32))
        assert gathered == {"m0": [1.5, 0.0, 64.0, 1.0], "m1": [2.5, 10.0, 64.0, 1.0]}


def _datasets_worker(rank, world, port, blobs, out):
    """Ranks ask for different dataset sets, in different orders; rank 1 holds one only as metadata."""
    import torch
    import torch.distributed as dist

    from paper_2408_01331_b200.parallel import DatasetMeta

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = RankGroup(rank, world, torch.device("cpu"))
    a, b, c = (store.from_splits(s) for s in blobs)
    if rank == 0:
        mine = [b, a]
    else:
        mine = [c, DatasetMeta(a.content_hash, a.sample_count, a.test_x.shape[0], a.sample_shape)]
    got = comm.share_datasets(mine, torch.device("cpu"))
    out[rank] = {h: (d.train_x.numpy().copy(), d.train_y.numpy().copy(), d.test_x.numpy().copy()) for h, d in got.items()}
    dist.barrier()
    dist.destroy_process_group()


def test_share_datasets_agrees_on_the_set_before_broadcasting():
    """each rank must receive exactly the datasets it asked for, under their own hash,
    whatever order the ranks list them in (src/store.py:55-56 content hashes)."""
    import torch.multiprocessing as mp

    blobs = [oracle.blob_splits("t", f"set{i}", 3, 5 + i, 12 + i, 4) for i in range(3)]
    ref = [store.from_splits(s) for s in blobs]
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_datasets_worker, args=(2, _free_port(), blobs, out), nprocs=2, join=True)
        res = dict(out)
    a, b, c = ref
    assert sorted(res[0]) == sorted([a.content_hash, b.content_hash])
    assert sorted(res[1]) == sorted([a.content_hash, c.content_hash])
    for rank, got in res.items():
        for d in ref:
            if d.content_hash in got:
                x, y, tx = got[d.content_hash]
                assert np.array_equal(x, d.train_x) and np.array_equal(tx, d.test_x)
                assert np.array_equal(y, d.train_y.astype(np.int32))

