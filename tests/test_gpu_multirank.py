"""Model-identity sharding end to end (VERDICT r01 "Next round" item 2).

Two ranks (torch.distributed, gloo, both on cuda:0 — the GPU box has one GPU, the NCCL path is
the same code with device-to-device collectives) run ``Trainer(..., comm=RankGroup)`` over a
C3-style job mix: each trains only its ``shard_jobs`` share, then results, slice log and final
model states are gathered.  Both ranks must return the report a single process over all jobs
returns, and hold every job's parameters and optimizer moments bit-identical to it (sub-models
share nothing, src/unify.py:1-9, so the partition cannot change a trajectory).
"""
import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup():
    from paper_2408_01331_b200 import make_plan, merge, store, zoo

    blob = store.from_splits(oracle.blob_splits("mr", "blob", 10, 784, 700, 150))
    other = store.from_splits(oracle.blob_splits("mr", "other", 10, 784, 530, 90))
    jobs = []
    for i in range(6):
        h = 64 * (1 + i % 4)
        ds = other if i == 4 else blob
        opt = "sgd" if i == 5 else "adam"
        jobs.append(zoo.job(f"m{i}", zoo.mlp(784, (h, h), 10), ds, i, epochs=2 + (i % 2), batch_size=64 + 32 * (i % 3),
                            lr=(1e-3 if opt == "adam" else 0.05), optimizer=opt, seed=i, milestones=(1,)))
    datasets = {j.job_id: (other if j.job_id == "m4" else blob) for j in jobs}
    return jobs, datasets, merge, make_plan


def _state(hybrid, jobs):
    snap = hybrid.snapshot()
    out = {}
    for j in jobs:
        sub = snap.sub(j.job_id)
        opt = sub.optimizer
        out[j.job_id] = ({k: v.copy() for k, v in snap.sub_params(j.job_id).items()},
                         {k: v.copy() for k, v in (opt.m1 or opt.velocity).items()},
                         {k: v.copy() for k, v in opt.m2.items()}, opt.step, sub.completed_epochs)
    return out


def _run(comm=None):
    from paper_2408_01331_b200 import Trainer

    jobs, datasets, merge, make_plan = _setup()
    hybrid = merge(jobs)
    report = Trainer(hybrid, make_plan("rr", jobs), jobs, datasets, comm=comm).run()
    return report.to_dict(), _state(hybrid, jobs), (report.steps, report.samples)


def _rank(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_2408_01331_b200.parallel import RankGroup

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = RankGroup(rank, world, torch.device("cuda", 0))
    out[rank] = _run(comm)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_trainer_matches_one_process_bit_exactly():
    import torch.multiprocessing as mp

    from paper_2408_01331_b200.parallel import shard_jobs

    jobs = _setup()[0]
    parts = shard_jobs(jobs, 2)
    assert all(parts), "both ranks must own jobs"
    ref_report, ref_state, (ref_steps, ref_samples) = _run()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_rank, args=(2, _free_port(), out), nprocs=2, join=True)
        res = dict(out)
    for rank in (0, 1):
        report, state, (steps, samples) = res[rank]
        assert report == ref_report, f"rank {rank}: report differs"
        assert samples == ref_samples and steps <= ref_steps
        for jid, (params, m1, m2, step, epochs) in ref_state.items():
            got = state[jid]
            assert got[3] == step and got[4] == epochs, (rank, jid)
            for ref_d, got_d in ((params, got[0]), (m1, got[1]), (m2, got[2])):
                assert sorted(ref_d) == sorted(got_d), (rank, jid)
                for k in ref_d:
                    assert np.array_equal(ref_d[k].view(np.uint32), got_d[k].view(np.uint32)), (rank, jid, k)
