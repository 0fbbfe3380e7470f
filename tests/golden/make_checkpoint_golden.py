"""Golden UNND v3 checkpoints written by the unmodified reference (hybridnn.train.Checkpoint.encode).

Run in the build container (the reference is importable from /root/reference/pkg/src):
    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 python tests/golden/make_checkpoint_golden.py
Writes
* checkpoint_synthetic_{adam,momentum}.bin: checkpoints of keyed-init parameters and closed-form
  moments (no training), so tests/test_host.py can build the same Checkpoint and compare bytes;
* checkpoint_paused_{adam,sgd}.bin + checkpoint_resumed.npz: a job trained by the reference
  Trainer, paused after epoch 1 (src/train.py:374-392), and the reference's own final parameters
  after restoring that checkpoint into a fresh hybrid and running the remaining two epochs (the lr milestone falls after the resume)
  (tests/test_gpu_parity.py resumes the same bytes on the device and compares).
"""
from pathlib import Path

import numpy as np

from hybridnn import engine, formats, store
from hybridnn.model import HyperParams, ModelGraph, OpNode, TrainingJob
from hybridnn.schedule import make_plan
from hybridnn.train import Checkpoint, Trainer, restore_checkpoint
from hybridnn.unify import merge

HERE = Path(__file__).resolve().parent


def chain(name, input_shape, spec):
    nodes, prev = [], "input"
    for nid, op, attrs in spec:
        nodes.append(OpNode(nid, op, [prev], dict(attrs)))
        prev = nid
    return ModelGraph(name, tuple(input_shape), nodes, prev)


GRAPH = chain("ckpt-mlp", (12,), [("fc1", "dense", {"units": 16}), ("act", "relu", {}),
                                  ("fc2", "dense", {"units": 4})])


def synthetic(kind):
    params = engine.init_params(GRAPH, 5)
    m = {k: (np.arange(v.size, dtype=np.float32).reshape(v.shape) * np.float32(0.001)) for k, v in params.items()}
    if kind == "adam":
        v = {k: a * a for k, a in m.items()}
        return Checkpoint("job-a", 2, 2, "adam", 17, 0.0, params, slot_m=m, slot_v=v)
    return Checkpoint("job-m", 1, 1, "sgd", 9, 0.9, params, slot_momentum=m)


def dataset():
    g = np.random.default_rng(11)
    centres = g.uniform(-2, 2, size=(4, 12))
    out = {}
    for split, n in (("train", 96), ("test", 40)):
        y = g.integers(0, 4, size=n)
        out[f"{split}_x"] = (centres[y] + g.normal(0, 0.5, size=(n, 12))).astype(np.float32)
        out[f"{split}_y"] = y.astype(np.float32)
    return store.decode(formats.encode_dataset(out)), out


def paused(kind):
    ds, _ = dataset()
    lr = 0.01 if kind == "adam" else 0.1
    job = TrainingJob(f"p-{kind}", GRAPH, ds.content_hash, HyperParams(3, 16, lr, kind, (2,), 3), 0, 0)
    h = merge([job])
    tr = Trainer(h, make_plan("fcfs", [job]), [job], {job.job_id: ds},
                 slice_observer=lambda jid, e: tr.request_pause(jid))
    tr.run()
    ckpt = tr.checkpoints[job.job_id]
    h2 = merge([job])
    restore_checkpoint(h2, ckpt)
    job2 = TrainingJob(job.job_id, GRAPH, ds.content_hash, job.hypers, 0, 0, completed_epochs=1)
    Trainer(h2, make_plan("fcfs", [job2]), [job2], {job.job_id: ds}).run()
    final = {pid: h2.params[pid].copy() for pid in h2.sub(job.job_id).param_ids()}
    return ckpt.encode(), final


if __name__ == "__main__":
    for kind in ("adam", "momentum"):
        (HERE / f"checkpoint_synthetic_{kind}.bin").write_bytes(synthetic(kind).encode())
    finals = {}
    for kind in ("adam", "sgd"):
        blob, final = paused(kind)
        (HERE / f"checkpoint_paused_{kind}.bin").write_bytes(blob)
        finals.update({f"{kind}/{k}": v for k, v in final.items()})
    _, splits = dataset()
    np.savez(HERE / "checkpoint_resumed.npz", **finals, **{f"data/{k}": v for k, v in splits.items()})
    print(sorted(finals))
