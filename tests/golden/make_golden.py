"""Regenerate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs only in the build container, where /root/reference exists:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

The reference package ``hybridnn`` is imported from baseline/_ref (if
installed) or /root/reference/pkg/src and driven through its public API
(``train_standalone``, ``Trainer``, ``evaluate``, ``OP_KINDS``).  Datasets
come from keyed generators (oracle.blob_splits / image_splits) so the GPU
box can regenerate identical bytes; each fixture stores the dataset digest
to prove it.  Outputs: *.npz / *.json next to this script.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
for cand in (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (cand / "hybridnn").exists():
        sys.path.insert(0, str(cand))
        break

import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

import hybridnn  # noqa: E402
from hybridnn import formats, store, unify  # noqa: E402
from hybridnn.model import HyperParams, ModelGraph, TrainingJob  # noqa: E402
from hybridnn.ops import OP_KINDS  # noqa: E402
from hybridnn.schedule import make_plan  # noqa: E402
from hybridnn.train import Trainer, train_standalone  # noqa: E402

import oracle  # noqa: E402
from paper_2408_01331_b200 import zoo  # noqa: E402

# the fixture cases; tests import this table to rebuild identical inputs
CASES = {
    "c1_mlp": dict(graph="mlp784", data=("blob", "c1-mini", 10, 784, 640, 200), epochs=2, batch=64, lr=0.05,
                   opt="sgd", seed=1),
    "deep_adam": dict(graph="mlp12", data=("blob", "four", 4, 12, 96, 32), epochs=3, batch=16, lr=0.01,
                      opt="adam", seed=2),
    "lenet": dict(graph="lenet", data=("image", "cifar-mini", 10, (3, 32, 32), 384, 128), epochs=2, batch=128,
                  lr=0.01, opt="sgd", seed=3),
    "c3_mlp": dict(graph="c3h128", data=("blob", "c1-mini", 10, 784, 640, 200), epochs=1, batch=256, lr=1e-3,
                   opt="adam", seed=5),
}


def case_graph(kind):
    if kind == "mlp784":
        return zoo.mlp(784, (256,), 10)
    if kind == "mlp12":
        return zoo.mlp(12, (24, 16), 4, name="mlp-3")
    if kind == "lenet":
        return zoo.lenet5()
    if kind == "c3h128":
        return zoo.mlp(784, (128, 128), 10)
    raise ValueError(kind)


def case_splits(data):
    if data[0] == "blob":
        _, name, classes, feats, ntr, nte = data
        return oracle.blob_splits("golden", name, classes, feats, ntr, nte)
    _, name, classes, shape, ntr, nte = data
    return oracle.image_splits("golden", name, classes, shape, ntr, nte)


def ref_graph(g):
    return ModelGraph.from_dict(g.to_dict())


def ref_dataset(splits):
    return store.decode(formats.encode_dataset(splits))


def ref_job(job_id, graph, ds, c, seq=0):
    return TrainingJob(job_id, ref_graph(graph), ds.content_hash,
                       HyperParams(c["epochs"], c["batch"], c["lr"], c["opt"], (), c["seed"]), seq, seq)


def trajectory_case(name, c, snapshot_steps=(0,)):
    graph = case_graph(c["graph"])
    splits = case_splits(c["data"])
    ds = ref_dataset(splits)
    job = ref_job(name, graph, ds, c)
    losses, snaps = [], {}
    step = [0]

    def observe(_jid, params):
        if step[0] in snapshot_steps:
            for pid, arr in params.items():
                snaps[f"step{step[0]}/{pid}"] = arr.copy()
        step[0] += 1

    params, opt = train_standalone(job, ds, step_observer=observe)
    # per-step losses + the trainer's curve/test metrics via the Trainer API
    trainer = Trainer(unify.merge([job]), make_plan("fcfs", [job]), [job], {name: ds})
    report = trainer.run().jobs[name]
    out = {f"final/{pid}": arr for pid, arr in params.items()}
    out.update(snaps)
    # losses of every step, recomputed through the reference's run_batch on a fresh model
    from hybridnn import engine
    from hybridnn.optim import OptimizerState, lr_at_epoch
    from hybridnn.train import run_batch

    p2 = engine.init_params(job.graph, c["seed"])
    o2 = OptimizerState.fresh(c["opt"])
    order = hybridnn.validate_graph(job.graph)
    corrects = []
    for e in range(c["epochs"]):
        for b in store.batches(ds, c["batch"], c["seed"], e):
            loss, corr = run_batch(job.graph, p2, order, b, o2, lr_at_epoch(c["lr"], (), e))
            losses.append(loss)
            corrects.append(corr)
    for pid in params:
        assert np.array_equal(p2[pid], params[pid])
    out["losses"] = np.asarray(losses, dtype=np.float64)
    out["corrects"] = np.asarray(corrects, dtype=np.int64)
    out["perm_epoch0"] = hybridnn.rng.permutation(ds.sample_count, "shuffle", ds.content_hash, c["seed"], 0)
    out["curve"] = np.asarray(report.curve, dtype=np.float64)
    out["test"] = np.asarray([report.final_test_loss, report.final_test_accuracy], dtype=np.float64)
    out["opt_step"] = np.asarray(opt.step)
    meta = {"digest": ds.content_hash, "case": {k: (list(v) if isinstance(v, tuple) else v) for k, v in c.items()}}
    out["meta"] = np.asarray(json.dumps(meta, default=list))
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "steps", len(losses), "final loss", losses[-1])


def ops_case():
    """Op-level vectors through the reference registry (forward + backward)."""
    g = oracle.keyed_generator("golden", "ops")
    out = {}

    def run(tag, op, x, params, attrs, dy, targets=None):
        kind = OP_KINDS[op]
        x32 = np.asarray(x, dtype=np.float32)
        p32 = {k: np.asarray(v, dtype=np.float32) for k, v in params.items()}
        if kind.takes_targets:
            y, aux = kind.forward(x32, p32, attrs, targets=targets)
        else:
            y, aux = kind.forward(x32, p32, attrs)
        dx, dp = kind.backward(np.asarray(dy, dtype=np.float32), aux, p32, attrs)
        out[f"{tag}/x"] = x32
        for k, v in p32.items():
            out[f"{tag}/p_{k}"] = v
        out[f"{tag}/dy"] = np.asarray(dy, dtype=np.float32)
        out[f"{tag}/y"] = np.asarray(y)
        if dx is not None:
            out[f"{tag}/dx"] = dx
        for k, v in dp.items():
            out[f"{tag}/d_{k}"] = v
        out[f"{tag}/attrs"] = np.asarray(json.dumps(attrs))
        if targets is not None:
            out[f"{tag}/targets"] = np.asarray(targets, dtype=np.float32)

    run("dense", "dense", g.normal(size=(7, 13)), {"weight": g.normal(size=(5, 13)), "bias": g.normal(size=5)},
        {"units": 5}, g.normal(size=(7, 5)))
    xr = g.normal(size=(6, 9))
    xr[0, :3] = 0.0
    run("relu", "relu", xr, {}, {}, g.normal(size=(6, 9)))
    run("conv_k3s2p1", "conv2d", g.normal(size=(2, 3, 9, 9)),
        {"weight": g.normal(size=(4, 3, 3, 3)), "bias": g.normal(size=4)},
        {"filters": 4, "kernel": 3, "stride": 2, "padding": 1}, g.normal(size=(2, 4, 5, 5)))
    run("conv_k5", "conv2d", g.normal(size=(2, 3, 12, 12)),
        {"weight": g.normal(size=(6, 3, 5, 5)), "bias": g.normal(size=6)},
        {"filters": 6, "kernel": 5}, g.normal(size=(2, 6, 8, 8)))
    xp = np.round(g.normal(size=(2, 3, 9, 9)) * 2) / 2  # many ties
    run("pool_k3s2", "maxpool2d", xp, {}, {"kernel": 3, "stride": 2}, g.normal(size=(2, 3, 4, 4)))
    run("pool_k2", "maxpool2d", g.normal(size=(3, 2, 8, 8)), {}, {"kernel": 2}, g.normal(size=(3, 2, 4, 4)))
    logits = g.normal(size=(9, 10)) * 3
    logits[0] = [800.0, -800.0] + [0.0] * 8
    run("sce", "softmax-cross-entropy", logits, {}, {}, np.float32(1.0),
        targets=g.integers(0, 10, size=9).astype(np.float64))
    np.savez_compressed(HERE / "ops.npz", **out)
    print("ops", len(out), "arrays")


def trainer_case():
    """Two jobs through Trainer (rr) plus a poison job that must abort alone."""
    ga, gb = case_graph("mlp12"), zoo.mlp(8, (16,), 2, name="mlp-2")
    sa = oracle.blob_splits("golden", "four", 4, 12, 96, 32)
    sb = oracle.blob_splits("golden", "two", 2, 8, 64, 32)
    da, db = ref_dataset(sa), ref_dataset(sb)
    ja = TrainingJob("a", ref_graph(ga), da.content_hash, HyperParams(3, 16, 0.01, "adam", (2,), 2), 0, 0)
    jb = TrainingJob("b", ref_graph(gb), db.content_hash, HyperParams(2, 16, 0.05, "sgd", (), 1), 1, 1)
    jbad = TrainingJob("bad", ref_graph(gb), db.content_hash, HyperParams(3, 16, 1e8, "sgd", (), 0), 2, 2)
    jobs = [ja, jb, jbad]
    trainer = Trainer(unify.merge(jobs), make_plan("rr", jobs), jobs, {"a": da, "b": db, "bad": db})
    report = trainer.run()
    rows = {}
    for jid, res in report.jobs.items():
        rows[jid] = {
            "status": res.status,
            "curve": [list(r) for r in res.curve],
            "final_test_loss": res.final_test_loss,
            "final_test_accuracy": res.final_test_accuracy,
            "abort_reason": res.abort_reason,
            "epochs_completed": res.epochs_completed,
        }
    params = {pid: arr.tolist() for pid, arr in trainer.hybrid.params.items() if not pid.startswith("bad/")}
    (HERE / "trainer_rr.json").write_text(json.dumps({"jobs": rows, "params": params}, sort_keys=True))
    print("trainer", {k: v["status"] for k, v in rows.items()})


def main():
    with threadpool_limits(1):
        for name, c in CASES.items():
            trajectory_case(name, c, snapshot_steps=(0,))
        ops_case()
        trainer_case()


if __name__ == "__main__":
    main()
