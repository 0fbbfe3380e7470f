"""Golden results of whole training runs at BASELINE configs, from the UNMODIFIED reference.

Runs only in the build container, where /root/reference exists:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_training_golden.py

Writes tests/golden/baseline_training.json.  Each case is trained through the reference's
public API (``merge`` + ``Trainer(...).run()``, src/train.py:294-446), one BLAS thread; the GPU
tests (tests/test_gpu_baseline_parity.py) rebuild the same inputs from the keyed generators and
compare their per-epoch curves, test metrics and parameter checksums with these numbers:

* ``c1``   BASELINE C1 exactly: 2 x MLP 784-256-10 on the 60,000 x 784 MNIST-shaped blob set
           (bench data, 10,000 test samples), batch 64, SGD lr 0.01 / 0.05, seeds 0 / 1, one epoch
           = 938 steps per model.
* ``bf16`` the C4-style short run the bf16 path is held to: LeNet-5 and a VGG slice
           (conv3x3x64 > pool4 > conv3x3x64 > pool2 > fc10) on CIFAR-shaped 32x32x3 images
           (2,048 train / 1,000 test), batch 32, SGD lr 0.03, 3 epochs (192 steps per model).
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

from hybridnn import formats, store, unify  # noqa: E402
from hybridnn.model import HyperParams, ModelGraph, TrainingJob  # noqa: E402
from hybridnn.schedule import make_plan  # noqa: E402
from hybridnn.train import Trainer  # noqa: E402

import oracle  # noqa: E402
from paper_2408_01331_b200 import zoo  # noqa: E402

sys.path.insert(0, str(HERE))
from training_cases import BF16_CASE, bf16_jobs_spec  # noqa: E402


def checksums(params: dict) -> dict:
    """Per-parameter float64 sum, sum of |x| and 64 fixed elements (flat indices spread over the tensor)."""
    out = {}
    for pid, arr in params.items():
        flat = np.asarray(arr, dtype=np.float32).reshape(-1)
        idx = np.linspace(0, flat.size - 1, num=min(64, flat.size)).astype(np.int64)
        out[pid] = {"sum": float(flat.astype(np.float64).sum()), "abs": float(np.abs(flat.astype(np.float64)).sum()),
                    "idx": idx.tolist(), "val": flat[idx].astype(np.float64).tolist()}
    return out


def run_reference(jobs_spec, splits, batch, lrs, epochs, seeds):
    ds = store.decode(formats.encode_dataset(splits))
    jobs = [TrainingJob(jid, ModelGraph.from_dict(g.to_dict()), ds.content_hash,
                        HyperParams(epochs, batch, lr, "sgd", (), seed), i, i)
            for i, ((jid, g), lr, seed) in enumerate(zip(jobs_spec, lrs, seeds))]
    hybrid = unify.merge(jobs)
    report = Trainer(hybrid, make_plan("rr", jobs), jobs, {j.job_id: ds for j in jobs}).run()
    out = {"digest": ds.content_hash, "jobs": {}}
    for j in jobs:
        r = report.jobs[j.job_id]
        sub = {k.split("/", 1)[1]: v for k, v in hybrid.sub_params(j.job_id).items()}
        out["jobs"][j.job_id] = {"status": r.status, "curve": [list(map(float, c)) for c in r.curve],
                                 "final_test_loss": r.final_test_loss, "final_test_accuracy": r.final_test_accuracy,
                                 "params": checksums(sub)}
    return out


def main():
    res = {}
    with threadpool_limits(1):
        ds = zoo.blob_dataset()  # the bench's C1 data (keyed "bench-data" generators)
        splits = {"train_x": ds.train_x, "train_y": ds.train_y, "test_x": ds.test_x, "test_y": ds.test_y}
        cfg = zoo.config_jobs("c1", ds)
        res["c1"] = run_reference([(j.job_id, j.graph) for j in cfg], splits, 64,
                                  [j.hypers.learning_rate for j in cfg], 1, [j.hypers.seed for j in cfg])
        print("c1", {k: (v["final_test_loss"], v["final_test_accuracy"]) for k, v in res["c1"]["jobs"].items()})
        c = BF16_CASE
        splits = oracle.image_splits(*c["data"])
        spec = bf16_jobs_spec()
        res["bf16"] = run_reference([(jid, g) for jid, g, _ in spec], splits, c["batch"], [c["lr"]] * len(spec),
                                    c["epochs"], [s for _, _, s in spec])
        print("bf16", {k: (v["final_test_loss"], v["final_test_accuracy"]) for k, v in res["bf16"]["jobs"].items()})
    (HERE / "baseline_training.json").write_text(json.dumps(res, sort_keys=True))


if __name__ == "__main__":
    main()
