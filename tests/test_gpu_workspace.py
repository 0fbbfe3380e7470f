"""The reference's own end-to-end workflow on the B200 trainer.

The unmodified reference package, installed offline into baseline/_ref (DESIGN.md "Reference
install"), runs ``Workspace.run`` twice over the same submissions: once as shipped (numpy, CPU)
and once with ``paper_2408_01331_b200.backend.install`` routing its training path to the GPU.
Everything around training — queue, dataset store, separator thread, report files, memory model,
pause markers, checkpoint files, resume — is the reference's code in both runs.

Compared: job statuses and epochs, per-epoch curves and test metrics (rel 1e-3, the trajectory bound of
test_gpu_parity.py; test accuracy within one sample of the tiny test splits), the packaged output models (UNND v2) parameter by
parameter (rel 1e-3), and a job paused by a marker file, whose UNND v3 checkpoint the reference's
``Workspace.resume`` re-queues and the GPU run then finishes.
"""
import json
import sys

import numpy as np
import pytest

import oracle
from conftest import REPO

pytestmark = pytest.mark.gpu

REF = REPO / "baseline" / "_ref"


@pytest.fixture(scope="module")
def hybridnn():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not (REF / "hybridnn").exists():
        pytest.skip("reference not installed in baseline/_ref (python -m pip install --target baseline/_ref ...)")
    sys.path.insert(0, str(REF))
    try:
        import hybridnn as mod
    finally:
        sys.path.remove(str(REF))
    return mod


def rel(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-6)) if ref.size else 0.0


def _submissions(hn):
    from paper_2408_01331_b200 import zoo

    blob = hn.formats.encode_dataset(oracle.blob_splits("ws", "blob", 4, 20, 160, 64))
    image = hn.formats.encode_dataset(oracle.image_splits("ws", "img", 10, (1, 12, 12), 96, 48))
    to_ref = lambda g: hn.ModelGraph.from_dict(g.to_dict())
    mlp = hn.workspace.architecture_blob(to_ref(zoo.mlp(20, (32, 16), 4)))
    cnn = to_ref(zoo._seq("tiny-cnn", (1, 12, 12), [
        ("conv1", "conv2d", {"filters": 4, "kernel": 3, "padding": 1}), ("act1", "relu", {}),
        ("pool1", "maxpool2d", {"kernel": 2}), ("flat", "flatten", {}), ("fc", "dense", {"units": 10})]))
    cnn = hn.workspace.architecture_blob(cnn)
    hyp = lambda **kw: json.dumps(dict({"epochs": 3, "batch_size": 32, "learning_rate": 0.05, "optimizer": "sgd",
                                        "seed": 1}, **kw))
    return [(mlp, blob, hyp()), (mlp, blob, hyp(optimizer="adam", learning_rate=1e-3, lr_milestones=[2], seed=2)),
            (cnn, image, hyp(batch_size=16, seed=3)), (mlp, blob, hyp(epochs=2, seed=4))]


def _run(hn, root, pause=None):
    ws = hn.Workspace(root)
    ids = [ws.submit(*s) for s in _submissions(hn)]
    if pause is not None:  # a marker present when the run starts: paused before its first slice
        ws._marker(ids[pause]).touch()
    report = ws.run("rr")
    return ws, ids, report


def _outputs(ws, ids):
    from paper_2408_01331_b200 import load_package

    return {j: load_package((ws.root / "outputs" / f"{j}.unnd").read_bytes())[1] for j in ids
            if (ws.root / "outputs" / f"{j}.unnd").exists()}


def test_reference_workspace_runs_on_the_b200_trainer(hybridnn, tmp_path):
    from paper_2408_01331_b200 import backend
    from paper_2408_01331_b200.train import Trainer

    ref_ws, ids, ref_report = _run(hybridnn, tmp_path / "ref", pause=3)
    backend.install(hybridnn)
    try:
        assert backend.installed(hybridnn) and hybridnn.workspace.Trainer is Trainer
        gpu_ws, gids, report = _run(hybridnn, tmp_path / "gpu", pause=3)
        paused = ids[3]
        assert ids == gids
        # the paused job: the reference's checkpoint file, re-queued by the reference's resume
        blob = (gpu_ws.root / "checkpoints" / f"{paused}.unnd").read_bytes()
        assert blob == (ref_ws.root / "checkpoints" / f"{paused}.unnd").read_bytes()  # init state, same bytes
        gpu_ws.resume(paused, blob)
        resumed = gpu_ws.run("rr")
    finally:
        backend.uninstall(hybridnn)
    assert not backend.installed(hybridnn)
    ref_ws.resume(paused, blob)
    ref_resumed = ref_ws.run("rr")

    for rep, ref in ((report, ref_report), (resumed, ref_resumed)):
        got, want = rep.to_dict(), ref.to_dict()
        assert sorted(got["jobs"]) == sorted(want["jobs"])
        for j, r in want["jobs"].items():
            g = got["jobs"][j]
            assert (g["status"], g["epochs_completed"]) == (r["status"], r["epochs_completed"]), j
            for (e, l, a), (re_, rl, ra) in zip(g["curve"], r["curve"]):
                assert e == re_ and abs(l - rl) <= 1e-3 * abs(rl) and abs(a - ra) <= 0.01, (j, e)
            if r["status"] == "complete":
                assert abs(g["final_test_loss"] - r["final_test_loss"]) <= 1e-3 * abs(r["final_test_loss"])
                # (48- / 64-sample test splits: one prediction is 1.6-2.1%; allow at most one flip)
                assert abs(g["final_test_accuracy"] - r["final_test_accuracy"]) <= 1 / 48 + 1e-12
    assert report.jobs[paused].status == "paused" and resumed.jobs[paused].status == "complete"
    got, want = _outputs(gpu_ws, ids), _outputs(ref_ws, ids)
    assert sorted(got) == sorted(want) == sorted(ids)
    for j in ids:
        for pid, v in want[j].items():
            assert rel(got[j][pid], v) <= 1e-3, (j, pid, rel(got[j][pid], v))
    for name in ("report.json", "memory.json", "training_curves.csv"):
        assert (gpu_ws.root / "reports" / name).exists()
    assert json.loads((gpu_ws.root / "queue.json").read_text())["jobs"][3]["status"] == "complete"
