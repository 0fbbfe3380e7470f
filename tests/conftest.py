"""Shared test fixtures.  ``gpu``-marked tests need a B200; everything else runs on CPU."""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402
import pytest  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(autouse=True)
def _single_blas_thread():
    """The oracle's bits depend on the BLAS thread count (SURVEY finding 5): pin 1."""
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        yield


def load_case(name):
    """(fixture arrays, case dict, graph, splits) for a tests/golden trajectory case."""
    import oracle
    from paper_2408_01331_b200 import zoo

    arr = np.load(GOLDEN / f"{name}.npz")
    meta = json.loads(str(arr["meta"]))
    c = meta["case"]
    graph = {
        "mlp784": lambda: zoo.mlp(784, (256,), 10),
        "mlp12": lambda: zoo.mlp(12, (24, 16), 4, name="mlp-3"),
        "lenet": lambda: zoo.lenet5(),
        "c3h128": lambda: zoo.mlp(784, (128, 128), 10),
    }[c["graph"]]()
    data = c["data"]
    if data[0] == "blob":
        splits = oracle.blob_splits("golden", *data[1:])
    else:
        splits = oracle.image_splits("golden", data[1], data[2], tuple(data[3]), data[4], data[5])
    assert oracle.dataset_digest(splits) == meta["digest"], "regenerated golden data drifted"
    return arr, c, graph, splits, meta["digest"]


def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
