"""Benchmark model graphs and synthetic datasets (BASELINE.md "Configs" table).

Graphs use only the reference op set, so every one of them also runs
through the CPU oracle.  ResNet-18 is the "plain" 17-conv variant (no
residual add / batch-norm exist in the reference IR, SURVEY.md finding 6).
Datasets use the reference's generator forms (blob: pkg/tests/conftest.py:59-70,
image: src/demo.py:113-124) on keyed streams ``("bench-data", name, split)``.
"""
from __future__ import annotations

import numpy as np

from . import rng, store
from .model import HyperParams, ModelGraph, OpNode, TrainingJob


def _seq(name, input_shape, spec):
    """Build a chain graph from [(id, op, attrs)]."""
    nodes, prev = [], "input"
    for nid, op, attrs in spec:
        nodes.append(OpNode(nid, op, [prev], dict(attrs)))
        prev = nid
    return ModelGraph(name, tuple(input_shape), nodes, prev)


def mlp(features=784, hidden=(256,), classes=10, name=None):
    spec = []
    for i, h in enumerate(hidden, 1):
        spec += [(f"fc{i}", "dense", {"units": h}), (f"act{i}", "relu", {})]
    spec.append((f"fc{len(hidden) + 1}", "dense", {"units": classes}))
    return _seq(name or "mlp-" + "-".join(map(str, (features, *hidden, classes))), (features,), spec)


def lenet5(channels=3, side=32, classes=10):
    """conv5x6 > pool2 > conv5x16 > pool2 > fc120 > fc84 > fc10 (62,006 params at 3x32x32)."""
    return _seq("lenet-5", (channels, side, side), [
        ("conv1", "conv2d", {"filters": 6, "kernel": 5}), ("act1", "relu", {}),
        ("pool1", "maxpool2d", {"kernel": 2}),
        ("conv2", "conv2d", {"filters": 16, "kernel": 5}), ("act2", "relu", {}),
        ("pool2", "maxpool2d", {"kernel": 2}),
        ("flat", "flatten", {}),
        ("fc1", "dense", {"units": 120}), ("act3", "relu", {}),
        ("fc2", "dense", {"units": 84}), ("act4", "relu", {}),
        ("fc3", "dense", {"units": classes}),
    ])


def vgg11_nobn(classes=10):
    spec, cin, i = [], 3, 0
    for v in (64, "M", 128, "M", 256, 256, "M", 512, 512, "M", 512, 512, "M"):
        if v == "M":
            spec.append((f"pool{i}", "maxpool2d", {"kernel": 2}))
        else:
            spec += [(f"conv{i}", "conv2d", {"filters": v, "kernel": 3, "padding": 1}), (f"act{i}", "relu", {})]
        i += 1
    spec += [("flat", "flatten", {}), ("fc", "dense", {"units": classes})]
    return _seq("vgg-11-nobn", (3, 32, 32), spec)


def resnet18_plain(classes=10):
    spec = [("conv0", "conv2d", {"filters": 64, "kernel": 3, "padding": 1}), ("act0", "relu", {})]
    i = 1
    for width, first_stride in ((64, 1), (128, 2), (256, 2), (512, 2)):
        for j in range(4):
            s = first_stride if j == 0 else 1
            spec += [(f"conv{i}", "conv2d", {"filters": width, "kernel": 3, "padding": 1, "stride": s}),
                     (f"act{i}", "relu", {})]
            i += 1
    spec += [("pool", "maxpool2d", {"kernel": 4}), ("flat", "flatten", {}), ("fc", "dense", {"units": classes})]
    return _seq("resnet-18-plain", (3, 32, 32), spec)


# ------------------------------------------------------------------ datasets


def blob_dataset(name="mnist", classes=10, features=784, train_n=60000, test_n=10000, sigma=0.5, tag="bench-data"):
    centres = rng.stream(tag, name, "centers").uniform(-2.0, 2.0, size=(classes, features))
    splits = {}
    for split, n in (("train", train_n), ("test", test_n)):
        g = rng.stream(tag, name, split)
        y = g.integers(0, classes, size=n)
        splits[f"{split}_x"] = (centres[y] + g.normal(0.0, sigma, size=(n, features))).astype(np.float32)
        splits[f"{split}_y"] = y.astype(np.float32)
    return store.from_splits(splits)


def image_dataset(name="cifar", classes=10, shape=(3, 32, 32), train_n=50000, test_n=10000, sigma=0.35,
                  tag="bench-data"):
    pats = rng.stream(tag, name, "patterns").uniform(0.0, 1.0, size=(classes,) + tuple(shape))
    splits = {}
    for split, n in (("train", train_n), ("test", test_n)):
        g = rng.stream(tag, name, split)
        y = g.integers(0, classes, size=n)
        splits[f"{split}_x"] = (pats[y] + g.normal(0.0, sigma, size=(n,) + tuple(shape))).astype(np.float32)
        splits[f"{split}_y"] = y.astype(np.float32)
    return store.from_splits(splits)


def job(job_id, graph, dataset, seq, epochs=1, batch_size=64, lr=0.01, optimizer="sgd", seed=0, milestones=()):
    return TrainingJob(job_id, graph, dataset.content_hash,
                       HyperParams(epochs, batch_size, lr, optimizer, tuple(milestones), seed), seq, seq)


# ------------------------------------------------------------ config builders


def c3_width(i: int) -> int:
    """C3 hidden width of model i: 128*(1 + i mod 16)."""
    return 128 * (1 + i % 16)


def config_jobs(config: str, dataset, first_model=0, count=None, epochs=1):
    """Jobs of a BASELINE config ("c1" .. "c5") with global model ids."""
    if config == "c1":
        ids, make = range(2), lambda i: job(f"m{i:03d}", mlp(), dataset, i, epochs, 64, (0.01, 0.05)[i], "sgd", i)
    elif config == "c2":
        ids, make = range(8), lambda i: job(f"m{i:03d}", lenet5(), dataset, i, epochs, 128, 0.01, "sgd", i)
    elif config == "c3":
        ids = range(32)

        def make(i):
            h = c3_width(i)
            return job(f"m{i:03d}", mlp(784, (h, h), 10), dataset, i, epochs, 256, 1e-3, "adam", i)
    elif config == "c4":
        # 32 mixed CNNs, 4 per GPU: {ResNet-18-plain, VGG-11-noBN, 2 x LeNet-5}
        ids = range(32)

        def make(i):
            graph = (resnet18_plain, vgg11_nobn, lenet5, lenet5)[i % 4]()
            return job(f"m{i:03d}", graph, dataset, i, epochs, 128, 1e-3, "sgd", i)
    elif config == "c5":
        ids = range(256)

        def make(i):
            return job(f"m{i:03d}", mlp(), dataset, i, epochs, 64, float(10 ** (-3 + 2 * i / 255)), "sgd", i)
    else:
        raise ValueError(config)
    n = len(ids) if count is None else count
    return [make(first_model + k) for k in range(n)]
