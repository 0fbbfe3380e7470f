"""Golden UNND v2 model files written by the unmodified reference (hybridnn.separate.package).

Run in the build container (the reference is importable from /root/reference/pkg/src):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_package_golden.py
Writes tests/golden/package_{mlp,conv}.bin; tests/test_host.py checks our package() is
byte-identical and load_package() round-trips them.
"""
from pathlib import Path

from hybridnn import engine
from hybridnn.model import ModelGraph, OpNode
from hybridnn.separate import package

HERE = Path(__file__).resolve().parent


def chain(name, input_shape, spec):
    nodes, prev = [], "input"
    for nid, op, attrs in spec:
        nodes.append(OpNode(nid, op, [prev], dict(attrs)))
        prev = nid
    return ModelGraph(name, tuple(input_shape), nodes, prev)


GRAPHS = {
    "mlp": chain("pkg-mlp", (12,), [("fc1", "dense", {"units": 6}), ("act", "relu", {}),
                                    ("fc2", "dense", {"units": 3})]),
    "conv": chain("pkg-conv", (2, 6, 6), [("conv", "conv2d", {"filters": 3, "kernel": 3, "padding": 1}),
                                          ("act", "relu", {}), ("pool", "maxpool2d", {"kernel": 2}),
                                          ("flat", "flatten", {}), ("fc", "dense", {"units": 4})]),
}

if __name__ == "__main__":
    for tag, graph in GRAPHS.items():
        params = engine.init_params(graph, 7)
        (HERE / f"package_{tag}.bin").write_bytes(package(graph, params))
        print(tag, sum(p.size for p in params.values()))
