"""Host-side logic and the C-ABI library surface (no GPU needed)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, REPO, load_case

import paper_2408_01331_b200 as h
from paper_2408_01331_b200 import _native, store, zoo
from paper_2408_01331_b200.runtime import lower_graph


def header_symbols():
    text = (REPO / "include" / "hnn_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(hnn_\w+)\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 14
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"binding misses {name}"
    assert lib.hnn_version().startswith(b"hnn_b200")


def test_abi_struct_layouts_match_binding():
    lib = _native.load()
    for name, cls in _native.STRUCTS.items():
        import ctypes

        assert lib.hnn_struct_size(name.encode()) == ctypes.sizeof(cls), name


def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_merge_validation_mirrors_reference():
    with pytest.raises(h.StateError, match="empty"):
        h.merge([])
    ds = store.from_splits(oracle.blob_splits("t", "v", 2, 8, 16, 4))
    good = zoo.job("a", zoo.mlp(8, (16,), 2), ds, 0)
    bad = zoo.job("b", zoo.mlp(8, (16,), 2), ds, 1)
    del bad.graph.nodes[0].attrs["units"]
    bad2 = zoo.job("c", zoo.mlp(8, (16,), 2), ds, 2)
    bad2.graph.nodes[1].inputs = ["ghost"]
    with pytest.raises(h.MergeError) as info:
        h.merge([good, bad, bad2])
    assert set(info.value.per_job) == {"b", "c"}
    assert any("missing attr" in p for p in info.value.per_job["b"])
    assert any("unknown input" in p for p in info.value.per_job["c"])
    with pytest.raises(h.MergeError) as info:
        h.merge([good, zoo.job("a", zoo.mlp(8, (16,), 2), ds, 3)])
    assert any("duplicate" in p for p in info.value.per_job["a"])


def test_init_is_bit_exact_and_merge_order_free():
    g1, g2 = zoo.mlp(784, (256,), 10), zoo.lenet5()
    ds = store.from_splits(oracle.blob_splits("t", "w", 2, 8, 16, 4))
    j1, j2 = zoo.job("x", g1, ds, 0, seed=3), zoo.job("y", g2, ds, 1, seed=4)
    a, b = h.merge([j1, j2]), h.merge([j2, j1])
    for pid in a.params:
        assert np.array_equal(a.params[pid], b.params[pid])
    for job in (j1, j2):
        ref = oracle.init_model(job.graph, job.hypers.seed)
        assert list(h.param_specs(job.graph)) == list(oracle.param_layout(job.graph))
        for pid, v in ref.items():
            assert np.array_equal(a.params[f"{job.job_id}/{pid}"], v)


def test_namespacing_and_routing_nodes():
    ds = store.from_splits(oracle.blob_splits("t", "w", 2, 8, 16, 4))
    hy = h.merge([zoo.job("a", zoo.mlp(8, (16,), 2), ds, 0), zoo.job("b", zoo.lenet5(), ds, 1)])
    assert hy.job_ids() == ["a", "b"]
    assert hy.global_input.node_id == "hybrid/input" and hy.global_output.routes["a"] == "a/fc2"
    assert hy.node_count() == 3 + 12 + 2
    assert hy.sub("a").graph.nodes[0].inputs == ["input"]
    with pytest.raises(h.UnknownJobError):
        hy.sub("zzz")
    snap = hy.snapshot()
    snap.params["a/fc1.weight"][0, 0] = 99.0
    assert hy.params["a/fc1.weight"][0, 0] != 99.0


def test_batches_and_hash_match_oracle():
    splits = oracle.blob_splits("t", "b", 3, 5, 23, 4)
    ds = store.from_splits(splits)
    assert ds.content_hash == oracle.dataset_digest(splits)
    got = store.batches(ds, 4, 7, 2)
    ref = oracle.epoch_batches(splits["train_x"], splits["train_y"], ds.content_hash, 4, 7, 2)
    assert [b.x.shape[0] for b in got] == [4, 4, 4, 4, 4, 3]
    for b, (x, y, _) in zip(got, ref):
        assert np.array_equal(b.x, x) and np.array_equal(b.y, y)
    assert store.batch_count(60000, 256) == 235


def test_lowering_fuses_relu_and_marks_masks():
    st, classes, head = lower_graph(zoo.lenet5())
    assert [s.kind for s in st] == ["conv", "pool", "conv", "pool", "dense", "dense", "dense"]
    assert [s.relu for s in st] == [True, False, True, False, True, True, False]
    assert [s.mask_input for s in st] == [False, True, False, True, False, True, True]
    assert [s.needs_dx for s in st] == [False, True, True, True, True, True, True]
    assert classes == 10 and not head
    # a relu that ends the graph stays a stand-alone stage
    g = zoo.mlp(8, (4,), 3)
    g.nodes.append(h.OpNode("act_out", "relu", [g.output]))
    g.output = "act_out"
    st, _, _ = lower_graph(g)
    assert [s.kind for s in st] == ["dense", "dense", "relu"]


def test_schedule_rows_follow_reference_batches_and_adam_steps():
    from paper_2408_01331_b200.train import Trainer, _Track

    splits = oracle.blob_splits("t", "s", 2, 8, 70, 4)
    ds = store.from_splits(splits)
    job = zoo.job("a", zoo.mlp(8, (16,), 2), ds, 0, epochs=3, batch_size=32, lr=0.1, optimizer="adam",
                  milestones=(2,))
    hy = h.merge([job])
    tr = Trainer(hy, h.make_plan("fcfs", [job]), [job], {"a": ds})
    track = _Track(job, 0, ds, [0, 1, 2])
    rows = tr._window_rows({"a": track}, 0, track.total)
    assert track.spe == 3 and track.total == 9
    assert rows["rows"][:, 0].tolist() == [32, 32, 6] * 3
    assert rows["perm_base"][:, 0].tolist() == [0, 32, 64] * 3
    assert rows["epoch"][:, 0].tolist() == [0, 0, 0, 1, 1, 1, 2, 2, 2]
    assert rows["opt_step"][:, 0].tolist() == list(range(1, 10))
    # milestone 2 (one-based) decays from zero-based epoch 1 on (src/optim.py:22-30)
    assert np.all(rows["lr"][:3, 0] == np.float32(0.1)) and np.all(rows["lr"][3:, 0] == np.float32(0.1 * 0.1))
    assert rows["bias1"][0, 0] == np.float32(1.0 - 0.9) and rows["bias2"][4, 0] == np.float32(1.0 - 0.999 ** 5)


@pytest.mark.parametrize("tag", ["mlp", "conv"])
def test_package_is_byte_identical_to_reference(tag):
    """package() writes the reference's UNND v2 bytes (src/separate.py:39-59) for the same graph and
    keyed init; load_package() round-trips them (fixtures: tests/golden/make_package_golden.py)."""
    from paper_2408_01331_b200 import init_params, load_package, package, zoo

    spec = {"mlp": ("pkg-mlp", (12,), [("fc1", "dense", {"units": 6}), ("act", "relu", {}),
                                       ("fc2", "dense", {"units": 3})]),
            "conv": ("pkg-conv", (2, 6, 6), [("conv", "conv2d", {"filters": 3, "kernel": 3, "padding": 1}),
                                             ("act", "relu", {}), ("pool", "maxpool2d", {"kernel": 2}),
                                             ("flat", "flatten", {}), ("fc", "dense", {"units": 4})])}[tag]
    graph = zoo._seq(*spec)
    golden = (GOLDEN / f"package_{tag}.bin").read_bytes()
    assert package(graph, init_params(graph, 7)) == golden
    g2, params = load_package(golden)
    assert g2.to_dict() == graph.to_dict()
    for pid, v in init_params(graph, 7).items():
        assert np.array_equal(params[pid], v)
    bad = dict(init_params(graph, 7))
    bad.pop(next(iter(bad)))
    with pytest.raises(Exception):
        package(graph, bad)


@pytest.mark.parametrize("kind", ["adam", "momentum"])
def test_checkpoint_encode_is_byte_identical_to_reference(kind):
    """Checkpoint.encode writes the reference's UNND v3 bytes (src/train.py:57-80,
    src/formats.py:188-201) for the same state; decode inverts it (fixtures:
    tests/golden/make_checkpoint_golden.py, written by the unmodified reference)."""
    from paper_2408_01331_b200 import Checkpoint, init_params, zoo

    graph = zoo.mlp(12, (16,), 4, name="ckpt-mlp")
    params = init_params(graph, 5)
    m = {k: np.arange(v.size, dtype=np.float32).reshape(v.shape) * np.float32(0.001) for k, v in params.items()}
    if kind == "adam":
        ours = Checkpoint("job-a", 2, 2, "adam", 17, 0.0, params, slot_m=m, slot_v={k: a * a for k, a in m.items()})
    else:
        ours = Checkpoint("job-m", 1, 1, "sgd", 9, 0.9, params, slot_momentum=m)
    golden = (GOLDEN / f"checkpoint_synthetic_{kind}.bin").read_bytes()
    assert ours.encode() == golden
    back = Checkpoint.decode(golden)
    assert (back.job_id, back.completed_epochs, back.data_cursor, back.optimizer_kind, back.optimizer_step,
            back.momentum) == (ours.job_id, ours.completed_epochs, ours.data_cursor, ours.optimizer_kind,
                               ours.optimizer_step, ours.momentum)
    for attr in ("params", "slot_m", "slot_v", "slot_momentum"):
        a, b = getattr(back, attr), getattr(ours, attr)
        assert sorted(a) == sorted(b) and all(np.array_equal(a[k], b[k]) for k in a), attr


@pytest.mark.parametrize("kind", ["adam", "sgd"])
def test_checkpoint_decode_reencodes_reference_bytes(kind):
    from paper_2408_01331_b200 import Checkpoint

    golden = (GOLDEN / f"checkpoint_paused_{kind}.bin").read_bytes()
    ck = Checkpoint.decode(golden)
    assert ck.completed_epochs == 1 and ck.data_cursor == 1 and ck.optimizer_kind == kind
    assert ck.encode() == golden


def test_checkpoint_decode_errors_match_reference():
    from paper_2408_01331_b200 import Checkpoint, FormatError, StateError
    from paper_2408_01331_b200 import formats

    golden = (GOLDEN / "checkpoint_paused_sgd.bin").read_bytes()
    with pytest.raises(FormatError, match="truncated container"):
        Checkpoint.decode(golden[:-3])
    with pytest.raises(FormatError, match="trailing bytes"):
        Checkpoint.decode(golden + b"\x00")
    with pytest.raises(FormatError, match="expected format version 3, got 2"):
        Checkpoint.decode(golden[:4] + b"\x02\x00" + golden[6:])
    bad = formats.encode_checkpoint({"job_id": "j", "completed_epochs": 0, "data_cursor": 0,
                                     "optimizer": {"kind": "sgd", "step": 0, "momentum": 0.0}},
                                    {"q/x": np.zeros(2, np.float32)}, ["q/x"])
    with pytest.raises(StateError, match="unrecognized checkpoint section"):
        Checkpoint.decode(bad)


def test_host_gather_rows_matches_store_batches():
    """hnn_host_gather_rows (the host-fed step's data loader) writes Batch(x=train_x[idx],
    y=train_y[idx]) (src/store.py:77-80) into a strided arena, labels as int32; host code only."""
    g = np.random.default_rng(3)
    src = g.normal(size=(50, 7)).astype(np.float32)
    ys = g.integers(0, 9, size=50).astype(np.float32)
    idx = g.permutation(50)[:13].astype(np.int64)
    ld = 8
    dst = np.full((16, ld), -1.0, dtype=np.float32)
    dy = np.full(16, -1, dtype=np.int32)
    _native.call("hnn_host_gather_rows", dst.ctypes.data, ld, dy.ctypes.data, src.ctypes.data, 7, ys.ctypes.data,
                 idx.ctypes.data, idx.size, 7)
    assert np.array_equal(dst[:13, :7], src[idx]) and np.all(dst[:13, 7] == -1) and np.all(dst[13:] == -1)
    assert np.array_equal(dy[:13], ys[idx].astype(np.int32)) and np.all(dy[13:] == -1)
    with pytest.raises(h.DeviceError):
        _native.call("hnn_host_gather_rows", dst.ctypes.data, 4, dy.ctypes.data, src.ctypes.data, 7, ys.ctypes.data,
                     idx.ctypes.data, idx.size, 7)


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_host_gather_batch_matches_per_model_gather(threads):
    """hnn_host_gather_batch (one native call per step for every model, rows split over host
    threads) writes each model's Batch(x=train_x[idx], y=train_y[idx]) (src/store.py:77-80) and
    zeroes the rows of a short final batch, independent of the thread count."""
    g = np.random.default_rng(5)
    items, dsts, expect = [], [], []
    for m, (rows, cap, cols, ld) in enumerate([(13, 16, 7, 8), (0, 4, 5, 5), (64, 64, 33, 36), (30, 32, 1, 4)]):
        src = g.normal(size=(90, cols)).astype(np.float32)
        ys = g.integers(0, 9, size=90).astype(np.float32)
        idx = g.permutation(90)[:rows].astype(np.int64)
        dst = np.full((cap, ld), -1.0, dtype=np.float32)
        dy = np.full(cap, -1, dtype=np.int32)
        keep = (src, ys, idx)
        items.append(_native.HostGatherItem(dst.ctypes.data, dy.ctypes.data, src.ctypes.data, ys.ctypes.data,
                                            idx.ctypes.data if rows else 0, ld, cols, cols, rows, cap))
        dsts.append((dst, dy, keep))
        ex = np.full((cap, ld), -1.0, dtype=np.float32)
        ex[:, :cols] = 0.0
        ex[:rows, :cols] = src[idx]
        ey = np.zeros(cap, dtype=np.int32)
        ey[:rows] = ys[idx].astype(np.int32)
        expect.append((ex, ey))
    arr = (_native.HostGatherItem * len(items))(*items)
    _native.call("hnn_host_gather_batch", C.addressof(arr), len(items), threads)
    for (dst, dy, _), (ex, ey) in zip(dsts, expect):
        assert np.array_equal(dst, ex) and np.array_equal(dy, ey)
    with pytest.raises(h.DeviceError):
        _native.call("hnn_host_gather_batch", C.addressof(arr), len(items), 0)


def test_backend_switch_rebinds_the_reference_workspace():
    """backend.install routes hybridnn.workspace's training names to this package and uninstall
    restores them (needs the reference installed in baseline/_ref; no GPU work)."""
    import sys

    ref = REPO / "baseline" / "_ref"
    if not (ref / "hybridnn").exists():
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, str(ref))
    try:
        import hybridnn
    finally:
        sys.path.remove(str(ref))
    from paper_2408_01331_b200 import backend
    from paper_2408_01331_b200.separate import package, separate

    ws = hybridnn.workspace
    before = {n: getattr(ws, n) for n in backend.ROUTED}
    backend.install(hybridnn)
    backend.install(hybridnn)  # idempotent: the saved bindings stay the reference's
    try:
        assert ws.Trainer is h.Trainer and ws.separate is separate and ws.package is package
        assert ws.Checkpoint is h.Checkpoint and ws.restore_checkpoint is h.restore_checkpoint
        assert ws.unify_jobs is backend.unify_jobs and backend.installed(hybridnn)
    finally:
        backend.uninstall(hybridnn)
    assert {n: getattr(ws, n) for n in backend.ROUTED} == before and not backend.installed(hybridnn)
