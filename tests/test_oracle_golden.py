"""Pin the CPU oracle to the reference's golden vectors (runs without a GPU).

(a) the reference's own frozen known answers (pkg/tests/expected_values.json,
    checked like pkg/tests/test_autograd.py:258-311 and test_store.py:105-107);
(b) trajectories produced by the unmodified reference (tests/golden/make_golden.py):
    the oracle must reproduce them BIT FOR BIT with one BLAS thread.
"""
import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, load_case

EXPECTED = json.loads((GOLDEN / "reference_expected_values.json").read_text())
F = np.float32


class _Node:
    def __init__(self, node_id, op, inputs, attrs=None):
        self.node_id, self.op, self.inputs, self.attrs = node_id, op, inputs, attrs or {}


class _Graph:
    def __init__(self, input_shape, nodes, output):
        self.input_shape, self.nodes, self.output = input_shape, nodes, output


def tiny_mlp():
    return _Graph((8,), [_Node("fc1", "dense", ["input"], {"units": 16}), _Node("act1", "relu", ["fc1"]),
                         _Node("fc2", "dense", ["act1"], {"units": 2})], "fc2")


class TestReferenceKnownAnswers:
    def test_init_row(self):
        p = oracle.init_model(tiny_mlp(), EXPECTED["seed"])
        np.testing.assert_allclose(p["fc1.weight"][0], EXPECTED["init_w1_row0"], rtol=1e-6)

    def test_step0_logits_and_loss(self):
        p = oracle.init_model(tiny_mlp(), EXPECTED["seed"])
        x = oracle.keyed_generator("test-batch", "x").normal(0.0, 1.0, size=(4, 8)).astype(F)
        y = np.array([0, 1, 1, 0], dtype=F)
        logits, _ = oracle.model_forward(tiny_mlp(), p, x)
        np.testing.assert_allclose(logits, EXPECTED["logits_step0"], rtol=1e-5)
        loss, _ = oracle.sce_loss_and_grad(logits, y)
        assert float(loss) == pytest.approx(EXPECTED["loss_step0"], rel=1e-6)

    def test_two_sgd_steps(self):
        g = tiny_mlp()
        p = oracle.init_model(g, EXPECTED["seed"])
        x = oracle.keyed_generator("test-batch", "x").normal(0.0, 1.0, size=(4, 8)).astype(F)
        y = np.array([0, 1, 1, 0], dtype=F)
        opt = oracle.OracleOptimizer("sgd")
        losses = []
        for _ in range(2):
            loss, _ = oracle.train_step(g, p, x, y, opt, 0.1)
            losses.append(loss)
        logits, _ = oracle.model_forward(g, p, x)
        losses.append(float(oracle.sce_loss_and_grad(logits, y)[0]))
        np.testing.assert_allclose(losses, EXPECTED["losses_two_sgd_steps"], rtol=1e-6)
        for pid, s in EXPECTED["param_sums_after"].items():
            assert float(np.sum(p[pid])) == pytest.approx(s, rel=1e-5, abs=1e-6)

    def test_frozen_permutation(self):
        assert oracle.keyed_permutation(10, "shuffle", "deadbeef", 7, 0).tolist() == EXPECTED["permutation_10"]


@pytest.mark.parametrize("name", ["c1_mlp", "deep_adam", "lenet", "c3_mlp"])
def test_oracle_reproduces_reference_trajectory_bit_for_bit(name):
    arr, c, graph, splits, digest = load_case(name)
    losses, corrects, step0 = [], [], {}

    def observe(step, params, loss):
        losses.append(loss)
        if step == 0:
            step0.update({k: v.copy() for k, v in params.items()})

    params, opt, curve, abort = oracle.standalone_training(
        graph, splits, digest, c["epochs"], c["batch"], c["lr"], c["opt"], c["seed"], observer=observe)
    assert abort is None
    assert np.array_equal(np.asarray(losses), arr["losses"])
    for pid, v in params.items():
        assert np.array_equal(v, arr[f"final/{pid}"]), pid
        assert np.array_equal(step0[pid], arr[f"step0/{pid}"]), pid
    assert np.array_equal(np.asarray(curve, dtype=np.float64), arr["curve"])
    assert opt.step == int(arr["opt_step"])
    perm = oracle.keyed_permutation(splits["train_x"].shape[0], "shuffle", digest, c["seed"], 0)
    assert np.array_equal(perm, arr["perm_epoch0"])
    tl, ta = oracle.evaluate_split(graph, params, splits["test_x"], splits["test_y"], c["batch"])
    assert (tl, ta) == tuple(arr["test"])


def test_oracle_ops_match_reference_registry():
    arr = np.load(GOLDEN / "ops.npz")
    tags = sorted({k.split("/")[0] for k in arr.files})
    ops = {"dense": "dense", "relu": "relu", "conv_k3s2p1": "conv2d", "conv_k5": "conv2d",
           "pool_k3s2": "maxpool2d", "pool_k2": "maxpool2d", "sce": "softmax-cross-entropy"}
    for tag in tags:
        op = ops[tag]
        attrs = json.loads(str(arr[f"{tag}/attrs"]))
        x = arr[f"{tag}/x"]
        p = {k.split("/p_")[1]: arr[k] for k in arr.files if k.startswith(f"{tag}/p_")}
        if op == "softmax-cross-entropy":
            loss, dx = oracle.sce_loss_and_grad(x, arr[f"{tag}/targets"])
            assert np.array_equal(loss, arr[f"{tag}/y"]) and np.array_equal(dx, arr[f"{tag}/dx"])
            continue
        y, saved = oracle.op_forward(op, x, p, attrs)
        assert np.array_equal(y, arr[f"{tag}/y"]), tag
        dx, dp = oracle.op_backward(op, arr[f"{tag}/dy"], saved, p, attrs)
        assert np.array_equal(dx, arr[f"{tag}/dx"]), tag
        for k, v in dp.items():
            assert np.array_equal(v, arr[f"{tag}/d_{k}"]), (tag, k)


def test_oracle_trainer_rr_curves():
    ref = json.loads((GOLDEN / "trainer_rr.json").read_text())
    from paper_2408_01331_b200 import zoo

    cases = {
        "a": (zoo.mlp(12, (24, 16), 4, name="mlp-3"), oracle.blob_splits("golden", "four", 4, 12, 96, 32),
              3, 16, 0.01, "adam", 2, (2,)),
        "b": (zoo.mlp(8, (16,), 2, name="mlp-2"), oracle.blob_splits("golden", "two", 2, 8, 64, 32),
              2, 16, 0.05, "sgd", 1, ()),
        "bad": (zoo.mlp(8, (16,), 2, name="mlp-2"), oracle.blob_splits("golden", "two", 2, 8, 64, 32),
                3, 16, 1e8, "sgd", 0, ()),
    }
    for jid, (g, s, ep, bs, lr, opt, seed, ms) in cases.items():
        params, _, curve, abort = oracle.standalone_training(g, s, oracle.dataset_digest(s), ep, bs, lr, opt, seed, ms)
        row = ref["jobs"][jid]
        if row["status"] == "aborted":
            assert abort is not None
            continue
        assert [list(r) for r in curve] == row["curve"]
        tl, ta = oracle.evaluate_split(g, params, s["test_x"], s["test_y"], bs)
        assert (tl, ta) == (row["final_test_loss"], row["final_test_accuracy"])
        for pid, v in params.items():
            assert np.array_equal(v, np.asarray(ref["params"][f"{jid}/{pid}"], dtype=F)), pid
