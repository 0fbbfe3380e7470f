"""GPU parity at BASELINE.json's own configs (VERDICT r01 "Next round" item 1).

* C3 widths h in {256, 1024, 2048} (K up to 2048 through the 3xTF32 pair GEMMs): first-step
  gradients and three Adam steps against the oracle;
* C4's VGG-11-noBN and ResNet-18-plain: first-step gradients on the fp32 (3xTF32) and the bf16
  tensor-core conv paths;
* C1 exactly as BASELINE states it (60,000 samples, 938 steps per model): curves, test metrics and
  weights against the unmodified reference's own run (tests/golden/baseline_training.json, made by
  tests/golden/make_training_golden.py);
* a bf16 C4-style short training run (LeNet-5 + a VGG slice): test accuracy after training within
  0.1% of the reference's fp32 run.

Error metric (pkg/tests/fd_oracle.py:86-88): rel(got, ref) = max|got - ref| / max|ref|.

Tolerances, stated per quantity:
* gradients (fp32 path): rel <= 1e-5 against the oracle, and as accurate as the reference's own
  fp32 BLAS: rel(gpu, float64) <= 2 * rel(oracle, float64) + 2e-7;
* losses: rel <= 1e-4 per step (north_star);
* Adam weights after step k: normwise relative error ||got - ref|| / ||ref|| <= 1e-4 per tensor
  (the north_star's "relative 1e-4 per step", measured; tools/adam_probe3.py saw <= 2.5e-6), and
  max-abs rel <= max(1e-4, 5 * J_k), where J_k is the reference's own sensitivity on the same
  case, measured here: the larger of (a) its change between 1 and 2 OpenBLAS threads and (b) its
  distance from the same Adam trajectory driven by float64-exact gradients.  Element-wise maxima
  are set by the few weights whose gradient is near eps: Adam's update lr * g / (|g| + eps) turns
  gradient noise of 1e-9 into weight changes of order lr there, so the reference itself moves by
  up to 8.7e-4 (rel) between BLAS thread counts / exact gradients at these widths, and the device
  path by 2-3.3x its J_k (probe3).  The update itself is bit-exact given the gradients
  (test_gpu_parity.py::test_optimizer_is_bit_exact_given_gradients).
* bf16 (accuracy class, SURVEY finding 4): stated per test below.
"""
import json

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

import oracle
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def rel(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-6)) if ref.size else 0.0


def normwise(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2408_01331_b200 as h

    return h


def _run_one(pkg, job, ds, **kw):
    """Train one job alone through the public Trainer; returns (first-step grads, params after each
    step, per-step losses, report, plan labels)."""
    h = pkg.merge([job])
    grads0, steps, losses = {}, [], []
    tr = pkg.Trainer(h, pkg.make_plan("fcfs", [job]), [job], {job.job_id: ds}, keep_grads=True,
                     loss_observer=lambda j, s, l, k: losses.append(l), **kw)

    def observe(j, p):
        if not grads0:
            grads0.update(tr.device.download_grads(0))
        steps.append({k.split("/", 1)[1]: v for k, v in p.items()})

    tr.step_observer = observe
    report = tr.run()
    return grads0, steps, losses, report, [l.label for l in tr.device.train_plan], h


# ----------------------------------------------------------------------------- C3 widths


def _mlp_grads_f64(params, x, y, n_layers):
    """First-step gradients of a dense/relu chain in float64 (the 'exact' yardstick)."""
    names = [f"fc{i + 1}" for i in range(n_layers)]
    acts, pre = [x.astype(np.float64)], []
    a = acts[0]
    for i, n in enumerate(names):
        z = a @ params[f"{n}.weight"].astype(np.float64).T + params[f"{n}.bias"].astype(np.float64)
        pre.append(z)
        a = np.maximum(z, 0.0) if i < n_layers - 1 else z
        acts.append(a)
    z = acts[-1] - acts[-1].max(axis=1, keepdims=True)
    p = np.exp(z) / np.exp(z).sum(axis=1, keepdims=True)
    t = y.astype(np.int64)
    p[np.arange(t.size), t] -= 1.0
    d = p / t.size
    g = {}
    for i in range(n_layers - 1, -1, -1):
        n = names[i]
        g[f"{n}.weight"] = d.T @ acts[i]
        g[f"{n}.bias"] = d.sum(axis=0)
        d = d @ params[f"{n}.weight"].astype(np.float64)
        if i > 0:
            d = d * (pre[i - 1] > 0)
    return g


def _oracle_adam_run(graph, batches, init, lr, steps, threads=1, exact=False):
    """The reference step (src/train.py:223-256) for `steps` batches; exact=True feeds the Adam
    update float64-exact gradients (rounded to f32) instead of the fp32 BLAS ones."""
    params = {k: v.copy() for k, v in init.items()}
    opt = oracle.OracleOptimizer("adam")
    states, losses, grads0 = [], [], None
    with threadpool_limits(threads):
        for k in range(steps):
            bx, by, _ = batches[k]
            logits, tape = oracle.model_forward(graph, params, bx)
            loss, dl = oracle.sce_loss_and_grad(logits, by)
            g = oracle.model_backward(tape, dl)
            if exact:
                g = {kk: v.astype(np.float32) for kk, v in _mlp_grads_f64(params, bx, by, 3).items()}
            if grads0 is None:
                grads0 = {kk: v.copy() for kk, v in g.items()}
            opt.apply(params, g, lr)
            states.append({kk: v.copy() for kk, v in params.items()})
            losses.append(float(loss))
    return states, losses, grads0


@pytest.mark.parametrize("h", [256, 1024, 2048])
def test_c3_width_gradients_and_adam_steps(pkg, h):
    """C3 model at width h (MLP 784-h-h-10, Adam lr 1e-3, batch 256): first-step gradients and three
    Adam steps (losses and weights per step) against the oracle, tolerances in the module doc."""
    from paper_2408_01331_b200 import store, zoo

    splits = oracle.blob_splits("c3-width", "mnist-768", 10, 784, 768, 64)
    ds = store.from_splits(splits)
    graph = zoo.mlp(784, (h, h), 10)
    seed, lr, B, steps = 5, 1e-3, 256, 3
    job = pkg.TrainingJob("c3", graph, ds.content_hash, pkg.HyperParams(1, B, lr, "adam", (), seed), 0, 0)
    g_gpu, p_gpu, l_gpu, report, labels, _ = _run_one(pkg, job, ds)
    assert sum(l.endswith("/tc2") for l in labels) >= 5, labels  # every dense GEMM on the CTA-pair kernel
    assert len(p_gpu) == steps and report.jobs["c3"].status == "complete"

    init = oracle.init_model(graph, seed)
    batches = oracle.epoch_batches(splits["train_x"], splits["train_y"], ds.content_hash, B, seed, 0)
    ref1, l_ref, g_ref = _oracle_adam_run(graph, batches, init, lr, steps, threads=1)
    ref2, _, _ = _oracle_adam_run(graph, batches, init, lr, steps, threads=2)
    exact, _, _ = _oracle_adam_run(graph, batches, init, lr, steps, exact=True)

    bx, by, _ = batches[0]
    g64 = _mlp_grads_f64(init, bx, by, 3)
    for pid, g in g_ref.items():
        e_gpu, e_ref = rel(g_gpu[pid], g64[pid]), rel(g, g64[pid])
        assert rel(g_gpu[pid], g) <= 1e-5, (h, pid, rel(g_gpu[pid], g))
        assert e_gpu <= 2 * e_ref + 2e-7, (h, pid, "vs float64", e_gpu, e_ref)
    for k in range(steps):
        assert abs(l_gpu[k] - l_ref[k]) / abs(l_ref[k]) <= 1e-4, (h, k, l_gpu[k], l_ref[k])
        for pid in ref1[k]:
            assert normwise(p_gpu[k][pid], ref1[k][pid]) <= 1e-4, (h, k, pid, normwise(p_gpu[k][pid], ref1[k][pid]))
            jit = max(rel(ref2[k][pid], ref1[k][pid]), rel(exact[k][pid], ref1[k][pid]))
            err = rel(p_gpu[k][pid], ref1[k][pid])
            assert err <= max(1e-4, 5 * jit), (h, k, pid, err, jit)


# ----------------------------------------------------------------------------- C4 CNNs, one step


_CNN_REF = {}


def _bf16(a):
    """Round fp32 to the nearest bf16 (ties to even), kept in fp32 storage."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _bf16_emulated_grads(graph, params, x, y):
    """The oracle's first-step gradients with the bf16 path's roundings applied (test
    infrastructure): every conv GEMM operand — the layer input, the weights and the upstream
    gradient — rounded to bf16; products and sums, the bias gradient, pooling, relu, the dense
    head and the loss in fp32 (bf16 operand copies, fp32 accumulation, fp32 master
    weights)."""
    tape, h = [], np.asarray(x, dtype=np.float32)
    for node in oracle.graph_chain(graph):
        if node.op == "softmax-cross-entropy":
            break
        p = {k.rsplit(".", 1)[1]: v for k, v in params.items() if k.rsplit(".", 1)[0] == node.node_id}
        if node.op == "conv2d":
            out, saved = oracle.op_forward("conv2d", _bf16(h), {"weight": _bf16(p["weight"]), "bias": p["bias"]},
                                           node.attrs)
        else:
            out, saved = oracle.op_forward(node.op, h, p, node.attrs)
        tape.append((node, p, saved))
        h = out
    _, d = oracle.sce_loss_and_grad(h, y)
    grads = {}
    for node, p, saved in reversed(tape):
        if node.op == "conv2d":
            dx, dp = oracle.op_backward("conv2d", _bf16(d), saved, {"weight": _bf16(p["weight"])}, node.attrs)
            dp["bias"] = d.sum(axis=(0, 2, 3))
        else:
            dx, dp = oracle.op_backward(node.op, d, saved, p, node.attrs)
        for k, g in dp.items():
            grads[f"{node.node_id}.{k}"] = g
        d = dx
    return grads


def _cnn_case(name):
    """(graph, splits, dataset, oracle first-step gradients fp32 / bf16-emulated) of a C4 network at
    batch 8 (cached)."""
    from paper_2408_01331_b200 import store, zoo

    if name not in _CNN_REF:
        graph = {"vgg11": zoo.vgg11_nobn, "resnet18": zoo.resnet18_plain}[name]()
        splits = oracle.image_splits("c4-grad", "cifar-8", 10, (3, 32, 32), 8, 8)
        ds = store.from_splits(splits)
        params = oracle.init_model(graph, 7)
        bx, by, _ = oracle.epoch_batches(splits["train_x"], splits["train_y"], ds.content_hash, 8, 7, 0)[0]
        logits, tape = oracle.model_forward(graph, params, bx)
        _, dl = oracle.sce_loss_and_grad(logits, by)
        _CNN_REF[name] = (graph, splits, ds, oracle.model_backward(tape, dl),
                          _bf16_emulated_grads(graph, params, bx, by))
    return _CNN_REF[name]


@pytest.mark.parametrize("precision", ["f32", "bf16"])
@pytest.mark.parametrize("name", ["vgg11", "resnet18"])
def test_c4_cnn_first_step_gradients(pkg, name, precision):
    """VGG-11-noBN / ResNet-18-plain (C4's networks), batch 8: first-step gradients of every layer
    against the fp32 oracle.  f32 (3xTF32 tensor-core convs): rel <= 1e-5 per tensor.

    bf16 operands (fp32 accumulation, BASELINE C4): accuracy class.  These plain (no batch-norm,
    no residual) deep nets are ill-conditioned at init: the oracle with the bf16 path's roundings
    emulated (_bf16_emulated_grads) is itself 13-30% (normwise) away from fp32 in the early layers'
    gradients.  So the criterion is that the device deviates from fp32 no more than bf16 arithmetic
    itself does: normwise(gpu, fp32) <= 1.5 * normwise(emulated bf16, fp32) + 1e-2 per tensor (a
    layout or indexing bug gives errors of order 1).  Measured: ratio <= 1.19."""
    graph, splits, ds, ref, emu = _cnn_case(name)
    job = pkg.TrainingJob(name, graph, ds.content_hash, pkg.HyperParams(1, 8, 1e-3, "sgd", (), 7), 0, 0)
    g_gpu, _, losses, _, labels, _ = _run_one(pkg, job, ds, fuse_optimizer=False, conv_precision=precision)
    tc = [l for l in labels if "/conv/tc" in l or l.endswith("/bf16")]
    assert len(tc) >= 6, labels
    errs = {pid: (rel(g_gpu[pid], g), normwise(g_gpu[pid], g)) for pid, g in ref.items()}
    print(name, precision, "worst max-abs", max(e[0] for e in errs.values()), "worst normwise",
          max(e[1] for e in errs.values()))
    if precision == "bf16":
        for pid, g in ref.items():
            print(f"  {pid:14s} gpu-vs-emu {normwise(g_gpu[pid], emu[pid]):.2e}  emu-vs-f32 {normwise(emu[pid], g):.2e}"
                  f"  gpu-vs-f32 {normwise(g_gpu[pid], g):.2e}")
    if precision == "f32":
        bad = {pid: e for pid, e in errs.items() if e[0] > 1e-5}
    else:
        bad = {pid: (e[1], normwise(emu[pid], ref[pid])) for pid, e in errs.items()
               if e[1] > 1.5 * normwise(emu[pid], ref[pid]) + 1e-2}
    assert not bad, bad


# ----------------------------------------------------------------------------- whole runs vs the reference


def _golden():
    return json.loads((GOLDEN / "baseline_training.json").read_text())


def _check_checksums(params, gold, tol):
    for pid, c in gold.items():
        flat = np.asarray(params[pid], dtype=np.float32).reshape(-1)
        got = flat[np.asarray(c["idx"])].astype(np.float64)
        ref = np.asarray(c["val"])
        assert rel(got, ref) <= tol, (pid, rel(got, ref))
        assert abs(float(np.abs(flat.astype(np.float64)).sum()) - c["abs"]) / c["abs"] <= tol, pid


def test_c1_full_epoch_matches_reference(pkg):
    """BASELINE C1 exactly (2 x MLP 784-256-10, 60,000 MNIST-shaped samples, batch 64, SGD lr
    0.01 / 0.05, one epoch = 938 steps each) in one hybrid, against the reference's own run:
    test accuracy within 0.1% (north_star), epoch train accuracy within 0.1%, train / test loss
    within rel 1e-4, and 64 sampled weights per tensor + the L1 norms within rel 1e-3 after 938 steps."""
    from paper_2408_01331_b200 import zoo

    gold = _golden()["c1"]
    ds = zoo.blob_dataset()
    assert ds.content_hash == gold["digest"]
    jobs = zoo.config_jobs("c1", ds)
    h = pkg.merge(jobs)
    report = pkg.Trainer(h, pkg.make_plan("rr", jobs), jobs, {j.job_id: ds for j in jobs}).run()
    assert report.steps == 938
    for j in jobs:
        got, ref = report.jobs[j.job_id], gold["jobs"][j.job_id]
        assert got.status == ref["status"] == "complete"
        (e, loss, acc), (re_, rloss, racc) = got.curve[0], ref["curve"][0]
        assert e == re_ == 0
        assert abs(loss - rloss) / rloss <= 1e-4, (j.job_id, loss, rloss)
        assert abs(acc - racc) <= 0.001, (j.job_id, acc, racc)
        assert abs(got.final_test_accuracy - ref["final_test_accuracy"]) <= 0.001, (j.job_id, got.final_test_accuracy)
        assert abs(got.final_test_loss - ref["final_test_loss"]) / ref["final_test_loss"] <= 1e-4
        _check_checksums(pkg.separate(h, j.job_id)[1], ref["params"], 1e-3)


def test_bf16_short_training_accuracy_matches_reference(pkg):
    """C4-style bf16 run (conv_precision="bf16": the VGG slice's convs on bf16 tensor cores incl. the
    implicit-GEMM 64-channel layer; LeNet's small convs stay fp32 direct kernels), 3 epochs of 2,048
    CIFAR-shaped images, batch 32, SGD lr 0.03, against the reference's fp32 run: test accuracy
    after training within 0.1% (north_star), per-epoch train loss within rel 5e-2 (bf16 accuracy
    class)."""
    from paper_2408_01331_b200 import store

    import sys
    sys.path.insert(0, str(GOLDEN))
    from training_cases import BF16_CASE, bf16_jobs_spec

    gold = _golden()["bf16"]
    c = BF16_CASE
    ds = store.from_splits(oracle.image_splits(*c["data"]))
    assert ds.content_hash == gold["digest"]
    jobs = [pkg.TrainingJob(jid, g, ds.content_hash, pkg.HyperParams(c["epochs"], c["batch"], c["lr"], "sgd", (), s),
                            i, i) for i, (jid, g, s) in enumerate(bf16_jobs_spec())]
    h = pkg.merge(jobs)
    tr = pkg.Trainer(h, pkg.make_plan("rr", jobs), jobs, {j.job_id: ds for j in jobs}, conv_precision="bf16")
    report = tr.run()
    labels = [l.label for l in tr.device.train_plan]
    assert sum(l.endswith("/bf16") for l in labels) >= 3, labels
    for j in jobs:
        got, ref = report.jobs[j.job_id], gold["jobs"][j.job_id]
        print(j.job_id, got.curve, got.final_test_accuracy, "ref", ref["curve"], ref["final_test_accuracy"])
        assert got.status == "complete"
        assert abs(got.final_test_accuracy - ref["final_test_accuracy"]) <= 0.001 + 1e-9, (j.job_id, got.final_test_accuracy,
                                                                                   ref["final_test_accuracy"])
        for (e, loss, acc), (re_, rloss, racc) in zip(got.curve, ref["curve"]):
            assert e == re_ and abs(loss - rloss) / rloss <= 5e-2, (j.job_id, e, loss, rloss)
