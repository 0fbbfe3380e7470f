"""Probe: where does the device Adam step differ from the oracle, and by how much does the
reference itself move between BLAS thread counts / against exact (float64) gradients?

    python tools/adam_probe2.py [h ...]      (GPU box)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from threadpoolctl import threadpool_limits

import oracle
from paper_2408_01331_b200 import store, zoo
import paper_2408_01331_b200 as h


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-6))


def f64_grads(params, x, y, hidden_layers):
    """Exact-ish first-step gradients of an MLP chain in float64."""
    names = [f"fc{i+1}" for i in range(hidden_layers + 1)]
    acts = [x.astype(np.float64)]
    pre = []
    a = acts[0]
    for i, n in enumerate(names):
        z = a @ params[f"{n}.weight"].astype(np.float64).T + params[f"{n}.bias"].astype(np.float64)
        pre.append(z)
        a = np.maximum(z, 0) if i < len(names) - 1 else z
        acts.append(a)
    z = acts[-1]
    z = z - z.max(1, keepdims=True)
    p = np.exp(z) / np.exp(z).sum(1, keepdims=True)
    t = y.astype(int)
    p[np.arange(len(t)), t] -= 1
    d = p / len(t)
    g = {}
    for i in range(len(names) - 1, -1, -1):
        n = names[i]
        g[f"{n}.weight"] = d.T @ acts[i]
        g[f"{n}.bias"] = d.sum(0)
        d = d @ params[f"{n}.weight"].astype(np.float64)
        if i > 0:
            d = d * (pre[i - 1] > 0)
    return g


def adam1(params, grads, lr):
    out = {}
    F = np.float32
    for k in params:
        g = grads[k]
        m = F(0.1) * g
        v = F(0.001) * g * g
        c1, c2 = F(1 - 0.9), F(1 - 0.999)
        out[k] = params[k] - F(lr) * (m / c1) / (np.sqrt(v / c2) + F(1e-8))
    return out


def main():
    hs = [int(a) for a in sys.argv[1:]] or [128, 256, 1024, 2048]
    splits = oracle.blob_splits("golden", "c1-mini", 10, 784, 768, 64)
    ds = store.from_splits(splits)
    for hid in hs:
        graph = zoo.mlp(784, (hid, hid), 10)
        seed, lr, B = 5, 1e-3, 256
        p0 = oracle.init_model(graph, seed)
        bx, by, _ = oracle.epoch_batches(splits["train_x"], splits["train_y"], ds.content_hash, B, seed, 0)[0]
        res = {}
        for th in (1, 2, 16):
            with threadpool_limits(th):
                logits, tape = oracle.model_forward(graph, p0, bx)
                _, dl = oracle.sce_loss_and_grad(logits, by)
                g = oracle.model_backward(tape, dl)
                p = {k: v.copy() for k, v in p0.items()}
                oracle.OracleOptimizer("adam").apply(p, {k: v.copy() for k, v in g.items()}, lr)
            res[th] = (g, p)
        gx = f64_grads(p0, bx, by, 2)
        px = adam1(p0, {k: v.astype(np.float32) for k, v in gx.items()}, lr)
        job = zoo.job("a", graph, ds, 0, epochs=1, batch_size=B, lr=lr, optimizer="adam", seed=seed)
        hy = h.merge([job])
        grabbed = {}
        tr = h.Trainer(hy, h.make_plan("fcfs", [job]), [job], {"a": ds}, keep_grads=True)
        tr.step_observer = lambda j, p: grabbed or grabbed.update(
            grads=tr.device.download_grads(0), params={k.split("/", 1)[1]: v for k, v in p.items()})
        tr.run()
        print(f"== h={hid}")
        for k in sorted(p0):
            g1, pp1 = res[1]
            line = (f"{k:12s} grad: gpu {rel(grabbed['grads'][k], g1[k]):.2e} t2 {rel(res[2][0][k], g1[k]):.2e} "
                    f"t16 {rel(res[16][0][k], g1[k]):.2e} | vs f64: gpu {rel(grabbed['grads'][k], gx[k]):.2e} "
                    f"t1 {rel(g1[k], gx[k]):.2e} || weights: gpu {rel(grabbed['params'][k], pp1[k]):.2e} "
                    f"t2 {rel(res[2][1][k], pp1[k]):.2e} t16 {rel(res[16][1][k], pp1[k]):.2e} | vs f64-grad: gpu "
                    f"{rel(grabbed['params'][k], px[k]):.2e} t1 {rel(pp1[k], px[k]):.2e}")
            print(line)
            d = np.abs(grabbed["params"][k].astype(np.float64) - pp1[k])
            i = np.unravel_index(np.argmax(d), d.shape)
            print(f"    worst elem {i}: g_gpu {grabbed['grads'][k][i]:.3e} g_t1 {g1[k][i]:.3e} g_f64 {gx[k][i]:.3e} "
                  f"dp {d[i]:.3e} |p|max {np.abs(pp1[k]).max():.3e}")


if __name__ == "__main__":
    main()
