"""Probe: per-step Adam weight errors at C3 widths, max-abs and normwise, against the reference's own
thread jitter and exact-gradient distance (numbers behind tests/test_gpu_baseline_parity.py)."""
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(REPO), str(REPO / "tests")]
import numpy as np
from threadpoolctl import threadpool_limits

import oracle
import paper_2408_01331_b200 as pkg
from paper_2408_01331_b200 import store, zoo
import test_gpu_baseline_parity as T

with threadpool_limits(1):
    for h in [int(a) for a in sys.argv[1:]] or [256, 1024, 2048]:
        splits = oracle.blob_splits("c3-width", "mnist-768", 10, 784, 768, 64)
        ds = store.from_splits(splits)
        graph = zoo.mlp(784, (h, h), 10)
        job = pkg.TrainingJob("c3", graph, ds.content_hash, pkg.HyperParams(1, 256, 1e-3, "adam", (), 5), 0, 0)
        g_gpu, p_gpu, l_gpu, report, labels, _ = T._run_one(pkg, job, ds)
        init = oracle.init_model(graph, 5)
        batches = oracle.epoch_batches(splits["train_x"], splits["train_y"], ds.content_hash, 256, 5, 0)
        ref1, l_ref, g_ref = T._oracle_adam_run(graph, batches, init, 1e-3, 3, threads=1)
        ref2, _, _ = T._oracle_adam_run(graph, batches, init, 1e-3, 3, threads=2)
        ex, _, _ = T._oracle_adam_run(graph, batches, init, 1e-3, 3, exact=True)
        for k in range(3):
            for pid in sorted(ref1[k]):
                if not pid.endswith("weight"):
                    continue
                f = lambda a: (T.rel(a, ref1[k][pid]), T.normwise(a, ref1[k][pid]))
                g, t2, e = f(p_gpu[k][pid]), f(ref2[k][pid]), f(ex[k][pid])
                gx = (T.rel(p_gpu[k][pid], ex[k][pid]), T.normwise(p_gpu[k][pid], ex[k][pid]))
                print(f"h={h} k={k} {pid:11s} gpu {g[0]:.2e}/{g[1]:.2e}  t2 {t2[0]:.2e}/{t2[1]:.2e}  "
                      f"exact {e[0]:.2e}/{e[1]:.2e}  gpu-vs-exact {gx[0]:.2e}/{gx[1]:.2e}  "
                      f"loss {abs(l_gpu[k]-l_ref[k])/l_ref[k]:.1e}")
