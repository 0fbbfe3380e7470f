"""Why do Adam weights differ after one step?  Compare device grads/weights vs the oracle (debug tool)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np

import oracle
import paper_2408_01331_b200 as pkg
from conftest import load_case
from paper_2408_01331_b200 import store

for name in ("c3_mlp",):
    arr, c, graph, splits, digest = load_case(name)
    ds = store.from_splits(splits)
    for tc in (True, False):
        job = pkg.TrainingJob(name, graph, digest, pkg.HyperParams(1, c["batch"], c["lr"], c["opt"], (), c["seed"]), 0, 0)
        h = pkg.merge([job])
        grads = {}
        tr = pkg.Trainer(h, pkg.make_plan("fcfs", [job]), [job], {name: ds}, use_tensor_cores=tc,
                         step_observer=lambda j, p: grads or grads.update(tr.device.download_grads(0)))
        tr.run()
        # oracle grads at step 0
        params = oracle.init_model(graph, c["seed"])
        bx, by, _ = oracle.epoch_batches(splits["train_x"], splits["train_y"], digest, c["batch"], c["seed"], 0)[0]
        logits, tape = oracle.model_forward(graph, params, bx)
        loss, dl = oracle.sce_loss_and_grad(logits, by)
        g_ref = oracle.model_backward(tape, dl)
        for pid in g_ref:
            g, r = grads[pid].astype(np.float64), g_ref[pid].astype(np.float64)
            rel = np.abs(g - r).max() / np.abs(r).max()
            flips = int(np.sum(np.sign(g) != np.sign(r)))
            tiny = int(np.sum(np.abs(r) < 1e-4 * np.abs(r).max()))
            print(f"tc={tc} {pid:12s} grad rel={rel:.2e} sign flips={flips} tiny(<1e-4 max)={tiny} of {r.size}")
        step0 = {k.split('/', 1)[1]: v for k, v in arr.items() if k.startswith("step0/")} if False else \
            {k.split("/", 1)[1]: arr[k] for k in arr.files if k.startswith("step0/")}
