"""Three eager training steps (the last on a ragged batch) of a small mixed hybrid for compute-sanitizer (racecheck / synccheck /
memcheck): an fp32 MLP on the CTA-pair 3xTF32 GEMMs (fwd / dgrad / wgrad, Adam), a LeNet-style CNN
on the direct conv + pool kernels, and a bf16 conv net on the tensor-core conv path (implicit-GEMM
forward, stride-2 parity-class input gradient, weight-gradient reduce).

usage: compute-sanitizer --tool racecheck python tools/sanitize_step.py [f32|bf16]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2408_01331_b200 import merge, store, zoo  # noqa: E402
from paper_2408_01331_b200.runtime import DeviceDataset, STEP_DTYPE  # noqa: E402
from paper_2408_01331_b200 import rng  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
torch.cuda.set_device(0)
dev_t = torch.device("cuda", 0)
img = store.from_splits(oracle.image_splits("san", "img", 10, (3, 16, 16), 128, 16))
blob = store.from_splits(oracle.blob_splits("san", "blob", 10, 784, 128, 16))
img32 = store.from_splits(oracle.image_splits("san", "img32", 10, (3, 32, 32), 128, 16))
convnet = zoo._seq("san-conv", (3, 16, 16), [
    ("c1", "conv2d", {"filters": 64, "kernel": 3, "padding": 1}), ("a1", "relu", {}),
    ("c2", "conv2d", {"filters": 64, "kernel": 3, "padding": 1, "stride": 2}), ("a2", "relu", {}),
    ("c3", "conv2d", {"filters": 64, "kernel": 3, "padding": 1}), ("a3", "relu", {}),
    ("p", "maxpool2d", {"kernel": 2}), ("f", "flatten", {}), ("fc", "dense", {"units": 10})])
jobs = [zoo.job("mlp", zoo.mlp(784, (256, 128), 10), blob, 0, batch_size=64, lr=1e-3, optimizer="adam"),
        zoo.job("cnn", convnet, img, 1, batch_size=32, lr=0.01),
        zoo.job("lenet", zoo.lenet5(), img32, 2, batch_size=32, lr=0.01)]
data = [blob, img, img32]
h = merge(jobs)
dev = h.materialize(dev_t, conv_precision=prec)
dev.bind_datasets([DeviceDataset(d, dev_t) for d in data], 128)
dev.build_plans()
rows = np.zeros((3, len(jobs)), dtype=STEP_DTYPE)
for m, j in enumerate(jobs):
    B = j.hypers.batch_size
    for t in range(3):  # (step 3: a ragged batch, rows < capacity)
        rows[t, m] = (1, B if t < 2 else B - 5, t * B, 0, t, t + 1, j.hypers.learning_rate, 0.1, 0.001, (0, 0, 0))
    d = data[m]
    dev.perm_upload(m, rng.permutation(d.sample_count, "shuffle", d.content_hash, j.hypers.seed, 0))
dev.load_schedule(rows)
dev.train_steps(3, use_graph=False)
torch.cuda.synchronize()
print("labels:", [l.label for l in dev.train_plan])
print("losses:", dev.loss_out.cpu().numpy())
