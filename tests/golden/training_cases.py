"""Inputs of the whole-run golden cases (tests/golden/make_training_golden.py writes the reference's
results for them; tests/test_gpu_baseline_parity.py rebuilds the same jobs on the GPU)."""
from paper_2408_01331_b200 import zoo

VGG_SLICE = [("conv1", "conv2d", {"filters": 64, "kernel": 3, "padding": 1}), ("act1", "relu", {}),
             ("pool1", "maxpool2d", {"kernel": 4}),
             ("conv2", "conv2d", {"filters": 64, "kernel": 3, "padding": 1}), ("act2", "relu", {}),
             ("pool2", "maxpool2d", {"kernel": 2}),
             ("flat", "flatten", {}), ("fc", "dense", {"units": 10})]
BF16_CASE = dict(data=("golden", "cifar-2048", 10, (3, 32, 32), 2048, 1000), batch=32, lr=0.03, epochs=3)


def bf16_jobs_spec():
    """(job_id, graph, seed) of the bf16 short run."""
    return [("vgg-slice", zoo._seq("vgg-slice", (3, 32, 32), VGG_SLICE), 3), ("lenet", zoo.lenet5(), 4)]
