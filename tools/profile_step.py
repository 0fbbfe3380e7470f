"""One eager training step of a bench workload between cudaProfilerStart/Stop, for
``ncu --profile-from-start off --set full`` (the capture behind bench.py's roofline `traffic`).

usage: ncu --set full --profile-from-start off --clock-control none -o gpurun_out/step_c3 \
           python tools/profile_step.py c3
Also writes gpurun_out/plan_<workload>.json: the step's launches in order (family, entry, label,
algorithmic bytes / FLOPs), which tools/ncu_traffic.py aligns with the captured kernels."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
torch.cuda.set_device(0)
_, jobs, hy, dev, ddev, ds, comm = bench.build_rank(wl, 0, 1, torch.device("cuda", 0))
rows = bench.schedule(jobs, ds, 16)
bench.upload_perms(dev, jobs, ds)
dev.load_schedule(rows)
dev.train_steps(4, use_graph=False)  # warm: first-touch, lazy module loads
torch.cuda.synchronize()
plan = [{"family": l.family, "entry": l.entry, "label": l.label, "nbytes": l.nbytes, "flops": l.flops}
        for l in dev.train_plan]
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/plan_{wl}.json").write_text(json.dumps(plan, indent=0))
torch.cuda.profiler.start()
dev.run_plan(dev.train_plan)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"profiled one {wl} step: {len(plan)} launches")
