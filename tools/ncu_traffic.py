"""DRAM traffic per kernel family of one profiled step (tools/profile_step.py under ncu --set full).

usage: python tools/ncu_traffic.py REPORT.ncu-rep PLAN.json WORKLOAD > profiles/rNN/traffic_WORKLOAD.json

The ncu rows (launch order) are aligned with the step's plan: the first kernel is step_begin, then
one kernel per launch, except that a tensor-core WGRAD launch also runs colsum_kernel (its bias
gradient), which is charged to that launch.  Per family: dram__bytes_read.sum +
dram__bytes_write.sum summed over the step, the kernels' ncu durations, and the plan's
algorithmic bytes / FLOPs, so `traffic / algorithmic` shows re-reads."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    table = list(csv.reader(io.StringIO(out)))
    hdr, units = table[0], table[1]

    def val(r, key):
        if key not in hdr:
            return 0.0
        i = hdr.index(key)
        v = r[i].replace(",", "")
        return float(v) * UNIT.get(units[i], 1.0) if v not in ("", "n/a") else 0.0

    for r in table[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("hnn::", "")
        yield name, val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"), val(r, "gpu__time_duration.sum")


def main():
    rep, plan_path, wl = sys.argv[1:4]
    plan = json.load(open(plan_path))
    kernels = list(rows(rep))
    assert kernels and kernels[0][0].startswith("step_begin"), kernels[:2]
    fam = defaultdict(lambda: {"dram_bytes_per_step": 0.0, "ncu_us": 0.0, "kernels": 0, "algorithmic_bytes": 0,
                               "flops": 0, "launches": 0})
    for p in plan:
        f = fam[p["family"]]
        f["algorithmic_bytes"] += p["nbytes"]
        f["flops"] += p["flops"]
        f["launches"] += 1
    i = 1
    current = None
    for name, dram, us in kernels[1:]:
        if name.startswith("colsum_kernel") and current is not None:
            f = fam[current]
        else:
            assert i < len(plan) + 1, f"more kernels than launches at {name}"
            current = plan[i - 1]["family"]
            f = fam[current]
            i += 1
        f["dram_bytes_per_step"] += dram
        f["ncu_us"] += us
        f["kernels"] += 1
    assert i == len(plan) + 1, f"{i - 1} launches matched of {len(plan)}"
    total_us = sum(f["ncu_us"] for f in fam.values())
    for f in fam.values():
        f["dram_bytes_per_step"] = int(f["dram_bytes_per_step"])
        f["ncu_share"] = round(f["ncu_us"] / total_us, 4)
        f["ncu_us"] = round(f["ncu_us"], 2)
        if f["algorithmic_bytes"]:
            f["traffic_over_algorithmic"] = round(f["dram_bytes_per_step"] / f["algorithmic_bytes"], 3)
    print(json.dumps({"workload": wl, "report": rep, "kernels": len(kernels),
                      "families": dict(sorted(fam.items(), key=lambda kv: -kv[1]["ncu_us"]))}, indent=1))


if __name__ == "__main__":
    main()
