"""Summarise an ncu report (--set full) and/or an ncu launch list into a compact text file for
profiles/.  usage: python tools/ncu_summary.py [--rep X.ncu-rep] [--launches X.csv] > out.txt"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "dur_us", 1e-3),
    ("dram__bytes_read.sum", "dram_rd_MB", None),
    ("dram__bytes_write.sum", "dram_wr_MB", None),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%", None),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_%", None),
    ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "l2_%", None),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%", None),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_lsu_%", None),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%", None),
    ("launch__registers_per_thread", "regs", None),
    ("launch__grid_size", "grid", None),
]


def rep_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        yield hdr, units, r


def summarize_rep(path):
    print(f"# ncu --set full: {path}")
    cols = ["kernel"] + [m[1] for m in METRICS]
    print(" | ".join(cols))
    for hdr, units, r in rep_rows(path):
        name = r[hdr.index("Kernel Name")]
        name = name.split("(")[0].replace("void ", "").replace("hnn::", "")
        vals = [name[:34]]
        for key, short, _ in METRICS:
            if key not in hdr:
                vals.append("-")
                continue
            v = r[hdr.index(key)].replace(",", "")
            u = units[hdr.index(key)]
            try:
                x = float(v)
                if u == "Gbyte":
                    x *= 1e3
                elif u == "Kbyte":
                    x *= 1e-3
                elif u == "byte":
                    x *= 1e-6
                if key == "gpu__time_duration.sum" and u in ("nsecond", "ns"):
                    x *= 1e-3
                elif key == "gpu__time_duration.sum" and u in ("msecond", "ms"):
                    x *= 1e3
                vals.append(f"{x:.2f}")
            except ValueError:
                vals.append(v)
        print(" | ".join(vals))


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    order = []
    for r in rows[h + 1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("hnn::", "")
        t = float(r[vi].replace(",", ""))
        t = t / 1e3 if r[ui] in ("nsecond", "ns") else t
        if name not in tot:
            order.append(name)
        tot[name] += t
        cnt[name] += 1
    allt = sum(tot.values())
    print(f"# ncu launch list (gpu__time_duration, cold-cache serialised): {path}, {len(rows) - h - 1} launches")
    print("kernel | launches | total_us | share")
    for n in sorted(order, key=lambda n: -tot[n]):
        print(f"{n[:40]} | {cnt[n]} | {tot[n]:.1f} | {tot[n] / allt:.3f}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches", action="append", default=[])
    a = ap.parse_args()
    for p in a.launches:
        summarize_launches(p)
        print()
    for p in a.rep:
        summarize_rep(p)
        print()
