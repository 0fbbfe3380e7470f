"""Map ncu per-instruction stall samples (source page CSV) to CUDA source lines via nvdisasm -g.
usage: python tools/stall_lines.py SRC_CSV CUBIN KERNEL_MANGLED CU_FILE [top]   (debug tool)"""
import csv
import re
import subprocess
import sys

src_csv, cubin, kern, cu = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 20
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
inside, line, lines = False, None, {}
for l in sass:
    if l.startswith(".text."):
        inside = l.startswith(f".text.{kern}:")
        continue
    if not inside:
        continue
    m = re.search(r'//## File ".*", line (\d+)', l)
    if m:
        line = int(m.group(1))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        lines[int(m.group(1), 16)] = line
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ai, wi = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
addrs = [int(r[ai], 16) for r in rows[2:] if r[ai].startswith("0x")]
base = min(addrs)
agg = {}
for r in rows[2:]:
    try:
        v, a = int(r[wi]), int(r[ai], 16) - base
    except ValueError:
        continue
    ln = lines.get(a)
    agg[ln] = agg.get(ln, 0) + v
text = open(cu).read().split("\n")
tot = sum(agg.values())
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:6d} {v / tot:5.1%} line {ln}: {text[ln - 1].strip()[:100] if ln else '?'}")
