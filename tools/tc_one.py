"""One tcgen05 GEMM launch of a given op/shape (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import tc_probe

op, M, N, K = (int(a) for a in sys.argv[1:5])
tc_probe.run(op, 1, M, N, K)
