"""CPU oracle for the hybrid-training hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the arithmetic of the reference
package ``hybridnn`` (/root/reference/pkg/src/hybridnn) for exactly the path
this repository accelerates: keyed initialisation, per-epoch batch order,
forward/backward through the op kinds, softmax-cross-entropy, and the
SGD/Adam update.  Every function cites the reference file:line it follows.

Who may import it: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` — as the
checker or the timed CPU baseline, never as the product.  The product
package ``paper_2408_01331_b200`` never imports anything from here; if its
CUDA library is missing it raises instead of falling back to this code.

Parity pinning: ``tests/test_oracle_golden.py`` checks this restatement
against (a) the reference's own frozen known-answer vectors
(pkg/tests/expected_values.json, copied verbatim as data into
``tests/golden/reference_expected_values.json``) and (b) trajectories
produced by importing the unmodified reference in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), which must
match this oracle bit for bit with OPENBLAS_NUM_THREADS=1.
"""
from .reference_oracle import *  # noqa: F401,F403
from .reference_oracle import __all__  # noqa: F401
