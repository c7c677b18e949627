"""one_flip_pass on one ER(1024, d=16) body (bench_core's case), repeated:
for an ncu launch list of the local-search path's kernels."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06921_b200 as P  # noqa: E402
from paper_2605_06921_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = P.generate(P.ErSpec(n, 16.0 / n), 3)
b = P.ChainBatch(g, 1)
side = (np.random.default_rng(11).integers(0, 2, n)).astype(np.uint8)
pk = P.pack_bodies(side[None, :])
for i in range(6):
    t = time.perf_counter()
    _, gain = P.local_search(b, _lib.LS_ONE_FLIP, pk)
    print(i, round((time.perf_counter() - t) * 1e6, 1), "us", int(gain[0]))
