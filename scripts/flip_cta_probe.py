"""One-body one_flip_pass on the reference micro-benchmark shape
(ER(1024, d=16) seed 3, random sides): two identical calls, for an ncu capture
of the second k_one_flip_cta launch (-k regex:k_one_flip_cta -s 1 -c 1)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06921_b200 as P  # noqa: E402
from paper_2605_06921_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
pg = P.generate(P.ErSpec(n, 16.0 / n), 3)
sides = np.random.default_rng(11).integers(0, 2, size=(1, n), dtype=np.uint8)
b = P.ChainBatch(pg, 1)
pk = P.pack_bodies(sides)
for _ in range(2):
    out, gain = P.local_search(b, _lib.LS_ONE_FLIP, pk.copy())
print("gain", int(gain[0]))
