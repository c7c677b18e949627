"""Single-call latency of one_two_swap (and one_flip_pass) at bench_core's
shapes, for a launch-list breakdown under ncu:
    python scripts/ls_swap_probe.py [--reps N]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06921_b200 as P  # noqa: E402
from paper_2605_06921_b200 import _lib  # noqa: E402


def greedy_mis(g):
    """greedy_maximalize from the empty set (localsearch.cpp order: ascending
    ids), on the host CSR"""
    off, nbr = g.csr()
    n = g.n()
    ind = np.zeros(n, np.uint8)
    blocked = np.zeros(n, bool)
    for v in range(n):
        if not blocked[v]:
            ind[v] = 1
            blocked[nbr[off[v]:off[v + 1]]] = True
    return ind


ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=0, help="fixed repetitions (0: time for 0.3 s)")
a = ap.parse_args()
for n in (1024, 4096):
    g = P.generate(P.ErSpec(n, 8.0 / n), 5)
    b = P.ChainBatch(g, 1)
    pk = P.pack_bodies(greedy_mis(g)[None, :])
    g16 = P.generate(P.ErSpec(n, 16.0 / n), 3)
    b16 = P.ChainBatch(g16, 1)
    sides = P.pack_bodies(np.random.default_rng(11).integers(0, 2, (1, n)).astype(np.uint8))
    row = {"n": n}
    for name, bb, op, body in (("one_two_swap", b, _lib.LS_ONE_TWO_SWAP, pk),
                               ("one_flip", b16, _lib.LS_ONE_FLIP, sides)):
        fn = lambda: P.local_search(bb, op, body.copy())  # noqa: E731
        fn()
        if a.reps:
            t0 = time.perf_counter()
            for _ in range(a.reps):
                fn()
            row[name + "_us"] = round(1e6 * (time.perf_counter() - t0) / a.reps, 1)
        else:
            reps, t0 = 0, time.perf_counter()
            while time.perf_counter() - t0 < 0.3:
                fn()
                reps += 1
            row[name + "_us"] = round(1e6 * (time.perf_counter() - t0) / reps, 1)
    print(json.dumps(row), flush=True)
