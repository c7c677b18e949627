"""Single-call latency of mqo_local_search on small bodies (random sides /
greedy MIS starts), per op and n, with the single-launch kernels on and off
(MQO_LS_SMALL=0 in a second run).  python scripts/ls_small_probe.py"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06921_b200 as P  # noqa: E402
from paper_2605_06921_b200 import _lib  # noqa: E402


def timeit(fn, min_time=0.3):
    fn()
    reps, t0 = 0, time.perf_counter()
    while True:
        fn()
        reps += 1
        if time.perf_counter() - t0 >= min_time:
            return (time.perf_counter() - t0) / reps


for n in (1024, 2000, 4096, 16384):
    g = P.generate(P.ErSpec(n, 8.0 / n), 3)
    b = P.ChainBatch(g, 1)
    sides = np.random.default_rng(n).integers(0, 2, (1, n)).astype(np.uint8)
    pk = P.pack_bodies(sides)
    row = {"n": n, "small": os.environ.get("MQO_LS_SMALL", "1")}
    for name, op in (("one_flip", _lib.LS_ONE_FLIP), ("two_flip", _lib.LS_TWO_FLIP),
                     ("one_two_flip", _lib.LS_ONE_TWO_FLIP)):
        row[name + "_us"] = round(1e6 * timeit(lambda: P.local_search(b, op, pk.copy())), 1)
        done, _ = P.local_search(b, op, pk.copy())
        row[name + "_optimal_us"] = round(1e6 * timeit(lambda: P.local_search(b, op, done.copy())), 1)
    print(json.dumps(row), flush=True)
