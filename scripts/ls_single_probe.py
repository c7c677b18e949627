"""Single-body local-search latency on the reference micro-benchmark shapes
(bench_core.py's one_flip_pass / one_two_swap cases): wall time per
mqo_local_search call for 1 and 16 bodies, and for 1 body that is already
locally optimal (the fixed cost of the call: copies, launches, round trips).
Run it once per variant knob, e.g. MQO_SWAP_CTA=0 python scripts/ls_single_probe.py.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06921_b200 as P  # noqa: E402
from paper_2605_06921_b200 import _lib  # noqa: E402


def timeit(fn, min_time=0.3, max_reps=5000):
    fn()
    reps, t0 = 0, time.perf_counter()
    while True:
        fn()
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_time or reps >= max_reps:
            return dt / reps


def main():
    tag = os.environ.get("TAG", "default")
    for n in (1 << 10, 1 << 12, 1 << 14):
        pg = P.generate(P.ErSpec(n, 16.0 / n), 3)
        rng = np.random.default_rng(11)
        sides = rng.integers(0, 2, size=(1, n), dtype=np.uint8)
        b1 = P.ChainBatch(pg, 1)
        pk = P.pack_bodies(sides)
        done, _ = P.local_search(b1, _lib.LS_ONE_FLIP, pk.copy())
        t1 = timeit(lambda: P.local_search(b1, _lib.LS_ONE_FLIP, pk.copy()))
        t0 = timeit(lambda: P.local_search(b1, _lib.LS_ONE_FLIP, done.copy()))
        many = np.repeat(pk, 16, axis=0)
        tb = timeit(lambda: P.local_search(b1, _lib.LS_ONE_FLIP, many.copy())) / 16
        print(json.dumps({"tag": tag, "case": "one_flip_pass", "n": n, "us_1": t1 * 1e6,
                          "us_fixed": t0 * 1e6, "us_per_body_16": tb * 1e6}), flush=True)
    for n in (1 << 10, 1 << 12, 1 << 14):
        pg = P.generate(P.ErSpec(n, 8.0 / n), 5)
        b1 = P.ChainBatch(pg, 1)
        # a maximal start: the harvested greedy completion of one trajectory
        b1.seed_streams(5)
        b1.init_states(P.PROBLEM_MIS, 0.15)
        b1.run_trajectories(P.MisQubo(2.0), P.OptimizerConfig(0.8, 0.3))
        sc, valid, packed = b1.harvest(P.PROBLEM_MIS)
        if not valid[0]:
            continue
        pk = packed[:1]
        done, _ = P.local_search(b1, _lib.LS_ONE_TWO_SWAP, pk.copy())
        t1 = timeit(lambda: P.local_search(b1, _lib.LS_ONE_TWO_SWAP, pk.copy()))
        t0 = timeit(lambda: P.local_search(b1, _lib.LS_ONE_TWO_SWAP, done.copy()))
        many = np.repeat(pk, 16, axis=0)
        tb = timeit(lambda: P.local_search(b1, _lib.LS_ONE_TWO_SWAP, many.copy())) / 16
        print(json.dumps({"tag": tag, "case": "one_two_swap", "n": n, "us_1": t1 * 1e6,
                          "us_fixed": t0 * 1e6, "us_per_body_16": tb * 1e6}), flush=True)


if __name__ == "__main__":
    main()
