"""Wall time per trajectory pass of the two launch forms for mid-size
problems (persistent cooperative kernel vs one launch per pass), MIS and
f_B, to place the `persistent_cells` threshold.

    python scripts/traj_paths.py
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06921_b200 as P  # noqa: E402
from paper_2605_06921_b200 import _lib  # noqa: E402


def main():
    iters = 300
    sizes = ((20000, 10, 32), (20000, 10, 128), (50000, 10, 64), (100000, 10, 16),
             (100000, 10, 32), (200000, 10, 16), (200000, 10, 32), (100000, 10, 128),
             (400000, 10, 32), (1000000, 10, 16), (1000000, 10, 32))
    only = sys.argv[1:] and int(sys.argv[1])
    for n, d, B in sizes[only:] if only else sizes:
        g = P.generate(P.ErFastSpec(n, d / n), 1)
        for name, spec, cfg, lo in (
                ("mis", P.MisQubo(2.0), P.OptimizerConfig(1e-9, 0.0, max_iters=iters), 0.0),
                ("fB", P.PerturbedBias(0.001), P.OptimizerConfig(0.0025, 0.8, max_iters=iters,
                                                                conv_tol=0.0), -1.0)):
            X = np.random.default_rng(1).uniform(lo, 1.0, (B, n))
            b = P.ChainBatch(g, B)
            row = {"n": n, "B": B, "obj": name, "cells": n * b.chains}
            for label, cells in (("persistent", 1 << 40), ("per_pass", 0)):
                _lib.check(_lib.lib.mqo_tune(b"persistent_cells", cells))
                _lib.check(_lib.lib.mqo_tune(b"cta_traj", 0))
                b.set_x(X)
                b.run_trajectories(spec, cfg)  # warm-up
                b.set_x(X)
                t = time.perf_counter()
                it, _ = b.run_trajectories(spec, cfg)
                dt = time.perf_counter() - t
                row[label + "_us_per_pass"] = round(dt / max(1, int(it.max())) * 1e6, 2)
            _lib.check(_lib.lib.mqo_tune(b"persistent_cells", 1 << 22))
            _lib.check(_lib.lib.mqo_tune(b"cta_traj", 1))
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
