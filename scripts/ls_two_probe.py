"""one_two_flip on 8 BA(1e6,5) bodies harvested from 200-iteration f_B
trajectories (the Phase-3 shape on the bench graph): for ncu captures of
the 2-flip sweep kernels."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06921_b200 as P  # noqa: E402

K = 8
g = P.generate(P.BaSpec(1_000_000, 5), 1)
b = P.ChainBatch(g, K)
b.set_x(np.random.default_rng(0).uniform(-1, 1, (K, g.n())))
b.run_trajectories(P.PerturbedBias(0.001), P.OptimizerConfig(alpha=0.0025, beta=0.8, max_iters=200))
scores, valid, packed = b.harvest(P.PROBLEM_MAXCUT)
t0 = time.time()
out, gains = P.local_search(b, 2, packed)
print("one_two_flip x8", round(time.time() - t0, 3), "s; gains", gains.tolist())
