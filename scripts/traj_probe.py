"""Small driver for profiling the trajectory kernels: BA(1e6,5) f_B, 128
chains, one bounded run_trajectories call (default 4 passes)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2605_06921_b200 as P
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    g = P.generate(P.BaSpec(1_000_000, 5), 1)
    b = P.ChainBatch(g, 128)
    b.set_x(np.random.default_rng(0).uniform(-1, 1, (128, g.n())))
    it, rs = b.run_trajectories(P.PerturbedBias(0.001),
                                P.OptimizerConfig(alpha=0.0025, beta=0.8, max_iters=iters))
    print("iterations", int(it.sum()))


if __name__ == "__main__":
    main()
