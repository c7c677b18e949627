"""Small driver for profiling the SMEM one-CTA-per-chain trajectory kernel:
ER(1000, p=0.01) MIS QUBO, B chains, 500 iterations to the cap."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2605_06921_b200 as P
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    g = P.generate(P.ErSpec(1000, 0.01), 1)
    b = P.ChainBatch(g, B)
    b.set_x(np.random.default_rng(0).uniform(0, 1, (B, g.n())))
    it, rs = b.run_trajectories(P.MisQubo(2.0), P.OptimizerConfig(
        alpha=1e-12, beta=0.3, max_iters=500, conv_tol=0.0))
    print("iterations", int(it.sum()))


if __name__ == "__main__":
    main()
