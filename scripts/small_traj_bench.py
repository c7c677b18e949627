"""Per-iteration latency of trajectories on the small configs (C1/C2): the
SMEM cluster-per-chain path (automatic and forced cluster sizes) vs the
cooperative persistent path."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2605_06921_b200 as P
    from paper_2605_06921_b200 import _lib
    cases = [("c1_mis", P.ErSpec(1000, 0.01), P.MisQubo(2.0), 0.0),
             ("c2_fB", P.ErSpec(2000, 6 / 2000), P.PerturbedBias(0.001), -1.0)]
    for name, gs, spec, lo in cases:
        g = P.generate(gs, 1)
        for B in (1, 32, 256):
            X = np.random.default_rng(B).uniform(lo, 1.0, (B, g.n()))
            for path, cta, clu in (("smem_auto", 1, 0), ("smem_c1", 1, 1), ("smem_c2", 1, 2),
                                   ("smem_c4", 1, 4), ("smem_c8", 1, 8), ("smem_c16", 1, 16),
                                   ("persistent", 0, 0)):
                if clu > 1 and B * clu > 1200:
                    continue
                _lib.check(_lib.lib.mqo_tune(b"cta_traj", cta))
                _lib.check(_lib.lib.mqo_tune(b"cta_cluster", clu))
                b = P.ChainBatch(g, B)
                # alpha tiny + conv_tol 0: every chain runs to the iteration cap
                cfg = P.OptimizerConfig(alpha=1e-12, beta=0.3, max_iters=2000, conv_tol=0.0)
                b.set_x(X)
                b.run_trajectories(spec, cfg)
                b.set_x(X)
                t0 = time.perf_counter()
                it, rs = b.run_trajectories(spec, cfg)
                dt = time.perf_counter() - t0
                print(json.dumps({"case": name, "B": B, "path": path, "iters": int(it.max()),
                                  "us_per_iter": round(dt / it.max() * 1e6, 3),
                                  "edge_chain_per_s": 2 * g.m() * int(it.sum()) / dt}), flush=True)
    _lib.check(_lib.lib.mqo_tune(b"cta_traj", 1))
    _lib.check(_lib.lib.mqo_tune(b"cta_cluster", 0))


if __name__ == "__main__":
    main()
