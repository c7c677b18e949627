"""Per-round stages of the engine at the large configs, one call each, for
timing and for the per-kernel ncu metric pass (scripts/profile_rounds.sh).

    python scripts/round_probe.py [c4|c3] [reps]

c4: MaxCut f_B on BA(1e6,5), 128 chains (bench workload); c3: MIS QUBO on
ER(1e5, d=10), 256 chains.  Stages: device init (K3), 200-iteration
trajectories, harvest (K5/K6), pool reset (K4), local search on 8 pool bodies
(K7 one_two_flip / K8 one_two_swap).  Prints one JSON line per stage with the
synchronised wall time and the stage's algorithmic bytes.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2605_06921_b200 as P
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    if cfgname == "c4":
        g = P.generate(P.BaSpec(1_000_000, 5), 1)
        B, problem, spec = 128, P.PROBLEM_MAXCUT, P.PerturbedBias(0.001)
        opt = P.OptimizerConfig(alpha=0.0025, beta=0.8, max_iters=200)
        rho, ls_op = 0.8, P.api._lib.LS_ONE_TWO_FLIP
    else:
        g = P.generate(P.ErFastSpec(100_000, 10 / 100_000), 1)
        B, problem, spec = 256, P.PROBLEM_MIS, P.MisQubo(2.0)
        opt = P.OptimizerConfig(alpha=0.8, beta=0.3, max_iters=200)
        rho, ls_op = 0.6, P.api._lib.LS_ONE_TWO_SWAP
    n, nnz = g.n(), 2 * g.m()
    b = P.ChainBatch(g, B)
    b.seed_streams(1)

    def timed(name, fn, algo_bytes):
        for _ in range(reps):
            b.sync()
            t = time.perf_counter()
            out = fn()
            b.sync()
            dt = time.perf_counter() - t
            print(json.dumps({"config": cfgname, "stage": name, "ms": round(dt * 1e3, 3),
                              "algo_bytes": algo_bytes,
                              "algo_GBps": round(algo_bytes / dt / 1e9, 1) if algo_bytes else None}),
                  flush=True)
        return out

    timed("init_states(device)", lambda: b.init_states(problem, 0.15), 8 * n * B + 8 * (n + 1))
    timed("run_trajectories(200)", lambda: b.run_trajectories(spec, opt), None)
    scores, valid, packed = timed("harvest", lambda: b.harvest(problem),
                                  8 * n * B + (4 * nnz + 8 * n if problem == P.PROBLEM_MIS else 0)
                                  + B * n // 8)
    order = np.argsort(-scores, kind="stable")[:8]
    pool = packed[order]
    b.set_pool(pool)
    k = int(rho * n)
    timed("reset_from_pool", lambda: b.reset_from_pool(problem, rho),
          B * (4 * k + 8 * k + 8 * (n - k) + 16 * n))
    timed("local_search(8 bodies)", lambda: P.local_search(b, ls_op, pool),
          None)


if __name__ == "__main__":
    main()
