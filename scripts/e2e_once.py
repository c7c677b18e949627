import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests/golden")
import paper_2605_06921_b200 as P
from make_engine_golden import RUNS
(kind, n, a, seed), oc = RUNS["c4"]
g = P.generate(P.BaSpec(n, a), seed)
spec = P.PerturbedBias(oc.param)
cfg = P.SolverConfig(objective=spec, optimizer=P.OptimizerConfig(oc.alpha, oc.beta, oc.max_iters),
                     reset_fraction=oc.reset_fraction, reset_rounds=oc.reset_rounds, seed=oc.seed,
                     time_budget_secs=3600, max_outer_loops=1, pool_batch=oc.pool_batch, pool_keep=oc.pool_keep)
r = P.solve_pooled(g, cfg)
print(r.best_score, r.elapsed_secs)
