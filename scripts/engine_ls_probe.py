import sys, time
sys.path.insert(0, "/root/repo")
import paper_2605_06921_b200 as P
g = P.generate(P.ErSpec(1000, 0.01), 1)
cfg = P.SolverConfig(objective=P.MisQubo(2.0), optimizer=P.OptimizerConfig(0.8, 0.3),
                     reset_fraction=0.7, reset_rounds=int(sys.argv[1]), seed=1, time_budget_secs=600,
                     max_outer_loops=1, pool_batch=256, pool_keep=8)
t = time.monotonic()
print("[mqo 0 %.6f] start" % t, file=sys.stderr)
r = P.solve_pooled(g, cfg)
print("[mqo 0 %.6f] end" % time.monotonic(), file=sys.stderr)
print(r.best_score, r.elapsed_secs)
