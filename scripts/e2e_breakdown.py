"""Wall-time breakdown of bench.py's e2e step (golden c4 solve): graph upload
from pinned host CSR, solve_pooled (wall vs the engine's own elapsed), and
the rest.  python scripts/e2e_breakdown.py [reps]"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def main():
    import torch
    import paper_2605_06921_b200 as P
    from paper_2605_06921_b200 import _lib
    from make_engine_golden import RUNS
    (kind, n, a, seed), oc = RUNS["c4"]
    g0 = P.generate(P.BaSpec(n, a), seed)
    off, nbr = g0.csr()
    h_off, h_nbr = torch.from_numpy(off).pin_memory(), torch.from_numpy(nbr).pin_memory()
    cfg = P.SolverConfig(objective=P.PerturbedBias(oc.param),
                         optimizer=P.OptimizerConfig(oc.alpha, oc.beta, oc.max_iters),
                         reset_fraction=oc.reset_fraction, reset_rounds=oc.reset_rounds,
                         seed=oc.seed, time_budget_secs=1e6, max_outer_loops=1,
                         pool_batch=oc.pool_batch, pool_keep=oc.pool_keep)
    for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = C.c_void_p()
        _lib.check(P.api.lib.mqo_graph_upload(n, C.cast(h_off.data_ptr(), C.POINTER(C.c_int64)),
                                              C.cast(h_nbr.data_ptr(), C.POINTER(C.c_int32)),
                                              0, C.byref(h)))
        g = P.Graph(h, 0)
        t1 = time.perf_counter()
        r = P.solve_pooled(g, cfg)
        t2 = time.perf_counter()
        del g
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"upload {1e3 * (t1 - t0):.1f} ms  solve wall {1e3 * (t2 - t1):.1f} ms "
              f"(engine {1e3 * r.elapsed_secs:.1f})  free {1e3 * (t3 - t2):.1f} ms  "
              f"total {1e3 * (t3 - t0):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
