"""Time-to-quality: best MIS size / cut at a fixed wall-clock budget, GPU
engine vs the reference's CPU solve_pooled on the same graph, seed and
config (BASELINE.json's second metric).

python scripts/ttq.py --budget 20 [--configs c1,c2,c3] [--out profiles/ttq.json]

The reference runs through oracle/_ref (the compiled reference core) with
MQO_THREADS = all host cores; the GPU runs the engine through the C ABI.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (generator, problem cfg, B, K)
    "c1": (("er", 1000, 0.01), dict(objective=0, param=2.0, alpha=0.8, beta=0.3,
                                    reset_fraction=0.7, reset_rounds=60), 1, 1),
    "c1_b256": (("er", 1000, 0.01), dict(objective=0, param=2.0, alpha=0.8, beta=0.3,
                                         reset_fraction=0.7, reset_rounds=60), 256, 8),
    "c2": (("er", 2000, 6 / 2000), dict(objective=4, param=0.001, alpha=0.0025, beta=0.8,
                                        reset_fraction=0.8, reset_rounds=90), 1, 1),
    "c2_b256": (("er", 2000, 6 / 2000), dict(objective=4, param=0.001, alpha=0.0025, beta=0.8,
                                             reset_fraction=0.8, reset_rounds=90), 256, 8),
    "c3": (("er", 100000, 1e-4), dict(objective=0, param=2.0, alpha=0.8, beta=0.3,
                                      reset_fraction=0.6, reset_rounds=60), 256, 8),
    "c4": (("ba", 1000000, 5), dict(objective=4, param=0.001, alpha=0.0025, beta=0.8,
                                    reset_fraction=0.8, reset_rounds=90), 128, 8),
    # ER(1e7, d=16) from the O(m) generator (the reference's O(n^2) ER would
    # take ~49 h); isolated vertices stripped; the reference gets the same
    # edge list through Graph::from_edges
    "c5": (("erfast", 10_000_000, 16 / 10_000_000), dict(objective=0, param=2.0, alpha=0.8,
                                                         beta=0.3, reset_fraction=0.6,
                                                         reset_rounds=60), 64, 8),
}


def stripped_edges(g):
    """(n_core, edges u<v) of g without its isolated vertices, relabelled in
    ascending order (strip_isolated, graph.cpp:180-198)."""
    import numpy as np
    off, nbr = g.csr()
    deg = np.diff(off)
    keep = np.flatnonzero(deg > 0)
    remap = np.full(g.n(), -1, np.int64)
    remap[keep] = np.arange(len(keep))
    src = np.repeat(np.arange(g.n()), deg)
    m = src < nbr
    return len(keep), np.stack([remap[src[m]], remap[nbr[m]]], 1).astype(np.int32)


def c5_graph(P, gen, seed, device):
    g = P.generate(P.ErFastSpec(gen[1], gen[2]), seed, device=device)
    return P.strip_isolated(g).core if device >= 0 else g


def run(name, budget, seed, which, local_search=True):
    import oracle
    gen, pc, B, K = CONFIGS[name]
    if which == "gpu":
        import paper_2605_06921_b200 as P
        g = (P.generate(P.ErSpec(gen[1], gen[2]), seed) if gen[0] == "er"
             else c5_graph(P, gen, seed, 0) if gen[0] == "erfast"
             else P.generate(P.BaSpec(gen[1], gen[2]), seed))
        spec = P.MisQubo(pc["param"]) if pc["objective"] == 0 else P.PerturbedBias(pc["param"])
        cfg = P.SolverConfig(objective=spec, optimizer=P.OptimizerConfig(pc["alpha"], pc["beta"]),
                             reset_fraction=pc["reset_fraction"], reset_rounds=pc["reset_rounds"],
                             time_budget_secs=budget, seed=seed, pool_batch=B, pool_keep=K,
                             local_search=local_search)
        t0 = time.time()
        r = P.solve_pooled(g, cfg)
        return dict(score=r.best_score, outer_loops=r.outer_loops, trajectories=r.trajectories,
                    iterations=r.total_iterations, wall=time.time() - t0,
                    edge_chain_per_s=r.total_iterations * 2 * g.m() / max(r.elapsed_secs, 1e-9))
    L = oracle.load("ref" if oracle.have_ref() else "oracle")
    os.environ["MQO_THREADS"] = str(os.cpu_count() or 1)
    if gen[0] == "erfast":  # the GPU side's edge list, stripped, through from_edges
        import numpy as np
        import paper_2605_06921_b200 as P
        hg = P.generate(P.ErFastSpec(gen[1], gen[2]), seed, device=-1)
        n_core, edges = stripped_edges(hg)
        del hg
        g = L.from_edges(n_core, edges)
    else:
        g = (L.generate_er(gen[1], gen[2], seed) if gen[0] == "er"
             else L.generate_ba(gen[1], gen[2], seed))
    c = oracle.Cfg(time_budget_secs=budget, seed=seed, pool_batch=B, pool_keep=K,
                   local_search=1 if local_search else 0, **pc)
    t0 = time.time()
    rep, _ = L.solve_pooled(g, c.to_c())
    return dict(score=rep["score"], outer_loops=rep["outer_loops"],
                trajectories=rep["trajectories"], iterations=rep["total_iterations"],
                wall=time.time() - t0,
                edge_chain_per_s=rep["total_iterations"] * 2 * g.m / max(rep["elapsed_secs"], 1e-9),
                ref_impl=L.name, threads=os.cpu_count())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=20.0)
    ap.add_argument("--configs", default="c1,c1_b256,c2,c2_b256")
    ap.add_argument("--seeds", default="1")
    ap.add_argument("--which", default="gpu,ref")
    ap.add_argument("--out", default="")
    ap.add_argument("--no-local-search", action="store_true",
                    help="both sides without local search (the reference's restart-from-0 "
                         "(1,2)-swap is O(swaps x n): hours at n = 1e7)")
    args = ap.parse_args()
    rows = []
    for name in args.configs.split(","):
        for seed in [int(s) for s in args.seeds.split(",")]:
            for which in args.which.split(","):
                res = run(name, args.budget, seed, which, not args.no_local_search)
                row = dict(config=name, seed=seed, impl=which, budget_secs=args.budget,
                           local_search=not args.no_local_search, **res)
                print(json.dumps(row), flush=True)
                rows.append(row)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
