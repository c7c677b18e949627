"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libref.so,
compiled from /root/reference/proj/core/src by `make -C oracle ref`).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are committed; tests/test_golden.py checks the plain-C oracle
and the CUDA path against them on any box (no reference tree needed).
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import MIS_QUBO, PERTURBED_BIAS, PERTURBED_LAPLACIAN, LAPLACIAN, ADJACENCY  # noqa

OUT = os.path.dirname(os.path.abspath(__file__))
KSEED = 20250801


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    oracle.build(ref=True)
    R = oracle.load("ref")
    assert R.name == "reference"

    # --- RNG streams (rng.hpp) -------------------------------------------
    streams = {}
    for seed in (1, KSEED):
        for b in range(1, 5):
            r = R.rng(R.derive_seed(seed, b))
            streams[f"u64_{seed}_{b}"] = np.array([r.next_u64() for _ in range(256)], np.uint64)
    r = R.rng(7)
    streams["normal_7"] = np.array([r.normal(0.0, 1.0) for _ in range(257)])
    r = R.rng(11)
    streams["index_11"] = np.array([r.uniform_index(n) for n in range(1, 300)], np.uint64)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **streams)

    # --- graphs (graph.cpp generators + from_edges) ------------------------
    graphs = {}
    specs = {
        "er1000": ("er", 1000, 0.01, 1), "er2000": ("er", 2000, 6 / 2000, 1),
        "ba10000": ("ba", 10000, 5, 1), "sbm300": ("sbm", 300, 3, 0.2, 0.01, 4),
        "er100": ("er", 100, 0.0166, 2400),
    }
    for name, s in specs.items():
        if s[0] == "er":
            g = R.generate_er(s[1], s[2], s[3])
        elif s[0] == "ba":
            g = R.generate_ba(s[1], s[2], s[3])
        else:
            g = R.generate_sbm(*s[1:])
        off, nbr = g.csr()
        graphs[f"{name}_nm"] = np.array([g.n, g.m, g.max_degree], np.int64)
        graphs[f"{name}_sha"] = np.array(sha(off, nbr))
        if g.n <= 2000:
            graphs[f"{name}_off"] = off
            graphs[f"{name}_nbr"] = nbr
    np.savez_compressed(os.path.join(OUT, "graphs.npz"), **graphs)

    # --- steps / gradients / trajectories on C1 and C2 ---------------------
    steps = {}
    g1 = R.generate_er(1000, 0.01, 1)
    g2 = R.generate_er(2000, 6 / 2000, 1)
    rng = np.random.default_rng(2024)
    for gname, g, kinds in (("c1", g1, [(MIS_QUBO, 2.0)]),
                            ("c2", g2, [(PERTURBED_BIAS, 0.001), (LAPLACIAN, 0.0),
                                        (PERTURBED_LAPLACIAN, 0.001), (ADJACENCY, 0.0)])):
        for kind, param in kinds:
            lo = 0.0 if kind == MIS_QUBO else -1.0
            x0 = rng.uniform(lo, 1.0, g.n)
            steps[f"{gname}_k{kind}_x0"] = x0
            steps[f"{gname}_k{kind}_grad"] = R.gradient(g, kind, param, x0)
            alpha, beta = (0.8, 0.3) if kind == MIS_QUBO else (0.0025, 0.8)
            x, v = x0.copy(), np.zeros(g.n)
            for t in range(1, 101):
                x, v = R.step(g, kind, param, x, v, alpha, beta)
                if t in (1, 10, 100):
                    steps[f"{gname}_k{kind}_x{t}"] = x
                    steps[f"{gname}_k{kind}_v{t}"] = v
            xt, it, rs = R.run_trajectory(g, kind, param, x0, alpha, beta, 5000, 1e-6, 1)
            steps[f"{gname}_k{kind}_traj"] = xt
            steps[f"{gname}_k{kind}_traj_ir"] = np.array([it, rs], np.int64)
    np.savez_compressed(os.path.join(OUT, "steps.npz"), **steps)

    # --- solver pieces: init_state, global_reset, harvest, local search -----
    pieces = {}
    for sig in (0.0, 0.15):
        r = R.rng(R.derive_seed(1, 1))
        pieces[f"init_mis_{sig}"] = R.init_state(g1, 0, sig, r)
        pieces[f"init_mis_{sig}_next"] = np.array([r.next_u64()], np.uint64)
        r = R.rng(R.derive_seed(1, 2))
        pieces[f"init_cut_{sig}"] = R.init_state(g2, 1, sig, r)
    for n in (1000, 2001, 100000):
        for rho in (0.5, 0.6, 0.8):
            r = R.rng(R.derive_seed(n, int(rho * 10)))
            x, chosen = R.global_reset(np.ones(n), rho, r)
            key = f"reset_{n}_{rho}"
            pieces[key + "_sha"] = np.array(sha(chosen))
            pieces[key + "_next"] = np.array([r.next_u64()], np.uint64)
            if n <= 2001:
                pieces[key] = chosen
    # harvested states of the C1/C2 trajectories, then the LS moves
    for gname, g, kind, param, prob in (("c1", g1, MIS_QUBO, 2.0, 0), ("c2", g2, PERTURBED_BIAS,
                                                                         0.001, 1)):
        xt = steps[f"{gname}_k{kind}_traj"]
        body, score = R.extract_solution(g, prob, xt)
        pieces[f"{gname}_harvest"] = body
        pieces[f"{gname}_harvest_score"] = np.array([score], np.int64)
        if prob == 0:
            pieces["c1_independent"] = np.array([R.is_independent(g, body)], np.int64)
            ind, size = R.greedy_maximalize(g, body)
            pieces["c1_greedy"] = ind
            ind2, size2 = R.one_two_swap(g, ind)
            pieces["c1_swap"] = ind2
            # from the empty set, greedy then (1,2)-swap
            ind, _ = R.greedy_maximalize(g, np.zeros(g.n, np.uint8))
            pieces["c1_greedy_empty"] = ind
            pieces["c1_swap_empty"] = R.one_two_swap(g, ind)[0]
        else:
            pieces["c2_tight"] = R.build_gain_table(g, body)
            s1, g1f = R.one_flip_pass(g, body)
            s2, g2f = R.two_flip_pass(g, body)
            s3, g3f = R.one_two_flip(g, body)
            pieces["c2_oneflip"], pieces["c2_twoflip"], pieces["c2_onetwo"] = s1, s2, s3
            pieces["c2_gains"] = np.array([g1f, g2f, g3f], np.int64)
    np.savez_compressed(os.path.join(OUT, "pieces.npz"), **pieces)

    # --- whole-engine RunReports (solve_pooled, pinned max_outer_loops) -----
    reports = {}
    runs = {
        "c1_s1": (g1, oracle.Cfg(objective=MIS_QUBO, param=2.0, alpha=0.8, beta=0.3,
                                 reset_fraction=0.7, reset_rounds=60, seed=1,
                                 time_budget_secs=600, max_outer_loops=1)),
        "c1_s2_b4": (R.generate_er(1000, 0.01, 2),
                     oracle.Cfg(objective=MIS_QUBO, param=2.0, alpha=0.8, beta=0.3,
                                reset_fraction=0.7, reset_rounds=10, seed=2,
                                time_budget_secs=600, max_outer_loops=2, pool_batch=4,
                                pool_keep=3)),
        "c2_s1_b4": (g2, oracle.Cfg(objective=PERTURBED_BIAS, param=0.001, alpha=0.0025,
                                    beta=0.8, reset_fraction=0.8, reset_rounds=6, seed=1,
                                    time_budget_secs=600, max_outer_loops=1, pool_batch=4,
                                    pool_keep=3, max_iters=2000)),
    }
    keys = oracle.REPORT_KEYS
    for name, (g, cfg) in runs.items():
        rep, body = R.solve_pooled(g, cfg.to_c())
        reports[name + "_report"] = np.array([rep[k] for k in keys], np.int64)
        reports[name + "_body"] = body
    reports["report_keys"] = np.array(keys)

    # acceptance criterion 5 (acceptance.cpp:192-219): per-graph final cuts
    cuts = {PERTURBED_LAPLACIAN: [], PERTURBED_BIAS: [], LAPLACIAN: []}
    for gi in range(10):
        g = R.generate_er(100, 1.66 / 100.0, R.derive_seed(KSEED, 2400 + gi))
        c = -1.0 + 2.0 * R.rng(R.derive_seed(KSEED, 2500 + gi)).uniform01()  # Rng::uniform(-1, 1)
        for kind in cuts:
            param = 0.001
            x, it, rs = R.run_trajectory(g, kind, param, np.full(g.n, c), 0.1, 0.0, 5000,
                                         1e-6, 1)
            cuts[kind].append(R.extract_solution(g, 1, x)[1])
    for kind, v in cuts.items():
        reports[f"crit5_k{kind}"] = np.array(v, np.int64)
    np.savez_compressed(os.path.join(OUT, "reports.npz"), **reports)
    print("crit5 means: fP", np.mean(cuts[PERTURBED_LAPLACIAN]), "fB",
          np.mean(cuts[PERTURBED_BIAS]))


if __name__ == "__main__":
    main()
