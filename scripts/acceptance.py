"""The reference's acceptance suite (/root/reference/proj/tests/acceptance.cpp)
rerun on the B200 backend: same instances, seeds, budgets and thresholds,
every solver-path quantity (gradients, trajectories, fixed-point checks,
local search, the pooled engine) computed through the C ABI on the GPU.

    python scripts/acceptance.py [--criteria 1,2,...] [--out FILE]

Output lines follow acceptance.cpp:28-35 ("[PASS] criterion N: name -- detail").
The reference's own recorded run is proj/test_output.txt (criterion 5's
perturbed-Laplacian leg fails there with mean 39.800; the B200 path is
bit-identical on that trajectory and reports the same value).
Differences in procedure, each forced by the backend and stated here:
* the dense census of criteria 3/4 (oracle.cpp:140-193) is a numpy dense
  product on the host -- an independent check of the GPU checker;
* the 60-second solves of criteria 9-11 and "extra" run concurrently (each
  is a B = K = 1 solve using a handful of SMs), each with its own 60 s
  wall-clock budget, instead of one after another;
* criterion 8 (toy_reset_experiment, a host-only double-well study with no
  graph) is reported as skipped, as `mqo verify` does.
"""
import argparse
import concurrent.futures
import json
import math
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_06921_b200 as P  # noqa: E402
from paper_2605_06921_b200 import _lib, cli, verify  # noqa: E402
from paper_2605_06921_b200.verify import Rng, derive_seed  # noqa: E402

K_SEED = 20250801
ESC_N, ESC_P = 100, 1.66 / 100.0
FAILS = []
OUT = []


def line(criterion, name, ok, detail):
    label = f"criterion {criterion}" if criterion > 0 else "extra"
    s = f"[{'PASS' if ok else 'FAIL'}] {label}: {name} — {detail}"
    print(s, flush=True)
    OUT.append(s)
    if not ok:
        FAILS.append(s)


def er(n, p, seed):
    return P.generate(P.ErSpec(n, p), seed)


def mis_preset(budget, seed):  # acceptance.cpp:42-54
    return P.SolverConfig(objective=P.MisQubo(2.0), optimizer=P.OptimizerConfig(0.8, 0.3),
                          reset_fraction=0.5, reset_rounds=60, init_noise=0.15,
                          time_budget_secs=budget, seed=seed)


def maxcut_preset(budget, seed):  # acceptance.cpp:56-67
    return P.SolverConfig(objective=P.PerturbedBias(0.001),
                          optimizer=P.OptimizerConfig(0.0025, 0.8), reset_fraction=0.8,
                          reset_rounds=90, init_noise=0.15, time_budget_secs=budget, seed=seed)


def dense(g):
    off, nbr = g.csr()
    A = np.zeros((g.n(), g.n()))
    A[np.repeat(np.arange(g.n()), np.diff(off)), nbr] = 1.0
    return A


def dense_grad(spec, A, X):
    """objectives.cpp:101-134 with a dense A (exact for binary / +-1 states)."""
    Y = X @ A.T
    d = A.sum(1)
    if isinstance(spec, P.MisQubo):
        return 1.0 - spec.gamma * Y
    if isinstance(spec, P.Laplacian):
        return 0.5 * (d * X - Y)
    if isinstance(spec, P.PerturbedLaplacian):
        return 2.0 * (d * X - Y + spec.lam * X)
    if isinstance(spec, P.Adjacency):
        return -2.0 * Y
    return -2.0 * Y - spec.lam


def gpu_binary_fixed(spec, g, X):
    """maxcut_binary_fixed_point_check (pga.cpp:137-152) for a batch of
    +-1 states: x_v * grad_v >= 0 for every v, gradients on the GPU."""
    b = P.ChainBatch(g, len(X))
    b.set_x(X)
    return ~np.any(X * b.gradient(spec) < 0.0, axis=1)


def c1():  # acceptance.cpp:71-100
    mis_hits = cut_hits = 0
    never = True
    for i in range(100):
        n, p = 8 + i % 7, 0.3 if (i // 7) % 2 == 0 else 0.5
        g = er(n, p, derive_seed(K_SEED, 1000 + i))
        mis_opt, cut_opt = verify.exact_optima(g)
        cfg = mis_preset(5.0, derive_seed(K_SEED, 2000 + i))
        cfg.stop_at_score = mis_opt
        r = P.solve_mis(g, cfg)
        never &= r.best_score <= mis_opt
        mis_hits += r.best_score == mis_opt
        cfg = maxcut_preset(5.0, derive_seed(K_SEED, 3000 + i))
        cfg.stop_at_score = cut_opt
        r = P.solve_maxcut(g, cfg)
        never &= r.best_score <= cut_opt
        cut_hits += r.best_score == cut_opt
    line(1, "solver never exceeds the exact optimum", never, "hard bound")
    line(1, "MIS matches exact on >= 95/100", mis_hits >= 95, f"{mis_hits}/100")
    line(1, "MaxCut matches exact on >= 95/100", cut_hits >= 95, f"{cut_hits}/100")


def c2():  # acceptance.cpp:102-122
    rng = Rng(derive_seed(K_SEED, 20))
    states, all_fixed = 0, True
    for gi in range(20):
        n = 16 + 3 * gi
        p = rng.uniform(0.1, 0.6)
        g = er(min(n, 64), p, derive_seed(K_SEED, 2100 + gi))
        X = np.array([[1.0 if rng.next_u64() & 1 else -1.0 for _ in range(g.n())]
                      for _ in range(50)])
        for lam in (0.001, 0.1, 1.0):
            all_fixed &= bool(gpu_binary_fixed(P.PerturbedLaplacian(lam), g, X).all())
        states += 50
    line(2, "1000 random binary states, lambda in {0.001, 0.1, 1}", all_fixed,
         f"{states} states, zero tolerance")


def c3():  # acceptance.cpp:124-152
    never_fixed = bias_ok = matches = True
    states = 0
    for gi in range(20):
        n = 6 + gi % 5
        g = er(n, 0.5 if gi % 2 else 0.35, derive_seed(K_SEED, 2200 + gi))
        A = dense(g)
        for spec in (P.Adjacency(), P.PerturbedBias(0.001)):
            c = verify.census(spec, g)  # GPU gradients of all 2^n states
            bits = verify._bits(n)
            X = 2.0 * bits - 1.0
            dense_fixed = ~np.any(X * dense_grad(spec, A, X) < 0.0, axis=1)
            states += len(X)
            never_fixed &= not np.any(c["repairable"] & dense_fixed)
            if isinstance(spec, P.PerturbedBias):
                bias_ok &= not np.any(dense_fixed & c["repairable"])
            matches &= bool(np.array_equal(gpu_binary_fixed(spec, g, X), dense_fixed))
    line(3, "1-flip repairable => not fixed (f_A, f_B)", never_fixed,
         f"{states} states exhaustively")
    line(3, "f_B fixed => 1-flip irreparable", bias_ok, "zero tolerance")
    line(3, "implementation checker agrees with the dense census", matches, "every state")


def c4():  # acceptance.cpp:154-190
    all_fixed = True
    maximal_count = swap_rep = 0
    for gi in range(20):
        n = 8 + gi % 5
        g = er(n, 0.45 if gi % 2 else 0.25, derive_seed(K_SEED, 2300 + gi))
        A = dense(g)
        bits = verify._bits(n).astype(np.float64)
        Y = bits @ A.T
        independent = ~np.any((bits == 1) & (Y > 0), axis=1)
        maximal = independent & ~np.any((bits == 0) & (Y == 0), axis=1)
        M = bits[maximal]
        maximal_count += len(M)
        b = P.ChainBatch(g, len(M))
        b.set_x(M)
        all_fixed &= bool(b.mis_fixed_point_check(2.0, 0.8).all())
        packed = P.pack_bodies(M.astype(np.uint8))
        _, sizes = P.local_search(b, _lib.LS_ONE_TWO_SWAP, packed)
        swap_rep += int(np.sum(sizes > M.sum(1)))  # a (1,2)-swap exists iff one is taken
    line(4, "every maximal IS is a PGA fixed point", all_fixed,
         f"{maximal_count} maximal sets, {swap_rep} of them (1,2)-swap repairable")
    line(4, "swap-repairable sets were exercised", swap_rep > 0, f"{swap_rep} witnesses")


def _run(g, spec, init, alpha, iters):  # experiments.cpp:11-26
    return verify._escape(g, spec, np.asarray(init, np.float64), alpha, iters)


def c5():  # acceptance.cpp:192-214
    zero, pm, bm = True, 0.0, 0.0
    for gi in range(10):
        g = er(ESC_N, ESC_P, derive_seed(K_SEED, 2400 + gi))
        c = Rng(derive_seed(K_SEED, 2500 + gi)).uniform(-1.0, 1.0)
        const = np.full(g.n(), c)
        il, fl = _run(g, P.Laplacian(), const, 0.1, 5000)
        _, fp = _run(g, P.PerturbedLaplacian(0.001), const, 0.1, 5000)
        _, fb = _run(g, P.PerturbedBias(0.001), const, 0.1, 5000)
        zero &= fl == 0 and il == 0
        pm += fp / 10
        bm += fb / 10
    line(5, "Laplacian stays at cut 0 exactly", zero, "10/10 graphs")
    line(5, "perturbed Laplacian mean final cut >= 40", pm >= 40.0, f"mean {pm:.3f}")
    line(5, "perturbed bias mean final cut >= 40", bm >= 40.0, f"mean {bm:.3f}")


def c6():  # acceptance.cpp:216-237
    ls = ps = True
    gain = 0.0
    for gi in range(10):
        g = er(ESC_N, ESC_P, derive_seed(K_SEED, 2400 + gi))
        side = verify._repairable_side(g, Rng(derive_seed(K_SEED, 2600 + gi)))
        init = np.where(side == 1, 1.0, -1.0)
        il, fl = _run(g, P.Laplacian(), init, 0.1, 5000)
        ip, fp = _run(g, P.PerturbedLaplacian(0.001), init, 0.1, 5000)
        ib, fb = _run(g, P.PerturbedBias(0.001), init, 0.1, 5000)
        ls &= fl == il
        ps &= fp == ip
        gain += (fb - ib) / 10
    line(6, "Laplacian is stuck exactly at the initial cut", ls, "10/10")
    line(6, "perturbed Laplacian is stuck exactly", ps, "10/10")
    line(6, "perturbed bias mean improvement >= 4", gain >= 4.0, f"mean gain {gain:.3f}")


def c7():  # acceptance.cpp:239-280
    bl = bp = ba = True
    detail = ""
    for n, d in ((100, 50.0), (1000, 100.0)):
        means = {"l": 0.0, "p": 0.0, "a": 0.0, "b": 0.0}
        for gi in range(3):
            g = er(n, d / n, derive_seed(K_SEED, 2700 + gi))
            r = Rng(derive_seed(K_SEED, 2800 + gi))
            st = np.zeros(1, dtype=_lib.RNG_DTYPE)
            st[0]["s"] = r.st
            init, _ = P.init_state_host(g, P.PROBLEM_MAXCUT, 0.15, st)
            opt = P.OptimizerConfig(alpha=0.0025, beta=0.8, max_iters=20000)
            for key, spec in (("l", P.Laplacian()), ("p", P.PerturbedLaplacian(0.001)),
                              ("a", P.Adjacency()), ("b", P.PerturbedBias(0.001))):
                out = P.run_trajectory(spec, g, init, opt)
                means[key] += verify._cut(g, (out.state > 0).astype(np.uint8)) / 3
        bl &= means["b"] >= 1.05 * means["l"]
        bp &= means["b"] >= 1.05 * means["p"]
        ba &= means["b"] >= means["a"]
        detail += (f"(n={n}: fL {means['l']:.3f}, fP {means['p']:.3f}, fA {means['a']:.3f}, "
                   f"fB {means['b']:.3f}) ")
    line(7, "f_B beats f_L by >= 5%", bl, detail)
    line(7, "f_B beats f_P by >= 5%", bp, detail)
    line(7, "f_B >= f_A", ba, detail)


def _parallel(jobs):
    with concurrent.futures.ThreadPoolExecutor(len(jobs)) as ex:
        return list(ex.map(lambda f: f(), jobs))


def c9_10_11_extra(which):  # acceptance.cpp:296-385
    jobs, tags = [], []
    if 9 in which:
        graphs = [er(3000, 100.0 / 3000.0, derive_seed(K_SEED, s)) for s in (3100, 3200, 3300)]
        for ri, rho in enumerate((0.0, 0.4, 0.5, 0.6, 0.7)):
            for si in range(3):
                cfg = mis_preset(60.0, derive_seed(K_SEED, 3400 + 10 * ri + si))
                cfg.reset_fraction = rho
                jobs.append(lambda g=graphs[si], c=cfg: P.solve_mis(g, c))
                tags.append(("c9", rho, si))
    if 10 in which:
        g10 = er(3000, 100.0 / 3000.0, derive_seed(K_SEED, 3500))
        cfg = mis_preset(60.0, derive_seed(K_SEED, 3501))
        cfg.reset_fraction = 0.6
        jobs.append(lambda g=g10, c=cfg: P.solve_mis(g, c))
        tags.append(("c10", 0, 0))
    if 11 in which:
        g11 = er(1000, 0.1, derive_seed(K_SEED, 3600))
        for si in range(8):
            cfg = mis_preset(60.0, derive_seed(K_SEED, 3700 + si))
            cfg.reset_fraction = 0.7
            jobs.append(lambda g=g11, c=cfg: P.solve_mis(g, c))
            tags.append(("c11", 0, si))
    if 0 in which:
        for si in range(3):
            g = er(100, 0.5, derive_seed(K_SEED, 3800 + si))
            jobs.append(lambda g=g, c=maxcut_preset(60.0, derive_seed(K_SEED, 3900 + si)):
                        P.solve_maxcut(g, c))
            tags.append(("extra", 0, si))
    if not jobs:
        return
    # at most 16 concurrent B = K = 1 solves at a time
    reps = []
    for k in range(0, len(jobs), 16):
        reps += _parallel(jobs[k:k + 16])
    res = dict(zip(tags, reps))
    if 9 in which:
        means = [sum(res[("c9", rho, si)].best_score for si in range(3)) / 3
                 for rho in (0.0, 0.4, 0.5, 0.6, 0.7)]
        detail = "  ".join(f"rho={rho:.3f}: {m:.3f}" for rho, m in
                           zip((0.0, 0.4, 0.5, 0.6, 0.7), means))
        line(9, "best rho in {0.4..0.7} strictly beats rho = 0", max(means[1:]) > means[0],
             detail)
    if 10 in which:
        r = res[("c10", 0, 0)]
        rg = r.after_reset_loop - r.after_gradient
        lg = r.after_local_search - r.after_reset_loop
        line(10, "reset gain > local-search gain >= 0", rg > lg >= 0,
             f"gradient {r.after_gradient} -> reset +{rg} -> local search +{lg}")
    if 11 in which:
        sc = [res[("c11", 0, si)].best_score for si in range(8)]
        mean = sum(sc) / 8
        line(11, "mean MIS size >= 63 over 8 seeds at 60 s", mean >= 63.0,
             f"mean {mean:.3f} [{' '.join(map(str, sc))} ]")
    if 0 in which:
        sc = [res[("extra", 0, si)].best_score for si in range(3)]
        mean = sum(sc) / 3
        line(0, "mean cut >= 1425 on ER(100, d=50)", mean >= 1425.0,
             f"mean {mean:.3f} [{' '.join(map(str, sc))} ]")


def c12():  # acceptance.cpp:387-404
    def run(flags):
        r = subprocess.run([sys.executable, "-m", "paper_2605_06921_b200.cli", *flags.split()],
                           capture_output=True, text=True, cwd=ROOT)
        rec = json.loads(r.stdout)
        rec.pop("timing")
        return cli.dump_record(rec), len(r.stdout)
    mis = ("solve --problem mis --gen er:80:6 --seed 11 --budget-secs 120 --max-outer 2 "
           "--tgs 10 --report json")
    a, b = run(mis), run(mis)
    line(12, "MIS records match byte for byte (timing excluded)", a[0] == b[0], f"{a[1]} bytes")
    cut = ("solve --problem maxcut --gen er:80:6 --seed 11 --budget-secs 120 --max-outer 1 "
           "--tgs 10 --report json")
    c, d = run(cut), run(cut)
    line(12, "MaxCut records match byte for byte (timing excluded)", c[0] == d[0],
         f"{c[1]} bytes")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--criteria", default="1,2,3,4,5,6,7,8,9,10,11,0,12")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    which = {int(x) for x in a.criteria.split(",") if x}
    for k, fn in ((1, c1), (2, c2), (3, c3), (4, c4), (5, c5), (6, c6), (7, c7)):
        if k in which:
            fn()
    if 8 in which:
        s = ("[SKIP] criterion 8: coordinate resets beat full restarts on the double well — "
             "toy_reset_experiment is a host-only study with no graph path (DESIGN.md §7)")
        print(s, flush=True)
        OUT.append(s)
    c9_10_11_extra(which & {9, 10, 11, 0})
    if 12 in which:
        c12()
    summary = f"{len(FAILS)} check(s) failed" if FAILS else "all checks passed"
    print(summary)
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(OUT + [summary]) + "\n")
    return 1 if FAILS else 0


if __name__ == "__main__":
    sys.exit(main())
