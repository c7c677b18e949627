"""Parity of the integration points at BASELINE.json's config sizes.

* The whole engine (solve_pooled, run_engine solver.cpp:192-372) on C3
  (ER(1e5) MIS, B=16) and C4 (BA(1e6) f_B, B=16) against reports produced by
  the compiled reference itself (tests/golden/engine_large.npz,
  tests/golden/make_engine_golden.py): identical counters, phase gains,
  iterations, last stop and best body.  At these sizes the engine runs the
  per-pass chain-tiled trajectories, the grid-round 1-flip, the look-ahead
  2-flip, the CTA (1,2)-swap without SMEM staging and multi-candidate body
  copies -- combinations the small-graph engine tests never reach.  Parity
  template: tests/test_solver.cpp:192-214 (same_report).
* C3 x 256 chains through the automatic chain tiler (pga.cu group sizing):
  fp64 steps and trajectories bit-exact against the oracle on sampled chains.
* C5, ER(1e7, d=16) from the O(m) generator, 64 chains: fp64 steps and
  MIS trajectories bit-exact against the oracle on sampled chains
  (pga.cpp:51-111).
"""
import hashlib
import os

import numpy as np
import pytest

import oracle
from oracle import MIS_QUBO, PERTURBED_BIAS

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2605_06921_b200 as P
    return P


def same(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                          np.ascontiguousarray(b).view(np.uint64))


def _report(r):
    return {"score": r.best_score, "found_solution": int(r.found_solution),
            "after_gradient": r.after_gradient, "after_reset_loop": r.after_reset_loop,
            "after_local_search": r.after_local_search, "outer_loops": r.outer_loops,
            "trajectories": r.trajectories, "resets_accepted": r.resets_accepted,
            "resets_rejected": r.resets_rejected, "total_iterations": r.total_iterations,
            "last_trajectory_stop": r.last_trajectory_stop, "n_warnings": len(r.warnings)}


def _cfg(P, oc):
    spec = P.MisQubo(oc.param) if oc.objective == MIS_QUBO else P.PerturbedBias(oc.param)
    return P.SolverConfig(
        objective=spec, optimizer=P.OptimizerConfig(oc.alpha, oc.beta, oc.max_iters, oc.conv_tol,
                                                     oc.check_every),
        reset_fraction=oc.reset_fraction, reset_rounds=oc.reset_rounds, init_noise=oc.init_noise,
        time_budget_secs=oc.time_budget_secs, seed=oc.seed, local_search=oc.local_search,
        pool_batch=oc.pool_batch, pool_keep=oc.pool_keep, max_outer_loops=oc.max_outer_loops)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name", ["c3", "c4"])
def test_engine_config_scale_vs_reference(P, name):
    import sys
    sys.path.insert(0, GOLD)
    from make_engine_golden import RUNS
    z = np.load(os.path.join(GOLD, "engine_large.npz"))
    (kind, n, a, seed), oc = RUNS[name]
    g = P.generate(P.ErSpec(n, a) if kind == "er" else P.BaSpec(n, a), seed)
    r = P.solve_pooled(g, _cfg(P, oc))
    keys = [str(k) for k in z["report_keys"]]
    got = _report(r)
    assert [got[k] for k in keys] == z[name + "_report"].tolist(), (got, z[name + "_report"])
    body = np.ascontiguousarray(r.best_body, np.uint8)
    assert hashlib.sha256(body.tobytes()).hexdigest() == str(z[name + "_body_sha"])
    print(f"{name}: {r.elapsed_secs:.2f} s on the GPU vs {float(z[name + '_elapsed'][0]):.1f} s "
          "for the reference (8 threads, golden generation)")


@pytest.mark.timeout(900)
def test_c3_256_chains_auto_tiler_bit_exact(O, P):
    og = O.generate_er(100_000, 1e-4, 1)
    pg = P.generate(P.ErSpec(100_000, 1e-4), 1)
    B = 256
    X = np.random.default_rng(256).uniform(0.0, 1.0, (B, og.n))
    b = P.ChainBatch(pg, B)  # MQO_GROUP_QUADS at its default: the automatic tiler
    b.set_x(X)
    b.zero_v()
    cfg = P.OptimizerConfig(alpha=0.8, beta=0.3)
    for _ in range(3):
        b.step(P.MisQubo(2.0), cfg)
    gx, gv = b.get_x(), b.get_v()
    for c in (0, 31, 32, 127, 200, 255):
        x, v = X[c].copy(), np.zeros(og.n)
        for _ in range(3):
            x, v = O.step(og, MIS_QUBO, 2.0, x, v, 0.8, 0.3)
        assert same(gx[c], x) and same(gv[c], v), c
    # trajectories with the fused checker, capped: iterations / reasons /
    # final states of sampled chains
    b.set_x(X)
    tcfg = P.OptimizerConfig(alpha=0.8, beta=0.3, max_iters=40)
    it, rs = b.run_trajectories(P.MisQubo(2.0), tcfg)
    gx = b.get_x()
    for c in (5, 64, 250):
        x, i, r = O.run_trajectory(og, MIS_QUBO, 2.0, X[c], 0.8, 0.3, 40)
        assert (int(it[c]), int(rs[c])) == (i, r) and same(gx[c], x), c


@pytest.mark.timeout(1200)
def test_c5_sampled_chains_bit_exact(O, P):
    n = 10_000_000
    pg = P.generate(P.ErFastSpec(n, 16.0 / n), 1)
    off, nbr = pg.csr()
    og = O.from_csr(n, off, nbr)
    del nbr
    B = 64
    rng = np.random.default_rng(5)
    b = P.ChainBatch(pg, B)
    X = np.empty((B, n))
    for c in range(B):
        X[c] = rng.uniform(0.0, 1.0, n)
    b.set_x(X)
    b.zero_v()
    cfg = P.OptimizerConfig(alpha=0.8, beta=0.3)
    for _ in range(3):
        b.step(P.MisQubo(2.0), cfg)
    gx, gv = b.get_x(), b.get_v()
    for c in (0, 33, 63):
        x, v = X[c].copy(), np.zeros(n)
        for _ in range(3):
            x, v = O.step(og, MIS_QUBO, 2.0, x, v, 0.8, 0.3)
        assert same(gx[c], x) and same(gv[c], v), c
    b.set_x(X)
    tcfg = P.OptimizerConfig(alpha=0.8, beta=0.3, max_iters=3)
    it, rs = b.run_trajectories(P.MisQubo(2.0), tcfg)
    gx = b.get_x()
    for c in (7, 50):
        x, i, r = O.run_trajectory(og, MIS_QUBO, 2.0, X[c], 0.8, 0.3, 3)
        assert (int(it[c]), int(rs[c])) == (i, r) and same(gx[c], x), c
