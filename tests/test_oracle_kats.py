"""Pins the plain-C oracle (oracle/mqo_oracle.c) against the reference's own
known-answer tests (re-hosted from /root/reference/proj/tests/*.cpp, cited
per case) and, where oracle/_ref is built, against the reference itself.
CPU only."""
import numpy as np
import pytest

import oracle as orc
from oracle import (ADJACENCY, CHECKER_ACCEPTED, CONVERGED, ITER_CAP, LAPLACIAN, MIS_QUBO,
                    PERTURBED_BIAS, PERTURBED_LAPLACIAN, PROBLEM_MAXCUT, PROBLEM_MIS,
                    OracleError)


def path(L, n):
    return L.from_edges(n, [(v, v + 1) for v in range(n - 1)])


def cycle(L, n):
    return L.from_edges(n, [(v, (v + 1) % n) for v in range(n)])


def complete(L, n):
    return L.from_edges(n, [(u, v) for u in range(n) for v in range(u + 1, n)])


def star(L, leaves):
    return L.from_edges(leaves + 1, [(0, v) for v in range(1, leaves + 1)])


# ---------------------------------------------------------------- graph
def test_graph_canonicalisation(O):  # test_graph.cpp canonicalization
    g = O.from_edges(4, [(1, 0), (0, 1), (2, 3), (3, 2), (1, 3)])
    off, nbr = g.csr()
    assert g.m == 3
    assert off.tolist() == [0, 1, 3, 4, 6]
    assert nbr.tolist() == [1, 0, 3, 3, 1, 2]
    with pytest.raises(OracleError) as e:
        O.from_edges(3, [(1, 1)])
    assert e.value.code == 1 and "self-loop" in e.value.msg
    with pytest.raises(OracleError):
        O.from_edges(3, [(0, 3)])


def test_spmv_kats(O):  # test_graph.cpp:71-97
    k3 = complete(O, 3)
    x = np.array([1.0, -1.0, -1.0])
    assert O.adjacency_apply(k3, x).tolist() == [-2.0, 0.0, 0.0]
    assert O.laplacian_apply(k3, x).tolist() == [4.0, -2.0, -2.0]
    g = O.generate_er(30, 0.3, 5)
    for c in (0.3, -0.7, 1.0):
        assert (O.laplacian_apply(g, np.full(30, c)) == 0.0).all()


def test_spmv_dense(O):  # test_graph.cpp:99-114: agrees with a dense product
    rng = np.random.default_rng(1)
    for t in range(10):
        g = O.generate_er(40, 0.2, 100 + t)
        off, nbr = g.csr()
        A = np.zeros((g.n, g.n))
        for v in range(g.n):
            A[v, nbr[off[v]:off[v + 1]]] = 1
        x = rng.uniform(-1, 1, g.n)
        np.testing.assert_allclose(O.adjacency_apply(g, x), A @ x, rtol=0, atol=1e-12)
        L = np.diag(A.sum(1)) - A
        np.testing.assert_allclose(O.laplacian_apply(g, x), L @ x, rtol=0, atol=1e-12)


# ----------------------------------------------------------- objectives
def test_gradient_kats(O):  # test_objectives.cpp:71-79
    k3 = complete(O, 3)
    assert O.gradient(k3, MIS_QUBO, 2.0, [1, 0, 0]).tolist() == [1.0, -1.0, -1.0]
    assert O.gradient(k3, PERTURBED_BIAS, 0.25, [0, 0, 0]).tolist() == [-0.25] * 3


@pytest.mark.parametrize("kind,param", [(MIS_QUBO, 2.0), (LAPLACIAN, 0.0),
                                        (PERTURBED_LAPLACIAN, 0.001), (ADJACENCY, 0.0),
                                        (PERTURBED_BIAS, 0.001)])
def test_gradient_finite_differences(O, kind, param):  # test_objectives.cpp:81-102
    rng = np.random.default_rng(kind)
    g = O.generate_er(20, 0.3, 7)
    lo = 0.0 if kind == MIS_QUBO else -1.0
    x = rng.uniform(lo + 0.1, 0.9, g.n)
    grad = O.gradient(g, kind, param, x)
    h = 1e-6
    for v in range(g.n):
        xp, xm = x.copy(), x.copy()
        xp[v] += h
        xm[v] -= h
        fd = (O.value(g, kind, param, xp) - O.value(g, kind, param, xm)) / (2 * h)
        assert abs(fd - grad[v]) < 1e-5


def test_threshold_ties(O):  # test_objectives.cpp:104-130
    k3 = complete(O, 3)
    body, score = O.extract_solution(k3, PROBLEM_MIS, [0.5, 0.5, 0.5])
    assert score == 0 and body.sum() == 0
    body, score = O.extract_solution(k3, PROBLEM_MAXCUT, [0.0, 0.0, 0.0])
    assert score == 0 and body.tolist() == [0, 0, 0]


def test_cut_identities(O):  # test_objectives.cpp:160-175 (binary identities)
    g = O.generate_er(10, 0.5, 3)
    rng = np.random.default_rng(0)
    for _ in range(50):
        side = rng.integers(0, 2, g.n).astype(np.uint8)
        x = np.where(side == 1, 1.0, -1.0)
        cut = O.cut_value(g, side)
        assert O.value(g, LAPLACIAN, 0.0, x) == cut
        assert O.value(g, ADJACENCY, 0.0, x) == 4 * cut - 2 * g.m


# ------------------------------------------------------------------ pga
def test_project(O):  # test_pga.cpp:25-37
    assert O.project([1.3, -0.2, 0.5], PROBLEM_MIS).tolist() == [1.0, 0.0, 0.5]
    assert O.project([2.0, -2.0, 0.0], PROBLEM_MAXCUT).tolist() == [1.0, -1.0, 0.0]


def test_step_kats(O):  # test_pga.cpp:39-72
    k3 = complete(O, 3)
    x, _ = O.step(k3, MIS_QUBO, 2.0, [1.0, 0.0, 0.0], np.zeros(3), 0.1, 0.0)
    assert x.tolist() == [1.0, 0.0, 0.0]
    x, _ = O.step(k3, MIS_QUBO, 2.0, [0.3, 0.7, 0.2], np.zeros(3), 0.0, 0.0)
    assert x.tolist() == [0.3, 0.7, 0.2]


def test_trajectory_kats(O):  # test_pga.cpp:77-119
    k3 = complete(O, 3)
    x, it, r = O.run_trajectory(k3, MIS_QUBO, 2.0, [0.9, 0.1, 0.1], 0.8)
    assert r == CHECKER_ACCEPTED and x.tolist() == [1.0, 0.0, 0.0]
    x, it, r = O.run_trajectory(k3, PERTURBED_BIAS, 0.001, [0.6, -0.5, -0.4], 0.1)
    assert r == CONVERGED and x.tolist() == [1.0, -1.0, -1.0]
    assert O.extract_solution(k3, PROBLEM_MAXCUT, x)[1] == 2
    g = O.generate_er(24, 0.3, 73)
    for c in (0.3, -0.62, 0.97):
        x, it, r = O.run_trajectory(g, LAPLACIAN, 0.0, np.full(g.n, c), 0.1)
        assert (x == c).all() and r == CONVERGED
    x, it, r = O.run_trajectory(k3, MIS_QUBO, 2.0, [0.4, 0.4, 0.4], 1e-9, max_iters=12)
    assert r == ITER_CAP and it == 12


def test_checker_kats(O):  # test_pga.cpp:138-148
    assert O.mis_fixed_point_check(complete(O, 3), [1, 0, 0])
    assert not O.mis_fixed_point_check(path(O, 3), [1, 0, 0])
    assert O.mis_fixed_point_check(cycle(O, 5), [1, 0, 1, 0, 0])
    assert not O.mis_fixed_point_check(complete(O, 3), [1, 1, 0])
    with pytest.raises(OracleError) as e:
        O.mis_fixed_point_check(complete(O, 3), [0.5, 0, 0])
    assert e.value.code == 1


# ------------------------------------------------------ solver pieces
def test_init_state_kats(O):  # test_solver.cpp:55-81
    g = star(O, 3)
    x = O.init_state(g, PROBLEM_MIS, 0.0, O.rng(1))
    assert x[0] == 0.0
    assert np.allclose(x[1:], 1 - 1 / 3)
    x = O.init_state(cycle(O, 4), PROBLEM_MAXCUT, 0.0, O.rng(1))
    assert (x == -1.0).all()
    with pytest.raises(OracleError):
        O.init_state(O.from_edges(4, []), PROBLEM_MIS, 0.1, O.rng(1))


def test_global_reset_kats(O):  # test_solver.cpp:83-118
    x, chosen = O.global_reset(np.ones(10), 0.5, O.rng(5))
    assert len(chosen) == 5 and (x == 0).sum() == 5
    x, chosen = O.global_reset(np.ones(5), 0.1, O.rng(5))
    assert len(chosen) == 0 and (x == 1).all()


# -------------------------------------------------------- local search
def test_local_search_kats(O):  # test_localsearch.cpp:37-105
    c5 = cycle(O, 5)
    ind, s = O.greedy_maximalize(c5, [1, 0, 0, 0, 0])
    assert ind.tolist() == [1, 0, 1, 0, 0]
    with pytest.raises(OracleError):
        O.greedy_maximalize(complete(O, 3), [1, 1, 0])
    ind, s = O.one_two_swap(c5, [1, 0, 1, 0, 0])
    assert ind.tolist() == [1, 0, 1, 0, 0]
    ind, s = O.one_two_swap(star(O, 4), [1, 0, 0, 0, 0])
    assert ind.tolist() == [0, 1, 1, 1, 1]
    ind, s = O.one_two_swap(path(O, 5), [0, 1, 0, 1, 0])
    assert ind.tolist() == [0, 1, 0, 1, 0]
    with pytest.raises(OracleError):
        O.one_two_swap(path(O, 3), [1, 0, 0])
    side, gain = O.one_flip_pass(complete(O, 3), [0, 0, 0])
    assert gain == 2 and O.cut_value(complete(O, 3), side) == 2
    side, gain = O.one_flip_pass(cycle(O, 4), [0, 1, 0, 1])
    assert gain == 0 and side.tolist() == [0, 1, 0, 1]
    side, gain = O.two_flip_pass(path(O, 3), [0, 1, 0])
    assert gain == 0


def test_gain_table_joint(O):  # test_localsearch.cpp:169-184
    rng = np.random.default_rng(131)
    for t in range(10):
        g = O.generate_er(10, 0.45, O.derive_seed(131, t))
        side = rng.integers(0, 2, g.n).astype(np.uint8)
        d = O.build_gain_table(g, side)
        base = O.cut_value(g, side)
        for u, v in g.edges():
            if side[u] == side[v]:
                continue
            f = side.copy()
            f[u] ^= 1
            f[v] ^= 1
            assert O.cut_value(g, f) - base == d[u] + d[v] + 2


# -------------------------------------------------------- engine KATs
def test_engine_small_optima(O):  # test_solver.cpp:120-142
    cfg = orc.Cfg(objective=MIS_QUBO, param=2.0, alpha=0.8, beta=0.3, reset_fraction=0.5,
                  reset_rounds=20, time_budget_secs=1.0, seed=3)
    rep, body = O.solve_pooled(cycle(O, 5), cfg.to_c())
    assert rep["score"] == 2 and rep["found_solution"]
    cfg = orc.Cfg(objective=PERTURBED_BIAS, param=0.001, alpha=0.0025, beta=0.8,
                  reset_fraction=0.8, reset_rounds=20, time_budget_secs=1.0, seed=5)
    rep, body = O.solve_pooled(complete(O, 3), cfg.to_c())
    assert rep["score"] == 2


def test_engine_edgeless(O):  # test_solver.cpp:159-165
    g = O.from_edges(6, [])
    rep, body = O.solve_pooled(g, orc.Cfg(time_budget_secs=0.5).to_c())
    assert rep["score"] == 6 and rep["n_warnings"] == 1
    rep, body = O.solve_pooled(g, orc.Cfg(objective=PERTURBED_BIAS, param=0.001,
                                          time_budget_secs=0.5).to_c())
    assert rep["score"] == 0


def test_engine_guards(O):  # test_solver.cpp:146-157
    with pytest.raises(OracleError) as e:
        O.solve_pooled(cycle(O, 5), orc.Cfg(reset_fraction=1.0).to_c())
    assert e.value.code == 1
    with pytest.raises(OracleError):
        O.solve_pooled(O.from_edges(0, []), orc.Cfg().to_c())


def test_presets(O):  # presets.cpp:17-60 rows used by BASELINE configs
    assert O.preset_for(PROBLEM_MIS, 1000, 9.938) == (0.8, 0.3, 0.7, 60)
    assert O.preset_for(PROBLEM_MIS, 100000, 10.0) == (0.8, 0.3, 0.6, 60)
    assert O.preset_for(PROBLEM_MAXCUT, 1000000, 10.0) == (0.0025, 0.8, 0.8, 90)


def test_strip_and_components_kats(O):  # test_graph.cpp:201-250
    core, rem, c2o, o2c = O.strip_isolated(O.from_edges(3, [(0, 1)]))
    assert core.n == 2 and rem.tolist() == [2] and c2o.tolist() == [0, 1]
    assert o2c.tolist() == [0, 1, -1]
    cyc = O.from_edges(5, [(v, (v + 1) % 5) for v in range(5)])
    core, rem, _, _ = O.strip_isolated(cyc)
    assert len(rem) == 0 and core.edges() == cyc.edges()
    star = O.from_edges(4, [(0, v) for v in range(1, 4)])
    core, rem, _, _ = O.strip_isolated(star)
    assert len(rem) == 0 and core.n == 4
    tri = O.from_edges(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])
    comps = O.connected_components(tri)
    assert [c.tolist() for c in comps] == [[0, 1, 2], [3, 4, 5]]
    assert len(O.connected_components(O.from_edges(5, []))) == 5
    assert len(O.connected_components(O.generate_er(50, 0.2, 1))) == 1


def test_strip_and_components_vs_reference(O, R):
    """The C restatement equals the compiled reference on sparse graphs with
    isolated vertices and many components."""
    for trial in range(12):
        n, p = 300 + 37 * trial, 0.8 / (300 + 37 * trial)
        seed = O.derive_seed(29, trial)
        og, rg = O.generate_er(n, p, seed), R.generate_er(n, p, seed)
        a, b = O.strip_isolated(og), R.strip_isolated(rg)
        assert a[0].edges() == b[0].edges() and a[0].n == b[0].n
        for x, y in zip(a[1:], b[1:]):
            assert (x == y).all()
        ca, cb = O.connected_components(og), R.connected_components(rg)
        assert len(ca) == len(cb) and all((x == y).all() for x, y in zip(ca, cb))
