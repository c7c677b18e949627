"""GPU parity of the fused PGA kernels (K1/K2) against the oracle, through the
C ABI.  Bit-exact: every fp64 iterate, gradient and velocity must equal the
reference's, chain by chain (the north star allows 1e-5 relative per step;
the design achieves 0 ulp, which is what these tests assert)."""
import os

import numpy as np
import pytest

from oracle import (ADJACENCY, LAPLACIAN, MIS_QUBO, PERTURBED_BIAS, PERTURBED_LAPLACIAN,
                    problem_of)

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KINDS = [(MIS_QUBO, 2.0), (LAPLACIAN, 0.0), (PERTURBED_LAPLACIAN, 0.001), (ADJACENCY, 0.0),
         (PERTURBED_BIAS, 0.001)]


class Spec:
    def __init__(self, kind, param):
        self.kind, self.param = kind, param


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2605_06921_b200 as P
    return P


def graphs(O, P):
    out = {}
    for name, (n, p, s) in {"c1": (1000, 0.01, 1), "c2": (2000, 6 / 2000, 1)}.items():
        og = O.generate_er(n, p, s)
        pg = P.generate(P.ErSpec(n, p), s)
        assert (og.csr()[0] == pg.csr()[0]).all() and (og.csr()[1] == pg.csr()[1]).all()
        out[name] = (og, pg)
    return out


def test_gradient_golden(O, P):
    z = np.load(os.path.join(GOLD, "steps.npz"))
    g = graphs(O, P)
    for gname, kinds in (("c1", [MIS_QUBO]), ("c2", [PERTURBED_BIAS, LAPLACIAN,
                                                      PERTURBED_LAPLACIAN, ADJACENCY])):
        for kind in kinds:
            param = dict(KINDS)[kind]
            b = P.ChainBatch(g[gname][1], 1)
            b.set_x(z[f"{gname}_k{kind}_x0"][None])
            assert same(b.gradient(Spec(kind, param))[0], z[f"{gname}_k{kind}_grad"])


def test_steps_golden(O, P):
    """100 fused steps from the golden x0 equal the reference's step()."""
    z = np.load(os.path.join(GOLD, "steps.npz"))
    g = graphs(O, P)
    for gname, kinds in (("c1", [MIS_QUBO]), ("c2", [PERTURBED_BIAS, LAPLACIAN,
                                                      PERTURBED_LAPLACIAN, ADJACENCY])):
        for kind in kinds:
            param = dict(KINDS)[kind]
            alpha, beta = (0.8, 0.3) if kind == MIS_QUBO else (0.0025, 0.8)
            b = P.ChainBatch(g[gname][1], 1)
            b.set_x(z[f"{gname}_k{kind}_x0"][None])
            b.zero_v()
            cfg = P.OptimizerConfig(alpha=alpha, beta=beta)
            for t in range(1, 101):
                b.step(Spec(kind, param), cfg)
                if t in (1, 10, 100):
                    assert same(b.get_x()[0], z[f"{gname}_k{kind}_x{t}"]), (kind, t)
                    assert same(b.get_v()[0], z[f"{gname}_k{kind}_v{t}"]), (kind, t)


@pytest.mark.parametrize("B", [1, 2, 3, 4, 7, 33, 128, 256])
@pytest.mark.parametrize("kind,param", KINDS)
def test_batched_steps_vs_oracle(O, P, B, kind, param):
    og = O.generate_er(300, 0.03, 5)
    pg = P.generate(P.ErSpec(300, 0.03), 5)
    rng = np.random.default_rng(B * 10 + kind)
    lo = 0.0 if kind == MIS_QUBO else -1.0
    X = rng.uniform(lo, 1.0, (B, og.n))
    V = rng.uniform(-0.5, 0.5, (B, og.n))
    b = P.ChainBatch(pg, B)
    b.set_x(X)
    b.set_v(V)
    cfg = P.OptimizerConfig(alpha=0.05, beta=0.7)
    for _ in range(5):
        b.step(Spec(kind, param), cfg)
    gx, gv = b.get_x(), b.get_v()
    for c in range(B):
        x, v = X[c].copy(), V[c].copy()
        for _ in range(5):
            x, v = O.step(og, kind, param, x, v, 0.05, 0.7)
        assert same(gx[c], x) and same(gv[c], v), c


@pytest.mark.parametrize("fuse", [1, 0])
@pytest.mark.parametrize("gq", [1, 2, 8])
@pytest.mark.parametrize("B", [33, 256])
def test_chain_tiled_steps_vs_oracle(O, P, B, gq, fuse):
    """Chain tiling (one graph sweep per group of gq quads; all groups in one
    launch or one launch per group) keeps every iterate bit-identical."""
    from paper_2605_06921_b200 import _lib
    og = O.generate_er(300, 0.03, 6)
    pg = P.generate(P.ErSpec(300, 0.03), 6)
    rng = np.random.default_rng(B + gq)
    for kind, param in ((MIS_QUBO, 2.0), (PERTURBED_BIAS, 0.001)):
        lo = 0.0 if kind == MIS_QUBO else -1.0
        X = rng.uniform(lo, 1.0, (B, og.n))
        b = P.ChainBatch(pg, B)
        b.set_x(X)
        cfg = P.OptimizerConfig(alpha=0.05, beta=0.7)
        _lib.check(_lib.lib.mqo_tune(b"group_quads", gq))
        _lib.check(_lib.lib.mqo_tune(b"fuse_groups", fuse))
        try:
            for _ in range(4):
                b.step(Spec(kind, param), cfg)
        finally:
            _lib.check(_lib.lib.mqo_tune(b"group_quads", 0))
            _lib.check(_lib.lib.mqo_tune(b"fuse_groups", 1))
        gx = b.get_x()
        for c in range(0, B, 7):
            x, v = X[c].copy(), np.zeros(og.n)
            for _ in range(4):
                x, v = O.step(og, kind, param, x, v, 0.05, 0.7)
            assert same(gx[c], x), (kind, c)


def test_hub_rows_ba(O, P):
    """BA(1e5, 5): power-law hub rows (deg in the hundreds), B=128 chains."""
    og = O.generate_ba(100000, 5, 3)
    pg = P.generate(P.BaSpec(100000, 5), 3)
    B = 128
    rng = np.random.default_rng(9)
    X = rng.uniform(-1, 1, (B, og.n))
    b = P.ChainBatch(pg, B)
    b.set_x(X)
    b.zero_v()
    cfg = P.OptimizerConfig(alpha=0.0025, beta=0.8)
    for _ in range(3):
        b.step(Spec(PERTURBED_BIAS, 0.001), cfg)
    gx = b.get_x()
    for c in (0, 1, 63, 127):
        x, v = X[c].copy(), np.zeros(og.n)
        for _ in range(3):
            x, v = O.step(og, PERTURBED_BIAS, 0.001, x, v, 0.0025, 0.8)
        assert same(gx[c], x), c


def test_checker_kats(P):  # test_pga.cpp:138-148
    def g(n, edges):
        return P.Graph.from_edges(n, edges)
    k3 = g(3, [(0, 1), (1, 2), (0, 2)])
    p3 = g(3, [(0, 1), (1, 2)])
    c5 = g(5, [(v, (v + 1) % 5) for v in range(5)])
    assert P.mis_fixed_point_check(k3, [1, 0, 0], 2.0, 0.8)
    assert not P.mis_fixed_point_check(p3, [1, 0, 0], 2.0, 0.8)
    assert P.mis_fixed_point_check(c5, [1, 0, 1, 0, 0], 2.0, 0.8)
    assert not P.mis_fixed_point_check(k3, [1, 1, 0], 2.0, 0.8)
    with pytest.raises(P.InvalidArgument, match="not binary"):
        P.mis_fixed_point_check(k3, [0.5, 0, 0], 2.0, 0.8)


def test_trajectory_kats(P):  # test_pga.cpp:77-119
    k3 = P.Graph.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    out = P.run_trajectory(P.MisQubo(2.0), k3, [0.9, 0.1, 0.1], P.OptimizerConfig(alpha=0.8))
    assert out.reason == P.StopReason.CheckerAccepted and out.state.tolist() == [1, 0, 0]
    out = P.run_trajectory(P.PerturbedBias(0.001), k3, [0.6, -0.5, -0.4],
                           P.OptimizerConfig(alpha=0.1))
    assert out.reason == P.StopReason.Converged and out.state.tolist() == [1, -1, -1]
    out = P.run_trajectory(P.MisQubo(2.0), k3, [0.4, 0.4, 0.4],
                           P.OptimizerConfig(alpha=1e-9, max_iters=12))
    assert out.reason == P.StopReason.IterCap and out.iterations == 12
    with pytest.raises(P.InvalidArgument, match="alpha"):
        P.run_trajectory(P.MisQubo(2.0), k3, [0.4, 0.4, 0.4], P.OptimizerConfig(alpha=0.0))


# (cta_traj, persistent_cells, cta_cluster, group_quads)
PATHS = {"cta": (1, 1 << 22, 0, 0), "cta_c1": (1, 1 << 22, 1, 0), "cta_c3": (1, 1 << 22, 3, 0),
         "cta_c16": (1, 1 << 22, 16, 0), "persistent": (0, 1 << 22, 0, 0),
         "perpass": (0, 0, 0, 0), "perpass_tiled": (0, 0, 0, 1)}


@pytest.fixture(params=list(PATHS))
def traj_path(request, P):
    """Run the trajectory parity tests through each device path: SMEM
    cluster-per-chain (automatic cluster size, and forced 1 / 3 / 16 CTAs
    per chain -- 16 is clamped to the slice count), cooperative persistent,
    launch-per-pass (untiled and one sweep per 4-chain group)."""
    from paper_2605_06921_b200 import _lib
    cta, cells, clu, gq = PATHS[request.param]
    _lib.check(_lib.lib.mqo_tune(b"cta_traj", cta))
    _lib.check(_lib.lib.mqo_tune(b"persistent_cells", cells))
    _lib.check(_lib.lib.mqo_tune(b"cta_cluster", clu))
    _lib.check(_lib.lib.mqo_tune(b"group_quads", gq))
    yield request.param
    _lib.check(_lib.lib.mqo_tune(b"cta_traj", 1))
    _lib.check(_lib.lib.mqo_tune(b"persistent_cells", 1 << 22))
    _lib.check(_lib.lib.mqo_tune(b"cta_cluster", 0))
    _lib.check(_lib.lib.mqo_tune(b"group_quads", 0))


@pytest.mark.parametrize("kind,param,alpha,beta,ce", [
    (MIS_QUBO, 2.0, 0.8, 0.3, 1), (MIS_QUBO, 2.0, 0.8, 0.3, 3), (MIS_QUBO, 2.0, 0.3, 0.0, 1),
    (PERTURBED_BIAS, 0.001, 0.0025, 0.8, 1), (PERTURBED_BIAS, 0.001, 0.1, 0.0, 1),
    (PERTURBED_BIAS, 0.001, 0.02, 0.5, 1),
    (LAPLACIAN, 0.0, 0.1, 0.0, 1), (PERTURBED_LAPLACIAN, 0.001, 0.1, 0.0, 1),
    (ADJACENCY, 0.0, 0.05, 0.5, 1)])
def test_batched_trajectories_vs_oracle(O, P, traj_path, kind, param, alpha, beta, ce):
    """Per-chain TrajectoryOutcome (state bits, iterations, reason) equal
    run_trajectory's for chains that stop at different iterations."""
    og = O.generate_er(400, 0.02, 11)
    pg = P.generate(P.ErSpec(400, 0.02), 11)
    B = 24
    rng = np.random.default_rng(kind * 7 + ce)
    lo = 0.0 if kind == MIS_QUBO else -1.0
    X = rng.uniform(lo, 1.0, (B, og.n))
    X[0] = 0.5  # edge cases: a constant start
    X[1] = np.where(rng.random(og.n) < 0.5, 1.0, lo)
    b = P.ChainBatch(pg, B)
    b.set_x(X)
    cfg = P.OptimizerConfig(alpha=alpha, beta=beta, max_iters=700, check_every=ce)
    it, rs = b.run_trajectories(Spec(kind, param), cfg)
    gx = b.get_x()
    for c in range(B):
        x, i, r = O.run_trajectory(og, kind, param, X[c], alpha, beta, 700, 1e-6, ce)
        assert (it[c], rs[c]) == (i, r), c
        assert same(gx[c], x), c


def test_trajectory_golden(O, P, traj_path):
    z = np.load(os.path.join(GOLD, "steps.npz"))
    g = graphs(O, P)
    for gname, kind in (("c1", MIS_QUBO), ("c2", PERTURBED_BIAS), ("c2", LAPLACIAN),
                        ("c2", PERTURBED_LAPLACIAN), ("c2", ADJACENCY)):
        param = dict(KINDS)[kind]
        alpha, beta = (0.8, 0.3) if kind == MIS_QUBO else (0.0025, 0.8)
        out = P.run_trajectory(Spec(kind, param), g[gname][1], z[f"{gname}_k{kind}_x0"],
                               P.OptimizerConfig(alpha=alpha, beta=beta))
        assert [out.iterations, out.reason] == z[f"{gname}_k{kind}_traj_ir"].tolist()
        assert same(out.state, z[f"{gname}_k{kind}_traj"])


def test_edgeless_vs_oracle(O, P):
    og, pg = O.from_edges(5, []), P.Graph.from_edges(5, [])
    b = P.ChainBatch(pg, 4)
    X = np.linspace(-0.9, 0.9, 20).reshape(4, 5)
    b.set_x(X)
    it, rs = b.run_trajectories(P.PerturbedBias(0.001), P.OptimizerConfig(alpha=0.1))
    gx = b.get_x()
    for c in range(4):
        x, i, r = O.run_trajectory(og, PERTURBED_BIAS, 0.001, X[c], 0.1, 0.0)
        assert (it[c], rs[c]) == (i, r) and same(gx[c], x)
