"""Heavy rows (csrc/pga.cu heavy_row): rows of high degree are staged
through SMEM by a whole CTA and summed in CSR order by one thread per chain.
Bit-exact against the oracle for every objective (incl. the Laplacian's
(x_v - x_u) terms and the fused MIS checker), few and odd chain counts (the
CPL = 1 kernels, ragged quads), steps and per-pass trajectories, with the
threshold forced low so most of the graph is staged."""
import numpy as np
import pytest

import oracle
from oracle import ADJACENCY, LAPLACIAN, MIS_QUBO, PERTURBED_BIAS, PERTURBED_LAPLACIAN

pytestmark = pytest.mark.gpu

PARAM = {MIS_QUBO: 2.0, LAPLACIAN: 0.0, PERTURBED_LAPLACIAN: 0.3, ADJACENCY: 0.0,
         PERTURBED_BIAS: 0.001}


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2605_06921_b200 as P
    return P


@pytest.fixture(scope="module")
def graphs(O, P):
    og = O.generate_ba(20_000, 5, 3)
    pg = P.generate(P.BaSpec(20_000, 5), 3)
    return og, pg


class Spec:
    def __init__(self, kind, param):
        self.kind, self.param = kind, param


def same(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                          np.ascontiguousarray(b).view(np.uint64))


@pytest.mark.parametrize("heavy_deg", [0, 24])
@pytest.mark.parametrize("B", [1, 3, 4, 9, 16, 40])
@pytest.mark.parametrize("kind", [MIS_QUBO, LAPLACIAN, PERTURBED_LAPLACIAN, PERTURBED_BIAS])
def test_heavy_rows_steps_and_trajectories(O, P, graphs, heavy_deg, B, kind):
    og, pg = graphs
    P.tune("heavy_deg", heavy_deg)
    P.tune("persistent_cells", 0)  # the per-pass kernels (the heavy-row launches)
    P.tune("cta_traj", 0)
    try:
        lo = 0.0 if kind == MIS_QUBO else -1.0
        rng = np.random.default_rng(B * 7 + kind)
        X = rng.uniform(lo, 1.0, (B, og.n))
        b = P.ChainBatch(pg, B)
        b.set_x(X)
        b.zero_v()
        alpha, beta = (0.8, 0.3) if kind == MIS_QUBO else (0.05, 0.5)
        cfg = P.OptimizerConfig(alpha=alpha, beta=beta)
        for _ in range(2):
            b.step(Spec(kind, PARAM[kind]), cfg)
        gx, gv = b.get_x(), b.get_v()
        for c in sorted({0, B // 2, B - 1}):
            x, v = X[c].copy(), np.zeros(og.n)
            for _ in range(2):
                x, v = O.step(og, kind, PARAM[kind], x, v, alpha, beta)
            assert same(gx[c], x) and same(gv[c], v), (c, heavy_deg)
        b.set_x(X)
        tcfg = P.OptimizerConfig(alpha=alpha, beta=beta, max_iters=7)
        it, rs = b.run_trajectories(Spec(kind, PARAM[kind]), tcfg)
        gx = b.get_x()
        for c in sorted({0, B - 1}):
            x, i, r = O.run_trajectory(og, kind, PARAM[kind], X[c], alpha, beta, 7)
            assert (int(it[c]), int(rs[c])) == (i, r) and same(gx[c], x), (c, heavy_deg)
    finally:
        P.tune("heavy_deg", 0)
        P.tune("persistent_cells", 1 << 22)
        P.tune("cta_traj", 1)
