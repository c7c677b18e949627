"""Parity at BASELINE.json's full sizes.

* C4 -- the bench workload, BA(n=1e6, m'=5) x 128 chains, f_B: fused steps
  and the per-pass trajectory path, bit-exact against the oracle on sampled
  chains (the oracle finishes a 1e6-vertex step in tens of ms).
* C4 / C5 -- size-independent property over EVERY chain: with integer-valued
  states every SpMV sum is exact in fp64, so the device gradients must equal
  a scipy CSR product exactly and be linear (grad(X1 + X2) = grad(X1) +
  grad(X2) - grad(0)) bit for bit.  C5 is ER(n=1e7, d=16) (the O(m)
  generator), 16 chains.
"""
import numpy as np
import pytest

from oracle import PERTURBED_BIAS

pytestmark = pytest.mark.gpu


class Spec:
    def __init__(self, kind, param):
        self.kind, self.param = kind, param


def same(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                          np.ascontiguousarray(b).view(np.uint64))


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2605_06921_b200 as P
    return P


@pytest.fixture(scope="module")
def c4(O, P):
    og = O.generate_ba(1_000_000, 5, 1)
    pg = P.generate(P.BaSpec(1_000_000, 5), 1)
    off, nbr = pg.csr()
    assert og.m == pg.m() == 4_999_975
    return og, pg


def test_c4_steps_and_trajectories_bit_exact(O, P, c4):
    og, pg = c4
    B = 128
    rng = np.random.default_rng(44)
    X = rng.uniform(-1, 1, (B, og.n))
    b = P.ChainBatch(pg, B)
    b.set_x(X)
    b.zero_v()
    cfg = P.OptimizerConfig(alpha=0.0025, beta=0.8)
    for _ in range(2):
        b.step(Spec(PERTURBED_BIAS, 0.001), cfg)
    gx, gv = b.get_x(), b.get_v()
    for c in (0, 77, 127):
        x, v = X[c].copy(), np.zeros(og.n)
        for _ in range(2):
            x, v = O.step(og, PERTURBED_BIAS, 0.001, x, v, 0.0025, 0.8)
        assert same(gx[c], x) and same(gv[c], v), c
    # trajectory path (per-pass launches at this size), capped at 6 iterations
    b.set_x(X)
    tcfg = P.OptimizerConfig(alpha=0.0025, beta=0.8, max_iters=6)
    it, rs = b.run_trajectories(P.PerturbedBias(0.001), tcfg)
    gx = b.get_x()
    for c in (3, 100):
        x, i, r = O.run_trajectory(og, PERTURBED_BIAS, 0.001, X[c], 0.0025, 0.8, 6)
        assert (int(it[c]), int(rs[c])) == (i, r) and same(gx[c], x), c


def _csr_matrix(g):
    import scipy.sparse as sp
    off, nbr = g.csr()
    return sp.csr_matrix((np.ones(len(nbr)), nbr, off), shape=(g.n(), g.n()))


def _integer_property(P, g, B, spec, coef, shift, seed):
    """gradient = coef * (A x) + shift elementwise for integer x; exact."""
    A = _csr_matrix(g)
    rng = np.random.default_rng(seed)
    X1 = rng.integers(-3, 4, (B, g.n())).astype(np.float64)
    X2 = rng.integers(-3, 4, (B, g.n())).astype(np.float64)
    b = P.ChainBatch(g, B)
    grads = []
    for X in (X1, X2, X1 + X2, np.zeros_like(X1)):
        b.set_x(X)
        grads.append(b.gradient(spec))
    g1, g2, g12, g0 = grads
    assert same(g12 - g0, (g1 - g0) + (g2 - g0))  # linear part, exact in fp64
    for X, G in ((X1, g1), (X2, g2)):
        want = coef * (A @ X.T).T + shift
        assert same(G, want)


def test_c4_integer_gradients_all_chains(P, c4):
    _, pg = c4
    # f_B gradient = -2 (A x) - lambda (objectives.cpp:131-133); lambda = 0.5 keeps it exact
    _integer_property(P, pg, 128, P.PerturbedBias(0.5), -2.0, -0.5, 1)


@pytest.mark.timeout(900)
def test_c5_integer_gradients_all_chains(P):
    g = P.generate(P.ErFastSpec(10_000_000, 16.0 / 10_000_000), 1)
    assert abs(2 * g.m() / g.n() - 16.0) < 0.05
    # MIS QUBO gradient = 1 - gamma (A x) (objectives.cpp:109-113), gamma = 2
    _integer_property(P, g, 16, P.MisQubo(2.0), -2.0, 1.0, 2)


def _sha(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _xoshiro_next(s):
    m = (1 << 64) - 1
    rotl = lambda x, k: ((x << k) | (x >> (64 - k))) & m  # noqa: E731
    return (rotl((s[1] * 5) & m, 7) * 9) & m


def test_large_goldens_gpu(P):
    """The GPU path against tests/golden/large.npz (the compiled reference):
    1e6-vertex resets, C3 (ER(1e5)) CSR / steps / greedy / (1,2)-swap, and
    one_two_flip on BA(1e5)."""
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "large.npz"))
    g6 = P.Graph.from_edges(1_000_000, [(0, 1)])
    for rho in (0.5, 0.8):
        b = P.ChainBatch(g6, 1)
        b.seed_streams(1_000_000, int(rho * 10))
        b.set_x(np.ones((1, 1_000_000)))
        b.global_reset(rho)
        x = b.get_x()[0]
        assert _sha(np.flatnonzero(x == 0).astype(np.int32)) == str(z[f"reset_1e6_{rho}_sha"])
        s = [int(w) for w in b.get_streams()[0]["s"]]
        assert _xoshiro_next(s) == int(z[f"reset_1e6_{rho}_next"][0])
    g = P.generate(P.ErSpec(100_000, 1e-4), 1)
    assert _sha(*g.csr()) == str(z["c3_csr_sha"])
    b = P.ChainBatch(g, 1)
    b.set_x(np.random.default_rng(33).uniform(0.0, 1.0, (1, g.n())))
    b.zero_v()
    cfg = P.OptimizerConfig(alpha=0.8, beta=0.3)
    for t in range(1, 11):
        b.step(P.MisQubo(2.0), cfg)
        if t in (1, 10):
            assert _sha(b.get_x()[0]) == str(z[f"c3_x{t}_sha"])
            assert _sha(b.get_v()[0]) == str(z[f"c3_v{t}_sha"])
    b.set_x(np.zeros((1, g.n())))  # harvest of the empty set = greedy_maximalize(g, {})
    _, valid, packed = b.harvest(P.PROBLEM_MIS)
    ind = P.unpack_bodies(packed, g.n())[0]
    assert valid[0] and _sha(ind) == str(z["c3_greedy_sha"])
    ind2, size = P.one_two_swap(g, ind)
    assert _sha(np.asarray(ind2, np.uint8)) == str(z["c3_swap_sha"])
    assert size == int(z["c3_swap_size"][0])
    gb = P.generate(P.BaSpec(100_000, 5), 2)
    side = np.random.default_rng(1).integers(0, 2, gb.n()).astype(np.uint8)
    s3, gain = P.one_two_flip(gb, side)
    assert _sha(np.asarray(s3, np.uint8)) == str(z["ba1e5_onetwo_sha"])
    assert gain == int(z["ba1e5_onetwo_gain"][0])
