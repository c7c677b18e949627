"""The independent dense census used by scripts/acceptance.py (criteria 3/4)
agrees with the oracle's gradients (objectives.cpp:101-134) on binary and
+-1 states, and its repairability / maximality predicates with brute force."""
import importlib.util
import os

import numpy as np

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _acceptance():
    spec = importlib.util.spec_from_file_location("acceptance",
                                                  os.path.join(ROOT, "scripts", "acceptance.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_dense_grad_matches_oracle(O):
    A = _acceptance()
    P = A.P
    rng = np.random.default_rng(3)
    for n, p, seed in ((9, 0.4, 1), (12, 0.3, 2)):
        og = O.generate_er(n, p, seed)
        pg = P.generate(P.ErSpec(n, p), seed, device=-1)
        D = A.dense(pg)
        for spec, kind, param in ((P.MisQubo(2.0), oracle.MIS_QUBO, 2.0),
                                  (P.Laplacian(), oracle.LAPLACIAN, 0.0),
                                  (P.PerturbedLaplacian(0.1), oracle.PERTURBED_LAPLACIAN, 0.1),
                                  (P.Adjacency(), oracle.ADJACENCY, 0.0),
                                  (P.PerturbedBias(0.001), oracle.PERTURBED_BIAS, 0.001)):
            for _ in range(5):
                b = rng.integers(0, 2, n).astype(np.float64)
                x = b if kind == oracle.MIS_QUBO else 2.0 * b - 1.0
                want = O.gradient(og, kind, param, x)
                got = A.dense_grad(spec, D, x[None, :])[0]
                assert np.array_equal(got, want), (kind, x)


def test_ttq_stripped_edges_match_strip_isolated(O):
    """scripts/ttq.py hands the reference the GPU side's stripped graph."""
    spec = importlib.util.spec_from_file_location("ttq", os.path.join(ROOT, "scripts", "ttq.py"))
    ttq = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ttq)
    import paper_2605_06921_b200 as P
    hg = P.generate(P.ErFastSpec(3000, 1.5 / 3000), 4, device=-1)
    n_core, edges = ttq.stripped_edges(hg)
    off, nbr = hg.csr()
    og = O.from_edges(hg.n(), np.stack([np.repeat(np.arange(hg.n()), np.diff(off)), nbr], 1))
    ref_core = O.strip_isolated(og)[0]
    mine = O.from_edges(n_core, edges)
    assert mine.n == ref_core.n < hg.n()
    assert all((a == b).all() for a, b in zip(mine.csr(), ref_core.csr()))
