"""The O(m) stochastic block model (MQO_GEN_SBM_FAST, csrc/graph_build.cu):
every pair is an independent Bernoulli(p_in | p_out) draw -- the
distribution of the reference's O(n^2) pair loop (graph.cpp:148-165) -- so
edge counts inside and across blocks match their expectations, as do the
reference generator's own counts; edge cases and error messages follow the
reference.  Host-only graphs (device -1): runs on CPU."""
import math

import numpy as np
import pytest

import paper_2605_06921_b200 as P


def blocks(n, k):
    return (np.arange(n, dtype=np.int64) * k) // n


def split_counts(off, nbr, n, k):
    b = blocks(n, k)
    u = np.repeat(np.arange(n), np.diff(off))
    keep = u < nbr
    u, v = u[keep], nbr[keep]
    same = b[u] == b[v]
    return int(same.sum()), int((~same).sum())


def expected(n, k, p_in, p_out):
    sizes = np.bincount(blocks(n, k), minlength=k).astype(np.float64)
    pin_pairs = float((sizes * (sizes - 1) / 2).sum())
    pout_pairs = n * (n - 1) / 2 - pin_pairs
    return pin_pairs, pout_pairs


@pytest.mark.parametrize("n,k,p_in,p_out,seed", [(4000, 4, 0.05, 0.005, 1), (3001, 7, 0.2, 0.01, 2),
                                                 (2000, 1, 0.03, 0.0, 3), (50000, 10, 0.002, 2e-5, 4)])
def test_sbm_fast_block_counts(O, n, k, p_in, p_out, seed):
    g = P.generate(P.SbmFastSpec(n, k, p_in, p_out), seed, device=-1)
    off, nbr = g.csr()
    ins, outs = split_counts(off, nbr, n, k)
    pin_pairs, pout_pairs = expected(n, k, p_in, p_out)
    for got, pairs, p in ((ins, pin_pairs, p_in), (outs, pout_pairs, p_out)):
        mean, sd = pairs * p, math.sqrt(max(pairs * p * (1 - p), 1e-9))
        assert abs(got - mean) <= 5 * sd + 1e-9, (got, mean, sd)
    if n <= 4000:  # the reference's generator lands in the same window
        og = O.generate_sbm(n, k, p_in, p_out, seed)
        r_in, r_out = split_counts(*og.csr(), n, k)
        mean, sd = pin_pairs * p_in, math.sqrt(pin_pairs * p_in * (1 - p_in))
        assert abs(r_in - mean) <= 5 * sd


def test_sbm_fast_degenerate_probabilities():
    n, k = 200, 3
    g = P.generate(P.SbmFastSpec(n, k, 1.0, 0.0), 5, device=-1)
    off, nbr = g.csr()
    ins, outs = split_counts(off, nbr, n, k)
    assert outs == 0 and ins == int(expected(n, k, 1, 0)[0])  # complete blocks
    g0 = P.generate(P.SbmFastSpec(n, k, 0.5, 0.0), 5, device=-1)
    assert split_counts(*g0.csr(), n, k)[1] == 0


def test_sbm_fast_errors_match_reference():
    for spec, msg in [((10, 0, 0.5, 0.1), "sbm: k must be >= 1"),
                      ((10, 2, 1.5, 0.1), "sbm: probabilities outside"),
                      ((10, 2, 0.1, 0.1), "sbm: requires p_in > p_out")]:
        with pytest.raises(P.InvalidArgument, match=msg):
            P.generate(P.SbmFastSpec(*spec), 1, device=-1)


def test_sbm_fast_is_linear_time():
    import time
    t0 = time.time()
    g = P.generate(P.SbmFastSpec(2_000_000, 20, 1e-4, 1e-6), 9, device=-1)
    assert time.time() - t0 < 30  # the O(n^2) loop would need ~2e12 draws
    assert 0.5 * 2e6 * 1e5 * 1e-4 * 0.8 < g.m() < 0.5 * 2e6 * (1e5 * 1e-4 + 2e6 * 1e-6) * 1.2
