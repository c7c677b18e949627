"""GPU device pre-processing against the oracle:
strip_isolated and connected_components (graph.cpp:180-224) -- identical
maps, core CSR and component lists.  KATs re-hosted from
/root/reference/proj/tests/test_graph.cpp:201-250."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2605_06921_b200 as P
    return P


def test_kats(P):  # test_graph.cpp:201-250
    r = P.strip_isolated(P.Graph.from_edges(3, [(0, 1)]))
    assert r.core.n() == 2 and r.removed.tolist() == [2]
    assert r.core_to_orig.tolist() == [0, 1] and r.orig_to_core.tolist() == [0, 1, -1]
    cyc = P.Graph.from_edges(5, [(v, (v + 1) % 5) for v in range(5)])
    r = P.strip_isolated(cyc)
    assert len(r.removed) == 0
    assert all((x == y).all() for x, y in zip(r.core.csr(), cyc.csr()))
    r = P.strip_isolated(P.Graph.from_edges(4, [(0, v) for v in range(1, 4)]))
    assert len(r.removed) == 0 and r.core.n() == 4
    tri = P.Graph.from_edges(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])
    assert [c.tolist() for c in P.connected_components(tri)] == [[0, 1, 2], [3, 4, 5]]
    assert len(P.connected_components(P.Graph.from_edges(5, []))) == 5
    assert len(P.connected_components(P.generate(P.ErSpec(50, 0.2), 1))) == 1
    empty = P.strip_isolated(P.Graph.from_edges(4, []))
    assert empty.core.n() == 0 and empty.removed.tolist() == [0, 1, 2, 3]
    assert P.connected_components(P.Graph.from_edges(0, [])) == []


def test_host_only_graph_rejected(P):
    g = P.Graph.from_edges(3, [(0, 1)], device=-1)
    with pytest.raises(P.InvalidArgument, match="host-only"):
        P.strip_isolated(g)


@pytest.mark.parametrize("n,deg", [(500, 0.5), (2000, 1.0), (20000, 1.5), (100000, 3.0)])
def test_random_vs_oracle(O, P, n, deg):
    """Sparse ER graphs (many isolated vertices and components, giant
    component at deg > 1) plus an SBM."""
    seed = O.derive_seed(31, n)
    og = O.generate_er(n, deg / n, seed)
    pg = P.generate(P.ErSpec(n, deg / n), seed)
    core, rem, c2o, o2c = O.strip_isolated(og)
    r = P.strip_isolated(pg)
    assert (r.removed == rem).all() and (r.core_to_orig == c2o).all()
    assert (r.orig_to_core == o2c).all()
    off, nbr = r.core.csr()
    ooff, onbr = core.csr()
    assert (off == ooff).all() and (nbr == onbr).all()
    ca, cb = P.connected_components(pg), O.connected_components(og)
    assert len(ca) == len(cb) and all((x == y).all() for x, y in zip(ca, cb))


def test_sbm_components(O, P):
    og = O.generate_sbm(3000, 6, 0.004, 0.0, 5)
    pg = P.generate(P.SbmSpec(3000, 6, 0.004, 0.0), 5)
    ca, cb = P.connected_components(pg), O.connected_components(og)
    assert len(ca) == len(cb) and all((x == y).all() for x, y in zip(ca, cb))
