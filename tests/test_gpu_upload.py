"""Device-side upload of a CSR (graph.cu upload_device): the invariant and
symmetry checks run on the device and must report exactly what the host
path reports (Graph::check_invariants, graph.cpp:44-56: the first violation
in (row, entry) order); the degree-descending row order comes from a device
radix sort and must be the stable host order."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2605_06921_b200 as P
    return P


def _err(P, off, nbr, device):
    try:
        P.Graph.from_csr(off, nbr, device=device)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__, str(e)
    return None


BROKEN = [
    ("not monotone", [0, 2, 1, 2], [1, 2]),
    ("not monotone, later row", [0, 1, 2, 4, 3, 4], [1, 0, 3, 4]),
    ("negative index", [0, 1, 2], [-1, 0]),
    ("index >= n", [0, 1, 2], [5, 0]),
    ("self-loop", [0, 1, 2], [0, 0]),
    ("duplicate entry", [0, 2, 3, 4], [1, 1, 0, 0]),
    ("descending row", [0, 2, 3, 4], [2, 1, 0, 0]),
    ("self-loop before a later range error", [0, 1, 2, 3, 4], [1, 1, 3, 9]),
    ("row order wins over entry order", [0, 2, 4, 5, 6], [1, 3, 0, 9, 0, 0]),
    ("first bad entry inside a row", [0, 4, 5, 6, 7, 8], [1, 3, 3, 9, 0, 0, 0, 0]),
    ("asymmetric", [0, 1, 2, 3, 4], [1, 2, 3, 0]),
    ("one-sided edge among good ones", [0, 2, 3, 3, 4], [1, 2, 0, 0]),
]


@pytest.mark.parametrize("name,off,nbr", BROKEN, ids=[b[0] for b in BROKEN])
def test_device_checks_match_host(P, name, off, nbr):
    host = _err(P, off, nbr, -1)
    dev = _err(P, off, nbr, 0)
    assert host is not None, name
    assert dev == host, (name, dev, host)


def _stable_order(off):
    deg = np.diff(off)
    return np.lexsort((np.arange(len(deg)), -deg)).astype(np.int32)


@pytest.mark.parametrize("spec", ["er", "ba_small", "ba_large", "edgeless", "single"])
def test_device_row_order_and_csr(P, spec):
    if spec == "er":
        g0 = P.generate(P.ErSpec(3000, 0.004), 3)
    elif spec == "ba_small":
        g0 = P.generate(P.BaSpec(2000, 3), 3)
    elif spec == "ba_large":
        g0 = P.generate(P.BaSpec(200_000, 5), 1)
    elif spec == "edgeless":
        g0 = P.Graph.from_csr(np.zeros(6, np.int64), np.zeros(0, np.int32), device=-1)
    else:
        g0 = P.Graph.from_edges(2, [(0, 1)], device=-1)
    off, nbr = g0.csr()
    g = P.Graph.from_csr(off, nbr, device=0)
    assert (g.n(), g.m(), g.max_degree()) == (g0.n(), g0.m(), g0.max_degree())
    o2, n2 = g.csr()
    assert np.array_equal(o2, off) and np.array_equal(n2, nbr)
    assert np.array_equal(g.row_order(), _stable_order(off))
