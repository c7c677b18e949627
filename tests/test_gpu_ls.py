"""GPU parity of the local-search kernels (K7/K8) against the oracle:
identical final bodies and gains / sizes (bit-exact integer paths).  KATs
re-hosted from /root/reference/proj/tests/test_localsearch.cpp."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2605_06921_b200 as P
    return P


def G(P, n, edges):
    return P.Graph.from_edges(n, edges)


def test_kats(P):  # test_localsearch.cpp:43-105, 138-160
    c5 = G(P, 5, [(v, (v + 1) % 5) for v in range(5)])
    assert P.one_two_swap(c5, [1, 0, 1, 0, 0])[0].tolist() == [1, 0, 1, 0, 0]
    star = G(P, 5, [(0, v) for v in range(1, 5)])
    body, size = P.one_two_swap(star, [1, 0, 0, 0, 0])
    assert body.tolist() == [0, 1, 1, 1, 1] and size == 4
    p5 = G(P, 5, [(v, v + 1) for v in range(4)])
    assert P.one_two_swap(p5, [0, 1, 0, 1, 0])[0].tolist() == [0, 1, 0, 1, 0]
    k3 = G(P, 3, [(0, 1), (1, 2), (0, 2)])
    with pytest.raises(P.InvalidArgument, match="not an independent set"):
        P.one_two_swap(k3, [1, 1, 0])
    p3 = G(P, 3, [(0, 1), (1, 2)])
    with pytest.raises(P.InvalidArgument, match="not maximal"):
        P.one_two_swap(p3, [1, 0, 0])
    side, gain = P.one_flip_pass(k3, [0, 0, 0])
    assert gain == 2
    c4 = G(P, 4, [(v, (v + 1) % 4) for v in range(4)])
    side, gain = P.one_flip_pass(c4, [0, 1, 0, 1])
    assert gain == 0 and side.tolist() == [0, 1, 0, 1]
    side, gain = P.two_flip_pass(p3, [0, 1, 0])
    assert gain == 0 and side.tolist() == [0, 1, 0]
    c6 = G(P, 6, [(v, (v + 1) % 6) for v in range(6)])
    assert P.two_flip_pass(c6, [0, 1, 0, 1, 0, 1])[1] == 0
    assert P.one_two_flip(c6, [0, 1, 0, 1, 0, 1])[1] == 0
    e4 = G(P, 4, [(0, 1)])
    e4 = P.Graph.from_edges(4, [])
    assert P.one_two_flip(e4, [0, 1, 0, 1])[1] == 0


@pytest.mark.parametrize("op", ["one_flip_pass", "two_flip_pass", "one_two_flip"])
def test_flips_random_vs_oracle(O, P, op):
    rng = np.random.default_rng(107)
    for trial in range(20):
        n = int(rng.integers(6, 60))
        seed = O.derive_seed(107, trial)
        og = O.generate_er(n, 0.4 if n < 20 else 0.15, seed)
        pg = P.generate(P.ErSpec(n, 0.4 if n < 20 else 0.15), seed)
        # several random sides at once through one batched call
        sides = rng.integers(0, 2, (7, n)).astype(np.uint8)
        b = P.ChainBatch(pg, 1)
        opcode = {"one_flip_pass": 0, "two_flip_pass": 1, "one_two_flip": 2}[op]
        packed, gains = P.local_search(b, opcode, P.pack_bodies(sides))
        got = P.unpack_bodies(packed, n)
        for k in range(7):
            ref_side, ref_gain = getattr(O, op)(og, sides[k])
            assert gains[k] == ref_gain and (got[k] == ref_side).all(), (trial, k)


def test_swap_random_vs_oracle(O, P):
    rng = np.random.default_rng(103)
    for trial in range(30):
        n = 24 if trial < 20 else 200
        p = float(rng.uniform(0.08, 0.35)) if n == 24 else 0.03
        seed = O.derive_seed(103, trial)
        og = O.generate_er(n, p, seed)
        pg = P.generate(P.ErSpec(n, p), seed)
        starts = []
        for k in range(5):  # greedy completions of random independent seeds
            ind = np.zeros(n, np.uint8)
            for v in rng.permutation(n)[: n // 6]:
                ind[v] = 1
                if not O.is_independent(og, ind):
                    ind[v] = 0
            starts.append(O.greedy_maximalize(og, ind)[0])
        starts = np.array(starts)
        b = P.ChainBatch(pg, 1)
        packed, sizes = P.local_search(b, 3, P.pack_bodies(starts))
        got = P.unpack_bodies(packed, n)
        for k in range(5):
            ref, size = O.one_two_swap(og, starts[k])
            assert sizes[k] == size and (got[k] == ref).all(), (trial, k)


def test_goldens(P):
    z = np.load(os.path.join(GOLD, "pieces.npz"))
    g1 = P.generate(P.ErSpec(1000, 0.01), 1)
    g2 = P.generate(P.ErSpec(2000, 6 / 2000), 1)
    assert (P.one_two_swap(g1, z["c1_greedy"])[0] == z["c1_swap"]).all()
    assert (P.one_two_swap(g1, z["c1_greedy_empty"])[0] == z["c1_swap_empty"]).all()
    s1, a = P.one_flip_pass(g2, z["c2_harvest"])
    s2, b = P.two_flip_pass(g2, z["c2_harvest"])
    s3, c = P.one_two_flip(g2, z["c2_harvest"])
    assert (s1 == z["c2_oneflip"]).all() and (s2 == z["c2_twoflip"]).all()
    assert (s3 == z["c2_onetwo"]).all() and [a, b, c] == z["c2_gains"].tolist()


def test_large_vs_oracle(O, P):
    """BA(1e5,5) one_two_flip from random sides; ER(2e4, d=10) one_two_swap
    from the greedy completion of the empty set."""
    og = O.generate_ba(100000, 5, 2)
    pg = P.generate(P.BaSpec(100000, 5), 2)
    side = np.random.default_rng(1).integers(0, 2, 100000).astype(np.uint8)
    got, gain = P.one_two_flip(pg, side)
    ref, rgain = O.one_two_flip(og, side)
    assert gain == rgain and (got == ref).all()
    got, gain = P.one_flip_pass(pg, side)  # round-parallel passes alone
    ref, rgain = O.one_flip_pass(og, side)
    assert gain == rgain and (got == ref).all()
    og = O.generate_er(20000, 10 / 20000, 3)
    pg = P.generate(P.ErSpec(20000, 10 / 20000), 3)
    start, _ = O.greedy_maximalize(og, np.zeros(20000, np.uint8))
    got, size = P.one_two_swap(pg, start)
    ref, rsize = O.one_two_swap(og, start)
    assert size == rsize and (got == ref).all()


def test_swap_batch_input_check_leaves_caller_buffer(P):
    # one_two_swap on several bodies with one invalid: the call raises the
    # reference's message and the caller's packed bodies are not modified
    # (the input check is read back with the results, after the kernels)
    import ctypes as C
    from paper_2605_06921_b200 import _lib
    star = G(P, 5, [(0, v) for v in range(1, 5)])
    b = P.ChainBatch(star, 1)
    good = [1, 0, 0, 0, 0]
    for bad, msg in (([1, 1, 0, 0, 0], "not an independent set"), ([0, 1, 1, 0, 0], "not maximal")):
        pk = P.pack_bodies(np.array([good, bad, good], np.uint8))
        before = pk.copy()
        out = np.zeros(3, np.int64)
        rc = _lib.lib.mqo_local_search(b._h, _lib.LS_ONE_TWO_SWAP, 3,
                                       pk.ctypes.data_as(C.POINTER(C.c_uint64)),
                                       out.ctypes.data_as(C.POINTER(C.c_int64)))
        assert rc != 0 and msg in _lib.lib.mqo_last_error().decode()
        assert np.array_equal(pk, before)
    pk, out = P.local_search(b, _lib.LS_ONE_TWO_SWAP, P.pack_bodies(np.array([good, good], np.uint8)))
    assert out.tolist() == [4, 4]


@pytest.mark.parametrize("n,d,bodies", [(1024, 16, 1), (8000, 16, 1), (16384, 16, 16), (4096, 8, 20),
                                         (20000, 8, 16)])
def test_one_flip_cta_variants_vs_oracle(O, P, n, d, bodies):
    # k_one_flip_cta with the CSR in shared memory (n = 1024, 4096) and read
    # from global memory (ER(8000, d=16): 512 KB of rows; 16 bodies at 16384),
    # one body per call and batched, against the oracle's one_flip_pass
    from paper_2605_06921_b200 import _lib
    og = O.generate_er(n, d / n, 3)
    pg = P.generate(P.ErSpec(n, d / n), 3)
    sides = np.random.default_rng(n + bodies).integers(0, 2, (bodies, n)).astype(np.uint8)
    b = P.ChainBatch(pg, 1)
    packed, gains = P.local_search(b, _lib.LS_ONE_FLIP, P.pack_bodies(sides))
    got = P.unpack_bodies(packed, n)
    for k in range(bodies):
        ref_side, ref_gain = O.one_flip_pass(og, sides[k])
        assert gains[k] == ref_gain and (got[k] == ref_side).all(), k


@pytest.mark.parametrize("n,d", [(1024, 16), (4096, 8), (16384, 8)])
@pytest.mark.parametrize("op", ["one_flip", "two_flip", "one_two_flip", "swap"])
@pytest.mark.parametrize("bodies", [1, 5])
def test_single_launch_small_bodies_vs_oracle(O, P, n, d, op, bodies):
    """The single-launch kernels (k_flip_small / k_swap_small, n <= 16384;
    CSR staged in SMEM or read from global memory) against the oracle."""
    from paper_2605_06921_b200 import _lib
    og = O.generate_er(n, d / n, 5)
    pg = P.generate(P.ErSpec(n, d / n), 5)
    b = P.ChainBatch(pg, 1)
    rng = np.random.default_rng(n * 7 + bodies)
    if op == "swap":
        starts = []
        for k in range(bodies):  # greedy completions of random independent seeds
            ind = np.zeros(n, np.uint8)
            ind[rng.choice(n, 3, replace=False)] = 1
            off, nbr = pg.csr()
            for v in np.flatnonzero(ind):
                if ind[nbr[off[v]:off[v + 1]]].any():
                    ind[v] = 0
            starts.append(O.greedy_maximalize(og, ind)[0])
        start = np.array(starts, np.uint8)
        packed, out = P.local_search(b, _lib.LS_ONE_TWO_SWAP, P.pack_bodies(start))
        got = P.unpack_bodies(packed, n)
        for k in range(bodies):
            ref, size = O.one_two_swap(og, start[k])
            assert out[k] == size and (got[k] == ref).all(), k
        return
    opc = {"one_flip": _lib.LS_ONE_FLIP, "two_flip": _lib.LS_TWO_FLIP,
           "one_two_flip": _lib.LS_ONE_TWO_FLIP}[op]
    sides = rng.integers(0, 2, (bodies, n)).astype(np.uint8)
    packed, gains = P.local_search(b, opc, P.pack_bodies(sides))
    got = P.unpack_bodies(packed, n)
    for k in range(bodies):
        fn = {"one_flip": O.one_flip_pass, "two_flip": O.two_flip_pass,
              "one_two_flip": O.one_two_flip}[op]
        ref, gain = fn(og, sides[k])
        assert gains[k] == gain and (got[k] == ref).all(), k


@pytest.mark.parametrize("graph", ["ba", "er_dense"])
def test_small_bodies_hubs_and_dense_vs_oracle(O, P, graph):
    """Single-launch 1-flip (closure + grouped rounds) and the swap kernel's
    batched pair search where rows are long and candidate pairs are often
    adjacent: BA(3000, 6) hubs, ER(400, 0.15)."""
    from paper_2605_06921_b200 import _lib
    if graph == "ba":
        og, pg, n = O.generate_ba(3000, 6, 9), P.generate(P.BaSpec(3000, 6), 9), 3000
    else:
        og, pg, n = O.generate_er(400, 0.15, 9), P.generate(P.ErSpec(400, 0.15), 9), 400
    b = P.ChainBatch(pg, 1)
    rng = np.random.default_rng(5)
    sides = rng.integers(0, 2, (4, n)).astype(np.uint8)
    for opc, fn in ((_lib.LS_ONE_FLIP, O.one_flip_pass), (_lib.LS_ONE_TWO_FLIP, O.one_two_flip)):
        packed, gains = P.local_search(b, opc, P.pack_bodies(sides))
        got = P.unpack_bodies(packed, n)
        for k in range(4):
            ref, gain = fn(og, sides[k])
            assert gains[k] == gain and (got[k] == ref).all(), (opc, k)
    starts = []
    for k in range(4):
        ind = np.zeros(n, np.uint8)
        for v in rng.permutation(n)[: n // 10]:
            ind[v] = 1
            if not O.is_independent(og, ind):
                ind[v] = 0
        starts.append(O.greedy_maximalize(og, ind)[0])
    starts = np.array(starts, np.uint8)
    packed, sizes = P.local_search(b, _lib.LS_ONE_TWO_SWAP, P.pack_bodies(starts))
    got = P.unpack_bodies(packed, n)
    for k in range(4):
        ref, size = O.one_two_swap(og, starts[k])
        assert sizes[k] == size and (got[k] == ref).all(), k
