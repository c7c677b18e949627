"""`mqo verify` on the B200 backend.

The reference's verification suites (tools/src/cmd_verify.cpp:27-176) rerun
with every solver-path quantity computed on the GPU: gradients of all 2^n
binary states as one chain batch (fixed-points), trajectories (escapability)
and the pooled engine (exact).  The brute-force optima and the census
predicates are small host computations over bitmasks, as in the
reference's oracle module (oracle.cpp:140-193), which shares no code with
the solver path.  Output lines, check names and exit codes (0 all passed,
1 a check failed, 2 usage) follow cmd_verify.cpp; the toy-reset study
(experiments outside the hot path) is reported as skipped.
"""
from __future__ import annotations

import argparse

import numpy as np

from . import api as P

EXIT_OK, EXIT_FAIL, EXIT_USAGE = 0, 1, 2
_M64 = (1 << 64) - 1


def derive_seed(master: int, stream: int) -> int:  # rng.hpp:77-84
    s = (master ^ ((0x9E3779B97F4A7C15 + stream * 0xD1342543DE82EF95) & _M64)) & _M64
    z = (s + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class Rng:
    """xoshiro256** with splitmix64 seeding (rng.hpp:13-46): the experiment
    set-up draws of the suites (constant starts, random sides)."""

    def __init__(self, seed: int):
        s = seed & _M64
        self.st = []
        for _ in range(4):
            s = (s + 0x9E3779B97F4A7C15) & _M64
            z = s
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
            self.st.append(z ^ (z >> 31))

    @staticmethod
    def _rotl(x, k):
        return ((x << k) | (x >> (64 - k))) & _M64

    def next_u64(self) -> int:
        s = self.st
        result = (self._rotl((s[1] * 5) & _M64, 7) * 9) & _M64
        t = (s[1] << 17) & _M64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return result

    def uniform01(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.uniform01()


class Suite:
    def __init__(self):
        self.failures = 0

    def check(self, ok: bool, name: str, detail: str = "") -> None:
        print(("[PASS] " if ok else "[FAIL] ") + name + (f": {detail}" if detail else ""))
        if not ok:
            self.failures += 1


def _census_graph(n: int, p: float, seed: int) -> P.Graph:
    return P.generate(P.ErSpec(n, p), seed)


def _adj_masks(g: P.Graph) -> np.ndarray:
    off, nbr = g.csr()
    adj = np.zeros(g.n(), np.int64)
    for v in range(g.n()):
        for u in nbr[off[v]:off[v + 1]]:
            adj[v] |= 1 << int(u)
    return adj


def _bits(n: int) -> np.ndarray:
    """[2^n][n] 0/1 matrix: row = mask, column v = bit v."""
    masks = np.arange(1 << n, dtype=np.int64)
    return ((masks[:, None] >> np.arange(n)) & 1).astype(np.int64)


def census(spec, g: P.Graph) -> dict:
    """enumerate_fixed_points (oracle.cpp:140-193) with the gradients of all
    2^n binary states computed by the GPU as one chain batch."""
    n = g.n()
    mis = P.problem_of(spec) == P.PROBLEM_MIS
    bits = _bits(n)
    x = bits.astype(np.float64) if mis else 2.0 * bits - 1.0
    b = P.ChainBatch(g, 1 << n)
    b.set_x(x)
    grad = b.gradient(spec)
    adj = _adj_masks(g)
    masks = np.arange(1 << n, dtype=np.int64)
    nb_on = np.stack([(adj[v] & masks) != 0 for v in range(n)], 1)  # a neighbour is set
    if mis:
        independent = ~np.any((bits == 1) & nb_on, axis=1)
        maximal = independent & ~np.any((bits == 0) & ~nb_on, axis=1)
        fixed = ~np.any(np.where(bits == 1, grad < 0.0, grad > 0.0), axis=1)
        return {"fixed": fixed, "independent": independent, "maximal": maximal}
    fixed = ~np.any(x * grad < 0.0, axis=1)
    deg = np.diff(g.csr()[0])
    on1 = np.stack([np.array([bin(int(a)).count("1") for a in (adj[v] & masks)]) for v in range(n)], 1)
    same = np.where(bits == 1, on1, deg[None, :] - on1)
    repairable = np.any(2 * same - deg[None, :] > 0, axis=1)
    return {"fixed": fixed, "repairable": repairable}


def suite_fixed_points(st: Suite, max_n: int, seed: int) -> None:  # cmd_verify.cpp:27-57
    cap = min(max_n, 12)
    ok = {"perturbed": True, "adjacency": True, "bias": True, "mis": True}
    graphs = 0
    for i in range(10):
        n = 6 + (i % (cap - 5))
        p = 0.3 if i % 2 == 0 else 0.5
        g = _census_graph(n, p, derive_seed(seed, 100 + i))
        graphs += 1
        for lam in (0.001, 0.1, 1.0):
            if not census(P.PerturbedLaplacian(lam), g)["fixed"].all():
                ok["perturbed"] = False
        c = census(P.Adjacency(), g)
        if np.any(c["repairable"] & c["fixed"]):
            ok["adjacency"] = False
        c = census(P.PerturbedBias(0.001), g)
        if np.any(c["repairable"] & c["fixed"]):
            ok["bias"] = False
        c = census(P.MisQubo(2.0), g)
        if np.any(c["fixed"] != c["maximal"]):
            ok["mis"] = False
    scope = f"over {graphs} graphs"
    st.check(ok["perturbed"], "fixed-points/perturbed-laplacian-all-binary-fixed", scope)
    st.check(ok["adjacency"], "fixed-points/adjacency-repairable-never-fixed", scope)
    st.check(ok["bias"], "fixed-points/perturbed-bias-fixed-iff-irreparable", scope)
    st.check(ok["mis"], "fixed-points/mis-fixed-iff-maximal", scope)


def _cut(g: P.Graph, side: np.ndarray) -> int:
    off, nbr = g.csr()
    src = np.repeat(np.arange(g.n()), np.diff(off))
    return int(np.sum((src < nbr) & (side[src] != side[nbr])))


def _escape(g: P.Graph, spec, init: np.ndarray, alpha: float, iters: int) -> tuple:
    """experiments.cpp:11-26: init cut, final cut after a PGA trajectory."""
    out = P.run_trajectory(spec, g, init, P.OptimizerConfig(alpha=alpha, beta=0.0,
                                                            max_iters=iters))
    return _cut(g, (init > 0).astype(np.uint8)), _cut(g, (out.state > 0).astype(np.uint8))


def _repairable_side(g: P.Graph, rng: Rng) -> np.ndarray:  # experiments.cpp:46-57
    off, nbr = g.csr()
    deg = np.diff(off)
    src = np.repeat(np.arange(g.n()), deg)
    for _ in range(10000):
        side = np.array([rng.next_u64() & 1 for _ in range(g.n())], np.uint8)
        same = np.zeros(g.n(), np.int64)
        np.add.at(same, src, (side[src] == side[nbr]).astype(np.int64))
        if np.any(2 * same - deg > 0):
            return side
    raise RuntimeError("no 1-flip repairable state found (degenerate graph?)")


def suite_escapability(st: Suite, n: int, p: float, seed: int) -> None:  # cmd_verify.cpp:59-109
    alpha, lam, iters, graphs = 0.1, 0.001, 5000, 10
    lap_stuck, flip_stuck = True, True
    pert_mean = bias_mean = flip_gain = flip_init = 0.0
    for i in range(graphs):
        g = _census_graph(n, p, derive_seed(seed, 200 + i))
        rng = Rng(derive_seed(seed, 300 + i))
        c = rng.uniform(-1.0, 1.0)
        const = np.full(g.n(), c)
        _, fl = _escape(g, P.Laplacian(), const, alpha, iters)
        _, fp = _escape(g, P.PerturbedLaplacian(lam), const, alpha, iters)
        _, fb = _escape(g, P.PerturbedBias(lam), const, alpha, iters)
        lap_stuck &= fl == 0
        pert_mean += fp / graphs
        bias_mean += fb / graphs
        side = _repairable_side(g, rng)
        init = np.where(side == 1, 1.0, -1.0)
        il, rl = _escape(g, P.Laplacian(), init, alpha, iters)
        ip, rp = _escape(g, P.PerturbedLaplacian(lam), init, alpha, iters)
        ib, rb = _escape(g, P.PerturbedBias(lam), init, alpha, iters)
        if rl != il or rp != ip:
            flip_stuck = False
        flip_gain += (rb - ib) / graphs
        flip_init += ib / graphs
    print(f"escapability on er(n={n}, p={p}), {graphs} graphs")
    print(f"  stationary init:  laplacian stuck={'yes' if lap_stuck else 'no'}"
          f"  perturbed-laplacian mean final={pert_mean:g}  perturbed-bias mean final={bias_mean:g}")
    print(f"  repairable init (mean {flip_init:g}): laplacian/perturbed stuck="
          f"{'yes' if flip_stuck else 'no'}  perturbed-bias mean gain={flip_gain:g}")
    st.check(lap_stuck, "escapability/laplacian-stationary-stuck", "final cut 0")
    st.check(pert_mean > 0.0, "escapability/perturbed-laplacian-escapes", f"mean final {pert_mean:f}")
    st.check(bias_mean > 0.0, "escapability/perturbed-bias-escapes", f"mean final {bias_mean:f}")
    st.check(flip_stuck, "escapability/laplacian-perturbed-flip-stuck")
    st.check(flip_gain > 0.0, "escapability/perturbed-bias-flip-gain", f"mean gain {flip_gain:f}")


def exact_optima(g: P.Graph) -> tuple:
    """Exhaustive MIS size and max cut over all 2^n states (n <= 20)."""
    n = g.n()
    if n > 20:
        raise P.InvalidArgument("exact: instance too large (n > 20)")
    bits = _bits(n)
    adj = _adj_masks(g)
    masks = np.arange(1 << n, dtype=np.int64)
    nb_on = np.stack([(adj[v] & masks) != 0 for v in range(n)], 1)
    independent = ~np.any((bits == 1) & nb_on, axis=1)
    mis = int(bits[independent].sum(axis=1).max())
    off, nbr = g.csr()
    src = np.repeat(np.arange(n), np.diff(off))
    e = src < nbr
    cut = np.zeros(1 << n, np.int64)
    for u, v in zip(src[e], nbr[e]):
        cut += bits[:, u] ^ bits[:, v]
    return mis, int(cut.max())


def suite_exact(st: Suite, max_n: int, seed: int) -> None:  # cmd_verify.cpp:111-145
    from . import cli
    hi = min(max_n, 14)
    k = 30
    mis_match = cut_match = 0
    never_exceed = True
    for i in range(k):
        n = 8 + (i % (hi - 7))
        p = 0.3 if i % 2 == 0 else 0.5
        g = _census_graph(n, p, derive_seed(seed, 400 + i))
        mis_opt, cut_opt = exact_optima(g)
        for problem, opt in (("mis", mis_opt), ("maxcut", cut_opt)):
            a = cli.solve_defaults(problem=problem, budget_secs=3.0,
                                   seed=derive_seed(seed, 500 + i), stop_at_score=opt)
            rep = P.solve_pooled(g, cli.build_config(a, g))
            never_exceed &= rep.best_score <= opt
            if rep.best_score == opt:
                if problem == "mis":
                    mis_match += 1
                else:
                    cut_match += 1
    st.check(never_exceed, "exact/never-exceeds-optimum")
    st.check(mis_match * 100 >= k * 95, "exact/mis-agreement", f"{mis_match}/{k}")
    st.check(cut_match * 100 >= k * 95, "exact/maxcut-agreement", f"{cut_match}/{k}")


def cmd_verify(suite: str, max_n: int, n: int, p: float, seed: int) -> int:  # cmd_verify.cpp:149-176
    if suite not in ("all", "fixed-points", "escapability", "exact", "toy-reset"):
        raise ValueError(f"unknown --suite '{suite}'")
    st = Suite()
    if suite in ("all", "fixed-points"):
        suite_fixed_points(st, max_n, seed)
    if suite in ("all", "escapability"):
        suite_escapability(st, n, p, seed)
    if suite in ("all", "exact"):
        suite_exact(st, max_n, seed)
    if suite in ("all", "toy-reset"):
        print("[SKIP] toy-reset: host-only reset study, outside the GPU hot path (DESIGN.md §7)")
    if st.failures:
        print(f"{st.failures} check(s) failed")
        return EXIT_FAIL
    print("all checks passed")
    return EXIT_OK


def add_parser(sub: argparse._SubParsersAction) -> None:  # main.cpp:94-106
    v = sub.add_parser("verify", help="oracle-backed verification suites on the GPU path")
    v.add_argument("--suite", default="all")
    v.add_argument("--max-n", type=int, default=12)
    v.add_argument("--n", type=int, default=100)
    v.add_argument("--p", type=float, default=0.0166)
    v.add_argument("--seed", type=int, default=1)
