"""TEST INFRASTRUCTURE ONLY -- ctypes front-end for the CPU checkers.

Two libraries expose the same C interface (oracle/mqo_oracle.h):

* ``oracle/liboracle.so``  -- the plain-C restatement of the reference
  algorithm (oracle/mqo_oracle.c);
* ``oracle/_ref/libref.so`` -- the reference core itself, compiled from
  /root/reference/proj/core/src by ``make -C oracle ref`` (only where the
  reference tree exists; the built .so travels to the GPU box).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this package.  The product package
(paper_2605_06921_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref.so")

MIS_QUBO, LAPLACIAN, PERTURBED_LAPLACIAN, ADJACENCY, PERTURBED_BIAS = range(5)
PROBLEM_MIS, PROBLEM_MAXCUT = 0, 1
CONVERGED, CHECKER_ACCEPTED, ITER_CAP = 0, 1, 2


def problem_of(kind: int) -> int:
    return PROBLEM_MIS if kind == MIS_QUBO else PROBLEM_MAXCUT


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class SolverCfg(C.Structure):
    _fields_ = [
        ("objective", C.c_int32), ("param", C.c_double),
        ("alpha", C.c_double), ("beta", C.c_double),
        ("max_iters", C.c_int32), ("conv_tol", C.c_double), ("check_every", C.c_int32),
        ("reset_fraction", C.c_double), ("reset_rounds", C.c_int32),
        ("init_noise", C.c_double), ("time_budget_secs", C.c_double),
        ("seed", C.c_uint64), ("local_search", C.c_int32),
        ("pool_batch", C.c_int32), ("pool_keep", C.c_int32),
        ("has_init_constant", C.c_int32), ("init_constant", C.c_double),
        ("has_stop_at_score", C.c_int32), ("stop_at_score", C.c_int64),
        ("has_max_outer_loops", C.c_int32), ("max_outer_loops", C.c_int32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("score", C.c_int64), ("found_solution", C.c_int32),
        ("after_gradient", C.c_int64), ("after_reset_loop", C.c_int64),
        ("after_local_search", C.c_int64),
        ("outer_loops", C.c_int32), ("trajectories", C.c_int32),
        ("resets_accepted", C.c_int64), ("resets_rejected", C.c_int64),
        ("total_iterations", C.c_int64), ("last_trajectory_stop", C.c_int32),
        ("elapsed_secs", C.c_double), ("n_warnings", C.c_int32),
    ]


REPORT_KEYS = ("score", "found_solution", "after_gradient", "after_reset_loop",
               "after_local_search", "outer_loops", "trajectories", "resets_accepted",
               "resets_rejected", "total_iterations", "last_trajectory_stop", "n_warnings")


def build(ref: bool | None = None) -> None:
    """Compile the checkers (make -C oracle [ref])."""
    targets = ["all"]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/core/src")
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)
_U8 = C.POINTER(C.c_uint8)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class Lib:
    """One checker library (oracle restatement or compiled reference)."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        L = C.CDLL(path)
        self.L = L
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_impl_name": (C.c_char_p, []),
            "orc_rng_new": (_P, [C.c_uint64]),
            "orc_rng_free": (None, [_P]),
            "orc_rng_next_u64": (C.c_uint64, [_P]),
            "orc_rng_uniform01": (C.c_double, [_P]),
            "orc_rng_uniform_index": (C.c_uint64, [_P, C.c_uint64]),
            "orc_rng_normal": (C.c_double, [_P, C.c_double, C.c_double]),
            "orc_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "orc_graph_from_edges": (C.c_int, [C.c_int32, C.c_int64, _I32, _I32, C.POINTER(_P)]),
            "orc_generate_er": (C.c_int, [C.c_int32, C.c_double, C.c_uint64, C.POINTER(_P)]),
            "orc_generate_ba": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, C.POINTER(_P)]),
            "orc_generate_sbm": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double,
                                           C.c_uint64, C.POINTER(_P)]),
            "orc_graph_free": (None, [_P]),
            "orc_graph_info": (None, [_P, _I32, _I64, _I32]),
            "orc_graph_csr": (None, [_P, _I64, _I32]),
            "orc_strip_isolated": (C.c_int, [_P, C.POINTER(_P), _I32, _I32, _I32, _I32, _I32]),
            "orc_components": (C.c_int, [_P, _I32, _I32]),
            "orc_adjacency_apply": (C.c_int, [_P, _D, _D]),
            "orc_laplacian_apply": (C.c_int, [_P, _D, _D]),
            "orc_validate_objective": (C.c_int, [C.c_int32, C.c_double]),
            "orc_gradient": (C.c_int, [_P, C.c_int32, C.c_double, _D, _D]),
            "orc_value": (C.c_int, [_P, C.c_int32, C.c_double, _D, _D]),
            "orc_extract_solution": (C.c_int, [_P, C.c_int32, _D, _U8, _I64]),
            "orc_cut_value": (C.c_int64, [_P, _U8]),
            "orc_is_independent": (C.c_int, [_P, _U8]),
            "orc_validate_optimizer": (C.c_int, [C.c_double, C.c_double, C.c_int32,
                                                 C.c_double, C.c_int32]),
            "orc_project": (None, [_D, C.c_int32, C.c_int32]),
            "orc_step": (C.c_int, [_P, C.c_int32, C.c_double, _D, _D, C.c_double, C.c_double]),
            "orc_run_trajectory": (C.c_int, [_P, C.c_int32, C.c_double, _D, C.c_double,
                                             C.c_double, C.c_int32, C.c_double, C.c_int32,
                                             _I32, _I32]),
            "orc_mis_fixed_point_check": (C.c_int, [_P, _D, C.c_double, C.c_double, _I32]),
            "orc_init_state": (C.c_int, [_P, C.c_int32, C.c_double, _P, _D]),
            "orc_global_reset": (C.c_int, [_D, C.c_int32, C.c_double, _P, _I32, _I32]),
            "orc_build_tightness": (C.c_int, [_P, _U8, _I32]),
            "orc_build_gain_table": (C.c_int, [_P, _U8, _I64]),
            "orc_greedy_maximalize": (C.c_int, [_P, _U8, _I32]),
            "orc_one_two_swap": (C.c_int, [_P, _U8, _I32]),
            "orc_one_flip_pass": (C.c_int, [_P, _U8, _I64]),
            "orc_two_flip_pass": (C.c_int, [_P, _U8, _I64]),
            "orc_one_two_flip": (C.c_int, [_P, _U8, _I64]),
            "orc_solve_pooled": (C.c_int, [_P, C.POINTER(SolverCfg), C.POINTER(Report), _U8]),
            "orc_preset_for": (C.c_int, [C.c_int32, C.c_int32, C.c_double, _D, _D, _D, _I32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if hasattr(L, "orc_graph_from_csr"):  # oracle-c only (test helper)
            L.orc_graph_from_csr.restype = C.c_int
            L.orc_graph_from_csr.argtypes = [C.c_int32, _I64, _I32, C.POINTER(_P)]
        self.name = L.orc_impl_name().decode()

    # ---------------------------------------------------------------- errors
    def _chk(self, rc: int) -> None:
        if rc != 0:
            raise OracleError(rc, self.L.orc_last_error().decode())

    # ------------------------------------------------------------------- rng
    def rng(self, seed: int) -> "Rng":
        return Rng(self, seed)

    def derive_seed(self, master: int, stream: int) -> int:
        return int(self.L.orc_derive_seed(master, stream))

    # ----------------------------------------------------------------- graph
    def _graph(self, fn, *args) -> "Graph":
        h = _P()
        self._chk(fn(*args, C.byref(h)))
        return Graph(self, h)

    def from_edges(self, n: int, edges) -> "Graph":
        e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
        u = np.ascontiguousarray(e[:, 0])
        v = np.ascontiguousarray(e[:, 1])
        return self._graph(self.L.orc_graph_from_edges, n, len(u), _ptr(u, _I32), _ptr(v, _I32))

    def from_csr(self, n: int, off, nbr) -> "Graph":
        """Wrap a canonical CSR (oracle-c test helper; no re-sort)."""
        off = np.ascontiguousarray(off, np.int64)
        nbr = np.ascontiguousarray(nbr, np.int32)
        return self._graph(self.L.orc_graph_from_csr, n, _ptr(off, _I64), _ptr(nbr, _I32))

    def generate_er(self, n: int, p: float, seed: int) -> "Graph":
        return self._graph(self.L.orc_generate_er, n, p, seed)

    def generate_ba(self, n: int, m_attach: int, seed: int) -> "Graph":
        return self._graph(self.L.orc_generate_ba, n, m_attach, seed)

    def generate_sbm(self, n, k, p_in, p_out, seed) -> "Graph":
        return self._graph(self.L.orc_generate_sbm, n, k, p_in, p_out, seed)

    def strip_isolated(self, g):
        """-> (core Graph, removed, core_to_orig, orig_to_core) (graph.cpp:180-198)."""
        n = g.n
        c2o, o2c, rem = (np.empty(max(n, 1), np.int32) for _ in range(3))
        nc, nr = C.c_int32(), C.c_int32()
        h = _P()
        self._chk(self.L.orc_strip_isolated(g.h, C.byref(h), _ptr(c2o, _I32), _ptr(o2c, _I32),
                                            _ptr(rem, _I32), C.byref(nc), C.byref(nr)))
        return Graph(self, h), rem[: nr.value].copy(), c2o[: nc.value].copy(), o2c[:n].copy()

    def connected_components(self, g):
        """-> list of sorted member arrays, in the reference's order (graph.cpp:200-224)."""
        comp = np.empty(max(g.n, 1), np.int32)
        cnt = C.c_int32()
        self._chk(self.L.orc_components(g.h, _ptr(comp, _I32), C.byref(cnt)))
        order = np.argsort(comp[: g.n], kind="stable")
        bounds = np.searchsorted(comp[: g.n][order], np.arange(cnt.value + 1))
        return [order[bounds[c]:bounds[c + 1]].astype(np.int32) for c in range(cnt.value)]

    # ------------------------------------------------------------ objectives
    def adjacency_apply(self, g, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        self._chk(self.L.orc_adjacency_apply(g.h, _ptr(x, _D), _ptr(y, _D)))
        return y

    def laplacian_apply(self, g, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        self._chk(self.L.orc_laplacian_apply(g.h, _ptr(x, _D), _ptr(y, _D)))
        return y

    def validate_objective(self, kind, param):
        self._chk(self.L.orc_validate_objective(kind, param))

    def gradient(self, g, kind, param, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        self._chk(self.L.orc_gradient(g.h, kind, param, _ptr(x, _D), _ptr(y, _D)))
        return y

    def value(self, g, kind, param, x) -> float:
        x = np.ascontiguousarray(x, np.float64)
        out = C.c_double()
        self._chk(self.L.orc_value(g.h, kind, param, _ptr(x, _D), C.byref(out)))
        return out.value

    def extract_solution(self, g, problem, x):
        x = np.ascontiguousarray(x, np.float64)
        body = np.zeros(g.n, np.uint8)
        score = C.c_int64()
        self._chk(self.L.orc_extract_solution(g.h, problem, _ptr(x, _D), _ptr(body, _U8),
                                              C.byref(score)))
        return body, score.value

    def cut_value(self, g, side) -> int:
        side = np.ascontiguousarray(side, np.uint8)
        return int(self.L.orc_cut_value(g.h, _ptr(side, _U8)))

    def is_independent(self, g, ind) -> bool:
        ind = np.ascontiguousarray(ind, np.uint8)
        return bool(self.L.orc_is_independent(g.h, _ptr(ind, _U8)))

    # ------------------------------------------------------------------- pga
    def validate_optimizer(self, alpha, beta, max_iters=5000, conv_tol=1e-6, check_every=1):
        self._chk(self.L.orc_validate_optimizer(alpha, beta, max_iters, conv_tol, check_every))

    def project(self, x, problem):
        x = np.array(x, np.float64)
        self.L.orc_project(_ptr(x, _D), len(x), problem)
        return x

    def step(self, g, kind, param, x, v, alpha, beta):
        x = np.array(x, np.float64)
        v = np.array(v, np.float64)
        self._chk(self.L.orc_step(g.h, kind, param, _ptr(x, _D), _ptr(v, _D), alpha, beta))
        return x, v

    def run_trajectory(self, g, kind, param, x, alpha, beta=0.0, max_iters=5000,
                       conv_tol=1e-6, check_every=1):
        x = np.array(x, np.float64)
        it = C.c_int32()
        rs = C.c_int32()
        self._chk(self.L.orc_run_trajectory(g.h, kind, param, _ptr(x, _D), alpha, beta,
                                            max_iters, conv_tol, check_every, C.byref(it),
                                            C.byref(rs)))
        return x, it.value, rs.value

    def mis_fixed_point_check(self, g, x, gamma=2.0, alpha=0.8) -> bool:
        x = np.ascontiguousarray(x, np.float64)
        f = C.c_int32()
        self._chk(self.L.orc_mis_fixed_point_check(g.h, _ptr(x, _D), gamma, alpha, C.byref(f)))
        return bool(f.value)

    # ---------------------------------------------------------------- solver
    def init_state(self, g, problem, sigma, rng: "Rng"):
        x = np.empty(g.n, np.float64)
        self._chk(self.L.orc_init_state(g.h, problem, sigma, rng.h, _ptr(x, _D)))
        return x

    def global_reset(self, x, rho, rng: "Rng"):
        x = np.array(x, np.float64)
        chosen = np.empty(max(len(x), 1), np.int32)
        k = C.c_int32()
        self._chk(self.L.orc_global_reset(_ptr(x, _D), len(x), rho, rng.h, _ptr(chosen, _I32),
                                          C.byref(k)))
        return x, chosen[: k.value].copy()

    # ---------------------------------------------------------- local search
    def build_tightness(self, g, ind):
        ind = np.ascontiguousarray(ind, np.uint8)
        t = np.empty(g.n, np.int32)
        self._chk(self.L.orc_build_tightness(g.h, _ptr(ind, _U8), _ptr(t, _I32)))
        return t

    def build_gain_table(self, g, side):
        side = np.ascontiguousarray(side, np.uint8)
        d = np.empty(g.n, np.int64)
        self._chk(self.L.orc_build_gain_table(g.h, _ptr(side, _U8), _ptr(d, _I64)))
        return d

    def greedy_maximalize(self, g, ind):
        ind = np.array(ind, np.uint8)
        s = C.c_int32()
        self._chk(self.L.orc_greedy_maximalize(g.h, _ptr(ind, _U8), C.byref(s)))
        return ind, s.value

    def one_two_swap(self, g, ind):
        ind = np.array(ind, np.uint8)
        s = C.c_int32()
        self._chk(self.L.orc_one_two_swap(g.h, _ptr(ind, _U8), C.byref(s)))
        return ind, s.value

    def _flip(self, fn, g, side):
        side = np.array(side, np.uint8)
        gain = C.c_int64()
        self._chk(fn(g.h, _ptr(side, _U8), C.byref(gain)))
        return side, gain.value

    def one_flip_pass(self, g, side):
        return self._flip(self.L.orc_one_flip_pass, g, side)

    def two_flip_pass(self, g, side):
        return self._flip(self.L.orc_two_flip_pass, g, side)

    def one_two_flip(self, g, side):
        return self._flip(self.L.orc_one_two_flip, g, side)

    # ---------------------------------------------------------------- engine
    def solve_pooled(self, g, cfg: SolverCfg):
        rep = Report()
        body = np.zeros(max(g.n, 1), np.uint8)
        self._chk(self.L.orc_solve_pooled(g.h, C.byref(cfg), C.byref(rep), _ptr(body, _U8)))
        return {k: getattr(rep, k) for k in REPORT_KEYS} | {
            "elapsed_secs": rep.elapsed_secs}, body[: g.n].copy()

    def preset_for(self, problem, n, mean_degree):
        a, m, r = C.c_double(), C.c_double(), C.c_double()
        t = C.c_int32()
        self._chk(self.L.orc_preset_for(problem, n, mean_degree, C.byref(a), C.byref(m),
                                        C.byref(r), C.byref(t)))
        return a.value, m.value, r.value, t.value


class Rng:
    def __init__(self, lib: Lib, seed: int):
        self.lib = lib
        self.h = lib.L.orc_rng_new(seed)

    def __del__(self):
        try:
            self.lib.L.orc_rng_free(self.h)
        except Exception:
            pass

    def next_u64(self) -> int:
        return int(self.lib.L.orc_rng_next_u64(self.h))

    def uniform01(self) -> float:
        return self.lib.L.orc_rng_uniform01(self.h)

    def uniform_index(self, n: int) -> int:
        return int(self.lib.L.orc_rng_uniform_index(self.h, n))

    def normal(self, mean: float, sd: float) -> float:
        return self.lib.L.orc_rng_normal(self.h, mean, sd)


class Graph:
    def __init__(self, lib: Lib, h):
        self.lib = lib
        self.h = h
        n, m, d = C.c_int32(), C.c_int64(), C.c_int32()
        lib.L.orc_graph_info(h, C.byref(n), C.byref(m), C.byref(d))
        self.n, self.m, self.max_degree = n.value, m.value, d.value
        self._csr = None

    def __del__(self):
        try:
            self.lib.L.orc_graph_free(self.h)
        except Exception:
            pass

    def csr(self):
        if self._csr is None:
            off = np.empty(self.n + 1, np.int64)
            nbr = np.empty(max(2 * self.m, 1), np.int32)
            self.lib.L.orc_graph_csr(self.h, _ptr(off, _I64), _ptr(nbr, _I32))
            self._csr = (off, nbr[: 2 * self.m].copy())
        return self._csr

    def edges(self):
        off, nbr = self.csr()
        out = []
        for v in range(self.n):
            for u in nbr[off[v]:off[v + 1]]:
                if v < u:
                    out.append((v, int(u)))
        return out


_cache: dict[str, Lib] = {}


def load(which: str = "oracle") -> Lib:
    """which = 'oracle' (C restatement) or 'ref' (compiled reference)."""
    path = ORACLE_SO if which == "oracle" else REF_SO
    if path not in _cache:
        if which == "oracle" and not os.path.exists(path):
            build(ref=False)
        _cache[path] = Lib(path)
    return _cache[path]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


@dataclass
class Cfg:
    """Python mirror of SolverConfig (solver.hpp:17-36) for the checkers."""
    objective: int = MIS_QUBO
    param: float = 2.0
    alpha: float = 0.8
    beta: float = 0.0
    max_iters: int = 5000
    conv_tol: float = 1e-6
    check_every: int = 1
    reset_fraction: float = 0.5
    reset_rounds: int = 60
    init_noise: float = 0.15
    time_budget_secs: float = 10.0
    seed: int = 1
    local_search: bool = True
    pool_batch: int = 1
    pool_keep: int = 1
    init_constant: float | None = None
    stop_at_score: int | None = None
    max_outer_loops: int | None = None

    def to_c(self) -> SolverCfg:
        c = SolverCfg()
        for f in ("objective", "param", "alpha", "beta", "max_iters", "conv_tol",
                  "check_every", "reset_fraction", "reset_rounds", "init_noise",
                  "time_budget_secs", "seed", "pool_batch", "pool_keep"):
            setattr(c, f, getattr(self, f))
        c.local_search = 1 if self.local_search else 0
        c.has_init_constant = self.init_constant is not None
        c.init_constant = self.init_constant or 0.0
        c.has_stop_at_score = self.stop_at_score is not None
        c.stop_at_score = self.stop_at_score or 0
        c.has_max_outer_loops = self.max_outer_loops is not None
        c.max_outer_loops = self.max_outer_loops or 0
        return c
