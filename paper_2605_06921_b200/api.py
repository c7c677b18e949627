"""Python mirror of the reference's public C++ API for the mQO hot path.

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/mqo/ (graph.hpp, objectives.hpp, pga.hpp,
solver.hpp); every call goes through the C ABI of include/mqo_gpu.h into
libmqo_b200.so.  ``std::invalid_argument`` surfaces as
:class:`InvalidArgument` (a ``ValueError``), ``std::logic_error`` as
:class:`LogicError`.

The batched entry points (:class:`ChainBatch`) are the B200-native shape of
the API: B independent chains of one graph advance together on the device.
The single-chain functions (``step``, ``run_trajectory`` ...) are the
reference signatures, implemented as a batch of one.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (ADJACENCY, CHECKER_ACCEPTED, CONVERGED, ITER_CAP, LAPLACIAN, MIS_QUBO,
                   PERTURBED_BIAS, PERTURBED_LAPLACIAN, PROBLEM_MAXCUT, PROBLEM_MIS,
                   InvalidArgument, LogicError, MqoError, Objective, Optimizer, ParseError, check,
                   lib)

__all__ = [
    "Graph", "ErSpec", "ErFastSpec", "BaSpec", "SbmSpec", "SbmFastSpec", "generate", "StripResult",
    "strip_isolated", "connected_components", "MisQubo", "Laplacian",
    "PerturbedLaplacian", "Adjacency", "PerturbedBias", "OptimizerConfig", "ChainBatch",
    "StopReason", "problem_of", "step", "gradient", "run_trajectory", "mis_fixed_point_check",
    "pack_bodies", "unpack_bodies", "local_search", "one_flip_pass", "two_flip_pass",
    "one_two_flip", "one_two_swap", "SolverConfig", "RunReport", "solve_pooled", "solve_mis",
    "solve_maxcut", "solve_replicas", "solve_devices", "NativeComm", "tune", "init_state_host", "INIT_EXACT", "INIT_DEVICE", "PROBLEM_MIS", "PROBLEM_MAXCUT",
    "InvalidArgument", "LogicError", "MqoError", "ParseError", "DimacsResult", "parse_dimacs_text",
    "read_canonical", "write_canonical", "load_graph_file", "write_graph_file",
]


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)
_U8 = C.POINTER(C.c_uint8)


class StopReason:  # pga.hpp:23
    Converged, CheckerAccepted, IterCap = CONVERGED, CHECKER_ACCEPTED, ITER_CAP
    names = {CONVERGED: "converged", CHECKER_ACCEPTED: "checker-accepted", ITER_CAP: "iter-cap"}


# ------------------------------------------------------------- objectives
@dataclass(frozen=True)
class MisQubo:  # objectives.hpp:22-24
    gamma: float = 2.0
    kind = MIS_QUBO

    @property
    def param(self):
        return self.gamma


@dataclass(frozen=True)
class Laplacian:
    kind = LAPLACIAN
    param = 0.0


@dataclass(frozen=True)
class PerturbedLaplacian:
    lam: float = 0.001
    kind = PERTURBED_LAPLACIAN

    @property
    def param(self):
        return self.lam


@dataclass(frozen=True)
class Adjacency:
    kind = ADJACENCY
    param = 0.0


@dataclass(frozen=True)
class PerturbedBias:  # the paper's new MaxCut objective f_B
    lam: float = 0.001
    kind = PERTURBED_BIAS

    @property
    def param(self):
        return self.lam


def problem_of(spec) -> int:  # objectives.cpp:8-10
    return PROBLEM_MIS if spec.kind == MIS_QUBO else PROBLEM_MAXCUT


def _obj(spec) -> Objective:
    return Objective(spec.kind, float(spec.param))


@dataclass
class OptimizerConfig:  # pga.hpp:13-19
    alpha: float = 0.8
    beta: float = 0.0
    max_iters: int = 5000
    conv_tol: float = 1e-6
    check_every: int = 1

    def to_c(self) -> Optimizer:
        return Optimizer(self.alpha, self.beta, self.max_iters, self.conv_tol, self.check_every)


# ------------------------------------------------------------------ graph
@dataclass(frozen=True)
class ErSpec:  # graph.hpp:67-70
    n: int
    p: float


@dataclass(frozen=True)
class ErFastSpec:
    """O(m) G(n, p) (geometric skipping); not the reference's draw sequence."""
    n: int
    p: float


@dataclass(frozen=True)
class BaSpec:  # graph.hpp:72-75
    n: int
    m_attach: int = 1


@dataclass(frozen=True)
class SbmSpec:  # graph.hpp:77-82
    n: int
    k: int = 2
    p_in: float = 0.0
    p_out: float = 0.0


@dataclass(frozen=True)
class SbmFastSpec:
    """O(m) stochastic block model (geometric skipping over the p_in / p_out
    pair runs); the reference's distribution, not its draw sequence."""
    n: int
    k: int = 2
    p_in: float = 0.0
    p_out: float = 0.0


class _GenSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("p", C.c_double),
                ("m_attach", C.c_int32), ("k", C.c_int32), ("p_in", C.c_double),
                ("p_out", C.c_double), ("seed", C.c_uint64)]


lib.mqo_generate.argtypes = [C.POINTER(_GenSpec), C.c_int32, C.POINTER(C.c_void_p)]
lib.mqo_generate.restype = C.c_int
lib.mqo_graph_from_edges.argtypes = [C.c_int32, C.c_int64, _I32, _I32, C.c_int32,
                                     C.POINTER(C.c_void_p)]
lib.mqo_graph_from_edges.restype = C.c_int
lib.mqo_graph_csr.argtypes = [C.c_void_p, _I64, _I32]
lib.mqo_graph_csr.restype = C.c_int
lib.mqo_graph_row_order.argtypes = [C.c_void_p, _I32]
lib.mqo_graph_row_order.restype = C.c_int
lib.mqo_graph_save.argtypes = [C.c_void_p, C.c_char_p, C.c_int32]
lib.mqo_graph_save.restype = C.c_int
lib.mqo_graph_load.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_void_p)]
lib.mqo_graph_load.restype = C.c_int


class Graph:
    """Immutable CSR graph (graph.hpp:20-63), resident in HBM on ``device``
    (``device=-1`` keeps a host-only graph: CSR readable, no chain batches)."""

    def __init__(self, handle: C.c_void_p, device: int):
        self._h = handle
        self.device = device
        n, m, d = C.c_int32(), C.c_int64(), C.c_int32()
        check(lib.mqo_graph_info(handle, C.byref(n), C.byref(m), C.byref(d)))
        self._n, self._m, self._dmax = n.value, m.value, d.value
        self._csr = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.mqo_graph_free(h)
            self._h = None

    # construction ---------------------------------------------------------
    @staticmethod
    def from_edges(n: int, edges, device: int = 0) -> "Graph":
        e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
        u = np.ascontiguousarray(e[:, 0])
        v = np.ascontiguousarray(e[:, 1])
        h = C.c_void_p()
        check(lib.mqo_graph_from_edges(n, len(u), _ptr(u, _I32), _ptr(v, _I32), device,
                                       C.byref(h)))
        return Graph(h, device)

    @staticmethod
    def from_csr(offsets, neighbors, device: int = 0) -> "Graph":
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.int32)
        if nbr.size == 0:
            nbr = np.zeros(1, np.int32)
        h = C.c_void_p()
        check(lib.mqo_graph_upload(len(off) - 1, _ptr(off, _I64), _ptr(nbr, _I32), device,
                                   C.byref(h)))
        return Graph(h, device)

    @staticmethod
    def load(path: str, device: int = 0) -> "Graph":
        """Binary CSR cache, DIMACS or the reference's canonical text
        (load_graph_file, graph_io.cpp:94-106)."""
        h = C.c_void_p()
        check(lib.mqo_graph_load(path.encode(), device, C.byref(h)))
        return Graph(h, device)

    def save(self, path: str, text: bool = False) -> None:
        check(lib.mqo_graph_save(self._h, path.encode(), 1 if text else 0))

    # accessors ------------------------------------------------------------
    def n(self) -> int:
        return self._n

    def m(self) -> int:
        return self._m

    def max_degree(self) -> int:
        return self._dmax

    def csr(self):
        if self._csr is None:
            off = np.empty(self._n + 1, np.int64)
            nbr = np.empty(max(2 * self._m, 1), np.int32)
            check(lib.mqo_graph_csr(self._h, _ptr(off, _I64), _ptr(nbr, _I32)))
            self._csr = (off, nbr[: 2 * self._m].copy())
        return self._csr

    def row_order(self) -> np.ndarray:
        """The kernels' row schedule (device graphs): degree descending, ties by id."""
        out = np.empty(max(self._n, 1), np.int32)
        check(lib.mqo_graph_row_order(self._h, _ptr(out, _I32)))
        return out[: self._n]

    def degree(self, v: int) -> int:
        off, _ = self.csr()
        return int(off[v + 1] - off[v])

    def neighbors(self, v: int) -> np.ndarray:
        off, nbr = self.csr()
        return nbr[off[v]:off[v + 1]]


def _load_warnings() -> list:
    k = lib.mqo_graph_load_warnings(None, 0)
    if k <= 0:
        return []
    buf = C.create_string_buffer(k + 1)
    lib.mqo_graph_load_warnings(buf, k + 1)
    return buf.value.decode().split("\n")


@dataclass
class DimacsResult:  # graph_io.hpp:23-28
    graph: Graph
    declared_edges: int
    parsed_edges: int
    warnings: list


def _parse(text, fmt: int, device: int):
    data = text.encode() if isinstance(text, str) else bytes(text)
    h, dm = C.c_void_p(), C.c_int64()
    check(lib.mqo_graph_parse(data, len(data), fmt, device, C.byref(dm), C.byref(h)))
    return Graph(h, device), dm.value


def parse_dimacs_text(text, device: int = 0) -> DimacsResult:
    """parse_dimacs_text (graph_io.hpp:35-36, graph_io.cpp:18-71): `c`
    comments, one `p edge <n> <m>` header, 1-based `e <u> <v>` lines;
    duplicates collapse, a declared/parsed m mismatch is a warning; raises
    :class:`ParseError` with the reference's line numbers and messages."""
    g, dm = _parse(text, 2, device)
    return DimacsResult(g, dm, g.m(), _load_warnings())


def read_canonical(text, device: int = 0) -> Graph:
    """read_canonical (graph_io.hpp:41, graph_io.cpp:74-87)."""
    return _parse(text, 1, device)[0]


def write_canonical(g: Graph) -> str:
    """write_canonical (graph_io.hpp:42, graph_io.cpp:89-92) as a string."""
    off, nbr = g.csr()
    src = np.repeat(np.arange(g.n(), dtype=np.int64), np.diff(off))
    keep = src < nbr
    lines = [f"{g.n()} {g.m()}"]
    lines += [f"{u} {v}" for u, v in zip(src[keep].tolist(), nbr[keep].tolist())]
    return "\n".join(lines) + "\n"


def load_graph_file(path: str, warnings: list | None = None, device: int = 0) -> Graph:
    """load_graph_file (graph_io.hpp:45, graph_io.cpp:94-106): sniffs DIMACS
    by a leading 'c'/'p' (else canonical; this backend's binary CSR cache by
    its magic); DIMACS warnings are appended to ``warnings``."""
    g = Graph.load(path, device)
    if warnings is not None:
        warnings.extend(_load_warnings())
    return g


def write_graph_file(g: Graph, path: str) -> None:
    """write_graph_file (graph_io.hpp:46): canonical text."""
    g.save(path, text=True)


@dataclass
class StripResult:  # graph.hpp:95-100
    core: Graph
    removed: np.ndarray        # isolated vertices, ascending
    core_to_orig: np.ndarray   # size core.n()
    orig_to_core: np.ndarray   # -1 for removed vertices


def strip_isolated(g: Graph) -> StripResult:
    """strip_isolated (graph.hpp:104, graph.cpp:180-198), computed on the
    graph's device (flag pass + scan + in-place relabelling)."""
    n = g.n()
    c2o, o2c, rem = (np.empty(max(n, 1), np.int32) for _ in range(3))
    nc, nr = C.c_int32(), C.c_int32()
    h = C.c_void_p()
    check(lib.mqo_graph_strip_isolated(g._h, C.byref(h), _ptr(c2o, _I32), _ptr(o2c, _I32),
                                       _ptr(rem, _I32), C.byref(nc), C.byref(nr)))
    return StripResult(Graph(h, g.device), rem[: nr.value].copy(), c2o[: nc.value].copy(),
                       o2c[:n].copy())


def connected_components(g: Graph) -> list:
    """connected_components (graph.hpp:106, graph.cpp:200-224) on the graph's
    device: sorted member arrays, ordered by smallest vertex."""
    n = g.n()
    comp = np.empty(max(n, 1), np.int32)
    cnt = C.c_int32()
    check(lib.mqo_graph_components(g._h, _ptr(comp, _I32), C.byref(cnt)))
    order = np.argsort(comp[:n], kind="stable")
    bounds = np.searchsorted(comp[:n][order], np.arange(cnt.value + 1))
    return [order[bounds[c]:bounds[c + 1]].astype(np.int32) for c in range(cnt.value)]


def generate(spec, seed: int, device: int = 0) -> Graph:
    """generate(GraphGenSpec) (graph.cpp:169-178), bit-identical graphs."""
    s = _GenSpec()
    s.seed = seed
    if isinstance(spec, ErSpec):
        s.kind, s.n, s.p = 0, spec.n, spec.p
    elif isinstance(spec, ErFastSpec):
        s.kind, s.n, s.p = 3, spec.n, spec.p
    elif isinstance(spec, BaSpec):
        s.kind, s.n, s.m_attach = 1, spec.n, spec.m_attach
    elif isinstance(spec, SbmSpec):
        s.kind, s.n, s.k, s.p_in, s.p_out = 2, spec.n, spec.k, spec.p_in, spec.p_out
    elif isinstance(spec, SbmFastSpec):
        s.kind, s.n, s.k, s.p_in, s.p_out = 4, spec.n, spec.k, spec.p_in, spec.p_out
    else:
        raise InvalidArgument(1, "generate: unknown spec")
    h = C.c_void_p()
    check(lib.mqo_generate(C.byref(s), device, C.byref(h)))
    return Graph(h, device)


# ------------------------------------------------------------ chain batch
class ChainBatch:
    """B chains (relaxed states + velocities) of one graph on its device."""

    def __init__(self, g: Graph, chains: int):
        self.g = g
        self.chains = chains
        h = C.c_void_p()
        check(lib.mqo_batch_create(g._h, chains, C.byref(h)))
        self._h = h
        pad = C.c_int32()
        check(lib.mqo_batch_chains(h, None, C.byref(pad)))
        self.padded = pad.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.mqo_batch_free(h)
            self._h = None

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        check(lib.mqo_batch_stream(self._h, C.byref(s)))
        return s.value or 0

    def sync(self) -> None:
        check(lib.mqo_batch_sync(self._h))

    def _shape_in(self, a) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.shape != (self.chains, self.g.n()):
            a = a.reshape(self.chains, self.g.n())
        return a

    def set_x(self, x) -> None:
        x = self._shape_in(x)
        check(lib.mqo_batch_set_x(self._h, _ptr(x, _D)))

    def get_x(self, out: np.ndarray | None = None) -> np.ndarray:
        out = np.empty((self.chains, self.g.n()), np.float64) if out is None else out
        check(lib.mqo_batch_get_x(self._h, _ptr(out, _D)))
        return out

    def set_v(self, v) -> None:
        v = self._shape_in(v)
        check(lib.mqo_batch_set_v(self._h, _ptr(v, _D)))

    def get_v(self) -> np.ndarray:
        out = np.empty((self.chains, self.g.n()), np.float64)
        check(lib.mqo_batch_get_v(self._h, _ptr(out, _D)))
        return out

    def zero_v(self) -> None:
        check(lib.mqo_batch_zero_v(self._h))

    def project(self, problem: int) -> None:
        check(lib.mqo_project(self._h, problem))

    def gradient(self, spec, out: np.ndarray | None = None) -> np.ndarray:
        """[B][n] gradients; `out` (C-contiguous float64, e.g. a view of
        pinned memory) avoids the pageable staging copy."""
        if out is None:
            out = np.empty((self.chains, self.g.n()), np.float64)
        elif out.shape != (self.chains, self.g.n()) or out.dtype != np.float64 \
                or not out.flags.c_contiguous:
            raise InvalidArgument(1, "gradient: out must be C-contiguous float64 [B][n]")
        o = _obj(spec)
        check(lib.mqo_gradient(self._h, C.byref(o), _ptr(out, _D)))
        return out

    def step(self, spec, cfg: OptimizerConfig) -> None:
        """One fused PGA step of every chain (asynchronous)."""
        o, c = _obj(spec), cfg.to_c()
        check(lib.mqo_step(self._h, C.byref(o), C.byref(c)))

    def run_trajectories(self, spec, cfg: OptimizerConfig, deadline: float = -1.0):
        o, c = _obj(spec), cfg.to_c()
        it = np.zeros(self.chains, np.int32)
        rs = np.zeros(self.chains, np.int32)
        check(lib.mqo_run_trajectories(self._h, C.byref(o), C.byref(c), deadline,
                                       _ptr(it, _I32), _ptr(rs, _I32)))
        return it, rs

    def mis_fixed_point_check(self, gamma: float, alpha: float) -> np.ndarray:
        f = np.zeros(self.chains, np.int32)
        check(lib.mqo_mis_fixed_point_check(self._h, gamma, alpha, _ptr(f, _I32)))
        return f.astype(bool)

    # -- streams, init, reset, harvest (solver.cpp) ------------------------
    def seed_streams(self, master_seed: int, first_stream: int = 1) -> None:
        """chain b <- Rng(derive_seed(master_seed, first_stream + b))."""
        check(lib.mqo_batch_seed_streams(self._h, master_seed, first_stream))

    def get_streams(self) -> np.ndarray:
        out = np.zeros(self.chains, dtype=_lib.RNG_DTYPE)
        check(lib.mqo_batch_get_streams(self._h, out.ctypes.data))
        return out

    def set_streams(self, states: np.ndarray) -> None:
        st = np.ascontiguousarray(states, dtype=_lib.RNG_DTYPE)
        check(lib.mqo_batch_set_streams(self._h, st.ctypes.data))

    def init_states(self, problem: int, sigma: float) -> None:
        check(lib.mqo_init_states(self._h, problem, sigma))

    def init_constant(self, problem: int, c: float) -> None:
        check(lib.mqo_init_constant(self._h, problem, c))

    def global_reset(self, rho: float) -> None:
        check(lib.mqo_global_reset(self._h, rho))

    def set_pool(self, packed: np.ndarray) -> None:
        p = np.ascontiguousarray(packed, dtype=np.uint64)
        check(lib.mqo_set_pool(self._h, p.shape[0], _ptr(p, C.POINTER(C.c_uint64))))

    def reset_from_pool(self, problem: int, rho: float) -> np.ndarray:
        picks = np.zeros(self.chains, np.int32)
        check(lib.mqo_reset_from_pool(self._h, problem, rho, _ptr(picks, _I32)))
        return picks

    def harvest(self, problem: int):
        """-> scores int64[B], valid bool[B], packed bodies uint64[B][W]."""
        W = (self.g.n() + 63) // 64
        scores = np.zeros(self.chains, np.int64)
        valid = np.zeros(self.chains, np.int32)
        packed = np.zeros((self.chains, max(W, 1)), np.uint64)
        check(lib.mqo_harvest(self._h, problem, _ptr(scores, _I64), _ptr(valid, _I32),
                              _ptr(packed, C.POINTER(C.c_uint64))))
        return scores, valid.astype(bool), packed[:, :W]


def pack_bodies(bodies: np.ndarray) -> np.ndarray:
    """uint8 [B][n] 0/1 -> packed uint64 [B][ceil(n/64)], vertex v at bit
    63-(v%64) of word v//64 (word order = lexicographic body order)."""
    b = np.atleast_2d(np.asarray(bodies, np.uint8))
    B, n = b.shape
    W = (n + 63) // 64
    pad = np.zeros((B, W * 64), np.uint8)
    pad[:, :n] = b
    bits = np.packbits(pad.reshape(B, W, 64), axis=2, bitorder="big")  # [B][W][8] bytes
    return bits.view(">u8").reshape(B, W).astype(np.uint64)


def unpack_bodies(packed: np.ndarray, n: int) -> np.ndarray:
    p = np.atleast_2d(np.asarray(packed, np.uint64))
    B, W = p.shape
    by = p.astype(">u8").view(np.uint8).reshape(B, W, 8)
    return np.unpackbits(by, axis=2, bitorder="big").reshape(B, W * 64)[:, :n].copy()


# ------------------------------------------- single-chain reference calls
@dataclass
class RelaxedState:  # objectives.hpp:45-48
    x: np.ndarray
    problem: int = PROBLEM_MIS


@dataclass
class TrajectoryOutcome:  # pga.hpp:26-30
    state: np.ndarray
    iterations: int = 0
    reason: int = ITER_CAP
    extra: dict = field(default_factory=dict)


def gradient(spec, g: Graph, x) -> np.ndarray:
    b = ChainBatch(g, 1)
    b.set_x(np.asarray(x, np.float64)[None, :])
    return b.gradient(spec)[0]


def step(spec, g: Graph, x, velocity, cfg: OptimizerConfig):
    """pga.hpp:36-37 -- returns (x, velocity) after one step."""
    b = ChainBatch(g, 1)
    b.set_x(np.asarray(x, np.float64)[None, :])
    v = np.zeros(g.n()) if velocity is None or len(velocity) == 0 else velocity
    b.set_v(np.asarray(v, np.float64)[None, :])
    b.step(spec, cfg)
    return b.get_x()[0], b.get_v()[0]


def run_trajectory(spec, g: Graph, init, cfg: OptimizerConfig,
                   deadline: float | None = None) -> TrajectoryOutcome:
    """pga.hpp:47-49 on one chain."""
    b = ChainBatch(g, 1)
    b.set_x(np.asarray(init, np.float64)[None, :])
    it, rs = b.run_trajectories(spec, cfg, -1.0 if deadline is None else deadline)
    return TrajectoryOutcome(b.get_x()[0], int(it[0]), int(rs[0]))


def mis_fixed_point_check(g: Graph, x, gamma: float, alpha: float) -> bool:
    b = ChainBatch(g, 1)
    b.set_x(np.asarray(x, np.float64)[None, :])
    return bool(b.mis_fixed_point_check(gamma, alpha)[0])


# ------------------------------------------------------------ local search
def local_search(batch: ChainBatch, op: int, bodies: np.ndarray):
    """Runs a local-search op (localsearch.hpp:28-48) on packed bodies
    [count][W] on the batch's device.  Returns (packed bodies, out) where out
    is the gain (flip ops) or the new set size (one_two_swap)."""
    p = np.array(np.atleast_2d(bodies), dtype=np.uint64, order="C")
    out = np.zeros(p.shape[0], np.int64)
    check(lib.mqo_local_search(batch._h, op, p.shape[0], _ptr(p, C.POINTER(C.c_uint64)),
                               _ptr(out, _I64)))
    return p, out


def _ls_single(g: Graph, op: int, body_u8) -> tuple:
    b = ChainBatch(g, 1)
    p, out = local_search(b, op, pack_bodies(np.asarray(body_u8, np.uint8)[None, :]))
    return unpack_bodies(p, g.n())[0], int(out[0])


def one_flip_pass(g: Graph, side):  # localsearch.hpp:39
    return _ls_single(g, _lib.LS_ONE_FLIP, side)


def two_flip_pass(g: Graph, side):  # localsearch.hpp:44
    return _ls_single(g, _lib.LS_TWO_FLIP, side)


def one_two_flip(g: Graph, side):  # localsearch.hpp:48
    return _ls_single(g, _lib.LS_ONE_TWO_FLIP, side)


def one_two_swap(g: Graph, indicator):  # localsearch.hpp:34
    return _ls_single(g, _lib.LS_ONE_TWO_SWAP, indicator)


# ------------------------------------------------------------------ solver
class _SolverCfg(C.Structure):
    _fields_ = [
        ("objective", C.c_int32), ("param", C.c_double), ("alpha", C.c_double),
        ("beta", C.c_double), ("max_iters", C.c_int32), ("conv_tol", C.c_double),
        ("check_every", C.c_int32), ("reset_fraction", C.c_double),
        ("reset_rounds", C.c_int32), ("init_noise", C.c_double),
        ("time_budget_secs", C.c_double), ("seed", C.c_uint64), ("local_search", C.c_int32),
        ("pool_batch", C.c_int32), ("pool_keep", C.c_int32),
        ("has_init_constant", C.c_int32), ("init_constant", C.c_double),
        ("has_stop_at_score", C.c_int32), ("stop_at_score", C.c_int64),
        ("has_max_outer_loops", C.c_int32), ("max_outer_loops", C.c_int32),
        ("init_mode", C.c_int32)]


class _RunReport(C.Structure):
    _fields_ = [
        ("score", C.c_int64), ("found_solution", C.c_int32), ("after_gradient", C.c_int64),
        ("after_reset_loop", C.c_int64), ("after_local_search", C.c_int64),
        ("outer_loops", C.c_int32), ("trajectories", C.c_int32),
        ("resets_accepted", C.c_int64), ("resets_rejected", C.c_int64),
        ("total_iterations", C.c_int64), ("last_trajectory_stop", C.c_int32),
        ("elapsed_secs", C.c_double), ("n_warnings", C.c_int32), ("warnings", C.c_int32)]


class _Comm(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_int32), ("world", C.c_int32),
                ("allgather", C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_size_t)),
                ("allreduce_max_u64", C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64),
                                                  C.c_size_t)),
                ("broadcast", C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t,
                                          C.c_int32))]


def _make_comm(comm) -> _Comm:
    """Wraps a Python communicator (.rank, .world, .allgather(bytes) -> bytes,
    optionally .allreduce_max(list[int]) -> list[int] and .broadcast(bytes,
    root) -> bytes) as an mqo_comm; the callbacks stay alive with the struct."""
    def _ag(ctx, send, recv, nbytes):
        try:
            out = comm.allgather(C.string_at(send, nbytes))
            C.memmove(recv, out, len(out))
            return 0
        except Exception:  # surfaced as an engine error
            return 1

    def _ar(ctx, data, count):
        try:
            vals = comm.allreduce_max([data[i] for i in range(count)])
            for i in range(count):
                data[i] = int(vals[i])
            return 0
        except Exception:
            return 1

    def _bc(ctx, buf, nbytes, root):
        try:
            out = comm.broadcast(C.string_at(buf, nbytes), root)
            C.memmove(buf, out, nbytes)
            return 0
        except Exception:
            return 1

    c = _Comm()
    c.ctx, c.rank, c.world = None, comm.rank, comm.world
    c.allgather = _Comm._fields_[3][1](_ag)
    # NULL callbacks are emulated with allgather by the engine
    c.allreduce_max_u64 = (_Comm._fields_[4][1](_ar) if hasattr(comm, "allreduce_max")
                           else _Comm._fields_[4][1]())
    c.broadcast = (_Comm._fields_[5][1](_bc) if hasattr(comm, "broadcast")
                   else _Comm._fields_[5][1]())
    return c


class NativeComm:
    """A communicator implemented inside libmqo_b200 (include/mqo_gpu.h):
    NCCL over NVLink (one process per GPU: `NativeComm.nccl`), or the
    in-process exchange for ranks that are threads of this process
    (`NativeComm.local_group`).  Pass it as `comm=` to solve_pooled /
    solve_replicas: the engine's collectives then run without Python."""

    def __init__(self, ptr):
        self._p = C.cast(ptr, C.POINTER(_Comm))
        self.rank, self.world = self._p.contents.rank, self._p.contents.world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib.mqo_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, rank: int, world: int, unique_id: bytes, device: int) -> "NativeComm":
        out = C.c_void_p()
        idb = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        check(lib.mqo_comm_nccl_create(rank, world, idb, device, C.byref(out)))
        return cls(out)

    @classmethod
    def local_group(cls, world: int) -> list:
        out = (C.c_void_p * world)()
        check(lib.mqo_comm_create_local(world, out))
        return [cls(out[i]) for i in range(world)]

    def close(self):
        if getattr(self, "_p", None) is not None:
            lib.mqo_comm_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


lib.mqo_nccl_unique_id.argtypes = [C.c_void_p]
lib.mqo_nccl_unique_id.restype = C.c_int
lib.mqo_comm_nccl_create.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                     C.POINTER(C.c_void_p)]
lib.mqo_comm_nccl_create.restype = C.c_int
lib.mqo_comm_create_local.argtypes = [C.c_int32, C.c_void_p]
lib.mqo_comm_create_local.restype = C.c_int
lib.mqo_comm_create_devices.argtypes = [C.c_int32, _I32, C.c_void_p]
lib.mqo_comm_create_devices.restype = C.c_int
lib.mqo_comm_free.argtypes = [C.c_void_p]
lib.mqo_comm_free.restype = C.c_int
lib.mqo_comm_last_error.restype = C.c_char_p


def _comm_arg(comm):
    """(ctypes argument, keep-alive) for a NativeComm, a Python comm or None."""
    if comm is None:
        return None, None
    if isinstance(comm, NativeComm):
        return comm._p, comm
    c = _make_comm(comm)
    return C.byref(c), c


lib.mqo_solve_pooled.argtypes = [C.c_void_p, C.POINTER(_SolverCfg), C.POINTER(_Comm),
                                 C.POINTER(_RunReport), _U8]
lib.mqo_solve_pooled.restype = C.c_int
lib.mqo_solve_replicas.argtypes = [C.c_void_p, C.POINTER(_SolverCfg), C.POINTER(_Comm),
                                   C.POINTER(_RunReport), _U8, _I64]
lib.mqo_solve_replicas.restype = C.c_int
lib.mqo_solve_devices.argtypes = [C.c_void_p, C.POINTER(_SolverCfg), _I32, C.c_int32, C.c_int32,
                                  C.POINTER(_RunReport), _U8, _I64]
lib.mqo_solve_devices.restype = C.c_int
lib.mqo_init_state_host.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_void_p, _D]
lib.mqo_init_state_host.restype = C.c_int

INIT_EXACT, INIT_DEVICE = 0, 1
WARNINGS = {1: "graph has no edges; returning the trivial solution",
            2: "floor(rho * n) = 0: global resets are no-ops",
            4: "budget exhausted before the first trajectory finished"}


@dataclass
class SolverConfig:  # solver.hpp:17-36
    objective: object = field(default_factory=MisQubo)
    optimizer: OptimizerConfig = field(default_factory=OptimizerConfig)
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
    init_mode: int = INIT_EXACT

    def to_c(self) -> _SolverCfg:
        c = _SolverCfg()
        c.objective, c.param = self.objective.kind, float(self.objective.param)
        o = self.optimizer
        c.alpha, c.beta, c.max_iters = o.alpha, o.beta, o.max_iters
        c.conv_tol, c.check_every = o.conv_tol, o.check_every
        c.reset_fraction, c.reset_rounds = self.reset_fraction, self.reset_rounds
        c.init_noise, c.time_budget_secs, c.seed = self.init_noise, self.time_budget_secs, self.seed
        c.local_search = 1 if self.local_search else 0
        c.pool_batch, c.pool_keep = self.pool_batch, self.pool_keep
        c.has_init_constant = self.init_constant is not None
        c.init_constant = self.init_constant or 0.0
        c.has_stop_at_score = self.stop_at_score is not None
        c.stop_at_score = self.stop_at_score or 0
        c.has_max_outer_loops = self.max_outer_loops is not None
        c.max_outer_loops = self.max_outer_loops or 0
        c.init_mode = self.init_mode
        return c


@dataclass
class RunReport:  # solver.hpp:48-61
    best_score: int
    best_body: np.ndarray
    found_solution: bool
    after_gradient: int
    after_reset_loop: int
    after_local_search: int
    outer_loops: int
    trajectories: int
    resets_accepted: int
    resets_rejected: int
    total_iterations: int
    last_trajectory_stop: int
    elapsed_secs: float
    warnings: list


def tune(key: str, value: float) -> None:
    """Measurement knobs of the kernels (include/mqo_gpu.h mqo_tune): e.g.
    "heavy_deg", "persistent_cells", "cta_traj", "group_quads"."""
    check(lib.mqo_tune(key.encode(), float(value)))


def solve_pooled(g: Graph, cfg: SolverConfig, comm=None) -> RunReport:
    """solve_pooled (solver.hpp:80) on g's device.  `comm` (optional) is an
    object with .rank, .world and .allgather(bytes) -> bytes (all ranks'
    contributions concatenated in rank order), e.g. a torch.distributed
    adapter; chains are then sharded over the ranks."""
    rep = _RunReport()
    body = np.zeros(max(g.n(), 1), np.uint8)
    arg, keep = _comm_arg(comm)  # kept alive for the call
    check(lib.mqo_solve_pooled(g._h, C.byref(cfg.to_c()), arg, C.byref(rep), _ptr(body, _U8)))
    del keep
    return _report(rep, body, g)


def solve_replicas(g: Graph, cfg: SolverConfig, comm=None):
    """Mode R (include/mqo_gpu.h mqo_solve_replicas):
    every rank solves its chain shard independently; one allreduce-max picks
    the best rank, whose body is broadcast.  Returns (RunReport, per-rank
    best scores)."""
    rep = _RunReport()
    body = np.zeros(max(g.n(), 1), np.uint8)
    arg, keep = _comm_arg(comm)
    world = comm.world if comm is not None else 1
    scores = np.zeros(world, np.int64)
    check(lib.mqo_solve_replicas(g._h, C.byref(cfg.to_c()), arg, C.byref(rep), _ptr(body, _U8),
                                 _ptr(scores, _I64)))
    del keep
    return _report(rep, body, g), scores


def solve_devices(g: Graph, cfg: SolverConfig, devices, mode: str = "pooled"):
    """One process, several GPUs (include/mqo_gpu.h mqo_solve_devices): rank
    r runs chains [r*ceil(B/N), ...) on devices[r] in its own host thread;
    "pooled" (Mode P) equals the single-GPU run, "replicas" (Mode R) ends
    with one argmax all-reduce.  Distinct devices exchange over NCCL.
    Returns (RunReport, per-rank best scores or None)."""
    devs = np.ascontiguousarray(devices, np.int32)
    m = {"pooled": 0, "replicas": 1}[mode]
    rep = _RunReport()
    body = np.zeros(max(g.n(), 1), np.uint8)
    scores = np.zeros(len(devs), np.int64)
    check(lib.mqo_solve_devices(g._h, C.byref(cfg.to_c()), _ptr(devs, _I32), len(devs), m,
                                C.byref(rep), _ptr(body, _U8), _ptr(scores, _I64)))
    return _report(rep, body, g), (scores if m == 1 else None)


def _report(rep, body, g) -> "RunReport":
    warns = [m for bit, m in WARNINGS.items() if rep.warnings & bit]
    return RunReport(rep.score, body[: g.n()].copy(), bool(rep.found_solution), rep.after_gradient,
                     rep.after_reset_loop, rep.after_local_search, rep.outer_loops,
                     rep.trajectories, rep.resets_accepted, rep.resets_rejected,
                     rep.total_iterations, rep.last_trajectory_stop, rep.elapsed_secs, warns)


def solve_mis(g: Graph, cfg: SolverConfig) -> RunReport:  # solver.cpp:376-381
    if problem_of(cfg.objective) != PROBLEM_MIS:
        raise InvalidArgument(1, "solve_mis: objective must be the MIS QUBO")
    if cfg.pool_batch != 1 or cfg.pool_keep != 1:
        raise InvalidArgument(1, "solve_mis: sequential solver requires batch = keep = 1")
    return solve_pooled(g, cfg)


def solve_maxcut(g: Graph, cfg: SolverConfig) -> RunReport:  # solver.cpp:383-389
    if problem_of(cfg.objective) != PROBLEM_MAXCUT:
        raise InvalidArgument(1, "solve_maxcut: objective must be a MaxCut formulation")
    if cfg.pool_batch != 1 or cfg.pool_keep != 1:
        raise InvalidArgument(1, "solve_maxcut: sequential solver requires batch = keep = 1")
    return solve_pooled(g, cfg)


def init_state_host(g: Graph, problem: int, sigma: float, state: np.ndarray):
    """init_state (solver.cpp:30-46) for one stream on the host (EXACT mode)."""
    st = np.array(state, dtype=_lib.RNG_DTYPE).reshape(1)
    x = np.empty(g.n(), np.float64)
    check(lib.mqo_init_state_host(g._h, problem, sigma, st.ctypes.data, _ptr(x, _D)))
    return x, st[0]
