"""ctypes binding of libmqo_b200.so (the C ABI in include/mqo_gpu.h).

The library is built in-tree (``make -C paper_2605_06921_b200`` or
``__graft_entry__.build()``).  There is no fallback: if the shared library is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmqo_b200.so")

(MQO_OK, MQO_ERR_INVALID, MQO_ERR_LOGIC, MQO_ERR_CUDA, MQO_ERR_NCCL, MQO_ERR_OTHER,
 MQO_ERR_PARSE) = range(7)
MIS_QUBO, LAPLACIAN, PERTURBED_LAPLACIAN, ADJACENCY, PERTURBED_BIAS = range(5)
PROBLEM_MIS, PROBLEM_MAXCUT = 0, 1
CONVERGED, CHECKER_ACCEPTED, ITER_CAP = 0, 1, 2


class MqoError(RuntimeError):
    """A failing C-ABI call; ``code`` is the MQO_ERR_* status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(MqoError, ValueError):
    """std::invalid_argument in the reference."""


class LogicError(MqoError):
    """std::logic_error in the reference."""


class ParseError(MqoError):
    """mqo::ParseError (graph_io.hpp:13-21): ``line`` is the 1-based line."""

    def __init__(self, code: int, msg: str, line: int):
        super().__init__(code, msg)
        self.line = line


class Objective(C.Structure):
    _fields_ = [("kind", C.c_int32), ("param", C.c_double)]


class Optimizer(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("max_iters", C.c_int32),
                ("conv_tol", C.c_double), ("check_every", C.c_int32)]


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)
_U8 = C.POINTER(C.c_uint8)
_U64 = C.POINTER(C.c_uint64)

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "mqo_last_error": (C.c_char_p, []),
    "mqo_last_error_line": (C.c_int32, []),
    "mqo_graph_parse": (C.c_int, [C.c_char_p, C.c_int64, C.c_int32, C.c_int32, _I64, _PP]),
    "mqo_graph_load_warnings": (C.c_int64, [C.c_char_p, C.c_int64]),
    "mqo_version": (C.c_char_p, []),
    "mqo_graph_upload": (C.c_int, [C.c_int32, _I64, _I32, C.c_int32, _PP]),
    "mqo_graph_free": (C.c_int, [_P]),
    "mqo_graph_info": (C.c_int, [_P, _I32, _I64, _I32]),
    "mqo_graph_strip_isolated": (C.c_int, [_P, _PP, _I32, _I32, _I32, _I32, _I32]),
    "mqo_graph_components": (C.c_int, [_P, _I32, _I32]),
    "mqo_batch_create": (C.c_int, [_P, C.c_int32, _PP]),
    "mqo_batch_free": (C.c_int, [_P]),
    "mqo_batch_chains": (C.c_int, [_P, _I32, _I32]),
    "mqo_batch_stream": (C.c_int, [_P, _PP]),
    "mqo_batch_sync": (C.c_int, [_P]),
    "mqo_batch_set_x": (C.c_int, [_P, _D]),
    "mqo_batch_get_x": (C.c_int, [_P, _D]),
    "mqo_batch_set_v": (C.c_int, [_P, _D]),
    "mqo_batch_get_v": (C.c_int, [_P, _D]),
    "mqo_batch_zero_v": (C.c_int, [_P]),
    "mqo_project": (C.c_int, [_P, C.c_int32]),
    "mqo_gradient": (C.c_int, [_P, C.POINTER(Objective), _D]),
    "mqo_step": (C.c_int, [_P, C.POINTER(Objective), C.POINTER(Optimizer)]),
    "mqo_run_trajectories": (C.c_int, [_P, C.POINTER(Objective), C.POINTER(Optimizer),
                                       C.c_double, _I32, _I32]),
    "mqo_mis_fixed_point_check": (C.c_int, [_P, C.c_double, C.c_double, _I32]),
    "mqo_batch_seed_streams": (C.c_int, [_P, C.c_uint64, C.c_uint64]),
    "mqo_batch_get_streams": (C.c_int, [_P, _P]),
    "mqo_batch_set_streams": (C.c_int, [_P, _P]),
    "mqo_init_states": (C.c_int, [_P, C.c_int32, C.c_double]),
    "mqo_init_constant": (C.c_int, [_P, C.c_int32, C.c_double]),
    "mqo_global_reset": (C.c_int, [_P, C.c_double]),
    "mqo_set_pool": (C.c_int, [_P, C.c_int32, _U64]),
    "mqo_reset_from_pool": (C.c_int, [_P, C.c_int32, C.c_double, _I32]),
    "mqo_harvest": (C.c_int, [_P, C.c_int32, _I64, _I32, _U64]),
    "mqo_local_search": (C.c_int, [_P, C.c_int32, C.c_int32, _U64, _I64]),
    "mqo_tune": (C.c_int, [C.c_char_p, C.c_double]),
}
LS_ONE_FLIP, LS_TWO_FLIP, LS_ONE_TWO_FLIP, LS_ONE_TWO_SWAP = range(4)

# mqo_rng_state as a numpy structured dtype (48 bytes)
RNG_DTYPE = [("s", "<u8", (4,)), ("spare", "<f8"), ("has_spare", "<i4"), ("flags", "<i4")]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc == MQO_OK:
        return
    msg = lib.mqo_last_error().decode()
    if rc == MQO_ERR_INVALID:
        raise InvalidArgument(rc, msg)
    if rc == MQO_ERR_LOGIC:
        raise LogicError(rc, msg)
    if rc == MQO_ERR_PARSE:
        raise ParseError(rc, msg, int(lib.mqo_last_error_line()))
    raise MqoError(rc, msg)
