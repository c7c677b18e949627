"""The C ABI library loads without a GPU and exports every function that
include/mqo_gpu.h declares; host-only entry points behave (CPU only)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "mqo_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mqo_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol():
    from paper_2605_06921_b200 import _lib
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing
    # and the ctypes signatures we bind are all declared in the header
    assert set(_lib.SIGNATURES) <= set(names)


def test_version_and_errors():
    from paper_2605_06921_b200 import _lib
    assert b"sm_100a" in _lib.lib.mqo_version()
    rc = _lib.lib.mqo_graph_info(None, None, None, None)
    assert rc == _lib.MQO_ERR_INVALID
    assert b"null graph" in _lib.lib.mqo_last_error()


def test_host_only_graph_has_no_batches():
    from paper_2605_06921_b200 import ChainBatch, Graph, InvalidArgument
    g = Graph.from_edges(3, [(0, 1), (1, 2)], device=-1)
    assert (g.n(), g.m(), g.max_degree()) == (3, 2, 2)
    with pytest.raises(InvalidArgument, match="host-only"):
        ChainBatch(g, 4)


def test_csr_invariants_are_checked():
    from paper_2605_06921_b200 import Graph, LogicError
    with pytest.raises(LogicError, match="strictly ascending"):
        Graph.from_csr([0, 2, 3, 4], [2, 1, 0, 0], device=-1)
    with pytest.raises(LogicError, match="self-loop"):
        Graph.from_csr([0, 1, 2], [0, 0], device=-1)
