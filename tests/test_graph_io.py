"""Graph text formats (graph_io.hpp:35-46) behind the C ABI
(mqo_graph_parse / mqo_graph_load), pinned to the REFERENCE's own parsers:
tests/golden/graph_io.json was produced by running graph_io.cpp itself
(tests/golden/make_graph_io_golden.py).  Host-only graphs (device=-1), so
these run without a GPU.  The KATs re-host test_graph.cpp:132-189."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2605_06921_b200 as P
from paper_2605_06921_b200 import _lib

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "graph_io.json")))["cases"]


def csr_sha(g):
    off, nbr = g.csr()
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(off, np.int64).tobytes())
    h.update(np.ascontiguousarray(nbr, np.int32).tobytes())
    return h.hexdigest()


def parse(fmt, text):
    if fmt == 2:
        r = P.parse_dimacs_text(text, device=-1)
        return r.graph, r.declared_edges, r.warnings
    if fmt == 1:
        return P.read_canonical(text, device=-1), -1, []
    g, dm = P.api._parse(text, 0, -1)
    return g, dm, P.api._load_warnings()


@pytest.mark.parametrize("case", GOLD, ids=[f"{i}" for i in range(len(GOLD))])
def test_parser_matches_reference(case):
    fmt, text = case["fmt"], case["text"]
    if case["rc"] == 0:
        g, dm, warnings = parse(fmt, text)
        assert (g.n(), g.m()) == (case["n"], case["m"])
        assert csr_sha(g) == case["csr"]
        assert warnings == case["warnings"]
        if case["declared"] >= 0:
            assert dm == case["declared"]
        return
    with pytest.raises(P.MqoError) as ei:
        parse(fmt, text)
    e = ei.value
    assert str(e) == case["msg"]
    if case["rc"] == 1:
        assert isinstance(e, P.ParseError) and e.line == case["line"]
    elif case["rc"] == 2:
        assert isinstance(e, P.InvalidArgument)
    else:
        assert e.code not in (_lib.MQO_ERR_PARSE, _lib.MQO_ERR_INVALID)


def test_load_graph_file_sniffs_the_format(tmp_path):
    """test_graph.cpp:173-189 + the binary cache of this backend."""
    g = P.generate(P.ErSpec(12, 0.3), 31, device=-1)
    canon = str(tmp_path / "canonical.g")
    P.write_graph_file(g, canon)
    assert (P.load_graph_file(canon, device=-1).csr()[1] == g.csr()[1]).all()
    dim = tmp_path / "dimacs.g"
    dim.write_text("c tiny triangle\np edge 3 3\ne 1 2\ne 2 3\ne 1 3\n")
    warnings = []
    k3 = P.load_graph_file(str(dim), warnings, device=-1)
    assert (k3.n(), k3.m()) == (3, 3) and warnings == []
    dim.write_text("p edge 3 2\ne 1 2\ne 2 1\n")
    k = P.load_graph_file(str(dim), warnings, device=-1)
    assert k.m() == 1 and warnings == ["declared m=2 but parsed m=1 after deduplication"]
    binp = str(tmp_path / "g.csr")
    g.save(binp)
    assert csr_sha(P.load_graph_file(binp, device=-1)) == csr_sha(g)
    with pytest.raises(P.MqoError, match="cannot open graph file"):
        P.load_graph_file(str(tmp_path / "missing.g"), device=-1)


def test_canonical_round_trip():
    """test_graph.cpp:163-171."""
    g = P.generate(P.ErSpec(37, 0.2), 21, device=-1)
    back = P.read_canonical(P.write_canonical(g), device=-1)
    assert back.n() == g.n() and csr_sha(back) == csr_sha(g)
