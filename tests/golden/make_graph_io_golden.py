"""Freezes the REFERENCE's graph text parsers (graph_io.cpp: parse_dimacs,
read_canonical, load_graph_file's sniffing) on a fixed set of inputs into
tests/golden/graph_io.json, via oracle/_ref/libref.so (`ref_parse_graph` in
oracle/ref_shim.cpp, compiled with the reference's graph.cpp/graph_io.cpp).

Run here (where /root/reference exists):
    python tests/golden/make_graph_io_golden.py
tests/test_graph_io.py checks the C ABI's parser (mqo_graph_parse /
mqo_graph_load) against the fixture on any box.
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "graph_io.json")


def csr_sha(off, nbr) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(off, np.int64).tobytes())
    h.update(np.ascontiguousarray(nbr, np.int32).tobytes())
    return h.hexdigest()


def cases():
    c = [
        (2, "c a comment\np edge 3 3\ne 1 2\ne 2 3\ne 1 3\n"),
        (2, "p edge 3 2\ne 1 2\ne 2 1\n"),
        (2, "e 1 2\n"), (2, "p edge 3 2\ne 1 2\ne 1 9\n"), (2, "p edge 3 1\ne 1 1\n"),
        (2, "p edge 3 1\nq 1 2\n"), (2, "p edge 3 1\ne one two\n"), (2, ""),
        (2, "c only comments\n\n  \n"), (2, "p edge 3 1\np edge 3 1\n"), (2, "p edge 3\n"),
        (2, "p edge -3 1\n"), (2, "p edge 3 -1\n"), (2, "p\n"),
        (2, "p edge 4 2\r\ne 1 2\r\n\r\ne 3 4\r\n"), (2, "p col 5 0\n"),
        (2, "p edge 3 1\ne 1 2x\n"), (2, "p edge 3 1\ne +1 2\n"), (2, "p edge 3 1\ne 1.5 2\n"),
        (2, "p edge 3 1\n   e 1 3   \n"), (2, "p edge 3 1\ncomment 1 2\n"),
        (2, "p edge 3 1\ne 0 2\n"), (2, "p edge 3 1\ne 1\n"), (2, "p edge 3 1\ne 1 2 3\n"),
        (2, "p edge 2 1\ne 1 2"), (2, "\n\np edge 2 1\n\ne 2 1\n\n"),
        (2, "p edge 99999999999 1\n"), (2, "p edge 3 1\ne 99999999999999999999 1\n"),
        (2, "c x\np edge 0 0\n"), (2, "p edge 5 0\n"),
        (1, "3 3\n0 1\n1 2\n0 2\n"), (1, "3 2\n0 1\n"), (1, ""), (1, "3"), (1, "3 1\n0 5\n"),
        (1, "3 1\n1 1\n"), (1, "-2 0\n"), (1, "4 -1\n"), (1, "4 2\n2 1\n1 2\n"),
        (1, "4 2 0 1 2 3"), (1, "4 1\n0 x\n"), (1, "x y\n"), (1, "5 0\n"),
        (0, "c sniffed\np edge 2 1\ne 1 2\n"), (0, "p edge 2 1\ne 2 1\n"), (0, "2 1\n0 1\n"),
        (0, " c leading space is canonical\n"), (0, "q\n"),
    ]
    rng = np.random.default_rng(5)
    for n, m in ((10, 20), (50, 300), (200, 900)):
        e = rng.integers(0, n, (m, 2))
        e = e[e[:, 0] != e[:, 1]]
        c.append((2, f"c random\np edge {n} {len(e)}\n" +
                  "".join(f"e {u + 1} {v + 1}\n" for u, v in e)))
        c.append((0, f"{n} {len(e)}\n" + "".join(f"{u} {v}\n" for u, v in e)))
    return c


def main():
    oracle.build(ref=True)
    L = C.CDLL(oracle.REF_SO)
    f = L.ref_parse_graph
    f.restype = C.c_int
    f.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                  C.POINTER(C.c_int64), C.c_void_p, C.c_void_p, C.c_char_p, C.c_int64,
                  C.POINTER(C.c_int32)]
    out = []
    for fmt, text in cases():
        b = text.encode()
        n, m, dm, line = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32()
        msg = C.create_string_buffer(4096)
        rc = f(b, len(b), fmt, C.byref(n), C.byref(m), C.byref(dm), None, None, msg, 4096,
               C.byref(line))
        rec = {"fmt": fmt, "text": text, "rc": rc, "msg": msg.value.decode(), "line": line.value}
        if rc == 0:
            off = np.zeros(n.value + 1, np.int64)
            nbr = np.zeros(max(1, 2 * m.value), np.int32)
            rc2 = f(b, len(b), fmt, C.byref(n), C.byref(m), C.byref(dm),
                    off.ctypes.data, nbr.ctypes.data, msg, 4096, C.byref(line))
            assert rc2 == 0
            rec.update(n=n.value, m=m.value, declared=dm.value,
                       csr=csr_sha(off, nbr[: 2 * m.value]),
                       warnings=[w for w in msg.value.decode().split("\n") if w])
            rec.pop("msg")
        out.append(rec)
    with open(OUT, "w") as fh:
        json.dump({"source": "reference graph_io.cpp via oracle/_ref/libref.so",
                   "cases": out}, fh, indent=0)
    print(f"wrote {len(out)} cases to {OUT}")


if __name__ == "__main__":
    main()
