"""Wall time of mqo_graph_upload from pinned host CSR (bench.py's e2e leg
uploads the C4 graph every step), with MQO_TRACE stage stamps on stderr.
    MQO_TRACE=1 python scripts/upload_probe.py"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2605_06921_b200 as P  # noqa: E402

g0 = P.generate(P.BaSpec(1_000_000, 5), 1)
off, nbr = g0.csr()
h_off, h_nbr = torch.from_numpy(off).pin_memory(), torch.from_numpy(nbr).pin_memory()
n = g0.n()
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = C.c_void_p()
    P._lib.check(P.api.lib.mqo_graph_upload(n, C.cast(h_off.data_ptr(), C.POINTER(C.c_int64)),
                                            C.cast(h_nbr.data_ptr(), C.POINTER(C.c_int32)), 0,
                                            C.byref(h)))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    g = P.Graph(h, 0)
    del g
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"upload {1e3 * (t1 - t0):.2f} ms  free {1e3 * (t2 - t1):.2f} ms", file=sys.stderr, flush=True)
