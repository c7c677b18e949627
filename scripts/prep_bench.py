"""Device pre-processing timings: strip_isolated and
connected_components on the GPU vs the reference's functions on the same
graph (oracle/_ref; same outputs checked).  Sparse ER (mean degree 1.5:
many isolated vertices and small components) and ER(1e7, d=16) (C5)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import oracle
    import paper_2605_06921_b200 as P
    L = oracle.load("ref" if oracle.have_ref() else "oracle")
    for n, d in ((2_000_000, 1.5), (10_000_000, 16.0)):
        g = P.generate(P.ErFastSpec(n, d / n), 1)
        P.strip_isolated(g)  # warm-up (module load)
        t0 = time.perf_counter()
        r = P.strip_isolated(g)
        t_strip = time.perf_counter() - t0
        t0 = time.perf_counter()
        comps = P.connected_components(g)
        t_cc = time.perf_counter() - t0
        off, nbr = g.csr()
        src = np.repeat(np.arange(n, dtype=np.int32), np.diff(off))
        mask = src < nbr
        og = L.from_edges(n, np.stack([src[mask], nbr[mask]], 1))
        t0 = time.perf_counter()
        core, rem, c2o, o2c = L.strip_isolated(og)
        c_strip = time.perf_counter() - t0
        t0 = time.perf_counter()
        ocomps = L.connected_components(og)
        c_cc = time.perf_counter() - t0
        same = ((r.removed == rem).all() and (r.core_to_orig == c2o).all()
                and (r.orig_to_core == o2c).all() and len(comps) == len(ocomps)
                and all((a == b).all() for a, b in zip(comps, ocomps)))
        print(json.dumps({"graph": f"er_fast:{n}:{d}", "m": g.m(), "removed": int(len(rem)),
                          "components": len(comps), "gpu_strip_s": round(t_strip, 4),
                          "gpu_components_s": round(t_cc, 4), "ref_strip_s": round(c_strip, 4),
                          "ref_components_s": round(c_cc, 4), "ref_impl": L.name,
                          "identical": bool(same)}), flush=True)


if __name__ == "__main__":
    main()
