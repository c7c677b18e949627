"""Config 5: MIS on ER(n = 1e7, mean degree 16), chain-count sweep on one
B200, with the reference's CPU step() on the same edge list beside it.

python scripts/sweep_c5.py [--n 10000000] [--chains 8,16,32,64,128] [--steps 20]

The graph comes from the O(m) generator (MQO_GEN_ER_FAST): the reference's
O(n^2) ER generator would take ~49 h at this size.
The same CSR is handed to the reference via Graph::from_edges.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--degree", type=float, default=16.0)
    ap.add_argument("--chains", default="8,16,32,64,128")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--cpu", action="store_true", help="also time the reference step()")
    args = ap.parse_args()
    import torch
    import paper_2605_06921_b200 as P
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    t0 = time.time()
    g = P.generate(P.ErFastSpec(args.n, args.degree / args.n), 1)
    n, nnz = g.n(), 2 * g.m()
    print(json.dumps({"graph": f"er_fast:{n}:{args.degree}", "m": g.m(),
                      "gen_secs": round(time.time() - t0, 1)}), flush=True)
    spec, cfg = P.MisQubo(2.0), P.OptimizerConfig(alpha=0.8, beta=0.3)
    for B in [int(c) for c in args.chains.split(",")]:
        batch = P.ChainBatch(g, B)
        X = np.random.default_rng(B).uniform(0.0, 1.0, (B, n))
        batch.set_x(X)
        del X
        batch.zero_v()
        stream = torch.cuda.ExternalStream(batch.stream)
        for _ in range(3):
            batch.step(spec, cfg)
        batch.sync()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(args.steps):
            batch.step(spec, cfg)
        e.record(stream)
        e.synchronize()
        ms = s.elapsed_time(e) / args.steps
        alg = 8 * (n + 1) + 4 * nnz + B * (8 * nnz + 32 * n)
        print(json.dumps({"chains": B, "ms_per_step": round(ms, 3),
                          "edge_chain_per_s": nnz * B / ms * 1e3,
                          "alg_GBps": round(alg / ms / 1e6, 1), "frac": round(alg / ms / 1e6 / peak, 4)}),
              flush=True)
        del batch
        torch.cuda.empty_cache()
    if args.cpu:
        import oracle
        L = oracle.load("ref" if oracle.have_ref() else "oracle")
        off, nbr = g.csr()
        src = np.repeat(np.arange(n, dtype=np.int32), np.diff(off))
        keep = src < nbr
        t0 = time.time()
        og = L.from_edges(n, np.stack([src[keep], nbr[keep]], 1))
        build = time.time() - t0
        threads = os.cpu_count() or 1
        xs = [np.random.default_rng(i).uniform(0, 1, n) for i in range(threads)]
        vs = [np.zeros(n) for _ in range(threads)]
        steps = 2

        def work(i):
            for _ in range(steps):
                xs[i], vs[i] = L.step(og, oracle.MIS_QUBO, 2.0, xs[i], vs[i], 0.8, 0.3)
        t0 = time.time()
        ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        dt = time.time() - t0
        print(json.dumps({"cpu_impl": L.name, "threads": threads, "from_edges_secs": round(build, 1),
                          "edge_chain_per_s": steps * threads * nnz / dt}), flush=True)


if __name__ == "__main__":
    main()
