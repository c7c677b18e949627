"""K1 in the small-chain regime: event-timed fused step and per-pass
trajectory cost vs chains per GPU, with the SURVEY 8d roofline fraction.

    python scripts/smallb_probe.py [--graph c4|c5] [--chains 4,8,16,32,64,128]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graph", default="c4")
    ap.add_argument("--chains", default="4,8,16,32,64,128")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--traj", type=int, default=50, help="trajectory iterations (0: skip)")
    ap.add_argument("--variant", type=int, default=0, help="mqo_tune k1_variant")
    args = ap.parse_args()
    import torch
    import paper_2605_06921_b200 as P
    c = bench.CONFIGS[args.graph]
    if args.variant:
        P.tune("k1_variant", args.variant)
    peak, _ = bench.load_peaks()
    g = bench.our_graph(P, c["graph"])
    n, nnz = g.n(), 2 * g.m()
    spec = P.MisQubo(c["param"]) if c["kind"] == bench.MIS else P.PerturbedBias(c["param"])
    lo = 0.0 if c["kind"] == bench.MIS else -1.0
    for B in [int(x) for x in args.chains.split(",")]:
        b = P.ChainBatch(g, B)
        b.set_x(np.random.default_rng(B).uniform(lo, 1.0, (B, n)))
        b.zero_v()
        cfg = P.OptimizerConfig(alpha=c["alpha"], beta=c["beta"])
        st = torch.cuda.ExternalStream(b.stream)
        for _ in range(3):
            b.step(spec, cfg)
        b.sync()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(args.steps):
            b.step(spec, cfg)
        e.record(st)
        e.synchronize()
        ms = s.elapsed_time(e) / args.steps
        alg = bench.bytes_per_step(n, nnz, B)
        row = {"graph": args.graph, "B": B, "step_ms": round(ms, 4),
               "rate": B * nnz / (ms / 1e3), "frac": alg / (ms / 1e3) / 1e9 / peak}
        if args.traj:
            tcfg = P.OptimizerConfig(alpha=c["alpha"], beta=c["beta"], max_iters=args.traj,
                                     conv_tol=0.0, check_every=args.traj + 1)
            b.run_trajectories(spec, tcfg)
            torch.cuda.synchronize()
            import time
            t0 = time.perf_counter()
            it, _ = b.run_trajectories(spec, tcfg)
            dt = time.perf_counter() - t0
            row["traj_ms_per_iter"] = round(1e3 * dt / max(1, int(it.max())), 4)
        print(json.dumps(row), flush=True)
        del b


if __name__ == "__main__":
    main()
