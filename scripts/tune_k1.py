"""Sweep the fused-step kernel's tuning knobs on the GPU (measurement only).

python scripts/tune_k1.py [--steps 60]
Prints ms/step, edge-chain updates/s and the algorithmic-bandwidth fraction
for each (variant, hot_frac, chain-group size) on the bench workload (BA(1e6,5) f_B, 128
chains) and on config 3 (ER(1e5, d=10) MIS, 256 chains), and checks every
variant produces bit-identical iterates.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--variants", default="0,1,2,3,4")
    ap.add_argument("--fracs", default="0,0.3,0.5,0.7")
    ap.add_argument("--grids", default="8")
    ap.add_argument("--groups", default="-1",
                    help="quads per chain group (-1 = untiled, 0 = automatic)")
    ap.add_argument("--traj", action="store_true", help="also time 20-pass trajectories")
    args = ap.parse_args()
    import torch
    import paper_2605_06921_b200 as P
    from paper_2605_06921_b200 import _lib
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    cases = [("ba1e6_fB_B128", P.generate(P.BaSpec(1_000_000, 5), 1), 128,
              P.PerturbedBias(0.001), P.OptimizerConfig(alpha=0.0025, beta=0.8), -1.0),
             ("er1e5_mis_B256", P.generate(P.ErSpec(100_000, 1e-4), 1), 256,
              P.MisQubo(2.0), P.OptimizerConfig(alpha=0.8, beta=0.3), 0.0)]
    for name, g, B, spec, cfg, lo in cases:
        n, nnz = g.n(), 2 * g.m()
        alg = 8 * (n + 1) + 4 * nnz + B * (8 * nnz + 32 * n)
        X = np.random.default_rng(0).uniform(lo, 1.0, (B, n))
        batch = P.ChainBatch(g, B)
        stream = torch.cuda.ExternalStream(batch.stream)
        ref = None
        combos = [(int(v), float(f), int(gr), int(gq)) for v in args.variants.split(",")
                  for f in args.fracs.split(",") for gr in args.grids.split(",")
                  for gq in args.groups.split(",")]
        for var, frac, grid, gq in combos:
            if True:
                _lib.check(_lib.lib.mqo_tune(b"group_quads", gq))
                _lib.check(_lib.lib.mqo_tune(b"k1_variant", var))
                _lib.check(_lib.lib.mqo_tune(b"hot_frac", frac))
                _lib.check(_lib.lib.mqo_tune(b"grid_per_sm", grid))
                batch.set_x(X)
                batch.zero_v()
                for _ in range(3):
                    batch.step(spec, cfg)
                got = batch.get_x()
                same = ref is None or np.array_equal(got.view(np.uint64), ref.view(np.uint64))
                if ref is None:
                    ref = got
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
                traj_ms = None
                if args.traj:
                    tcfg = P.OptimizerConfig(alpha=cfg.alpha, beta=cfg.beta, max_iters=20)
                    batch.set_x(X)
                    t0 = time.time()
                    batch.run_trajectories(spec, tcfg)
                    traj_ms = round((time.time() - t0) * 1e3 / 20, 4)
                print(json.dumps({"case": name, "variant": var, "hot_frac": frac, "grid": grid,
                                  "group_quads": gq,
                                  "traj_ms_per_pass_wall": traj_ms,
                                  "ms_per_step": round(ms, 4),
                                  "edge_chain_per_s": nnz * B / ms * 1e3,
                                  "alg_GBps": round(alg / ms / 1e6, 1),
                                  "frac": round(alg / ms / 1e6 / peak, 4), "bit_identical": same}),
                      flush=True)
        del batch


if __name__ == "__main__":
    main()
