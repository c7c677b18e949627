"""The reference's own micro-benchmark suite (proj/benchmarks/bench_core.cpp)
re-hosted: each case runs on the B200 through the C ABI and on the compiled
reference (oracle/_ref/libref.so, one host thread -- the reference's
functions are single-threaded) on the same graph and inputs.

    python scripts/bench_core.py [--out profiles/r08_bench_core.jsonl]

Cases (bench_core.cpp:11-88): ER(n, mean degree d) from the reference
generator, seeds as in the reference.  `items/s` follows SetItemsProcessed
(m per call) where the reference sets it.  GPU columns:
  gpu_1     one call = one vector (B = 1), the reference's shape, through the
            C ABI including its host<->device copies (latency-bound);
  gpu_b     the same op on B independent vectors per call (the B200 shape),
            reported per vector.
Gradient outputs are written to pinned host buffers (a pageable
destination costs the driver a staged copy at ~20 GB/s).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, min_time=0.3, max_reps=10000):
    fn()  # warm-up
    reps, t0 = 0, time.perf_counter()
    while True:
        fn()
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_time or reps >= max_reps:
            return dt / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--batch", type=int, default=128)
    a = ap.parse_args()
    import oracle
    import paper_2605_06921_b200 as P
    from paper_2605_06921_b200 import _lib
    R = oracle.load("ref" if oracle.have_ref() else "oracle")
    import torch

    def pinned(shape):
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    Bb = a.batch
    rows = []

    def emit(case, n, m, cpu_s, g1_s, gb_s, items=True, batch=None):
        row = {"case": case, "n": n, "m": m, "ref_cpu_us": cpu_s * 1e6, "gpu_1_us": g1_s * 1e6,
               "gpu_b_us_per_vector": gb_s * 1e6, "batch": batch or Bb,
               "speedup_1": cpu_s / g1_s, "speedup_b": cpu_s / gb_s}
        if items:
            row.update(ref_items_per_s=m / cpu_s, gpu_b_items_per_s=m / gb_s)
        rows.append(row)
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items()}),
              flush=True)

    def graphs(n, d, seed):
        return R.generate_er(n, d / n, seed), P.generate(P.ErSpec(n, d / n), seed)

    # BM_adjacency_apply / BM_laplacian_apply / BM_gradient_perturbed_bias (d = 16)
    for n in (1 << 10, 1 << 12, 1 << 14, 1 << 16):
        og, pg = graphs(n, 16.0, 1)
        for case, spec, kind, param, xval in (
                ("adjacency_apply", P.Adjacency(), oracle.ADJACENCY, 0.0, 0.5),
                ("laplacian_apply", P.Laplacian(), oracle.LAPLACIAN, 0.0, 0.5),
                ("gradient_perturbed_bias", P.PerturbedBias(0.001), oracle.PERTURBED_BIAS,
                 0.001, -0.25)):
            x = np.full(n, xval)
            if case == "adjacency_apply":
                cpu = timeit(lambda: R.adjacency_apply(og, x))
            elif case == "laplacian_apply":
                cpu = timeit(lambda: R.laplacian_apply(og, x))
            else:
                cpu = timeit(lambda: R.gradient(og, kind, param, x))
            b1 = P.ChainBatch(pg, 1)
            b1.set_x(x[None, :])
            o1 = pinned((1, n))
            g1 = timeit(lambda: b1.gradient(spec, out=o1))
            bb = P.ChainBatch(pg, Bb)
            bb.set_x(np.tile(x, (Bb, 1)))
            ob = pinned((Bb, n))
            gb = timeit(lambda: bb.gradient(spec, out=ob)) / Bb
            emit(case, n, og.m, cpu, g1, gb, items=case != "gradient_perturbed_bias")

    # BM_mis_trajectory (d = 32, seed 2; fresh init_state per run, not timed)
    for n in (1 << 10, 1 << 12):
        og, pg = graphs(n, 32.0, 2)
        rng = R.rng(7)
        inits = [R.init_state(og, 0, 0.15, R.rng(rng.next_u64())) for _ in range(8)]
        k = [0]

        def cpu_traj():
            R.run_trajectory(og, oracle.MIS_QUBO, 2.0, inits[k[0] % 8], 0.8, 0.3)
            k[0] += 1
        cpu = timeit(cpu_traj, min_time=1.0)
        cfg = P.OptimizerConfig(0.8, 0.3)
        b1 = P.ChainBatch(pg, 1)
        X1 = np.array(inits[0])[None, :]

        def g1_traj():
            b1.set_x(X1)
            b1.zero_v()
            b1.run_trajectories(P.MisQubo(2.0), cfg)
        g1 = timeit(g1_traj)
        bb = P.ChainBatch(pg, Bb)
        XB = np.array([inits[i % 8] for i in range(Bb)])

        def gb_traj():
            bb.set_x(XB)
            bb.zero_v()
            bb.run_trajectories(P.MisQubo(2.0), cfg)
        gb = timeit(gb_traj) / Bb
        emit("mis_trajectory", n, og.m, cpu, g1, gb, items=False)

    # BM_one_flip_pass (d = 16, seed 3; random sides)
    for n in (1 << 10, 1 << 12, 1 << 14):
        og, pg = graphs(n, 16.0, 3)
        rng = R.rng(11)
        sides = [np.array([rng.next_u64() & 1 for _ in range(n)], np.uint8) for _ in range(4)]
        k = [0]

        def cpu_flip():
            R.one_flip_pass(og, sides[k[0] % 4])
            k[0] += 1
        cpu = timeit(cpu_flip)
        b1 = P.ChainBatch(pg, 1)
        pk = P.pack_bodies(np.array(sides))
        g1 = timeit(lambda: P.local_search(b1, _lib.LS_ONE_FLIP, pk[:1]))
        many = np.repeat(pk, 16, axis=0)
        gb = timeit(lambda: P.local_search(b1, _lib.LS_ONE_FLIP, many)) / len(many)
        emit("one_flip_pass", n, og.m, cpu, g1, gb, items=False, batch=len(many))

    # BM_one_two_swap (d = 8, seed 5; from greedy_maximalize(g, {}))
    for n in (1 << 10, 1 << 12, 1 << 14):
        og, pg = graphs(n, 8.0, 5)
        start, _ = R.greedy_maximalize(og, np.zeros(n, np.uint8))
        cpu = timeit(lambda: R.one_two_swap(og, start))
        b1 = P.ChainBatch(pg, 1)
        pk = P.pack_bodies(np.array(start)[None, :])
        g1 = timeit(lambda: P.local_search(b1, _lib.LS_ONE_TWO_SWAP, pk))
        many = np.repeat(pk, 16, axis=0)
        gb = timeit(lambda: P.local_search(b1, _lib.LS_ONE_TWO_SWAP, many)) / len(many)
        emit("one_two_swap", n, og.m, cpu, g1, gb, items=False, batch=len(many))

    if a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
