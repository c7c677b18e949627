"""Local-search timing on the large configs, GPU kernels vs the reference CPU
functions on the same inputs (bodies must come out identical).

  one_two_flip on BA(1e6,5) sides harvested from 200-iteration f_B
  trajectories (8 bodies, one warp each) vs the reference one_two_flip;
  one_two_swap on ER(1e5, d=10) greedy MIS completions (8 bodies).
"""
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle
    import paper_2605_06921_b200 as P
    L = oracle.load("ref" if oracle.have_ref() else "oracle")
    K = 8
    # --- MaxCut: BA(1e6, 5)
    g = P.generate(P.BaSpec(1_000_000, 5), 1)
    b = P.ChainBatch(g, K)
    b.set_x(np.random.default_rng(0).uniform(-1, 1, (K, g.n())))
    b.run_trajectories(P.PerturbedBias(0.001), P.OptimizerConfig(alpha=0.0025, beta=0.8,
                                                                  max_iters=200))
    scores, valid, packed = b.harvest(P.PROBLEM_MAXCUT)
    P.local_search(b, 2, packed[:1])  # warm-up (module load, pools)
    t0 = time.time()
    out, gains = P.local_search(b, 2, packed)
    gpu = time.time() - t0
    og = L.generate_ba(1_000_000, 5, 1)
    sides = P.unpack_bodies(packed, g.n())
    res = [None] * K

    def work(i):
        res[i] = L.one_two_flip(og, sides[i])
    t0 = time.time()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(K)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    cpu = time.time() - t0
    got = P.unpack_bodies(out, g.n())
    same = all((got[i] == res[i][0]).all() and gains[i] == res[i][1] for i in range(K))
    print(json.dumps({"op": "one_two_flip", "graph": "ba:1e6:5", "bodies": K,
                      "gpu_secs": round(gpu, 3), "cpu_secs_8_threads": round(cpu, 3),
                      "mean_gain": float(np.mean(gains)), "identical": bool(same)}), flush=True)
    del b
    # --- MIS: ER(1e5, d=10)
    og = L.generate_er(100_000, 1e-4, 1)
    g = P.generate(P.ErSpec(100_000, 1e-4), 1)
    b = P.ChainBatch(g, K)
    starts = []
    rng = np.random.default_rng(1)
    for i in range(K):  # greedy completions of random independent seeds
        x = np.zeros(g.n())
        x[rng.choice(g.n(), 2000, replace=False)] = 1.0
        starts.append(x)
    b.set_x(np.array(starts))
    # independent seeds: harvest greedily completes them (dependent ones are dropped)
    scores, valid, packed = b.harvest(P.PROBLEM_MIS)
    keep = np.flatnonzero(valid)
    if len(keep) == 0:
        b.set_x(np.zeros((K, g.n())))
        scores, valid, packed = b.harvest(P.PROBLEM_MIS)
        keep = np.arange(K)
    packed = packed[keep]
    P.local_search(b, 3, packed[:1])  # warm-up
    t0 = time.time()
    out, sizes = P.local_search(b, 3, packed)
    gpu = time.time() - t0
    bodies = P.unpack_bodies(packed, g.n())
    res = [None] * len(keep)

    def work2(i):
        res[i] = L.one_two_swap(og, bodies[i])
    t0 = time.time()
    ths = [threading.Thread(target=work2, args=(i,)) for i in range(len(keep))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    cpu = time.time() - t0
    got = P.unpack_bodies(out, g.n())
    same = all((got[i] == res[i][0]).all() and sizes[i] == res[i][1] for i in range(len(keep)))
    print(json.dumps({"op": "one_two_swap", "graph": "er:1e5:10", "bodies": int(len(keep)),
                      "gpu_secs": round(gpu, 3), "cpu_secs_threads": round(cpu, 3),
                      "mean_size_gain": float(np.mean(sizes - scores[keep])),
                      "identical": bool(same)}), flush=True)


if __name__ == "__main__":
    main()
