import sys, numpy as np, time
sys.path.insert(0, "/root/repo")
import paper_2605_06921_b200 as P
from paper_2605_06921_b200 import _lib
n=1024
pg = P.generate(P.ErSpec(n, 16.0 / n), 3)
sides = np.random.default_rng(11).integers(0, 2, size=(1, n), dtype=np.uint8)
b1 = P.ChainBatch(pg, 1)
pk = P.pack_bodies(sides)
done, _ = P.local_search(b1, _lib.LS_ONE_FLIP, pk.copy())
for i in range(50): P.local_search(b1, _lib.LS_ONE_FLIP, done.copy())
print("----", file=sys.stderr, flush=True)
for i in range(3):
    t=time.perf_counter(); P.local_search(b1, _lib.LS_ONE_FLIP, done.copy()); print("py", (time.perf_counter()-t)*1e6, file=sys.stderr, flush=True)
pg = P.generate(P.ErSpec(n, 8.0 / n), 5)
b1 = P.ChainBatch(pg, 1); b1.seed_streams(5); b1.init_states(P.PROBLEM_MIS, 0.15)
b1.run_trajectories(P.MisQubo(2.0), P.OptimizerConfig(0.8, 0.3))
sc, valid, packed = b1.harvest(P.PROBLEM_MIS)
done, _ = P.local_search(b1, _lib.LS_ONE_TWO_SWAP, packed[:1].copy())
for i in range(50): P.local_search(b1, _lib.LS_ONE_TWO_SWAP, done.copy())
print("----", file=sys.stderr, flush=True)
for i in range(3):
    t=time.perf_counter(); P.local_search(b1, _lib.LS_ONE_TWO_SWAP, done.copy()); print("py", (time.perf_counter()-t)*1e6, file=sys.stderr, flush=True)
