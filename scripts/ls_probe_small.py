import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2605_06921_b200 as P
from paper_2605_06921_b200 import _lib
g = P.generate(P.ErSpec(1000, 0.01), 1)
B = 256
b = P.ChainBatch(g, B)
b.seed_streams(1)
b.init_states(P.PROBLEM_MIS, 0.15)
b.run_trajectories(P.MisQubo(2.0), P.OptimizerConfig(0.8, 0.3))
sc, valid, packed = b.harvest(P.PROBLEM_MIS)
print("valid", valid.sum(), "scores", sc[valid][:8])
bodies = packed[valid][:8]
for cnt in (1, 8, 8, 1):
    for rep in range(2):
        t = time.perf_counter()
        out, res = P.local_search(b, _lib.LS_ONE_TWO_SWAP, bodies[:cnt])
        dt = time.perf_counter() - t
        print(cnt, "bodies", round(dt * 1e3, 2), "ms", res[:cnt])
