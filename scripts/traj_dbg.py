import os, sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2605_06921_b200 as P
from paper_2605_06921_b200 import _lib
g = P.generate(P.BaSpec(1_000_000, 5), 1)
b = P.ChainBatch(g, 128)
X = np.random.default_rng(0).uniform(-1, 1, (128, g.n()))
spec, cfg = P.PerturbedBias(0.001), P.OptimizerConfig(alpha=0.0025, beta=0.8, max_iters=40)
for dbg in [0, 4, 5, 6, 7, 4]:
    _lib.check(_lib.lib.mqo_tune(b"traj_dbg", dbg))
    b.set_x(X); b.sync()
    t0 = time.time(); b.run_trajectories(spec, cfg); dt = time.time() - t0
    print("dbg", dbg, "ms/pass", round(dt * 1e3 / 40, 4), flush=True)
_lib.check(_lib.lib.mqo_tune(b"traj_dbg", 0))
import torch
st = torch.cuda.ExternalStream(b.stream)
b.set_x(X); b.zero_v()
for _ in range(3): b.step(spec, cfg)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(st)
for _ in range(40): b.step(spec, cfg)
e.record(st); e.synchronize()
print("k_pass ms/step", s.elapsed_time(e) / 40)
