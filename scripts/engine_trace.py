"""Per-stage wall time of the engine on a small config (MQO_TRACE)."""
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = f"""
import sys
sys.path.insert(0, {ROOT!r})
import paper_2605_06921_b200 as P
g = P.generate(P.ErSpec(1000, 0.01), 1)
cfg = P.SolverConfig(objective=P.MisQubo(2.0), optimizer=P.OptimizerConfig(0.8, 0.3),
                     reset_fraction=0.7, reset_rounds=60, seed=1, time_budget_secs=600,
                     max_outer_loops=1, pool_batch=int(sys.argv[1]), pool_keep=int(sys.argv[2]))
r = P.solve_pooled(g, cfg)
print("score", r.best_score, "secs", r.elapsed_secs, "iters", r.total_iterations)
"""
B, K = (sys.argv[1], sys.argv[2]) if len(sys.argv) > 2 else ("1", "1")
out = subprocess.run([sys.executable, "-c", CHILD, B, K], capture_output=True, text=True,
                     env=dict(os.environ, MQO_TRACE="1"))
print(out.stdout.strip())
lines = [l for l in out.stderr.splitlines() if l.startswith("[mqo")]
events = []
for l in lines:
    m = re.match(r"\[mqo \d+ ([\d.]+)\] (.*)", l)
    if m:
        events.append((float(m.group(1)), re.sub(r"\d+", "#", m.group(2))))
acc = defaultdict(float)
cnt = defaultdict(int)
for (t0, e0), (t1, _) in zip(events, events[1:]):
    acc[e0] += t1 - t0
    cnt[e0] += 1
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:15]:
    print(f"{v*1e3:10.1f} ms  {cnt[k]:6d}x  {k}")
