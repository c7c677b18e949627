"""Per-stage wall time of the engine (MQO_TRACE) for one outer loop.

    python scripts/engine_trace.py [c1|c1_b256|c2|c3|c4] [rounds]

Same instances and presets as scripts/ttq.py; prints the report line and
the top stages by accumulated wall time (time from a trace event to the
next one is charged to the first)."""
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = f"""
import sys, time
sys.path.insert(0, {ROOT!r})
sys.path.insert(0, {os.path.join(ROOT, 'scripts')!r})
import paper_2605_06921_b200 as P
from ttq import CONFIGS
gen, pc, B, K = CONFIGS[sys.argv[1]]
g = (P.generate(P.ErSpec(gen[1], gen[2]), 1) if gen[0] == "er"
     else P.generate(P.BaSpec(gen[1], gen[2]), 1))
spec = P.MisQubo(pc["param"]) if pc["objective"] == 0 else P.PerturbedBias(pc["param"])
cfg = P.SolverConfig(objective=spec, optimizer=P.OptimizerConfig(pc["alpha"], pc["beta"]),
                     reset_fraction=pc["reset_fraction"],
                     reset_rounds=int(sys.argv[2]) if len(sys.argv) > 2 else pc["reset_rounds"],
                     time_budget_secs=3600, seed=1, max_outer_loops=1, pool_batch=B, pool_keep=K)
print("[mqo 0 %.6f] start" % time.monotonic(), file=sys.stderr, flush=True)
r = P.solve_pooled(g, cfg)
print("[mqo 0 %.6f] end" % time.monotonic(), file=sys.stderr, flush=True)
print("score", r.best_score, "secs", round(r.elapsed_secs, 3), "iters", r.total_iterations,
      "trajectories", r.trajectories)
"""
args = sys.argv[1:] or ["c1"]
out = subprocess.run([sys.executable, "-c", CHILD, *args], capture_output=True, text=True,
                     env=dict(os.environ, MQO_TRACE="1"))
print(out.stdout.strip())
if out.returncode:
    print(out.stderr[-3000:])
lines = [l for l in out.stderr.splitlines() if l.startswith("[mqo")]
events = []
for l in lines:
    m = re.match(r"\[mqo \d+ ([\d.]+)\] (.*)", l)
    if m:
        events.append((float(m.group(1)), re.sub(r"\d+", "#", m.group(2))))
events = [e for e in events if e[1] != "start"] if len(events) > 2 else events
acc = defaultdict(float)
cnt = defaultdict(int)
for (t0, e0), (t1, _) in zip(events, events[1:]):
    acc[e0] += t1 - t0
    cnt[e0] += 1
total = sum(acc.values())
print(f"traced {total * 1e3:.1f} ms")
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:20]:
    print(f"{v*1e3:10.1f} ms  {cnt[k]:6d}x  {k}")
