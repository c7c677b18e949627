"""Per-stage wall time (MQO_TRACE) of bench.py's e2e solve: the golden
config tests/golden/make_engine_golden.py RUNS[name] (default c4), run
twice, the second traced.

    python scripts/e2e_trace.py [c3|c4]
"""
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = f"""
import sys, time, os
sys.path.insert(0, {ROOT!r})
sys.path.insert(0, {os.path.join(ROOT, 'tests', 'golden')!r})
import paper_2605_06921_b200 as P
from make_engine_golden import RUNS
(kind, n, a, seed), oc = RUNS[sys.argv[1]]
g = P.generate(P.ErSpec(n, a) if kind == "er" else P.BaSpec(n, a), seed)
spec = P.MisQubo(oc.param) if oc.objective == 0 else P.PerturbedBias(oc.param)
cfg = P.SolverConfig(objective=spec, optimizer=P.OptimizerConfig(oc.alpha, oc.beta, oc.max_iters),
                     reset_fraction=oc.reset_fraction, reset_rounds=oc.reset_rounds, seed=oc.seed,
                     time_budget_secs=3600, max_outer_loops=1, pool_batch=oc.pool_batch,
                     pool_keep=oc.pool_keep)
os.environ.pop("MQO_TRACE", None)
P.solve_pooled(g, cfg)
print("[mqo 0 %.6f] start" % time.monotonic(), file=sys.stderr, flush=True)
r = P.solve_pooled(g, cfg)
print("[mqo 0 %.6f] end" % time.monotonic(), file=sys.stderr, flush=True)
print("score", r.best_score, "secs", round(r.elapsed_secs, 3), "iters", r.total_iterations)
"""
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
out = subprocess.run([sys.executable, "-c", CHILD, name], capture_output=True, text=True,
                     env=dict(os.environ, MQO_TRACE="1"))
print(out.stdout.strip())
if out.returncode:
    print(out.stderr[-3000:])
lines = [l for l in out.stderr.splitlines() if l.startswith("[mqo")]
i0 = max(i for i, l in enumerate(lines) if l.endswith("] start"))
events = []
for l in lines[i0:]:
    m = re.match(r"\[mqo \d+ ([\d.]+)\] (.*)", l)
    if m:
        events.append((float(m.group(1)), m.group(2)))
acc, cnt = defaultdict(float), defaultdict(int)
for (t0, e0), (t1, _) in zip(events, events[1:]):
    k = re.sub(r"\d+", "#", e0)
    acc[k] += t1 - t0
    cnt[k] += 1
print(f"traced {sum(acc.values()) * 1e3:.1f} ms")
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:25]:
    print(f"{v * 1e3:10.1f} ms  {cnt[k]:6d}x  {k}")
print("--- timeline")
for t, e in events:
    print(f"{(t - events[0][0]) * 1e3:9.2f}  {e}")
