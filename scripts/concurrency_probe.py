"""Two independent processes solving on one GPU at the same time (no
communicator): checks that device-sharing alone never stalls the engine."""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = f"""
import sys, time
sys.path.insert(0, {ROOT!r})
import paper_2605_06921_b200 as P
g = P.generate(P.ErSpec(400, 0.03), 7)
cfg = P.SolverConfig(objective=P.MisQubo(2.0), optimizer=P.OptimizerConfig(0.8, 0.3),
                     reset_fraction=0.6, reset_rounds=6, seed=7, time_budget_secs=600,
                     max_outer_loops=2, pool_batch=int(sys.argv[1]), pool_keep=3)
t0 = time.time()
r = P.solve_pooled(g, cfg)
print("B", sys.argv[1], "score", r.best_score, "secs", round(time.time() - t0, 2), flush=True)
"""

if __name__ == "__main__":
    for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
        ps = [subprocess.Popen([sys.executable, "-c", CHILD, str(b)], stdout=subprocess.PIPE, env=dict(os.environ, MQO_TRACE="1"),
                               stderr=subprocess.STDOUT, text=True) for b in (4, 3)]
        t0 = time.time()
        outs = []
        for p in ps:
            try:
                outs.append(p.communicate(timeout=150)[0].strip().splitlines()[-1:])
            except subprocess.TimeoutExpired:
                diag = subprocess.run(
                    f"cat /proc/{p.pid}/wchan; echo; for t in /proc/{p.pid}/task/*; do "
                    f"echo $t $(cat $t/wchan) $(cat $t/stat | cut -d' ' -f3); done; "
                    f"(which gdb >/dev/null && gdb -batch -p {p.pid} -ex 'thread apply all bt 12' "
                    f"2>/dev/null | grep -E '^#|^Thread' | head -80)",
                    shell=True, capture_output=True, text=True).stdout
                print(diag, flush=True)
                p.kill()
                outs.append(["TIMEOUT", (p.communicate()[0] or "").strip().splitlines()[-4:]])
        print("trial", trial, round(time.time() - t0, 1), outs, flush=True)
