"""Config-scale solve_pooled goldens from the REFERENCE ITSELF
(oracle/_ref/libref.so = /root/reference/proj/core compiled by oracle/Makefile):
tests/golden/engine_large.npz.

The whole engine (run_engine, solver.cpp:192-372) on the BASELINE configs'
graphs, with pinned max_outer_loops so the run is deterministic and bounded:

* c3: MIS-QUBO (gamma 2) on ER(n=1e5, p=1e-4, seed 1) -- configs[2]'s graph --
  preset row (3000,100) alpha 0.8 / beta 0.3 / rho 0.6, B=16 chains, K=4,
  T_gs=2, one outer loop, max_iters 5000 (the reset rounds run to the cap).
* c4: MaxCut f_B (lambda 0.001) on BA(n=1e6, m'=5, seed 1) -- configs[3]'s
  graph -- preset row (1000,100) alpha 0.0025 / beta 0.8 / rho 0.8, B=16,
  K=4, T_gs=1, one outer loop, max_iters 200 (bounded so the reference run
  takes about a minute).  This is also bench.py's e2e (solve_pooled) config.

Stored: the RunReport counters (oracle.REPORT_KEYS) and the SHA-256 of the
best body (uint8[n]).  The reference's parity template is
tests/test_solver.cpp:192-214 (same_report).

Run here (where /root/reference exists):
    python tests/golden/make_engine_golden.py
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import MIS_QUBO, PERTURBED_BIAS  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "engine_large.npz")

RUNS = {
    "c3": (("er", 100_000, 1e-4, 1),
           oracle.Cfg(objective=MIS_QUBO, param=2.0, alpha=0.8, beta=0.3, reset_fraction=0.6,
                      reset_rounds=2, seed=1, time_budget_secs=1e6, max_outer_loops=1,
                      pool_batch=16, pool_keep=4)),
    "c4": (("ba", 1_000_000, 5, 1),
           oracle.Cfg(objective=PERTURBED_BIAS, param=0.001, alpha=0.0025, beta=0.8,
                      reset_fraction=0.8, reset_rounds=1, seed=1, time_budget_secs=1e6,
                      max_outer_loops=1, pool_batch=16, pool_keep=4, max_iters=200)),
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    oracle.build(ref=True)
    R = oracle.load("ref")
    assert R.name == "reference"
    z = {"report_keys": np.array(oracle.REPORT_KEYS)}
    only = set(sys.argv[1:]) or set(RUNS)
    if os.path.exists(OUT):
        old = np.load(OUT)
        z.update({k: old[k] for k in old.files})
    for name, (gspec, cfg) in RUNS.items():
        if name not in only:
            continue
        g = R.generate_er(*gspec[1:]) if gspec[0] == "er" else R.generate_ba(*gspec[1:])
        t0 = time.time()
        rep, body = R.solve_pooled(g, cfg.to_c())
        dt = time.time() - t0
        z[name + "_report"] = np.array([rep[k] for k in oracle.REPORT_KEYS], np.int64)
        z[name + "_body_sha"] = np.array(sha(body))
        z[name + "_elapsed"] = np.array([dt])
        print(name, f"{dt:.1f}s", {k: rep[k] for k in oracle.REPORT_KEYS}, flush=True)
    np.savez_compressed(OUT, **z)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
