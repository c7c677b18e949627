"""RunRecord / CSV / sweep output of the REFERENCE CLI itself
(tools/src/cli_common.cpp + cmd_basic.cpp + cmd_sweep.cpp + core
report_json.cpp, compiled into oracle/_ref/libref.so by oracle/Makefile and
driven through ref_shim.cpp's orc_cli_run) for tests/test_cli_records.py:
tests/golden/cli_records.json.  Every case pins max_outer, so the solve is
deterministic; timing fields are compared after masking.

Run here (where /root/reference exists): python tests/golden/make_cli_golden.py
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli_records.json")

# (name, {key: value}) -- keys are SolveOptions fields (cli_common.hpp:33-48)
CASES = [
    ("mis_er_json", {"problem": "mis", "gen": "er:200:4", "seed": "3", "tgs": "5",
                     "max_outer": "1", "budget_secs": "600"}),
    ("maxcut_er_json", {"problem": "maxcut", "gen": "er:150:5", "seed": "2", "tgs": "3",
                        "max_outer": "1", "max_iters": "400", "budget_secs": "600"}),
    ("mis_isolated", {"problem": "mis", "gen": "er:300:1.5", "seed": "5", "tgs": "4",
                      "max_outer": "1", "budget_secs": "600"}),
    ("maxcut_isolated", {"problem": "maxcut", "gen": "er:300:1.5", "seed": "6", "tgs": "2",
                         "max_outer": "1", "max_iters": "300", "budget_secs": "600"}),
    ("mis_csv", {"problem": "mis", "gen": "ba:500:3", "seed": "7", "tgs": "3", "max_outer": "1",
                 "report": "csv", "budget_secs": "600"}),
    ("mis_rle_pool", {"problem": "mis", "gen": "er:2000:6", "seed": "8", "tgs": "2",
                      "max_outer": "2", "pool_b": "4", "pool_k": "2", "sigma": "0.2",
                      "budget_secs": "600"}),
    ("maxcut_flags", {"problem": "maxcut", "gen": "sbm:400:4:0.1:0.01", "seed": "9",
                      "objective": "perturbed-laplacian", "lambda": "0.25", "alpha": "0.05",
                      "momentum": "0.5", "rho": "0.4", "tgs": "2", "max_outer": "1",
                      "max_iters": "300", "conv_tol": "1e-05", "no_local_search": "1",
                      "budget_secs": "600"}),
    ("mis_init_constant", {"problem": "mis", "gen": "er:120:3", "seed": "4", "tgs": "2",
                           "max_outer": "1", "init_constant": "0.4", "preset": "none",
                           "alpha": "0.7", "budget_secs": "600"}),
    ("sweep_rho", {"cmd": "sweep", "problem": "mis", "gen": "er:100:3", "seed": "1",
                   "tgs": "3", "max_outer": "1", "budget_secs": "600", "param": "rho",
                   "values": "0.3,0.6", "seeds": "1,2"}),
]

CHILD = r"""
import ctypes, sys
L = ctypes.CDLL(sys.argv[1])
L.orc_cli_run.argtypes = [ctypes.c_char_p]
L.orc_last_error.restype = ctypes.c_char_p
rc = L.orc_cli_run(sys.argv[2].encode())
sys.stdout.flush()
if rc < 0:
    print("ERR", L.orc_last_error().decode(), file=sys.stderr)
sys.exit(rc if rc >= 0 else 99)
"""


def main():
    sys.path.insert(0, ROOT)
    import oracle
    oracle.build(ref=True)
    out = []
    with tempfile.TemporaryDirectory() as tmp:
        for name, kv in CASES:
            kv = dict(kv)
            path = os.path.join(tmp, name + (".jsonl" if kv.get("cmd") == "sweep" else ".out"))
            kv["jsonl" if kv.get("cmd") == "sweep" else "out"] = path
            args = "\n".join(f"{k}={v}" for k, v in kv.items())
            r = subprocess.run([sys.executable, "-c", CHILD, oracle.REF_SO, args],
                               capture_output=True, text=True)
            assert r.returncode == 0, (name, r.returncode, r.stderr)
            file_text = open(path).read() if os.path.exists(path) else ""
            out.append({"name": name, "options": {k: v for k, v in kv.items()
                                                  if k not in ("out", "jsonl")},
                        "stdout": r.stdout, "file": file_text, "stderr": r.stderr})
            print(name, len(file_text), "bytes", r.stderr.strip()[:80])
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
