"""Byte-level parity of the B200 CLI's records with the reference CLI's own
(tests/golden/cli_records.json, made by tests/golden/make_cli_golden.py from
tools/src/cmd_basic.cpp / cmd_sweep.cpp + core/src/report_json.cpp:108-172
compiled into oracle/_ref): JSON RunRecords (incl. RLE bitmaps, stripped /
re-embedded isolated vertices, warnings), CSV rows and sweep output --
identical bytes once the wall-clock fields are masked."""
import json
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "cli_records.json")
CASES = json.load(open(GOLD))

FLAG = {"problem": "--problem", "gen": "--gen", "graph": "--graph", "objective": "--objective",
        "preset": "--preset", "report": "--report", "budget_secs": "--budget-secs",
        "seed": "--seed", "alpha": "--alpha", "momentum": "--momentum", "rho": "--rho",
        "lambda": "--lambda", "gamma": "--gamma", "sigma": "--sigma", "conv_tol": "--conv-tol",
        "tgs": "--tgs", "max_iters": "--max-iters", "check_every": "--check-every",
        "pool_b": "--pool-b", "pool_k": "--pool-k", "max_outer": "--max-outer",
        "init_constant": "--init-constant", "stop_at_score": "--stop-at-score",
        "param": "--param", "values": "--values", "seeds": "--seeds", "jobs": "--jobs"}


def mask(text: str) -> str:
    text = re.sub(r'"(solve_secs|graph_load_secs)":[-0-9.eE+]+', r'"\1":T', text)
    out = []
    for line in text.splitlines(keepends=True):  # CSV rows: elapsed_secs is the last column
        if line.count(",") == 14 and not line.startswith("problem,"):
            line = line[:line.rindex(",") + 1] + "T" + ("\n" if line.endswith("\n") else "")
        out.append(line)
    return "".join(out)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_cli_records_byte_identical(cuda_ok, case, tmp_path):
    opt = dict(case["options"])
    cmd = opt.pop("cmd", "solve")
    args = [sys.executable, "-m", "paper_2605_06921_b200.cli", cmd]
    for k, v in opt.items():
        if k == "no_local_search":
            if v == "1":
                args.append("--no-local-search")
            continue
        args += [FLAG[k], v]
    out_path = tmp_path / ("records.jsonl" if cmd == "sweep" else "record.out")
    args += ["--jsonl" if cmd == "sweep" else "--out", str(out_path)]
    r = subprocess.run(args, capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert mask(out_path.read_text()) == mask(case["file"])
    assert mask(r.stdout) == mask(case["stdout"])
    assert r.stderr == case["stderr"]
