"""The reference's CLI / record / scaling tests re-hosted on the B200 CLI
(/root/reference/proj/tests/test_cli.cpp, test_report.cpp, test_scaling.cpp;
same commands, instances and assertions).  `gen` and the record codec run on
CPU; solve / sweep / verify need the GPU."""
import json
import os
import subprocess
import sys
import time

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(*args):
    r = subprocess.run([sys.executable, "-m", "paper_2605_06921_b200.cli", *args],
                       capture_output=True, text=True, cwd=ROOT)
    return r.returncode, r.stdout


def canonical(text):
    import paper_2605_06921_b200 as P
    return P.read_canonical(text, device=-1)


# ---------------------------------------------------------------- test_cli.cpp
def test_cli_gen():  # test_cli.cpp:38-58
    code, out = run_cli("gen", "--kind", "er", "--n", "4", "--p", "1.0", "--seed", "1")
    g = canonical(out)
    assert code == 0 and g.n() == 4 and g.m() == 6
    code, out = run_cli("gen", "--kind", "er", "--n", "1000", "--d", "100", "--seed", "1")
    assert code == 0 and abs(canonical(out).m() - 49950.0) < 4 * 212.0
    assert run_cli("gen", "--kind", "er", "--p", "0.5")[0] == 2


@pytest.mark.gpu
def test_cli_solve(cuda_ok):  # test_cli.cpp:60-83
    code, out = run_cli("solve", "--problem", "maxcut", "--gen", "er:3:p1.0", "--budget-secs",
                        "1", "--seed", "1")
    assert code == 0 and json.loads(out)["best_score"] == 2
    code, out = run_cli("solve", "--problem", "maxcut", "--gen", "er:100:p0.66", "--objective",
                        "laplacian", "--init-constant", "0.3", "--tgs", "0", "--max-outer", "1",
                        "--no-local-search", "--budget-secs", "5", "--seed", "1")
    assert code == 0 and json.loads(out)["best_score"] == 0
    assert run_cli("solve", "--problem", "mis", "--graph", "/does/not/exist")[0] == 2
    assert run_cli("solve", "--problem", "mis", "--gen", "er:10:2", "--objective",
                   "laplacian")[0] == 2


@pytest.mark.gpu
def test_cli_sweep_single_point(cuda_ok):  # test_cli.cpp:85-104
    common = ["--problem", "mis", "--gen", "er:40:4", "--budget-secs", "60", "--max-outer", "1",
              "--tgs", "5", "--seed", "9"]
    code, out = run_cli("solve", *common)
    record = json.loads(out)
    code, swept = run_cli("sweep", *common, "--param", "rho", "--values", "0.5")
    assert code == 0
    row = swept.splitlines()[1].split(",")
    assert int(row[6]) == record["best_score"]


@pytest.mark.gpu
def test_cli_sweep_lambda_stable(cuda_ok):  # test_cli.cpp:106-124
    code, out = run_cli("sweep", "--problem", "maxcut", "--gen", "er:60:8", "--budget-secs", "60",
                        "--max-outer", "2", "--tgs", "10", "--seed", "4", "--param", "lambda",
                        "--values", "0.0001,0.001,0.01,0.1")
    assert code == 0
    bests = [float(line.split(",")[6]) for line in out.splitlines()[1:] if line[0] != "#"]
    assert len(bests) == 4
    assert (max(bests) - min(bests)) / max(bests) <= 0.1


@pytest.mark.gpu
def test_cli_verify_exact(cuda_ok):  # test_cli.cpp:126-130
    code, out = run_cli("verify", "--suite", "exact", "--max-n", "10", "--seed", "3")
    assert code == 0 and "[FAIL]" not in out


# ------------------------------------------------------------- test_report.cpp
def _tiny_record(problem, g, P, cli):
    """tiny_run (test_report.cpp:15-27) turned into a record."""
    spec = P.MisQubo(2.0) if problem == "mis" else P.PerturbedBias(0.001)
    opt = P.OptimizerConfig() if problem == "mis" else P.OptimizerConfig(0.0025, 0.8)
    cfg = P.SolverConfig(objective=spec, optimizer=opt, time_budget_secs=1.0, reset_rounds=5,
                         max_outer_loops=1, seed=7)
    rep = P.solve_pooled(g, cfg)
    key = "members" if problem == "mis" else "side"
    sol = {"kind": "independent_set" if problem == "mis" else "cut_partition",
           key: cli.encode_bits(rep.best_body), "score": rep.best_score}
    return {"schema_version": cli.SCHEMA_VERSION, "solution": sol}, rep


@pytest.mark.gpu
def test_records_round_trip(cuda_ok):  # test_report.cpp:42-68, 82-90
    import paper_2605_06921_b200 as P
    from paper_2605_06921_b200 import cli
    for problem, (n, p, seed) in (("mis", (30, 0.2, 401)), ("maxcut", (30, 0.2, 401)),
                                  ("maxcut", (600, 0.01, 403)), ("mis", (20, 0.2, 407))):
        g = P.generate(P.ErSpec(n, p), seed)
        rec, rep = _tiny_record(problem, g, P, cli)
        rec["future_field"] = {"nested": True}
        rec["solution"]["annotation"] = "ignored"
        kind, bits, score = cli.solution_from_record(rec, n)
        assert cli.rescore(g, problem, bits) == rep.best_score == score
        assert (bits == rep.best_body).all()
        if n == 600:
            assert rec["solution"]["side"]["encoding"] == "rle"


def test_bitmap_codec_identity():  # test_report.cpp:70-89
    from paper_2605_06921_b200 import cli
    rng = np.random.default_rng(405)
    for n in (1, 5, 511, 513, 2000):
        bits = rng.integers(0, 2, n).astype(np.uint8)
        rec = {"solution": {"kind": "independent_set", "members": cli.encode_bits(bits),
                            "score": int(bits.sum())}}
        assert (cli.solution_from_record(rec, n)[1] == bits).all()


def test_csv_arity():  # test_report.cpp:92-99
    from paper_2605_06921_b200 import cli
    rec = {"problem": "mis", "config": {"seed": 7}, "graph": {"n": 20, "m": 40},
           "best_score": 9, "phases": {"after_gradient": 8, "after_reset_loop": 9,
                                       "after_local_search": 9},
           "counters": {"resets_accepted": 1, "resets_rejected": 4, "outer_loops": 1,
                        "iterations": 77}, "timing": {"solve_secs": 0.5}}
    assert cli.CSV_HEADER.count(",") == cli.csv_row("rho", "0.5", rec).count(",")


# ------------------------------------------------------------ test_scaling.cpp
@pytest.mark.gpu
def test_objective_cost_scales_linearly(cuda_ok):  # test_scaling.cpp:41-57
    import paper_2605_06921_b200 as P
    small = P.generate(P.BaSpec(1 << 16, 8), 501)
    large = P.generate(P.BaSpec(1 << 18, 8), 503)
    scale = (large.m() + large.n()) / (small.m() + small.n())

    def eval_secs(g, spec, lo):
        b = P.ChainBatch(g, 1)
        b.set_x(np.random.default_rng(1).uniform(lo, 1.0, (1, g.n())))
        samples = []
        for _ in range(7):
            t0 = time.perf_counter()
            for _ in range(10):
                b.gradient(spec)
            samples.append(time.perf_counter() - t0)
        return sorted(samples)[3]

    for spec, lo in ((P.MisQubo(2.0), 0.0), (P.PerturbedBias(0.001), -1.0)):
        assert eval_secs(large, spec, lo) / eval_secs(small, spec, lo) < 4.0 * scale
