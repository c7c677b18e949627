"""The `mqo` CLI on the B200 backend: spec
parsing, presets, record encoding and exit codes on CPU; a full `solve`
(with isolated-vertex stripping and re-embedding, cli_common.cpp:163-198)
checked against the oracle on GPU."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2605_06921_b200.cli", *args],
                          capture_output=True, text=True, cwd=ROOT)


def test_gen_and_errors(tmp_path):
    r = cli("gen", "--gen", "er:2000:6", "--seed", "1", "--out", str(tmp_path / "g.csr"))
    assert r.returncode == 0 and json.loads(r.stdout)["m"] == 5952
    r = cli("gen", "--gen", "ba:100:3", "--seed", "2", "--out", str(tmp_path / "g.txt"), "--text")
    assert r.returncode == 0
    assert open(tmp_path / "g.txt").readline().split() == ["100", str(3 + 3 * 96)]
    assert cli("solve", "--gen", "er:10:p2").returncode == 2          # p outside [0,1]
    assert cli("solve", "--gen", "xx:10:2").returncode == 2           # unknown kind
    assert cli("solve").returncode == 2                               # no graph
    assert cli("solve", "--gen", "er:10:2", "--problem", "mis",
               "--objective", "perturbed-bias").returncode == 2       # objective/problem clash


def test_presets_and_bits():
    from paper_2605_06921_b200.cli import decode_bits, encode_bits, parse_gen_spec, preset_for
    O = oracle.load("oracle")
    for prob, code in (("mis", 0), ("maxcut", 1)):
        for n, d in ((1000, 9.9), (100000, 10.0), (1000000, 10.0), (3000, 700.0), (50, 1.0)):
            assert preset_for(prob, n, d) == O.preset_for(code, n, d)
    for n in (5, 512, 513, 4000):
        b = np.random.default_rng(n).integers(0, 2, n).astype(np.uint8)
        e = encode_bits(b)
        assert e["encoding"] == ("plain" if n <= 512 else "rle")
        assert (decode_bits(e, n) == b).all()
    s = parse_gen_spec("er:1000:10")
    assert s.n == 1000 and s.p == 10 / 1000
    assert parse_gen_spec("er:100:p0.5").p == 0.5


@pytest.mark.gpu
def test_solve_strips_isolated_vertices(cuda_ok, tmp_path):
    # ER(300, 1/300) has isolated vertices: the CLI strips, solves, re-embeds
    O = oracle.load("oracle")
    og = O.generate_er(300, 1.0 / 300, 5)
    off, nbr = og.csr()
    deg = np.diff(off)
    assert (deg == 0).any()
    out = tmp_path / "r.json"
    r = cli("solve", "--problem", "mis", "--gen", "er:300:1", "--seed", "5", "--max-outer", "1",
            "--budget-secs", "600", "--out", str(out))
    assert r.returncode == 0, r.stderr
    rec = json.loads(out.read_text())
    # the reference flow: strip, solve_pooled on the core, re-embed
    keep = np.flatnonzero(deg > 0)
    remap = np.full(300, -1)
    remap[keep] = np.arange(len(keep))
    src = np.repeat(np.arange(300), deg)
    m = src < nbr
    core = O.from_edges(len(keep), np.stack([remap[src[m]], remap[nbr[m]]], 1))
    a, mom, rho, tgs = O.preset_for(0, 300, 2 * og.m / 300)
    cfg = oracle.Cfg(objective=0, param=2.0, alpha=a, beta=mom, reset_fraction=rho,
                     reset_rounds=tgs, time_budget_secs=600, seed=5, max_outer_loops=1)
    rep, body = O.solve_pooled(core, cfg.to_c())
    full = np.zeros(300, np.uint8)
    full[keep] = body
    full[deg == 0] = 1
    from paper_2605_06921_b200.cli import decode_bits
    assert rec["best_score"] == rep["score"] + int((deg == 0).sum())
    assert (decode_bits(rec["solution"]["members"], 300) == full).all()
    assert rec["counters"]["iterations"] == rep["total_iterations"]
    assert any("stripped" in w for w in rec["warnings"])


def test_verify_rng_matches_reference_stream():
    """The suites' set-up draws (verify.Rng / derive_seed) follow rng.hpp."""
    from paper_2605_06921_b200 import verify
    O = oracle.load("oracle")
    for seed in (1, 20250801, 2**63 + 5):
        r, o = verify.Rng(seed), O.rng(seed)
        assert [r.next_u64() for _ in range(50)] == [o.next_u64() for _ in range(50)]
        assert r.uniform01() == o.uniform01()
        for stream in (0, 1, 400, 2**40):
            assert verify.derive_seed(seed, stream) == O.derive_seed(seed, stream)


def test_verify_usage_error():
    r = cli("verify", "--suite", "nope")
    assert r.returncode == 2 and "unknown --suite" in r.stderr


@pytest.mark.gpu
def test_verify_suites(cuda_ok):
    """cmd_verify.cpp's suites on the GPU path (reduced sizes)."""
    r = cli("verify", "--suite", "fixed-points", "--max-n", "9")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 4 and "all checks passed" in r.stdout
    r = cli("verify", "--suite", "escapability", "--n", "60", "--p", "0.05")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 5
    r = cli("verify", "--suite", "exact", "--max-n", "10")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 3


def test_gen_reference_flags_match_oracle(tmp_path):
    """cmd_basic.cpp:9-43: `gen --kind ...` writes the canonical text of
    the reference generator's graph (stdout or --out)."""
    O = oracle.load("oracle")
    r = cli("gen", "--kind", "ba", "--n", "60", "--m-attach", "3", "--seed", "77")
    assert r.returncode == 0, r.stderr
    og = O.generate_ba(60, 3, 77)
    off, nbr = og.csr()
    src = np.repeat(np.arange(60), np.diff(off))
    m = src < nbr
    want = f"60 {og.m}\n" + "".join(f"{u} {v}\n" for u, v in zip(src[m], nbr[m]))
    assert r.stdout == want
    out = tmp_path / "er.g"
    r = cli("gen", "--kind", "er", "--n", "80", "--d", "4", "--seed", "3", "--out", str(out))
    assert r.returncode == 0 and "wrote n=80" in r.stderr
    og = O.generate_er(80, 4 / 80, 3)
    assert out.read_text().splitlines()[0] == f"80 {og.m}"
    assert cli("gen", "--kind", "er", "--n", "80").returncode == 2           # neither --d nor --p
    assert cli("gen", "--kind", "ba", "--n", "5", "--m-attach", "9").returncode == 2


def test_sweep_usage_errors():
    base = ("sweep", "--gen", "er:100:3")
    assert cli(*base, "--param", "alpha", "--values", "1").returncode == 2
    assert cli(*base, "--param", "rho", "--values", ",").returncode == 2
    assert cli(*base, "--param", "local-search", "--values", "maybe").returncode == 2
    assert cli(*base, "--param", "rho", "--values", "abc").returncode == 2


def test_csv_row_format():
    from paper_2605_06921_b200.cli import CSV_HEADER, csv_row
    rec = {"problem": "mis", "config": {"seed": 3}, "graph": {"n": 10, "m": 12},
           "best_score": 4, "phases": {"after_gradient": 3, "after_reset_loop": 4,
                                       "after_local_search": 4},
           "counters": {"resets_accepted": 5, "resets_rejected": 6, "outer_loops": 1,
                        "iterations": 1234},
           "timing": {"solve_secs": 0.123456789}}
    assert CSV_HEADER.count(",") == csv_row("rho", "0.6", rec).count(",")
    assert csv_row("rho", "0.6", rec) == "mis,rho,0.6,3,10,12,4,3,4,4,5,6,1,1234,0.123457"


@pytest.mark.gpu
def test_sweep_rows_match_single_solves(cuda_ok, tmp_path):
    """cmd_sweep.cpp: every grid cell is exactly `solve` with that value and
    seed (also with --jobs 2), rows in grid order, '# mean' per value."""
    common = ("--problem", "maxcut", "--gen", "er:300:4", "--max-outer", "1",
              "--budget-secs", "600")
    jl = tmp_path / "s.jsonl"
    r = cli("sweep", *common, "--param", "rho", "--values", "0.5,0.8", "--seeds", "1,2",
            "--jobs", "2", "--jsonl", str(jl))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0].startswith("problem,param,value,seed")
    rows = [ln.split(",") for ln in lines[1:5]]
    assert [(x[2], x[3]) for x in rows] == [("0.5", "1"), ("0.5", "2"), ("0.8", "1"), ("0.8", "2")]
    recs = [json.loads(x) for x in jl.read_text().splitlines()]
    for row, rec in zip(rows, recs):
        single = cli("solve", *common, "--rho", row[2], "--seed", row[3])
        one = json.loads(single.stdout)
        assert int(row[6]) == rec["best_score"] == one["best_score"]
        assert one["counters"]["iterations"] == rec["counters"]["iterations"] == int(row[13])
        assert one["solution"] == rec["solution"]
    means = [ln for ln in lines if ln.startswith("# mean")]
    assert len(means) == 2 and means[0].startswith("# mean rho=0.5 best=")


@pytest.mark.gpu
def test_solve_dimacs_file_and_csv(cuda_ok, tmp_path):
    """--graph with a DIMACS file (warnings carried into the record) and
    --report csv."""
    O = oracle.load("oracle")
    og = O.generate_er(120, 0.05, 9)
    off, nbr = og.csr()
    src = np.repeat(np.arange(120), np.diff(off))
    m = src < nbr
    path = tmp_path / "g.dimacs"
    path.write_text(f"c test\np edge 120 {og.m + 1}\n" +
                    "".join(f"e {u + 1} {v + 1}\n" for u, v in zip(src[m], nbr[m])))
    r = cli("solve", "--graph", str(path), "--max-outer", "1", "--budget-secs", "600")
    assert r.returncode == 0, r.stderr
    rec = json.loads(r.stdout)
    assert rec["graph"] == {"source": "file", "n": 120, "m": og.m, "path": str(path)}
    assert f"declared m={og.m + 1} but parsed m={og.m} after deduplication" in rec["warnings"]
    r2 = cli("solve", "--graph", str(path), "--max-outer", "1", "--budget-secs", "600",
             "--report", "csv")
    hdr, row = r2.stdout.splitlines()
    assert hdr.startswith("problem,param") and row.split(",")[:7] == [
        "mis", "-", "-", "1", "120", str(og.m), str(rec["best_score"])]
