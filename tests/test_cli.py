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
