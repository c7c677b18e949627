"""`mqo solve` / `sweep` / `gen` / `verify` on the B200 backend (SURVEY.md
section 8f rows 2 and 4).

    python -m paper_2605_06921_b200.cli solve --problem mis --gen er:1000:10 --seed 1
    python -m paper_2605_06921_b200.cli sweep --problem maxcut --gen er:2000:6 \
        --param rho --values 0.6,0.8 --seeds 1,2,3
    python -m paper_2605_06921_b200.cli gen --kind ba --n 1000 --m-attach 4 --out ba.g
    python -m paper_2605_06921_b200.cli gen --gen ba:1000000:5 --seed 1 --out ba.csr

Flags, defaults and the flow follow the reference CLI
(tools/src/main.cpp:11-46, cli_common.cpp:44-203): generator spec strings,
preset `auto` (nearest Appendix-G row, explicit flags win), isolated vertices
stripped before solving and re-embedded after, a RunRecord JSON (report_json
.cpp:108-137: same fields, bitmaps run-length encoded above 512 vertices)
CSV rows (report_json.cpp:139-157), `sweep` over rho / lambda / momentum /
local-search (cmd_sweep.cpp:27-117) and exit codes 0 / 2.  Graph files:
DIMACS or the reference's canonical text (graph_io.cpp:94-106), or this
backend's binary CSR cache (`gen --gen ... --out x.csr`).
"""
from __future__ import annotations

import argparse
import concurrent.futures
import json
import math
import sys
import time

import numpy as np

from . import api as P

SCHEMA_VERSION = 1
EXIT_OK, EXIT_USAGE = 0, 2

MIS_ROWS = [(1000, 100, (0.80, 0.30, 0.70, 60)), (1000, 300, (0.80, 0.45, 0.70, 60)),
            (1000, 500, (0.80, 0.45, 0.60, 60)), (3000, 100, (0.80, 0.30, 0.60, 60)),
            (3000, 300, (0.80, 0.45, 0.60, 60)), (3000, 1000, (0.80, 0.45, 0.50, 60)),
            (10000, 5000, (0.80, 0.75, 0.50, 60)), (20000, 10000, (0.80, 0.75, 0.50, 60)),
            (30000, 15000, (0.80, 0.75, 0.50, 60))]
CUT_ROWS = [(100, 50, (0.0025, 0.90, 0.80, 90)), (1000, 100, (0.0025, 0.80, 0.80, 90)),
            (1000, 500, (0.0025, 0.80, 0.80, 90)), (1000, 800, (0.0025, 0.80, 0.80, 90)),
            (30000, 15000, (5e-5, 0.80, 0.80, 90)), (30000, 24000, (5e-5, 0.80, 0.80, 90)),
            (40000, 20000, (5e-5, 0.80, 0.80, 90)), (40000, 32000, (5e-5, 0.80, 0.80, 90))]


class UsageError(Exception):
    pass


def preset_for(problem: str, n: int, mean_degree: float):
    """presets.cpp:43-60: nearest row in (log n, log d) space."""
    rows = MIS_ROWS if problem == "mis" else CUT_ROWS
    ln, ld = math.log(max(1.0, n)), math.log(max(1.0, mean_degree))
    best, out = math.inf, rows[0][2]
    for rn, rd, p in rows:
        dist = (ln - math.log(rn)) ** 2 + (ld - math.log(rd)) ** 2
        if dist < best:
            best, out = dist, p
    return out


def parse_gen_spec(text: str):
    """cli_common.cpp:44-75 (+ er-fast:<n>:<d> and sbm-fast:<n>:<k>:<pin>:<pout>,
    the O(m) generators)."""
    parts = text.split(":")
    try:
        if parts[0] in ("er", "er-fast") and len(parts) == 3:
            n = int(parts[1])
            p = float(parts[2][1:]) if parts[2].startswith("p") else float(parts[2]) / n
            return (P.ErSpec if parts[0] == "er" else P.ErFastSpec)(n, p)
        if parts[0] == "ba" and len(parts) == 3:
            return P.BaSpec(int(parts[1]), int(parts[2]))
        if parts[0] in ("sbm", "sbm-fast") and len(parts) == 5:
            return (P.SbmSpec if parts[0] == "sbm" else P.SbmFastSpec)(
                int(parts[1]), int(parts[2]), float(parts[3]), float(parts[4]))
    except ValueError as e:
        raise UsageError(f"cannot parse generator spec '{text}': {e}")
    raise UsageError(f"unknown generator spec '{text}' (er, er-fast, ba, sbm, sbm-fast)")


def encode_bits(bits: np.ndarray) -> dict:
    """report_json.cpp:15-32."""
    bits = np.asarray(bits, np.uint8)
    if len(bits) <= 512:
        return {"encoding": "plain", "bits": [int(b) for b in bits]}
    change = np.flatnonzero(np.diff(bits)) + 1
    edges = np.concatenate([[0], change, [len(bits)]])
    return {"encoding": "rle", "first": int(bits[0]), "runs": np.diff(edges).tolist()}


def decode_bits(j: dict, n: int) -> np.ndarray:
    if j["encoding"] == "plain":
        out = np.array(j["bits"], np.uint8)
    else:
        vals, v = [], j["first"]
        for r in j["runs"]:
            vals.append(np.full(r, v, np.uint8))
            v ^= 1
        out = np.concatenate(vals) if vals else np.zeros(0, np.uint8)
    if len(out) != n:
        raise ValueError("solution bitmap length does not match n")
    return out


OBJECTIVES = {"mis-qubo": lambda a: P.MisQubo(a.gamma if a.gamma is not None else 2.0),
              "laplacian": lambda a: P.Laplacian(),
              "perturbed-laplacian": lambda a: P.PerturbedLaplacian(
                  a.lam if a.lam is not None else 0.001),
              "adjacency": lambda a: P.Adjacency(),
              "perturbed-bias": lambda a: P.PerturbedBias(a.lam if a.lam is not None else 0.001)}


def build_config(a, g) -> P.SolverConfig:
    """cli_common.cpp:100-152."""
    obj_name = a.objective or ("mis-qubo" if a.problem == "mis" else "perturbed-bias")
    spec = OBJECTIVES[obj_name](a)
    if (P.problem_of(spec) == P.PROBLEM_MIS) != (a.problem == "mis"):
        raise UsageError(f"objective '{obj_name}' does not fit problem '{a.problem}'")
    cfg = P.SolverConfig(objective=spec)
    if a.preset == "auto":
        md = 2.0 * g.m() / g.n() if g.n() > 0 else 0.0
        alpha, mom, rho, tgs = preset_for(a.problem, g.n(), md)
        cfg.optimizer.alpha, cfg.optimizer.beta = alpha, mom
        cfg.reset_fraction, cfg.reset_rounds = rho, tgs
    for flag, setter in (("alpha", lambda v: setattr(cfg.optimizer, "alpha", v)),
                         ("momentum", lambda v: setattr(cfg.optimizer, "beta", v)),
                         ("max_iters", lambda v: setattr(cfg.optimizer, "max_iters", v)),
                         ("conv_tol", lambda v: setattr(cfg.optimizer, "conv_tol", v)),
                         ("check_every", lambda v: setattr(cfg.optimizer, "check_every", v)),
                         ("rho", lambda v: setattr(cfg, "reset_fraction", v)),
                         ("tgs", lambda v: setattr(cfg, "reset_rounds", v)),
                         ("sigma", lambda v: setattr(cfg, "init_noise", v)),
                         ("pool_b", lambda v: setattr(cfg, "pool_batch", v)),
                         ("pool_k", lambda v: setattr(cfg, "pool_keep", v))):
        if getattr(a, flag) is not None:
            setter(getattr(a, flag))
    cfg.time_budget_secs, cfg.seed = a.budget_secs, a.seed
    cfg.local_search = not a.no_local_search
    cfg.init_constant, cfg.stop_at_score, cfg.max_outer_loops = (
        a.init_constant, a.stop_at_score, a.max_outer)
    return cfg


def run_solve(a) -> dict:
    """cli_common.cpp:154-203 + report_json.cpp:108-137."""
    if bool(a.graph) == bool(a.gen):
        raise UsageError("exactly one of --graph and --gen is required")
    t0 = time.time()
    load_warnings = []
    if a.graph:
        g = P.load_graph_file(a.graph, load_warnings, device=a.device)
        desc = {"source": "file", "n": g.n(), "m": g.m(), "path": a.graph}
    else:
        g = P.generate(parse_gen_spec(a.gen), a.seed, device=a.device)
        desc = {"source": "generator", "n": g.n(), "m": g.m(), "spec": a.gen, "seed": a.seed}
    load_secs = time.time() - t0
    cfg = build_config(a, g)
    off, _ = g.csr()
    deg = np.diff(off)
    warnings = []
    if g.m() > 0 and (deg == 0).any():  # strip isolated vertices, solve, re-embed
        strip = P.strip_isolated(g)  # on the device (cli_common.cpp:163-198)
        keep = strip.core_to_orig
        core = strip.core
        rep = P.solve_pooled(core, cfg)
        body = np.zeros(g.n(), np.uint8)
        body[keep] = rep.best_body
        removed = g.n() - len(keep)
        if a.problem == "mis":
            body[deg == 0] = 1
            rep.best_score += removed
            rep.after_gradient += removed
            rep.after_reset_loop += removed
            rep.after_local_search += removed
        rep.best_body = body
        rep.warnings.append(f"stripped {removed} isolated vertices before solving")
    else:
        rep = P.solve_pooled(g, cfg)
    warnings = list(rep.warnings) + load_warnings
    o = cfg.objective
    obj = {"name": [k for k, f in OBJECTIVES.items() if type(f(a)) is type(o)][0]}
    if isinstance(o, P.MisQubo):
        obj["gamma"] = o.gamma
    elif isinstance(o, (P.PerturbedLaplacian, P.PerturbedBias)):
        obj["lambda"] = o.lam
    config = {"objective": obj, "alpha": cfg.optimizer.alpha, "momentum": cfg.optimizer.beta,
              "max_iters": cfg.optimizer.max_iters, "conv_tol": cfg.optimizer.conv_tol,
              "check_every": cfg.optimizer.check_every, "rho": cfg.reset_fraction,
              "tgs": cfg.reset_rounds, "sigma": cfg.init_noise, "budget_secs": cfg.time_budget_secs,
              "seed": cfg.seed, "local_search": cfg.local_search, "pool_b": cfg.pool_batch,
              "pool_k": cfg.pool_keep}
    for k, v in (("init_constant", cfg.init_constant), ("stop_at_score", cfg.stop_at_score),
                 ("max_outer_loops", cfg.max_outer_loops)):
        if v is not None:
            config[k] = v
    sol = ({"kind": "independent_set", "members": encode_bits(rep.best_body)} if a.problem == "mis"
           else {"kind": "cut_partition", "side": encode_bits(rep.best_body)})
    sol["score"] = rep.best_score
    if rescore(g, a.problem, decode_bits(sol["members" if a.problem == "mis" else "side"],
                                         g.n())) != rep.best_score:  # report_json.cpp:133-135
        raise P.LogicError(2, "run record round-trip: re-scored solution != best score")
    return {"schema_version": SCHEMA_VERSION, "problem": a.problem, "graph": desc,
            "config": config, "best_score": rep.best_score,
            "found_solution": rep.found_solution, "solution": sol,
            "phases": {"after_gradient": rep.after_gradient,
                       "after_reset_loop": rep.after_reset_loop,
                       "after_local_search": rep.after_local_search},
            "counters": {"outer_loops": rep.outer_loops, "trajectories": rep.trajectories,
                         "resets_accepted": rep.resets_accepted,
                         "resets_rejected": rep.resets_rejected,
                         "iterations": rep.total_iterations},
            "stop": P.StopReason.names[rep.last_trajectory_stop],
            "timing": {"solve_secs": rep.elapsed_secs, "graph_load_secs": load_secs},
            "warnings": warnings}


def rescore(g, problem: str, bits: np.ndarray) -> int:
    """score_solution on a decoded record body (objectives.cpp:143-180):
    |I| for an independent set (-1 if dependent), the cut otherwise."""
    off, nbr = g.csr()
    src = np.repeat(np.arange(g.n()), np.diff(off))
    if problem == "mis":
        if (bits[src] & bits[nbr]).any():
            return -1
        return int(bits.sum())
    return int(((bits[src] != bits[nbr]) & (src < nbr)).sum())


def solution_from_record(record: dict, n: int) -> tuple:
    """solution_from_record (report_json.cpp:139-154): (kind, bits uint8[n],
    score); fields other than the ones it reads are ignored."""
    j = record["solution"]
    kind = j["kind"]
    bits = decode_bits(j["members"] if kind == "independent_set" else j["side"], n)
    return kind, bits, int(j["score"])


CSV_HEADER = ("problem,param,value,seed,n,m,best,after_gradient,after_reset_loop,"
              "after_local_search,resets_accepted,resets_rejected,outer_loops,"
              "iterations,elapsed_secs")


def _g(x: float) -> str:
    """std::ostream << double (default precision 6)."""
    return f"{x:g}"


def csv_row(param: str, value: str, rec: dict) -> str:
    """run_record_csv_row (report_json.cpp:145-157)."""
    ph, c = rec["phases"], rec["counters"]
    return ",".join(str(v) for v in (
        rec["problem"], param, value, rec["config"]["seed"], rec["graph"]["n"],
        rec["graph"]["m"], rec["best_score"], ph["after_gradient"], ph["after_reset_loop"],
        ph["after_local_search"], c["resets_accepted"], c["resets_rejected"], c["outer_loops"],
        c["iterations"], _g(rec["timing"]["solve_secs"])))


def dump_record(rec: dict) -> str:
    """nlohmann::json::dump(): keys sorted, no spaces."""
    return json.dumps(rec, sort_keys=True, separators=(",", ":"))


SWEEP_PARAMS = {"rho": ("rho", float), "lambda": ("lam", float),
                "momentum": ("momentum", float), "local-search": ("no_local_search", None)}


def cmd_sweep(a) -> int:
    """cmd_sweep.cpp:45-117: the grid values x seeds, solved with `--jobs`
    concurrent solves (each on its own streams of the same GPU), CSV rows in
    grid order, then one '# mean' line per value."""
    values = [v for v in a.values.split(",") if v]
    if not values:
        raise UsageError("--values is empty")
    seeds = [int(x) for x in a.seeds.split(",") if x] if a.seeds else [a.seed]
    if a.param not in SWEEP_PARAMS:
        raise UsageError("--param must be rho, lambda, momentum or local-search")
    grid = []
    for value in values:
        for seed in seeds:
            o = argparse.Namespace(**vars(a))
            field, conv = SWEEP_PARAMS[a.param]
            if conv is None:
                if value not in ("on", "off"):
                    raise UsageError("local-search values are on/off")
                o.no_local_search = value == "off"
            else:
                try:
                    setattr(o, field, conv(value))
                except ValueError as e:
                    raise UsageError(str(e))
            o.seed = seed
            grid.append((o, value))
    workers = max(1, min(a.jobs, len(grid)))
    with concurrent.futures.ThreadPoolExecutor(workers) as ex:
        results = list(ex.map(lambda job: run_solve(job[0]), grid))
    jsonl = None
    if a.jsonl:
        try:
            jsonl = open(a.jsonl, "w")
        except OSError:
            raise UsageError(f"cannot open --jsonl file {a.jsonl}")
    print(CSV_HEADER)
    totals = {}
    for (o, value), rec in zip(grid, results):
        print(csv_row(a.param, value, rec))
        sm, cnt = totals.get(value, (0, 0))
        totals[value] = (sm + rec["best_score"], cnt + 1)
        if jsonl:
            jsonl.write(dump_record(rec) + "\n")
    if jsonl:
        jsonl.close()
    for value in values:
        sm, cnt = totals[value]
        print(f"# mean {a.param}={value} best={_g(sm / cnt)} over {cnt} seeds")
    return EXIT_OK


def cmd_gen(a) -> int:
    """cmd_basic.cpp:9-43 (`--kind/--n/...`, canonical text to --out or
    stdout) or a generator spec (`--gen er:n:d`, binary CSR cache unless
    --text)."""
    if a.gen:
        g = P.generate(parse_gen_spec(a.gen), a.seed, device=-1)
        g.save(a.out, text=a.text)
        print(json.dumps({"n": g.n(), "m": g.m(), "out": a.out}))
        return EXIT_OK
    if a.n is None:
        raise UsageError("--n is required")
    if a.kind == "er":
        if (a.d is None) == (a.p is None):
            raise UsageError("er needs exactly one of --d and --p")
        spec = P.ErSpec(a.n, a.p if a.p is not None else a.d / a.n)
    elif a.kind == "ba":
        spec = P.BaSpec(a.n, a.m_attach)
    else:
        spec = P.SbmSpec(a.n, a.k, a.p_in, a.p_out)
    try:
        g = P.generate(spec, a.seed, device=-1)
    except P.InvalidArgument as e:
        raise UsageError(str(e))
    if a.out:
        P.write_graph_file(g, a.out)
        print(f"wrote n={g.n()} m={g.m()} to {a.out}", file=sys.stderr)
    else:
        sys.stdout.write(P.write_canonical(g))
    return EXIT_OK


def _add_solve_options(s) -> None:
    """add_solve_options (main.cpp:11-46)."""
    s.add_argument("--problem", choices=["mis", "maxcut"], default="mis")
    s.add_argument("--graph", default="")
    s.add_argument("--gen", default="")
    s.add_argument("--budget-secs", type=float, default=10.0)
    s.add_argument("--seed", type=int, default=1)
    for f, t in (("alpha", float), ("momentum", float), ("rho", float), ("lambda", float),
                 ("gamma", float), ("sigma", float), ("conv-tol", float), ("tgs", int),
                 ("max-iters", int), ("check-every", int), ("pool-b", int), ("pool-k", int),
                 ("init-constant", float), ("stop-at-score", int), ("max-outer", int)):
        s.add_argument(f"--{f}", type=t, default=None, dest=f.replace("-", "_").replace(
            "lambda", "lam"))
    s.add_argument("--no-local-search", action="store_true")
    s.add_argument("--objective", choices=list(OBJECTIVES), default="")
    s.add_argument("--preset", choices=["auto", "none"], default="auto")
    s.add_argument("--report", choices=["json", "csv"], default="json")
    s.add_argument("--out", default="")
    s.add_argument("--device", type=int, default=0)


def _parser() -> argparse.ArgumentParser:
    from . import verify
    ap = argparse.ArgumentParser(prog="mqo", description="mQO on the B200 backend")
    sub = ap.add_subparsers(dest="cmd", required=True)
    _add_solve_options(sub.add_parser("solve", help="run the mQO solver on one instance"))
    sw = sub.add_parser("sweep", help="sweep one parameter, emit CSV")
    _add_solve_options(sw)
    sw.add_argument("--param", required=True, help="rho | lambda | momentum | local-search")
    sw.add_argument("--values", required=True, help="comma-separated values")
    sw.add_argument("--seeds", default="", help="comma-separated seeds (default: --seed)")
    sw.add_argument("--jobs", type=int, default=1, help="parallel solves")
    sw.add_argument("--jsonl", default="", help="also write one JSON record per run")
    gsub = sub.add_parser("gen", help="generate a random graph file")
    gsub.add_argument("--gen", default="", help="generator spec (binary CSR cache unless --text)")
    gsub.add_argument("--kind", choices=["er", "ba", "sbm"], default="er")
    gsub.add_argument("--n", type=int, default=None)
    gsub.add_argument("--d", type=float, default=None)
    gsub.add_argument("--p", type=float, default=None)
    gsub.add_argument("--m-attach", type=int, default=1, dest="m_attach")
    gsub.add_argument("--k", type=int, default=2)
    gsub.add_argument("--p-in", type=float, default=0.5, dest="p_in")
    gsub.add_argument("--p-out", type=float, default=0.05, dest="p_out")
    gsub.add_argument("--seed", type=int, default=1)
    gsub.add_argument("--out", default="")
    gsub.add_argument("--text", action="store_true", help="canonical text instead of binary CSR")
    verify.add_parser(sub)
    return ap


def solve_defaults(**overrides) -> argparse.Namespace:
    """The `solve` flags at their defaults (SolveOptions, cli_common.hpp),
    with overrides -- for callers that build configs without a command line."""
    a = _parser().parse_args(["solve"])
    for k, v in overrides.items():
        setattr(a, k, v)
    return a


def main(argv=None) -> int:
    a = _parser().parse_args(argv)
    try:
        if a.cmd == "verify":
            from . import verify
            return verify.cmd_verify(a.suite, a.max_n, a.n, a.p, a.seed)
        if a.cmd == "gen":
            return cmd_gen(a)
        if a.cmd == "sweep":
            return cmd_sweep(a)
        rec = run_solve(a)
        text = (dump_record(rec) if a.report == "json"
                else CSV_HEADER + "\n" + csv_row("-", "-", rec))
        if a.out:
            with open(a.out, "w") as f:
                f.write(text + "\n")
        else:
            print(text)
        for w in rec["warnings"]:
            print(f"warning: {w}", file=sys.stderr)
        return EXIT_OK
    except (UsageError, P.MqoError, OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
