"""GPU parity of the whole solver engine (solve_pooled) against the oracle and
the reference's goldens: identical RunReports (best score and body, phase
gains, counters, iterations, last stop) for pinned max_outer_loops.  KATs
re-hosted from /root/reference/proj/tests/test_solver.cpp."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from oracle import MIS_QUBO, PERTURBED_BIAS

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
KEYS = ["score", "found_solution", "after_gradient", "after_reset_loop", "after_local_search",
        "outer_loops", "trajectories", "resets_accepted", "resets_rejected", "total_iterations",
        "last_trajectory_stop", "n_warnings"]


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2605_06921_b200 as P
    return P


def to_cfg(P, oc: oracle.Cfg):
    spec = P.MisQubo(oc.param) if oc.objective == MIS_QUBO else P.PerturbedBias(oc.param)
    return P.SolverConfig(
        objective=spec, optimizer=P.OptimizerConfig(oc.alpha, oc.beta, oc.max_iters, oc.conv_tol,
                                                     oc.check_every),
        reset_fraction=oc.reset_fraction, reset_rounds=oc.reset_rounds, init_noise=oc.init_noise,
        time_budget_secs=oc.time_budget_secs, seed=oc.seed, local_search=oc.local_search,
        pool_batch=oc.pool_batch, pool_keep=oc.pool_keep, init_constant=oc.init_constant,
        stop_at_score=oc.stop_at_score, max_outer_loops=oc.max_outer_loops)


def as_dict(r):
    return {"score": r.best_score, "found_solution": int(r.found_solution),
            "after_gradient": r.after_gradient, "after_reset_loop": r.after_reset_loop,
            "after_local_search": r.after_local_search, "outer_loops": r.outer_loops,
            "trajectories": r.trajectories, "resets_accepted": r.resets_accepted,
            "resets_rejected": r.resets_rejected, "total_iterations": r.total_iterations,
            "last_trajectory_stop": r.last_trajectory_stop, "n_warnings": len(r.warnings)}


GOLDEN_RUNS = {
    "c1_s1": ((1000, 0.01, 1), oracle.Cfg(objective=MIS_QUBO, param=2.0, alpha=0.8, beta=0.3,
                                          reset_fraction=0.7, reset_rounds=60, seed=1,
                                          time_budget_secs=600, max_outer_loops=1)),
    "c1_s2_b4": ((1000, 0.01, 2), oracle.Cfg(objective=MIS_QUBO, param=2.0, alpha=0.8, beta=0.3,
                                             reset_fraction=0.7, reset_rounds=10, seed=2,
                                             time_budget_secs=600, max_outer_loops=2,
                                             pool_batch=4, pool_keep=3)),
    "c2_s1_b4": ((2000, 6 / 2000, 1), oracle.Cfg(objective=PERTURBED_BIAS, param=0.001,
                                                 alpha=0.0025, beta=0.8, reset_fraction=0.8,
                                                 reset_rounds=6, seed=1, time_budget_secs=600,
                                                 max_outer_loops=1, pool_batch=4, pool_keep=3,
                                                 max_iters=2000)),
}


@pytest.mark.parametrize("name", list(GOLDEN_RUNS))
def test_engine_golden_reports(P, name):
    """Byte-identical reports vs the reference's own solve_pooled output."""
    z = np.load(os.path.join(GOLD, "reports.npz"))
    (n, p, s), oc = GOLDEN_RUNS[name]
    g = P.generate(P.ErSpec(n, p), s)
    r = P.solve_pooled(g, to_cfg(P, oc))
    keys = [str(k) for k in z["report_keys"]]
    assert [as_dict(r)[k] for k in keys] == z[name + "_report"].tolist()
    assert (r.best_body == z[name + "_body"]).all()


CASES = [
    dict(objective=MIS_QUBO, param=2.0, alpha=0.8, beta=0.3, reset_fraction=0.5, reset_rounds=8,
         pool_batch=1, pool_keep=1, max_outer_loops=2),
    dict(objective=MIS_QUBO, param=2.0, alpha=0.8, beta=0.3, reset_fraction=0.6, reset_rounds=5,
         pool_batch=8, pool_keep=4, max_outer_loops=1, check_every=2),
    dict(objective=MIS_QUBO, param=2.0, alpha=0.5, beta=0.0, reset_fraction=0.3, reset_rounds=4,
         pool_batch=5, pool_keep=2, max_outer_loops=2, local_search=False),
    dict(objective=PERTURBED_BIAS, param=0.001, alpha=0.0025, beta=0.8, reset_fraction=0.8,
         reset_rounds=4, pool_batch=6, pool_keep=3, max_outer_loops=1, max_iters=800),
    dict(objective=PERTURBED_BIAS, param=0.001, alpha=0.05, beta=0.5, reset_fraction=0.5,
         reset_rounds=6, pool_batch=3, pool_keep=3, max_outer_loops=2, max_iters=500),
    dict(objective=PERTURBED_BIAS, param=0.001, alpha=0.1, beta=0.0, reset_fraction=0.5,
         reset_rounds=3, pool_batch=4, pool_keep=2, max_outer_loops=1, init_constant=0.3),
]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("seed", [3, 11])
def test_engine_vs_oracle(O, P, case, seed):
    kw = dict(CASES[case])
    oc = oracle.Cfg(time_budget_secs=600, seed=seed, **kw)
    n = 300 if kw["objective"] == MIS_QUBO else 200
    og = O.generate_er(n, 0.04, seed)
    pg = P.generate(P.ErSpec(n, 0.04), seed)
    ref, body = O.solve_pooled(og, oc.to_c())
    r = P.solve_pooled(pg, to_cfg(P, oc))
    assert {k: ref[k] for k in KEYS} == as_dict(r)
    assert (r.best_body == body).all()


def test_solver_kats(P):  # test_solver.cpp:120-165
    def g(n, edges):
        return P.Graph.from_edges(n, edges)
    c5 = g(5, [(v, (v + 1) % 5) for v in range(5)])
    mis = dict(objective=P.MisQubo(2.0), optimizer=P.OptimizerConfig(alpha=0.8, beta=0.3),
               reset_fraction=0.5, reset_rounds=20)
    cut = dict(objective=P.PerturbedBias(0.001), optimizer=P.OptimizerConfig(alpha=0.0025, beta=0.8),
               reset_fraction=0.8, reset_rounds=20)
    r = P.solve_mis(c5, P.SolverConfig(**mis, seed=3, time_budget_secs=1.0))
    assert r.best_score == 2 and r.found_solution
    pet = []
    for v in range(5):
        pet += [(v, (v + 1) % 5), (v, v + 5), (v + 5, 5 + (v + 2) % 5)]
    r = P.solve_mis(g(10, pet), P.SolverConfig(**mis, seed=4, time_budget_secs=5.0, stop_at_score=4))
    assert r.best_score == 4
    k3 = g(3, [(0, 1), (1, 2), (0, 2)])
    assert P.solve_maxcut(k3, P.SolverConfig(**cut, seed=5, time_budget_secs=1.0)).best_score == 2
    assert P.solve_maxcut(c5, P.SolverConfig(**cut, seed=6, time_budget_secs=1.0)).best_score == 4
    with pytest.raises(P.InvalidArgument):
        P.solve_mis(c5, P.SolverConfig(**cut))
    with pytest.raises(P.InvalidArgument, match="reset_fraction"):
        P.solve_mis(c5, P.SolverConfig(**{**mis, "reset_fraction": 1.0}))
    with pytest.raises(P.InvalidArgument, match="batch = keep = 1"):
        P.solve_mis(c5, P.SolverConfig(**mis, pool_batch=4, pool_keep=2))
    e6 = P.Graph.from_edges(6, [])
    r = P.solve_mis(e6, P.SolverConfig(**mis, time_budget_secs=0.5))
    assert r.best_score == 6 and r.warnings
    assert P.solve_maxcut(e6, P.SolverConfig(**cut, time_budget_secs=0.5)).best_score == 0
    r = P.solve_mis(P.generate(P.ErSpec(30, 0.2), 311), P.SolverConfig(**mis, time_budget_secs=1e-9))
    assert not r.found_solution and r.best_score == 0 and r.warnings


def test_engine_init_modes_identical(O, P):
    """Both init_mode values run the bit-exact device K3 (no host path):
    identical reports, equal to the oracle's solve_pooled."""
    og = O.generate_er(1000, 0.01, 1)
    g = P.generate(P.ErSpec(1000, 0.01), 1)
    oc = oracle.Cfg(objective=MIS_QUBO, param=2.0, alpha=0.8, beta=0.3, reset_fraction=0.7,
                    reset_rounds=5, seed=1, time_budget_secs=600, max_outer_loops=1,
                    pool_batch=8, pool_keep=4)
    ref, body = O.solve_pooled(og, oc.to_c())
    for mode in (P.INIT_EXACT, P.INIT_DEVICE):
        cfg = to_cfg(P, oc)
        cfg.init_mode = mode
        r = P.solve_pooled(g, cfg)
        assert {k: ref[k] for k in KEYS} == as_dict(r)
        assert (r.best_body == body).all()


def test_engine_two_ranks_match_single(P, tmp_path):
    """Chains sharded over 2 ranks (2 processes, gloo all-gathers, one GPU)
    give the single-process report (cf. test_solver.cpp:221-233)."""
    script = tmp_path / "ranks.py"
    script.write_text(f"""
import os, sys, json
sys.path.insert(0, {ROOT!r})
import torch.distributed as dist
import paper_2605_06921_b200 as P
from paper_2605_06921_b200.dist import TorchComm
import datetime
dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=120))
g = P.generate(P.ErSpec(400, 0.03), 7)
cfg = P.SolverConfig(objective=P.MisQubo(2.0), optimizer=P.OptimizerConfig(0.8, 0.3),
                     reset_fraction=0.6, reset_rounds=6, seed=7, time_budget_secs=600,
                     max_outer_loops=2, pool_batch=7, pool_keep=3)
r = P.solve_pooled(g, cfg, comm=TorchComm())
out = dict(score=r.best_score, it=r.total_iterations, acc=r.resets_accepted,
           rej=r.resets_rejected, body=r.best_body.tolist(), stop=r.last_trajectory_stop)
open(os.environ["OUT"] + str(dist.get_rank()), "w").write(json.dumps(out))
dist.destroy_process_group()
""")
    # two ranks share this one GPU here: keep to the per-pass kernels (no
    # cooperative grid barriers competing for one device across processes)
    env = dict(os.environ, OUT=str(tmp_path / "r"), MQO_PERSISTENT_CELLS="0",
               MQO_COMM_TRACE="1")
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    proc = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           "--nproc-per-node=2", "--master-addr=127.0.0.1",
                           f"--master-port={port}", str(script)], env=env, timeout=400,
                          capture_output=True, text=True)
    if proc.returncode != 0:
        log = os.path.join(ROOT, "gpurun_out", "two_ranks_failure.log")
        os.makedirs(os.path.dirname(log), exist_ok=True)
        with open(log, "a") as f:
            f.write(proc.stdout + "\n----\n" + proc.stderr + "\n====\n")
    assert proc.returncode == 0, proc.stderr[-4000:]
    import json
    r0 = json.loads((tmp_path / "r0").read_text())
    r1 = json.loads((tmp_path / "r1").read_text())
    assert r0 == r1
    g = P.generate(P.ErSpec(400, 0.03), 7)
    cfg = P.SolverConfig(objective=P.MisQubo(2.0), optimizer=P.OptimizerConfig(0.8, 0.3),
                         reset_fraction=0.6, reset_rounds=6, seed=7, time_budget_secs=600,
                         max_outer_loops=2, pool_batch=7, pool_keep=3)
    r = P.solve_pooled(g, cfg)
    assert r0 == dict(score=r.best_score, it=r.total_iterations, acc=r.resets_accepted,
                      rej=r.resets_rejected, body=r.best_body.tolist(),
                      stop=r.last_trajectory_stop)


class _LoopbackComm:
    """A one-process stand-in for rank `rank` of `world`: every collective
    sees only this rank's contribution (used to obtain one rank's local
    Mode-R result in isolation)."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def allgather(self, data):
        return data * self.world

    def allreduce_max(self, values):
        return values

    def broadcast(self, data, root):
        return data


def _replica_cfg(P):
    return P.SolverConfig(objective=P.PerturbedBias(0.001),
                          optimizer=P.OptimizerConfig(0.0025, 0.8), reset_fraction=0.8,
                          reset_rounds=4, seed=3, time_budget_secs=600, max_outer_loops=1,
                          pool_batch=7, pool_keep=2)


def test_engine_replicas_mode(P, tmp_path):
    """Mode R (mqo_solve_replicas): each rank's shard is an independent
    pooled solve over its global chain streams; one allreduce-max picks the
    best rank (ties: lowest) and its body is broadcast to every rank."""
    g = P.generate(P.ErSpec(500, 0.02), 3)
    cfg = _replica_cfg(P)
    # rank 0's shard (chains 0..3) is the single-process solve with 4 chains
    r0, s0 = P.solve_replicas(g, cfg, comm=_LoopbackComm(0, 2))
    import dataclasses
    ref0 = P.solve_pooled(g, dataclasses.replace(cfg, pool_batch=4))
    assert s0[0] == ref0.best_score and (r0.best_body == ref0.best_body).all()
    assert r0.total_iterations == 2 * ref0.total_iterations  # loopback: both "ranks" are rank 0
    r1, s1 = P.solve_replicas(g, cfg, comm=_LoopbackComm(1, 2))
    # no comm: Mode R is solve_pooled
    rs, ss = P.solve_replicas(g, cfg)
    full = P.solve_pooled(g, cfg)
    assert ss[0] == full.best_score and (rs.best_body == full.best_body).all()
    script = tmp_path / "replicas.py"
    script.write_text(f"""
import os, sys, json, datetime
sys.path.insert(0, {ROOT!r})
import torch.distributed as dist
import paper_2605_06921_b200 as P
from paper_2605_06921_b200.dist import TorchComm
dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=120))
g = P.generate(P.ErSpec(500, 0.02), 3)
cfg = P.SolverConfig(objective=P.PerturbedBias(0.001), optimizer=P.OptimizerConfig(0.0025, 0.8),
                     reset_fraction=0.8, reset_rounds=4, seed=3, time_budget_secs=600,
                     max_outer_loops=1, pool_batch=7, pool_keep=2)
r, scores = P.solve_replicas(g, cfg, comm=TorchComm())
out = dict(score=r.best_score, body=r.best_body.tolist(), scores=scores.tolist(),
           it=r.total_iterations)
open(os.environ["OUT"] + str(dist.get_rank()), "w").write(json.dumps(out))
dist.destroy_process_group()
""")
    env = dict(os.environ, OUT=str(tmp_path / "q"), MQO_PERSISTENT_CELLS="0")
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    proc = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           "--nproc-per-node=2", "--master-addr=127.0.0.1",
                           f"--master-port={port}", str(script)], env=env, timeout=400,
                          capture_output=True, text=True)
    assert proc.returncode == 0, proc.stderr[-4000:]
    import json
    q0 = json.loads((tmp_path / "q0").read_text())
    q1 = json.loads((tmp_path / "q1").read_text())
    assert q0 == q1
    assert q0["scores"] == [int(s0[0]), int(s1[0])]
    win = r0 if s0[0] >= s1[0] else r1
    assert q0["score"] == max(s0[0], s1[0]) and q0["body"] == win.best_body.tolist()
    assert q0["it"] == (r0.total_iterations + r1.total_iterations) // 2


def test_concurrent_solves_on_host_threads(P):
    """Solves on several host threads (shared graphs, different graphs,
    SMEM-path kernels with different shared-memory sizes, local search)
    give exactly the serial results."""
    import concurrent.futures
    g1 = P.generate(P.ErSpec(600, 0.02), 5)
    g2 = P.generate(P.ErSpec(100, 0.5), 6)
    jobs = []
    for s in range(3):
        jobs.append((g1, P.SolverConfig(objective=P.MisQubo(2.0), optimizer=P.OptimizerConfig(0.8, 0.3),
                                        reset_fraction=0.6, reset_rounds=5, seed=10 + s,
                                        time_budget_secs=600, max_outer_loops=1)))
        jobs.append((g2, P.SolverConfig(objective=P.PerturbedBias(0.001),
                                        optimizer=P.OptimizerConfig(0.0025, 0.8), reset_fraction=0.8,
                                        reset_rounds=5, seed=20 + s, time_budget_secs=600,
                                        max_outer_loops=1)))
    serial = [P.solve_pooled(g, c) for g, c in jobs]
    with concurrent.futures.ThreadPoolExecutor(len(jobs)) as ex:
        conc = list(ex.map(lambda j: P.solve_pooled(*j), jobs))
    for a, b in zip(serial, conc):
        assert (a.best_score, a.total_iterations) == (b.best_score, b.total_iterations)
        assert (a.best_body == b.best_body).all()
