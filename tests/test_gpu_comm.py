"""The native communicators of libmqo_b200 (include/mqo_gpu.h, csrc/comm.cu)
and the multi-device engine (mqo_solve_devices).

One B200 per test box: NCCL refuses two ranks on one GPU, so the multi-rank
engine runs here over the in-process exchange (devices [0, 0]) and NCCL
itself at world size 1; an 8-GPU box takes the same code with distinct
devices.  Results must not depend on the rank count (the reference's
thread-count independence, tests/test_solver.cpp:221-233), and a failure on
one rank must fail every rank instead of hanging the others."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_2605_06921_b200 as P
    return P


def _key(r):
    return (r.best_score, r.after_gradient, r.after_reset_loop, r.after_local_search,
            r.outer_loops, r.trajectories, r.resets_accepted, r.resets_rejected,
            r.total_iterations, r.last_trajectory_stop, len(r.warnings))


def _cfgs(P):
    mis = P.SolverConfig(objective=P.MisQubo(2.0), optimizer=P.OptimizerConfig(0.8, 0.3),
                         reset_fraction=0.6, reset_rounds=4, seed=5, time_budget_secs=600,
                         max_outer_loops=2, pool_batch=6, pool_keep=3)
    cut = P.SolverConfig(objective=P.PerturbedBias(0.001),
                         optimizer=P.OptimizerConfig(0.0025, 0.8, 600),
                         reset_fraction=0.8, reset_rounds=3, seed=7, time_budget_secs=600,
                         max_outer_loops=1, pool_batch=5, pool_keep=3)
    return [(P.generate(P.ErSpec(400, 0.02), 3), mis), (P.generate(P.ErSpec(300, 0.03), 4), cut)]


def test_solve_devices_pooled_matches_single(P):
    for g, cfg in _cfgs(P):
        ref = P.solve_pooled(g, cfg)
        for devs in ([0, 0], [0, 0, 0]):
            r, _ = P.solve_devices(g, cfg, devs, "pooled")
            assert _key(r) == _key(ref), devs
            assert (r.best_body == ref.best_body).all()


def test_solve_devices_replicas(P):
    g, cfg = _cfgs(P)[0]
    r, scores = P.solve_devices(g, cfg, [0, 0], "replicas")
    assert r.best_score == scores.max()
    # rank 0's shard is chains 0..2: the single-process solve with B = 3
    half = P.SolverConfig(**{**cfg.__dict__, "pool_batch": 3})
    assert scores[0] == P.solve_pooled(g, half).best_score
    off, nbr = g.csr()
    for v in np.flatnonzero(r.best_body):  # the broadcast body is an independent set
        assert not r.best_body[nbr[off[v]:off[v + 1]]].any()
    assert int(r.best_body.sum()) == r.best_score


def test_nccl_world1_native_comm(P):
    """NCCL through the library (ncclCommInitRank, world 1): the engine's
    collectives run on device buffers and change nothing."""
    comm = P.NativeComm.nccl(0, 1, P.NativeComm.nccl_unique_id(), 0)
    for g, cfg in _cfgs(P):
        ref = P.solve_pooled(g, cfg)
        r = P.solve_pooled(g, cfg, comm=comm)
        assert _key(r) == _key(ref) and (r.best_body == ref.best_body).all()
        rr, scores = P.solve_replicas(g, cfg, comm=comm)
        assert _key(rr)[0] == ref.best_score and scores.tolist() == [ref.best_score]
    comm.close()


@pytest.mark.timeout(120)
@pytest.mark.parametrize("mode", ["pooled", "replicas"])
def test_rank_failure_fails_every_rank(P, mode, monkeypatch):
    """MQO_FAULT_RANK=1 makes rank 1 fail in its first reset round: the call
    returns rank 1's own error on time instead of leaving rank 0 blocked."""
    g, cfg = _cfgs(P)[0]
    monkeypatch.setenv("MQO_FAULT_RANK", "1")
    with pytest.raises(Exception, match="injected fault on rank 1"):
        P.solve_devices(g, cfg, [0, 0], mode)
    monkeypatch.delenv("MQO_FAULT_RANK")
    r, _ = P.solve_devices(g, cfg, [0, 0], mode)  # the library is still usable
    assert r.found_solution


@pytest.mark.timeout(300)
def test_solve_devices_shared_gpu_stress(P):
    """Two and three engine ranks on one GPU from host threads, repeatedly
    (the configuration in which the SMEM/cluster trajectory kernel faulted
    intermittently): every call completes and the pooled
    report equals the single-process solve."""
    cases = _cfgs(P)
    refs = [P.solve_pooled(g, cfg) for g, cfg in cases]
    for _ in range(15):
        for (g, cfg), ref in zip(cases, refs):
            for devs in ([0, 0], [0, 0, 0]):
                r, _ = P.solve_devices(g, cfg, devs, "pooled")
                assert _key(r) == _key(ref)
                P.solve_devices(g, cfg, devs, "replicas")
