"""Benchmark of the mQO hot path (BASELINE.json metric: "edge-chain
updates/sec of mQO gradient step; best MIS size / cut at fixed time").

Default workload (--config c4, BASELINE.json configs[3], per GPU): MaxCut with
the paper's perturbed-bias objective f_B (lambda 0.001) on the synthetic
Barabasi-Albert graph BA(n=1e6, m'=5, seed 1) -- nnz = 2m = 9,999,950 -- with
B = 128 independent chains per GPU (1024 over 8 GPUs), preset alpha 0.0025,
beta 0.8.  One "step" = one fused PGA iteration of every chain (gather-SpMM
over the CSR + f_B epilogue + momentum + box clip + the ||dx|| stop bit).

* value        device-timed K steps (CUDA events on the batch stream), inputs
               resident in HBM; the 1 GB chain state is > L2, no flush needed.
* roofline     algorithmic bytes of the fused kernel
               per launch / event-timed launch duration vs the measured HBM
               copy peak (MEASURED_PEAKS.json); `traffic` = ncu dram bytes.
* e2e          the whole solver through the public API: mqo_solve_pooled
               (Mode R mqo_solve_replicas over NCCL when N > 1) on the graph's
               host CSR, copied in every step, report + best body copied out;
               rate = total_iterations * nnz / wall time.  At N = 1 the config
               is tests/golden/make_engine_golden.py's "c4" (B 16, K 4, T_gs 1,
               max_iters 200, one outer loop) and the report is compared with
               the reference's own (tests/golden/engine_large.npz); the
               reference arm runs the same solve.
* ttq          best cut at a fixed wall-clock budget (--ttq-secs), preset
               solver (T_gs 90), both arms.
* cpu_baseline the reference's own run_trajectory (oracle/_ref) on the box's
               host cores, one chain per thread, bounded sample.
``--impl reference`` times that CPU implementation alone (the driver's
reference arm).  ``--config c3|c5`` print the other BASELINE roofline rows
(ER(1e5) MIS x 256 chains, chain-tiled; ER(1e7, d=16) MIS x 64 chains).
Multi-GPU: one process per GPU (``--gpus N`` spawns them through
torch.distributed.run when not already launched that way), chains sharded,
no collective in the step (weak scaling), time = max over ranks.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edge-chain updates/sec of mQO gradient step"
UNIT = "edge-chain updates/s"
MIS, FB = 0, 4  # objective kinds (objectives.hpp:22-35 variant order)

# the BASELINE roofline rows
CONFIGS = {
    "c4": dict(graph=("ba", 1_000_000, 5, 1), kind=FB, param=0.001, alpha=0.0025, beta=0.8,
               chains=128, name="MaxCut f_B (lambda=0.001) on BA(n=1e6, m=5)"),
    "c3": dict(graph=("er", 100_000, 1e-4, 1), kind=MIS, param=2.0, alpha=0.8, beta=0.3,
               chains=256, name="MIS-QUBO (gamma=2) on ER(n=1e5, p=1e-4)"),
    "c5": dict(graph=("erfast", 10_000_000, 16.0 / 10_000_000, 1), kind=MIS, param=2.0,
               alpha=0.8, beta=0.3, chains=64,
               name="MIS-QUBO (gamma=2) on ER(n=1e7, d=16) (O(m) generator)"),
}
TTQ_CHAINS = 128  # per GPU


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config):
    """ncu dram read+write bytes per launch of the fused kernel (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "latest_traffic.json")) as f:
            d = json.load(f)
        return d.get(config, d if config == "c4" else {})
    except Exception:
        return {}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def engine_golden(name):
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_engine_golden import RUNS
    z = np.load(os.path.join(ROOT, "tests", "golden", "engine_large.npz"))
    return RUNS[name], z


class ClockSampler:
    """In-process NVML sampling of SM clock and clock-event reasons (1 ms)."""

    NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
             "sw_power_cap": 0x4, "hw_power_brake": 0x80}

    def __init__(self, index: int):
        self.index, self.rows, self.stop = index, [], threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        while not self.stop.is_set():
            try:
                sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.001)

    def __exit__(self, *exc):
        self.stop.set()
        if self.nv is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({k for _, r in self.rows for k, bit in self.NAMES.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.rows),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.rows),
                "source": "nvml, 1 ms, during the timed steps"}


def bytes_per_step(n: int, nnz: int, B: int) -> int:
    """Algorithmic HBM bytes of one fused step, no-reuse model (SURVEY.md
    section 8d): CSR offsets + indices once, per chain the gathered
    neighbour values and read x, v / write x, v per vertex."""
    return 8 * (n + 1) + 4 * nnz + B * (8 * nnz + 32 * n)


def compulsory_bytes(n: int, nnz: int, B: int) -> int:
    """DRAM-compulsory bytes of one step when the gathered rows are
    L2-resident (C3's chain-tiled slices): CSR once (re-read per chain
    group from L2) plus x, v read and written once."""
    return 8 * (n + 1) + 4 * nnz + B * 32 * n


# ------------------------------------------------------------ graphs
def ref_graph(L, spec):
    kind, n, a, seed = spec
    if kind == "ba":
        return L.generate_ba(n, a, seed)
    if kind == "er":
        return L.generate_er(n, a, seed)
    raise ValueError(kind)


def our_graph(P, spec, device=0):
    kind, n, a, seed = spec
    s = {"ba": lambda: P.BaSpec(n, a), "er": lambda: P.ErSpec(n, a),
         "erfast": lambda: P.ErFastSpec(n, a)}[kind]()
    return P.generate(s, seed, device=device)


def ref_graph_for(L, spec):
    """The reference's graph for a config; C5's O(m) ER comes from the device
    generator's edge list (the reference ER is O(n^2))."""
    if spec[0] != "erfast":
        return ref_graph(L, spec)
    import paper_2605_06921_b200 as P
    g = our_graph(P, spec, device=-1)
    off, nbr = g.csr()
    u = np.repeat(np.arange(g.n(), dtype=np.int32), np.diff(off))
    keep = u < nbr
    return L.from_edges(g.n(), np.stack([u[keep], nbr[keep]], 1))


# ------------------------------------------------------------ CPU arms
def cpu_traj_rate(L, g, c, threads: int, iters: int, warm: int = 1):
    """The reference's own run_trajectory (pga.cpp:63-111), in place with
    conv_tol = 0 and a fixed iteration count, one chain per host thread
    (ctypes releases the GIL).  -> (rate, seconds)."""
    lo = 0.0 if c["kind"] == MIS else -1.0
    rng = np.random.default_rng(123)
    xs = [rng.uniform(lo, 1.0, g.n) for _ in range(threads)]

    done = [0] * threads

    def run(k):
        def work(i):  # MIS: check_every past the cap, so the checker never accepts
            _, it, _ = L.run_trajectory(g, c["kind"], c["param"], xs[i], c["alpha"], c["beta"],
                                        k, 0.0, k + 1 if c["kind"] == MIS else 1)
            done[i] = it
        ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return time.perf_counter() - t0

    if warm:
        run(warm)
    dt = run(iters)
    return sum(done) * 2 * g.m / dt, dt


def ref_solve(L, g, oc, threads):
    os.environ["MQO_THREADS"] = str(threads)
    t0 = time.perf_counter()
    rep, body = L.solve_pooled(g, oc.to_c())
    return rep, body, time.perf_counter() - t0


def report_digest(rep: dict, body) -> dict:
    return {"report": {k: int(rep[k]) for k in ("score", "after_gradient", "after_reset_loop",
                                                "after_local_search", "trajectories",
                                                "resets_accepted", "resets_rejected",
                                                "total_iterations", "last_trajectory_stop")},
            "body_sha256": hashlib.sha256(np.ascontiguousarray(body, np.uint8).tobytes())
            .hexdigest()}


def ttq_cfg_oracle(oracle, budget, chains, seed=1):
    return oracle.Cfg(objective=FB, param=0.001, alpha=0.0025, beta=0.8, reset_fraction=0.8,
                      reset_rounds=90, seed=seed, time_budget_secs=budget, pool_batch=chains,
                      pool_keep=8)


def run_reference(args, rank: int, world: int):
    """The driver's reference arm: the reference's own CPU implementation
    (oracle/_ref, compiled from /root/reference) on all host cores."""
    if rank != 0:
        return
    import oracle
    c = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    kind = "reference" if oracle.have_ref() else "port"
    L = oracle.load("ref" if kind == "reference" else "oracle")
    g = ref_graph_for(L, c["graph"])
    nnz = 2 * g.m
    rate, dt = cpu_traj_rate(L, g, c, threads, args.steps, warm=args.warmup)
    model = cpu_model()
    sample = (f"{threads} chains (one per host thread) x run_trajectory(max_iters={args.steps}, "
              f"conv_tol=0) on {c['name']}; warm-up {args.warmup} iterations; {model}, "
              f"nproc {threads}")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{c['name']}: reference CPU run_trajectory, one chain per core",
                   "chains": threads, "graph": ":".join(map(str, c["graph"])), "nnz": int(nnz),
                   "alpha": c["alpha"], "beta": c["beta"]},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "kind": "run_trajectory"},
    }
    if args.config in ("c3", "c4") and not args.no_e2e:
        (gspec, oc), z = engine_golden(args.config)
        rep, body, wall = ref_solve(L, g, oc, threads)
        d = report_digest(rep, body)
        line["e2e"] = {"value": rep["total_iterations"] * nnz / wall, "unit": UNIT,
                       "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0, "kind": "solve_pooled",
                       "wall_s": wall, "threads": threads,
                       "config": f"tests/golden/make_engine_golden.py RUNS['{args.config}']",
                       **d}
    if args.config == "c4" and not args.no_ttq:
        rep, body, wall = ref_solve(L, g, ttq_cfg_oracle(oracle, args.ttq_secs, threads), threads)
        line["ttq"] = {"budget_s": args.ttq_secs, "best_cut": int(rep["score"]), "wall_s": wall,
                       "chains": threads, "trajectories": int(rep["trajectories"]),
                       "total_iterations": int(rep["total_iterations"]),
                       "solver": "solve_pooled, preset row (1000,100): T_gs 90, rho 0.8, K 8"}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU arm
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import paper_2605_06921_b200 as P
    from paper_2605_06921_b200 import _lib

    c = CONFIGS[args.config]
    dist = world > 1
    if dist:
        import torch.distributed as tdist
    torch.cuda.set_device(local_rank)
    device = local_rank
    B = c["chains"]
    g = our_graph(P, c["graph"], device=device)
    n, nnz = g.n(), 2 * g.m()
    spec = P.MisQubo(c["param"]) if c["kind"] == MIS else P.PerturbedBias(c["param"])
    lo = 0.0 if c["kind"] == MIS else -1.0
    batch = P.ChainBatch(g, B)
    X = np.empty((B, n))
    for i in range(B):  # chains rank*B .. rank*B+B-1 of the global batch
        X[i] = np.random.default_rng(1000 + rank * B + i).uniform(lo, 1.0, n)
    batch.set_x(X)
    batch.zero_v()
    cfg = P.OptimizerConfig(alpha=c["alpha"], beta=c["beta"])
    stream = torch.cuda.ExternalStream(batch.stream, device=device)
    red_dev = f"cuda:{device}" if (not dist or tdist.get_backend() == "nccl") else "cpu"

    def maxed(v):
        t = torch.tensor([v], dtype=torch.float64, device=red_dev)
        if dist:
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def summed(v):
        t = torch.tensor([v], dtype=torch.float64, device=red_dev)
        if dist:
            tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
        return float(t.item())

    # ---- value: K fused steps, device-timed
    for _ in range(args.warmup):
        batch.step(spec, cfg)
    batch.sync()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clk:
        start.record(stream)
        for _ in range(args.steps):
            batch.step(spec, cfg)
        end.record(stream)
        end.synchronize()
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    ms = start.elapsed_time(end)
    ms_max = maxed(ms)
    value = world * B * nnz / (ms_max / 1e3 / args.steps)

    peak, peak_kind = load_peaks()
    launch_s = ms / 1e3 / args.steps
    traffic = load_traffic(args.config)
    if args.config == "c3":  # L2-resident gathers: DRAM-compulsory model
        alg, model = compulsory_bytes(n, nnz, B), "compulsory (x, v in/out + CSR; gathers from L2)"
    else:
        alg, model = bytes_per_step(n, nnz, B), "no-reuse (SURVEY.md section 8d)"
    achieved = alg / launch_s / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_kind": peak_kind,
                "traffic": traffic.get("dram_bytes_per_launch"),
                "algorithmic_bytes_per_launch": alg, "model": model,
                "bytes_per_edge_chain": alg / (nnz * B),
                "dram_frac": (traffic["dram_bytes_per_launch"] / launch_s / 1e9 / peak
                              if traffic.get("dram_bytes_per_launch") else None),
                "kernel": traffic.get("kernel", "k_pass (fused PGA step)")}
    if traffic.get("l2_bytes_per_launch"):
        # the chain-tiled gathers are served by L2: its bytes (ncu lts__t_bytes
        # of the same kernel) against the measured L2 read bandwidth
        l2 = traffic["l2_bytes_per_launch"] / launch_s / 1e9
        roofline["l2"] = {"bytes_per_launch": traffic["l2_bytes_per_launch"], "achieved": l2,
                          "peak": traffic["l2_read_peak_gbs"], "unit": "GB/s",
                          "frac": l2 / traffic["l2_read_peak_gbs"],
                          "peak_source": traffic.get("l2_peak_source")}
    del batch
    torch.cuda.synchronize()

    # ---- e2e: the solver through the public API, host in / host out
    e2e = None
    if not args.no_e2e:
        e2e = e2e_solve(args, P, _lib, c, g, rank, world, local_rank, maxed, summed)

    # ---- ttq: best cut at a fixed budget (MaxCut config only)
    ttq = None
    if args.config == "c4" and not args.no_ttq:
        ttq = ttq_solve(args, P, g, rank, world, maxed)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        kind = "reference" if oracle.have_ref() else "port"
        L = oracle.load("ref" if kind == "reference" else "oracle")
        threads = os.cpu_count() or 1
        rg = ref_graph_for(L, c["graph"])
        rate, dt = cpu_traj_rate(L, rg, c, threads, args.cpu_steps)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": (f"{threads} chains (one per host thread) x run_trajectory("
                          f"max_iters={args.cpu_steps}, conv_tol=0) on {c['name']} "
                          f"({dt:.1f} s); {cpu_model()}, nproc {threads}")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{c['name']}: fused PGA step, {B} chains per GPU",
                       "graph": ":".join(map(str, c["graph"])), "n": n, "nnz": nnz,
                       "chains_per_gpu": B, "global_chains": B * world,
                       "alpha": c["alpha"], "beta": c["beta"],
                       "parallelism": f"chains sharded x{world} (one process per GPU)",
                       "l2": ("chain state > 126 MB L2 between steps; no flush needed"
                              if args.config != "c3" else
                              "chain state 205 MB per array > L2; gathers tiled to stay in L2")},
            "roofline": roofline,
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if ttq:
            line["ttq"] = ttq
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)


def e2e_solve(args, P, _lib, c, g, rank, world, local_rank, maxed, summed):
    """solve_pooled (N = 1) / Mode R solve_replicas over native NCCL (N > 1)
    from the graph's host CSR: H2D of the CSR + solve + D2H of report and
    body each step."""
    import ctypes as C
    import torch
    if args.config == "c5":
        return e2e_trajectories(args, P, _lib, c, g, world, maxed, summed)
    (gspec, oc), z = engine_golden(args.config)
    off, nbr = g.csr()
    h_off = torch.from_numpy(off).pin_memory()
    h_nbr = torch.from_numpy(nbr).pin_memory()
    n, nnz = g.n(), int(len(nbr))
    spec = P.MisQubo(oc.param) if oc.objective == MIS else P.PerturbedBias(oc.param)
    B_rank = oc.pool_batch
    cfg = P.SolverConfig(objective=spec,
                         optimizer=P.OptimizerConfig(oc.alpha, oc.beta, oc.max_iters, oc.conv_tol,
                                                     oc.check_every),
                         reset_fraction=oc.reset_fraction, reset_rounds=oc.reset_rounds,
                         init_noise=oc.init_noise, time_budget_secs=oc.time_budget_secs,
                         seed=oc.seed, local_search=oc.local_search,
                         pool_batch=B_rank * world, pool_keep=oc.pool_keep,
                         max_outer_loops=oc.max_outer_loops)
    comm = make_comm(world, local_rank)

    def once():
        h = C.c_void_p()
        _lib.check(P.api.lib.mqo_graph_upload(n, C.cast(h_off.data_ptr(), C.POINTER(C.c_int64)),
                                              C.cast(h_nbr.data_ptr(), C.POINTER(C.c_int32)),
                                              local_rank, C.byref(h)))
        gg = P.Graph(h, local_rank)
        if world == 1:
            r = P.solve_pooled(gg, cfg)
        else:
            r, _ = P.solve_replicas(gg, cfg, comm=comm)
        del gg
        return r

    once()  # warm-up (lazy per-graph state, allocator)
    runs, walls = [], []
    for _ in range(args.e2e_steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = once()
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
        runs.append(r)
    wall = maxed(sum(walls)) / len(walls)
    r = runs[-1]
    its = r.total_iterations  # summed over ranks by Mode R / global in Mode P
    rep = {"score": r.best_score, "after_gradient": r.after_gradient,
           "after_reset_loop": r.after_reset_loop, "after_local_search": r.after_local_search,
           "trajectories": r.trajectories, "resets_accepted": r.resets_accepted,
           "resets_rejected": r.resets_rejected, "total_iterations": r.total_iterations,
           "last_trajectory_stop": r.last_trajectory_stop}
    d = report_digest(rep, r.best_body)
    out = {"value": its * nnz / wall, "unit": UNIT,
           "h2d_bytes_per_step": int(off.nbytes + nbr.nbytes) * world,
           "d2h_bytes_per_step": int(n + 128) * world,
           "kind": "solve_pooled" if world == 1 else "solve_replicas (Mode R, NCCL argmax)",
           "wall_s": wall, "steps": args.e2e_steps,
           "config": (f"tests/golden/make_engine_golden.py RUNS['{args.config}'], "
                      f"{B_rank} chains per GPU"),
           **d}
    if world == 1:
        keys = [str(k) for k in z["report_keys"]]
        gold = dict(zip(keys, z[args.config + "_report"].tolist()))
        out["matches_reference_golden"] = (
            all(rep[k] == gold[k] for k in rep) and
            d["body_sha256"] == str(z[args.config + "_body_sha"]))
        out["reference_golden_wall_s"] = float(z[args.config + "_elapsed"][0])
    if comm is not None and hasattr(comm, "close"):
        comm.close()
    return out


def e2e_trajectories(args, P, _lib, c, g, world, maxed, summed):
    """C5: mqo_run_trajectories from pinned host states (x in / x out)."""
    import ctypes as C
    import torch
    B, n, nnz = c["chains"], g.n(), 2 * g.m()
    batch = P.ChainBatch(g, B)
    lo = 0.0 if c["kind"] == MIS else -1.0
    hx = torch.empty((B, n), dtype=torch.float64, pin_memory=True)
    hx.numpy()[:] = np.random.default_rng(7).uniform(lo, 1.0, (B, n))
    hout = torch.empty((B, n), dtype=torch.float64, pin_memory=True)
    spec = P.MisQubo(c["param"]) if c["kind"] == MIS else P.PerturbedBias(c["param"])
    cfg = P.OptimizerConfig(alpha=c["alpha"], beta=c["beta"], max_iters=100)

    def once():
        _lib.check(_lib.lib.mqo_batch_set_x(batch._h, C.cast(hx.data_ptr(), _lib._D)))
        it, _ = batch.run_trajectories(spec, cfg)
        _lib.check(_lib.lib.mqo_batch_get_x(batch._h, C.cast(hout.data_ptr(), _lib._D)))
        return int(it.sum())

    once()
    t0 = time.perf_counter()
    its = sum(once() for _ in range(args.e2e_steps))
    wall = maxed(time.perf_counter() - t0)
    its = summed(its)
    return {"value": its * nnz / wall, "unit": UNIT, "h2d_bytes_per_step": int(hx.numel() * 8),
            "d2h_bytes_per_step": int(hout.numel() * 8 + 8 * B),
            "kind": "run_trajectories (max_iters 100, host x in / out)"}


def torch_device():
    import torch
    return torch.cuda.current_device()


def make_comm(world, device):
    """The engine's communicator at N > 1: the library's native NCCL
    communicator (one rank per GPU); under the gloo test hook (ranks sharing
    a GPU, where NCCL refuses) the torch.distributed adapter."""
    if world == 1:
        return None
    if os.environ.get("MQO_BENCH_BACKEND", "nccl") == "nccl":
        from paper_2605_06921_b200.dist import nccl_comm
        return nccl_comm(device)
    from paper_2605_06921_b200.dist import TorchComm
    return TorchComm()


def ttq_solve(args, P, g, rank, world, maxed):
    cfg = P.SolverConfig(objective=P.PerturbedBias(0.001),
                         optimizer=P.OptimizerConfig(0.0025, 0.8),
                         reset_fraction=0.8, reset_rounds=90, seed=1,
                         time_budget_secs=args.ttq_secs, pool_batch=TTQ_CHAINS * world,
                         pool_keep=8)
    comm = make_comm(world, torch_device())
    t0 = time.perf_counter()
    if world == 1:
        r = P.solve_pooled(g, cfg)
    else:
        r, _ = P.solve_replicas(g, cfg, comm=comm)
    wall = maxed(time.perf_counter() - t0)
    if comm is not None and hasattr(comm, "close"):
        comm.close()
    return {"budget_s": args.ttq_secs, "best_cut": int(r.best_score), "wall_s": wall,
            "chains": TTQ_CHAINS * world, "trajectories": r.trajectories,
            "total_iterations": r.total_iterations,
            "solver": ("solve_pooled" if world == 1 else "solve_replicas (Mode R)") +
                      ", preset row (1000,100): T_gs 90, rho 0.8, K 8"}


def spawn(args):
    """--gpus N without a torch.distributed launcher: start N ranks."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-steps", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--ttq-secs", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ttq", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="print each rank's (rank, world) and exit (launcher test)")
    args = ap.parse_args()
    if args.warmup < 1 and args.impl == "ours":
        ap.error("--warmup must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}")
    if args.dry_run:
        print(json.dumps({"rank": rank, "world": world, "local_rank": local_rank}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # test hook: several ranks sharing fewer GPUs (gloo for the timing
    # reductions); production runs one rank per GPU over NCCL
    backend = os.environ.get("MQO_BENCH_BACKEND", "nccl")
    if world > 1:
        import torch
        import torch.distributed as tdist
        if backend != "nccl":
            local_rank %= max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            tdist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as tdist
            tdist.destroy_process_group()


if __name__ == "__main__":
    main()
